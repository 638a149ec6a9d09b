/* C-ABI of the B200 PipeMax decode path (libpmb200.so).
 *
 * The reference (arxiv 2605.02189, pkg/src/pipemax) is a pure-Python
 * simulator: it has no native code and no FFI.  These entry points replace
 * the SIMULATED pieces of its decode engine (`_DecodeEngine.run`,
 * pipeline_sim.py:386-543) and are bound from Python with ctypes
 * (paper_2605_02189_b200/_C.py; INTEGRATION.md shows the binding):
 *
 *   stage compute  `estimate_decode_time(...) * noise / n`     pipeline_sim.py:423-427
 *       -> pm_embed, pm_rmsnorm, pm_gemm, pm_qkv_rope_append,
 *          pm_paged_attention, pm_argmax_reduce
 *   KV prefetch    `h2d.submit_stream(... "kv_prefetch")`       pipeline_sim.py:442-450
 *   KV offload     `d2h.submit_stream(... "kv_offload_decode")` pipeline_sim.py:486-490
 *       -> pm_copy_pieces (+ pm_host_alloc / pm_host_free for the host pool)
 *
 * Conventions: every function returns a cudaError_t as int (0 = success) and
 * pm_error_string() describes it; calls are asynchronous on the given CUDA
 * stream (cudaStream_t passed as void*); no function allocates device memory
 * (workspaces are caller-owned); tensor maps are 128-byte CUtensorMap images
 * built by pm_tmap_encode_2d.  bf16 tensors are passed as void*.
 */
#ifndef PM_B200_H
#define PM_B200_H
#ifdef __cplusplus
extern "C" {
#endif

int pm_abi_version(void);
const char* pm_error_string(int code);

/* ---- descriptors / memory ------------------------------------------------ */
int pm_tmap_encode_2d(void* tmap_out, const void* gaddr, unsigned long long inner, unsigned long long outer,
                      unsigned long long row_stride_bytes, unsigned box_inner, unsigned box_outer,
                      int swizzle128);
/* 5-D map over the block-first KV pool (n_rows = blocks*16 slots of L_s*2*Hkv*hd bf16): one copy moves one KV
 * block's K and V of one (layer, kv head); pm_paged_attention takes it with cfg bit 4 set */
int pm_tmap_encode_pool(void* tmap_out, const void* pool, unsigned long long n_rows, int L_s, int Hkv, int hd);
int pm_host_alloc(unsigned long long bytes, void** out);
int pm_host_free(void* p);
/* NUMA node of device `device`'s PCIe attachment (sysfs; -1 unknown) */
int pm_device_numa_node(int device, int* node);
/* pinned + mapped host memory bound to NUMA node `numa_node` (1 GB-aligned mmap + mbind, registered in 1 GB
 * pieces with retries; falls back to cudaHostAlloc; < 0: pm_host_alloc).  A single cudaMemcpy may not span two
 * pieces: pm_copy_pieces / pm_copy_2d cut copies at 1 GB boundaries; the mapped device address
 * (pm_host_device_ptr) covers the first piece.  Free with pm_host_free_numa(p, bytes, numa_node) */
int pm_host_alloc_numa(unsigned long long bytes, int numa_node, void** out);
int pm_host_free_numa(void* p, unsigned long long bytes, int numa_node);
/* eager decode offload: host_dev + offs[2i] <- pool + offs[2i+1], `bytes` each, one kernel (`ctas` CTAs) writing
 * through the mapped replica; host_dev / offs are pm_host_device_ptr addresses; bytes % 16 == 0 */
int pm_offload_rows(void* host_dev, const void* pool, const void* offs, int n, unsigned long long bytes, int ctas,
                    void* stream);
/* device address of pm_host_alloc memory (it is mapped: kernels may read it over PCIe) */
int pm_host_device_ptr(void* host, void** dev);
/* per-step metadata upload: dst[i][0..n[i]) <- src[i] (int32; src = pm_host_device_ptr addresses), a
 * kernel on `stream` instead of a copy-engine DMA so it never queues behind KV prefetch copies */
int pm_meta_upload(int count, void* const* dst, const void* const* src, const int* n, void* stream);
/* dst_base+dst_off[i] <- src_base+src_off[i], `bytes` each; contiguous runs merged */
/* decode offload in one DMA: gather the n rows (pool + pool_off[i], `bytes` each) into dev_stage, one
 * cudaMemcpyAsync to pinned host_stage, then a host function in stream order scatters them to
 * replica + rep_off[i] (pipeline_sim.py:486-490's eager offload); rep_off / pool_off are host arrays */
int pm_offload_gather(void* replica, const void* pool, const long long* rep_off, const long long* pool_off, int n,
                      unsigned long long bytes, void* dev_stage, void* host_stage, void* stream);
int pm_copy_pieces(void* dst_base, const void* src_base, const long long* dst_off, const long long* src_off,
                   int n, unsigned long long bytes, void* stream);

/* pitched copy (one layer's K/V of a run of tokens, pool <-> host replica; prefill offload) */
int pm_copy_2d(void* dst, unsigned long long dpitch, const void* src, unsigned long long spitch,
               unsigned long long width, unsigned long long height, void* stream);

/* ---- per-stage decode forward ---------------------------------------------- */
int pm_embed(const int* tok_table, const int* slots, const void* table, float* resid, int M, int d,
             void* stream);
int pm_rmsnorm(const float* x, const void* w, void* y, int M, int d, float eps, void* stream);
/* stream-K tcgen05 GEMM over a packed weight ([units][K/64][2][128][64], 128B-swizzled).  grid = CTAs.
 * cta_pair = 0: one CTA per stream-K worker computes whole 256-row units, tmap_x box [bn rows x 64];
 * cta_pair = 1: each worker is a (2,1,1) cluster (grid even), one 128-row half per CTA, tmap_x box
 * [bn/2 rows x 64] (each CTA loads half the activation tile and multicasts it to its partner).
 * max_segs = pm_gemm_max_segments(total, kb, workers); the argmax epilogue writes 2 tiles (128-row
 * halves) per 256-row unit. */
int pm_gemm(const void* w_packed, const void* tmap_x, int n_out, int n_units, int k, int m_tok, int bn,
            int grid, int cta_pair, int epilogue, void* out, int ld_out, float* ws, int max_segs, float* amax_val,
            int* amax_idx, int m_cap, const void* prefetch, unsigned long long prefetch_bytes,
            unsigned long long prefetch_span, int fix_mode, int* fix_counters, const int* fix_units, int n_fix,
            void* stream);
/* prefetch/prefetch_bytes: optional region the NEXT operation reads first; it is pulled into L2 while
 * this GEMM drains (keeps HBM busy across the kernel boundary); NULL/0 for none.  prefetch_span = 0:
 * the contiguous [prefetch, +prefetch_bytes); > 0: one stripe of prefetch_bytes / grid per CTA, stripe c
 * at prefetch + c * prefetch_span / grid -- the first bytes of every stream-K worker's range when the
 * next operation is a GEMM over prefetch_span bytes of packed weight (its workers start at evenly spaced
 * k-blocks). */
/* fix_mode: how the units the stream-K partition splits are finished.
 *   0: a post kernel on `stream` waits for the whole GEMM grid, then finishes them;
 *   2 (poll): the GEMM arrives on fix_counters[unit] as each part lands and every post-kernel CTA starts
 *      as soon as its own unit is complete (overlapping the GEMM's tail); the post kernel still completes
 *      only after the GEMM grid.  Deadlock-free (the post kernel launches after every GEMM CTA started);
 *   1 (fused): the GEMM kernel itself runs fixup tasks over the n_fix units in fix_units (the split
 *      units, pm_gemm_fix_units; every unit for pm_gemm_qkv_rope), each waiting on its unit's arrivals --
 *      needs every CTA of the grid resident at once (one stream of dependent kernels) and m_tok <= bn.
 * fix_counters: int[2 * n_units], zero at rest, left zero (modes 1 and 2). */
/* residual projection (O / down) fused with the next RMSNorm: resid += X W^T (fp32), then
 * xn = RMSNorm(resid) * norm_w (bf16) per row; row_counters int[m_cap], zero at rest, left zero.
 * split_norm = 0: the last unit to finish a row normalises it inside the fixup kernel;
 * 1: fixup kernel, then a row-parallel RMSNorm kernel (same result, bit for bit) */
int pm_gemm_resid_rmsnorm(const void* w_packed, const void* tmap_x, int n_out, int n_units, int k, int m_tok,
                          int bn, int grid, int cta_pair, float* resid, float* ws, int max_segs, int m_cap, const void* prefetch,
                          unsigned long long prefetch_bytes, unsigned long long prefetch_span, const void* norm_w, void* xn, float eps,
                          int* row_counters, int split_norm, int fix_mode, int* fix_counters, const int* fix_units,
                          int n_fix, void* stream);
/* QKV projection fused with (Qwen3 q/k RMSNorm) + RoPE + paged KV append (pm_qkv_rope_append's contract);
 * qkv_out [m_cap][n_out] bf16 is scratch */
int pm_gemm_qkv_rope(const void* w_packed, const void* tmap_x, int n_out, int n_units, int k, int m_tok, int bn,
                     int grid, int cta_pair, void* qkv_out, float* ws, int max_segs, int m_cap, const void* prefetch,
                     unsigned long long prefetch_bytes, unsigned long long prefetch_span, int fix_mode,
                     int* fix_counters, const int* fix_units, int n_fix, void* q_out, void* pool, const int* block_table,
                     const int* positions, const float* rope, const void* qn_w, const void* kn_w, int H, int Hkv,
                     int hd, int layer, int L_s, int max_blocks, float eps, void* stream);
/* stream-K geometry helpers over `workers` (= grid, or grid / 2 in pair mode) */
int pm_gemm_split_units(long long total, int kb, int workers);
int pm_gemm_max_segments(long long total, int kb, int workers);
/* the units a stream-K partition splits (ascending) into out[], returns their count */
int pm_gemm_fix_units(long long total, int kb, int workers, int* out);
int pm_qkv_rope_append(const void* qkv, void* q_out, void* pool, const int* block_table, const int* positions,
                       const float* rope, const void* qn_w, const void* kn_w, int M, int H, int Hkv, int hd,
                       int layer, int L_s, int max_blocks, float eps, void* stream);
int pm_paged_attention(const void* tmap_kv, const void* q, const int* block_table, const int* seq_lens,
                       const int* work, void* out, float* ws_o, float* ws_ml, int* counters, int M, int H,
                       int Hkv, int hd,
                       int layer, int L_s, int max_blocks, int max_chunks, int max_piece, int cfg,
                       void* stream);
/* tmap_kv: the 2-D view [blocks*16][L_s*2*Hkv*hd] with a [16][64] box (pm_tmap_encode_2d, four copies
 * per KV block), or -- cfg bit 4 (16) set -- pm_tmap_encode_pool's 5-D map (one copy per block).
 * cfg bit 5 (32): decode step -- every row is a distinct request whose only KV the preceding kernels write
 * is its current token, so blocks before each row's last load ahead of the PDL dependency wait.
 * cfg & 15: warps x KV-ring stages per SM (0: 6x4, 1: 12x2, 2: 8x3, 3: 4x2 at 2 CTAs/SM; -1: default);
 * the work list must be built for pm_attn_workers_cfg(hd, cfg) warps and pieces of at most max_piece
 * (<= pm_attn_max_piece()) blocks; max_chunks >= the most pieces of one (row, kv head). */
int pm_attn_max_piece(void);
/* host: a step's balanced attention work list -- every (row, kv head)'s KV blocks end to end, one equal
 * range per warp (at least minq blocks), cut into pieces of at most maxp blocks; work[0] = warps used,
 * work[1] = pieces, work[2 + w] = warp w's first piece, pieces (4 ints: row | kvh << 16, b0 | nblk << 16,
 * chunk | nchunks << 16, seq_len) from int (3 + used + 3) & ~3.  Returns the ints written (negative
 * cudaError_t when `cap` is too small). */
int pm_attn_work_list(const int* seq_lens, int M, int hkv, int workers, int maxp, int minq, int cap, int* work);
/* warps of a full attention launch on the current device (the `workers` above) */
int pm_attn_workers(int hd);
int pm_attn_workers_cfg(int hd, int cfg);
/* one-time kernel attributes; call once per device before CUDA-graph capture */
int pm_prepare_gemm(void);
/* profiling: record cudaEvent_t `event` between the next GEMM launch's main and fixup kernels (one-shot) */
int pm_gemm_split_event(void* event);
int pm_prepare_attention(void);
int pm_argmax_reduce(const float* val, const int* idx, int n_tiles, int M, int m_cap, int* out_ids,
                     int* tok_table, const int* slots, void* stream);

/* ---- pipeline hop (pipeline.py) -------------------------------------------------------------------- */
/* fp32 residual rows <-> bf16 wire format (n elements, n % 8 == 0) */
int pm_hop_pack(const float* resid, void* out, long long n, void* stream);
int pm_hop_unpack(const void* in, float* resid, long long n, void* stream);
/* stage 0: tok_table[slots[i]] = ids[i]; slots may be mapped pinned host memory (pm_host_device_ptr) */
int pm_scatter_tokens(const int* ids, const int* slots, int n, int* tok_table, void* stream);

/* ---- cluster split-K projection (gemm_cl.cu): split-K reduction and epilogue in ONE kernel ----------
 * cluster = 2 * slices CTAs (pair = the two 128-row halves of a 256-row unit, sharing a multicast
 * activation tile; slices split K); n_clusters clusters own consecutive units; the slices' fp32 partials
 * are summed in slice order (L2 scratch, cluster-scope mbarrier hand-off).  m_tok <= bn <= 128; tmap_x box
 * [bn/2 rows x 64].  epilogue: 0 bf16 store, 1 SiLU(gate)*up (interleaved rows), 2 resid += acc (fp32;
 * with norm_w: xn = bf16(resid * norm_w) and ssq_out[n_out/128][m_cap] = per-128-row sums of resid^2),
 * 3 logits (out may be NULL) + argmax tiles, 4 bf16 round + q/k norm + RoPE + q_out / paged KV append.
 * ssq_in (NULL = none): the input rows are bf16(x * w) of a folded RMSNorm; every token column is scaled
 * by rsqrt(sum_t ssq_in[t][m] / d_in + eps).  Replaces pm_gemm / pm_gemm_resid_rmsnorm /
 * pm_gemm_qkv_rope and their fixup kernels for m_tok <= 128. */
int pm_gemm_cl(const void* w_packed, const void* tmap_x, int n_out, int n_units, int k, int m_tok, int bn,
               int m_cap, int slices, int n_clusters, int epilogue, void* out, int ld_out, const float* ssq_in,
               int n_ht_in, int d_in, float eps, float* resid, const void* norm_w, void* xn, float* ssq_out,
               float* amax_val, int* amax_idx, void* q_out, void* pool, const int* block_table,
               const int* positions, const float* rope, const void* qn_w, const void* kn_w, int H, int Hkv, int hd,
               int layer, int L_s, int max_blocks, float* part, void* stream);
/* part: fp32 scratch, n_clusters * 2 * slices * bn * 128 floats (split-K partials, L2-resident) */
/* co-resident clusters of `cluster_size` CTAs of the bn instantiation (cudaOccupancyMaxActiveClusters) */
int pm_gemm_cl_max_clusters(int bn, int cluster_size, int* out);
/* profiling only: per-CTA globaltimer stamps of the last launch under PM_CL_TRACE=1 ([160][8] u64) */
int pm_gemm_cl_trace_read(void* dst);
/* weight-ring stages of the bn instantiation */
int pm_gemm_cl_stages(int bn);
/* one-time kernel attributes of the cluster GEMM */
int pm_prepare_gemm_cl(void);

#ifdef __cplusplus
}
#endif
#endif
