// Paged GQA decode attention over the block-first KV pool (one query token
// per request).  HBM-bound: every KV byte of the active micro-batch is read
// exactly once per layer, so the kernel is built to keep every SM streaming.
//
// Work split (host-built, pm_attn_work_list): the KV blocks of every (request
// row, kv head) unit are laid end to end and cut into one contiguous range of
// equal length per warp, each range into pieces of at most `maxp` blocks.
// Every warp therefore streams the same number of KV blocks whatever the rows'
// lengths (the previous fixed-size chunks left the busiest warp ~1.5x the
// mean).  Persistent grid; every WARP is an independent worker that walks its
// pieces with its own STAGES-deep TMA pipeline running straight across piece
// boundaries (no CTA-wide barriers on the hot path):
//   lane 0 issues, per KV block, four 128B-swizzled 2-D TMA boxes (K and V,
//   two 64-dim halves each); the warp consumes them with ldmatrix +
//   mma.sync.m16n8k16 in the transposed arrangement
//       S^T[16 tok x 8 heads] = K[16 x hd] . Q^T[hd x 8]
//       O^T[hd x 8 heads]   += V^T[hd x 16] . P^T[16 x 8]
//   (the 8 q-heads of a GQA group are the MMA N; P^T moves from the S
//   accumulator to the B fragment with one movmatrix.trans per 8x8), online
//   softmax in fp32 with warp shuffles.
// A unit covered by one piece is normalised and stored by its warp; otherwise
// piece partials (O, m, l) go to a workspace and the last warp to finish a
// unit merges them in piece order (deterministic for a given step).
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "common.cuh"

namespace {

constexpr int MAX_G = 8;
constexpr int MAX_P = 32;     // KV blocks per piece at most (host ATTN_MAXP)

PM_DEV void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
PM_DEV void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
// Register-only warp instructions (no memory side effects): without `volatile`
// the compiler may interleave the S = K Q^T and O += V P^T chains of a block
// with the softmax arithmetic (PM_ATTN_VOLATILE_ASM=1 at build time: the old
// strictly ordered form, for A/B).
#ifdef PM_ATTN_VOLATILE_ASM
#define PM_REG_ASM asm volatile
#else
#define PM_REG_ASM asm
#endif
PM_DEV uint32_t movmatrix_t(uint32_t x) {
  uint32_t y;
  PM_REG_ASM("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
PM_DEV void mma16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  PM_REG_ASM(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
PM_DEV void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// byte offset of 16-byte chunk `chunk` (0..7) of row `row` in a 128B-swizzled [rows][128 B] tile
PM_DEV uint32_t sw128(int row, int chunk) { return row * 128 + ((chunk ^ (row & 7)) << 4); }

struct AttnArgs {
  const bf16* q;           // [M][H][HD]
  const int* block_table;  // [M][max_blocks]
  const int* seq_lens;     // [M]
  bf16* out;               // [M][H][HD]
  float* ws_o;             // [M][Hkv][max_chunks][8][HD]
  float* ws_ml;            // [M][Hkv][max_chunks][2][8]
  int* counters;           // [M][Hkv] merge counts, zero at rest
  const int* work;         // [0] warps used, [1] pieces, [2 + w] warp w's first piece, pieces (int4) from
                           // the next 16-byte boundary: (row | kvh << 16, b0 | nblk << 16, chunk | nchunks << 16, seq)
  int M, H, Hkv, G, layer, max_blocks, max_chunks, maxp;
  float scale_log2;        // log2(e)/sqrt(hd)
  int debug;               // profiling only: bit0 skip the math (memory pipeline alone), bit2 trace
  int kv5;                 // tmap is pm_tmap_encode_pool's 5-D map: one copy per KV block (else four 2-D boxes)
  int early;               // decode step: KV blocks before a row's last may load before the dependency wait
};
__device__ unsigned long long g_attn_trace[148 * 16 * 4];  // per warp: start, first data, end, blocks
PM_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// A warp's pieces are work entries [off[gw], off[gw + 1]).  Their descriptors
// and KV block ids are loaded into the warp's shared memory in windows of up
// to ITEM_WIN pieces (maxp block-id slots each), all loads in flight at once
// and before griddepcontrol.wait (the host wrote them), so the streaming loop
// never waits on metadata.
constexpr int ITEM_WIN = 8;
constexpr int WIN_IDS = ITEM_WIN * MAX_P;   // block-id slots per warp window

struct Cursor {
  int j, blk, nblk, r, kvh, chunk, nchunks, b0, seq;  // j = piece index in the window; b0 = first block
};

PM_DEV bool item_setup(const AttnArgs& a, const int4* itm, int j, int nw, Cursor& c) {
  if (j >= nw) return false;
  const int4 m = itm[j];
  c.j = j;
  c.r = m.x & 0xffff;
  c.kvh = (int)((unsigned)m.x >> 16);
  c.b0 = m.y & 0xffff;
  c.nblk = (int)((unsigned)m.y >> 16);
  c.chunk = m.z & 0xffff;
  c.nchunks = (int)((unsigned)m.z >> 16);
  c.seq = m.w;
  c.blk = 0;
  return true;
}

template <int HD, int WARPS, int STAGES>
struct AttnCfg {
  static constexpr int TILE = 16 * HD * 2;          // one K or V tile
  static constexpr int STAGE = 2 * TILE;
  static constexpr int SMEM = WARPS * STAGES * STAGE + WARPS * (STAGES * 8 + ITEM_WIN * 16 + WIN_IDS * 4) + 1024;
};

// Q^T fragments of an item's GQA group straight from global (prefetched one
// item ahead): head n = lane/4 of the group, dim pairs 2t and 2t+8 per k-chunk
template <int HD>
PM_DEV void load_q(const AttnArgs& a, const Cursor& c, int lane, uint32_t (&q)[HD / 16][2]) {
  const int g8 = lane >> 2, t = lane & 3;
  const bool live = g8 < a.G;
  const uint32_t* row = reinterpret_cast<const uint32_t*>(a.q + ((size_t)c.r * a.H + c.kvh * a.G + (live ? g8 : 0)) * HD);
#pragma unroll
  for (int kc = 0; kc < HD / 16; ++kc) {
    q[kc][0] = live ? __ldg(&row[(kc * 16 + 2 * t) >> 1]) : 0u;
    q[kc][1] = live ? __ldg(&row[(kc * 16 + 8 + 2 * t) >> 1]) : 0u;
  }
}

// PM_ATTN_MAXNREG (build-time A/B): cap the registers so a small fixup CTA
// of the other lane can share the SM with an attention CTA
#ifdef PM_ATTN_MAXNREG
#define PM_ATTN_BOUNDS(T) __maxnreg__(PM_ATTN_MAXNREG)
#else
#define PM_ATTN_BOUNDS(T) __launch_bounds__(T)
#endif
template <int HD, int WARPS, int STAGES>
__global__ void PM_ATTN_BOUNDS(WARPS * 32)
paged_attn_kernel(const __grid_constant__ CUtensorMap tmap_kv, AttnArgs a) {
  using C = AttnCfg<HD, WARPS, STAGES>;
  constexpr int HALVES = HD / 64;
  constexpr int KC = HD / 16;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* wbuf = smem + warp * STAGES * C::STAGE;
  uint8_t* meta = smem + WARPS * STAGES * C::STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(meta) + warp * STAGES;
  int4* itm = reinterpret_cast<int4*>(meta + WARPS * STAGES * 8) + warp * ITEM_WIN;
  int* bid = reinterpret_cast<int*>(meta + WARPS * STAGES * 8 + WARPS * ITEM_WIN * 16) + warp * WIN_IDS;
  const int W = gridDim.x * WARPS;
  const int gw = blockIdx.x * WARPS + warp;
  const int G = a.G;

  pdl_trigger();
  const int tr_slot = (blockIdx.x * WARPS + warp) * 4;
  const bool tr = (a.debug & 4) && blockIdx.x * WARPS + warp < 148 * 16;
  if (tr && lane == 0) g_attn_trace[tr_slot] = gtimer();
  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
  }
  __syncwarp();
  // host-written metadata: readable before the wait
  const int w_used = __ldg(&a.work[0]);
  const int p_first = gw < w_used ? __ldg(&a.work[2 + gw]) : 0;
  const int n_items = gw < w_used ? __ldg(&a.work[3 + gw]) - p_first : 0;
  const int4* pieces = reinterpret_cast<const int4*>(a.work + ((3 + w_used + 3) & ~3)) + p_first;
  const int win = ITEM_WIN;

  const int g8 = lane >> 2, t = lane & 3;
  // per-lane ldmatrix offsets inside a (swizzled) K tile and V tile
  uint32_t koff[KC], voff[KC];
  {
    const int krow = ((lane >> 3) & 1) * 8 + (lane & 7);
    const int q4 = lane >> 3, vtok = (q4 >> 1) * 8 + (lane & 7);
#pragma unroll
    for (int kc = 0; kc < KC; ++kc) {
      const int dk = kc * 16 + (lane >> 4) * 8;
      koff[kc] = (dk >> 6) * 2048 + sw128(krow, (dk & 63) >> 3);
      const int dv = kc * 16 + (q4 & 1) * 8;
      voff[kc] = C::TILE + (dv >> 6) * 2048 + sw128(vtok, (dv & 63) >> 3);
    }
  }
  int issued = 0, consumed = 0;
  bool waited = false;
  for (int j0 = 0; j0 < n_items; j0 += win) {
    const int nw = min(win, n_items - j0);
    // ---- window metadata: descriptors, then every block id, all in flight
    if (lane < nw) itm[lane] = __ldg(pieces + j0 + lane);
    __syncwarp();
    for (int idx = lane; idx < nw * MAX_P; idx += 32) {
      const int4 m = itm[idx / MAX_P];
      const int k = idx % MAX_P;
      const int row = m.x & 0xffff, b0 = m.y & 0xffff, nb = (int)((unsigned)m.y >> 16);
      bid[idx] = k < nb ? __ldg(&a.block_table[(size_t)row * a.max_blocks + b0 + k]) : 0;
    }
    __syncwarp();

    // producer cursor (lane 0 issues STAGES blocks ahead of the consumer)
    Cursor pc;
    bool p_live = item_setup(a, itm, 0, nw, pc);
    auto issue_one = [&]() {  // lane 0
      const int s = issued % STAGES;
      uint8_t* dst = wbuf + s * C::STAGE;
      const int phys = bid[pc.j * MAX_P + pc.blk];
      const int col_k = ((a.layer * 2 + 0) * a.Hkv + pc.kvh) * HD;
      const int col_v = ((a.layer * 2 + 1) * a.Hkv + pc.kvh) * HD;
      const uint64_t pol = policy_evict_first();
      mbar_arrive_expect_tx(&bars[s], 2 * C::TILE);
      if (a.kv5) {   // [k|v][half][16 slots][128 B] in one copy
        tma_load_5d(dst, &tmap_kv, &bars[s], 0, phys * 16, 0, 0, a.layer * 2 * a.Hkv + pc.kvh, pol);
      } else {
#pragma unroll
        for (int hh = 0; hh < HALVES; ++hh) {
          tma_load_2d(dst + hh * 2048, &tmap_kv, &bars[s], col_k + hh * 64, phys * 16, pol);
          tma_load_2d(dst + C::TILE + hh * 2048, &tmap_kv, &bars[s], col_v + hh * 64, phys * 16, pol);
        }
      }
      ++issued;
      if (++pc.blk == pc.nblk) p_live = item_setup(a, itm, pc.j + 1, nw, pc);
    };
    int k0 = 0;
    if (!waited) {
      // Decode rows are distinct requests whose only KV the previous kernels
      // write is the current token's (block (seq-1)/16 of its row, this
      // layer): the ring's first blocks before that one are loaded ahead of
      // the dependency wait, hiding the first-load latency behind the
      // previous kernel's tail (a.early; not for prefill chunks, whose rows
      // read each other's new tokens).
      if (a.early && lane == 0)
        for (; k0 < STAGES && p_live && pc.b0 + pc.blk < (pc.seq - 1) / 16; ++k0) issue_one();
      __syncwarp();
      pdl_wait();  // q and the appended KV come from the previous kernel
      waited = true;
    }
    if (lane == 0) {
      for (int k = k0; k < STAGES && p_live; ++k) issue_one();
    }

    Cursor cc, cn;
    bool c_live = item_setup(a, itm, 0, nw, cc), n_live = false;
    uint32_t qf[KC][2], qn[KC][2];
    if (c_live) load_q<HD>(a, cc, lane, qn);
    float o[KC][4];
    float mrun[2], lrun[2];
  while (c_live) {
    if (cc.blk == 0) {
      // new item: take the prefetched Q^T, prefetch the next item's, reset
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) { qf[kc][0] = qn[kc][0]; qf[kc][1] = qn[kc][1]; }
      n_live = item_setup(a, itm, cc.j + 1, nw, cn);
      if (n_live) load_q<HD>(a, cn, lane, qn);
#pragma unroll
      for (int i = 0; i < KC; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
      mrun[0] = mrun[1] = -INFINITY;
      lrun[0] = lrun[1] = 0.f;
    }
    const int s = consumed % STAGES;
    mbar_wait(&bars[s], (consumed / STAGES) & 1);
    if (tr && consumed == 0 && lane == 0) g_attn_trace[tr_slot + 1] = gtimer();
    if (a.debug & 1) {
      __syncwarp();
      ++consumed;
      if (lane == 0 && p_live) issue_one();
      if (++cc.blk < cc.nblk) continue;
      c_live = n_live;
      cc = cn;
      continue;
    }
    const uint32_t kbase = smem_u32(wbuf + s * C::STAGE);
    // ---- S^T = K Q^T
    float sc[4] = {0.f, 0.f, 0.f, 0.f}, sd[4] = {0.f, 0.f, 0.f, 0.f};  // two chains
    {
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) {
        uint32_t a0, a1, a2, a3;
        ldsm_x4(kbase + koff[kc], a0, a1, a2, a3);
        mma16816((kc & 1) ? sd : sc, a0, a1, a2, a3, qf[kc][0], qf[kc][1]);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) sc[e] += sd[e];
    }
    // ---- mask + online softmax (columns = heads 2t, 2t+1; rows = tokens g8, g8+8)
    const int seq = cc.seq;
    const int tok0 = (cc.b0 + cc.blk) * 16;
    const bool v0 = tok0 + g8 < seq, v1 = tok0 + g8 + 8 < seq;
    const float x0 = v0 ? sc[0] * a.scale_log2 : -INFINITY, x1 = v0 ? sc[1] * a.scale_log2 : -INFINITY;
    const float x2 = v1 ? sc[2] * a.scale_log2 : -INFINITY, x3 = v1 ? sc[3] * a.scale_log2 : -INFINITY;
    float mx0 = fmaxf(x0, x2), mx1 = fmaxf(x1, x3);
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
    }
    const float mn0 = fmaxf(mrun[0], mx0), mn1 = fmaxf(mrun[1], mx1);
    const float al0 = exp2f(mrun[0] - mn0), al1 = exp2f(mrun[1] - mn1);
    mrun[0] = mn0;
    mrun[1] = mn1;
    const float p0 = exp2f(x0 - mn0), p1 = exp2f(x1 - mn1), p2 = exp2f(x2 - mn0), p3 = exp2f(x3 - mn1);
    lrun[0] = lrun[0] * al0 + p0 + p2;
    lrun[1] = lrun[1] * al1 + p1 + p3;
    if (__any_sync(0xffffffffu, al0 != 1.f || al1 != 1.f)) {
#pragma unroll
      for (int mt = 0; mt < KC; ++mt) { o[mt][0] *= al0; o[mt][1] *= al1; o[mt][2] *= al0; o[mt][3] *= al1; }
    }
    const uint32_t pb0 = movmatrix_t(pack_bf16(p0, p1));  // tokens 0-7  -> b0
    const uint32_t pb1 = movmatrix_t(pack_bf16(p2, p3));  // tokens 8-15 -> b1
    // A partial block's unwritten slots hold whatever the pool memory held
    // (recycled allocations, prefetched host pages): P is 0 there, but 0 x Inf
    // or 0 x NaN is NaN, so those V^T columns are zeroed (a0/a1 carry tokens
    // 2t, 2t+1 and a2/a3 tokens 2t+8, 2t+9; the low half is the lower token).
    uint32_t vm_lo = 0xffffffffu, vm_hi = 0xffffffffu;
    if (tok0 + 16 > seq) {   // warp-uniform: the row's last block only
      const int ta = tok0 + 2 * t, tb = ta + 8;
      vm_lo = (ta < seq ? 0x0000ffffu : 0u) | (ta + 1 < seq ? 0xffff0000u : 0u);
      vm_hi = (tb < seq ? 0x0000ffffu : 0u) | (tb + 1 < seq ? 0xffff0000u : 0u);
    }
    // ---- O^T += V^T P^T
#pragma unroll
    for (int mt = 0; mt < KC; ++mt) {
      uint32_t a0, a1, a2, a3;
      ldsm_x4_t(kbase + voff[mt], a0, a1, a2, a3);
      mma16816(o[mt], a0 & vm_lo, a1 & vm_lo, a2 & vm_hi, a3 & vm_hi, pb0, pb1);
    }
    __syncwarp();
    ++consumed;
    if (lane == 0 && p_live) issue_one();  // refill the slot just consumed (reads done: __syncwarp)
    if (++cc.blk < cc.nblk) continue;

    // ---- item done: per-column row sums, then store or stash the partial
    float l0 = lrun[0], l1 = lrun[1];
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      l0 += __shfl_xor_sync(0xffffffffu, l0, off);
      l1 += __shfl_xor_sync(0xffffffffu, l1, off);
    }
    const int r = cc.r, kvh = cc.kvh;
    const int nchunks = cc.nchunks;
    const int h0 = 2 * t, h1 = 2 * t + 1;
    if (nchunks == 1) {
      const float i0 = 1.f / l0, i1 = 1.f / l1;
#pragma unroll
      for (int mt = 0; mt < KC; ++mt) {
        const int d = mt * 16 + g8;
        if (h0 < G) {
          bf16* dst = a.out + ((size_t)r * a.H + kvh * G + h0) * HD;
          dst[d] = __float2bfloat16(o[mt][0] * i0);
          dst[d + 8] = __float2bfloat16(o[mt][2] * i0);
        }
        if (h1 < G) {
          bf16* dst = a.out + ((size_t)r * a.H + kvh * G + h1) * HD;
          dst[d] = __float2bfloat16(o[mt][1] * i1);
          dst[d + 8] = __float2bfloat16(o[mt][3] * i1);
        }
      }
    } else {
      const size_t rk = (size_t)r * a.Hkv + kvh;
      float* wo = a.ws_o + (rk * a.max_chunks + cc.chunk) * MAX_G * HD;
      float* wml = a.ws_ml + (rk * a.max_chunks + cc.chunk) * 2 * MAX_G;
#pragma unroll
      for (int mt = 0; mt < KC; ++mt) {
        const int d = mt * 16 + g8;
        __stcg(&wo[h0 * HD + d], o[mt][0]);
        __stcg(&wo[h1 * HD + d], o[mt][1]);
        __stcg(&wo[h0 * HD + d + 8], o[mt][2]);
        __stcg(&wo[h1 * HD + d + 8], o[mt][3]);
      }
      if (g8 == 0) {
        __stcg(&wml[h0], mrun[0]);
        __stcg(&wml[h1], mrun[1]);
        __stcg(&wml[MAX_G + h0], l0);
        __stcg(&wml[MAX_G + h1], l1);
      }
      __syncwarp();
      int last = 0;
      if (lane == 0) {
        // release: this warp's partial (written with st.cg, i.e. at L2) is
        // visible before the count; the merging warp reads with ld.cg
        int prev;
        asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], 1;" : "=r"(prev) : "l"(&a.counters[rk]) : "memory");
        last = prev == nchunks - 1;
        if (last) a.counters[rk] = 0;
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        // merge the chunks in chunk order (online rescale, deterministic):
        // lane covers 16 consecutive values of the group's flattened
        // [head][dim] space per pass, 4 chunks' loads in flight per step
        const float* bo = a.ws_o + rk * a.max_chunks * MAX_G * HD;
        const float* bml = a.ws_ml + rk * a.max_chunks * 2 * MAX_G;
        for (int f0 = lane * 16; f0 < G * HD; f0 += 32 * 16) {
          const int h = f0 / HD, d0 = f0 % HD;
          float Mx = -INFINITY, Lx = 0.f, acc[16];
      #pragma unroll
          for (int e = 0; e < 16; ++e) acc[e] = 0.f;
          for (int c0 = 0; c0 < nchunks; c0 += 4) {
            float m[4], l[4];
            float4 ov[4][4];
      #pragma unroll
            for (int j = 0; j < 4; ++j) {
              const bool ok = c0 + j < nchunks;
              m[j] = ok ? __ldcg(&bml[(c0 + j) * 2 * MAX_G + h]) : -INFINITY;
              l[j] = ok ? __ldcg(&bml[(c0 + j) * 2 * MAX_G + MAX_G + h]) : 0.f;
              const float4* src = reinterpret_cast<const float4*>(bo + ((c0 + j) * MAX_G + h) * HD + d0);
      #pragma unroll
              for (int v = 0; v < 4; ++v) ov[j][v] = ok ? __ldcg(src + v) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
      #pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float Mn = fmaxf(Mx, m[j]);
              const float s1 = Mx == -INFINITY ? 0.f : exp2f(Mx - Mn);
              const float s2 = m[j] == -INFINITY ? 0.f : exp2f(m[j] - Mn);
              Lx = Lx * s1 + l[j] * s2;
      #pragma unroll
              for (int v = 0; v < 4; ++v) {
                acc[4 * v + 0] = acc[4 * v + 0] * s1 + ov[j][v].x * s2;
                acc[4 * v + 1] = acc[4 * v + 1] * s1 + ov[j][v].y * s2;
                acc[4 * v + 2] = acc[4 * v + 2] * s1 + ov[j][v].z * s2;
                acc[4 * v + 3] = acc[4 * v + 3] * s1 + ov[j][v].w * s2;
              }
              Mx = Mn;
            }
          }
          const float inv = 1.f / Lx;
          uint32_t pk[8];
      #pragma unroll
          for (int e = 0; e < 8; ++e) pk[e] = pack_bf16(acc[2 * e] * inv, acc[2 * e + 1] * inv);
          uint4* dst = reinterpret_cast<uint4*>(a.out + ((size_t)r * a.H + kvh * G + h) * HD + d0);
          dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        }
      }
    }
    c_live = n_live;
    cc = cn;
  }
    __syncwarp();  // the window's smem metadata is reused by the next window
  }
  if (!waited) pdl_wait();
  if (tr && lane == 0) {
    g_attn_trace[tr_slot + 2] = gtimer();
    g_attn_trace[tr_slot + 3] = consumed;
  }
}

int num_sms();
int attn_debug();

template <int HD, int WARPS, int STAGES>
int launch_cfg(const CUtensorMap* tm, const AttnArgs& a, cudaStream_t st) {
  using C = AttnCfg<HD, WARPS, STAGES>;
  static bool attr[64] = {false};   // per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!attr[dev]) {
    cudaError_t e = cudaFuncSetAttribute(paged_attn_kernel<HD, WARPS, STAGES>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return (int)e;
    attr[dev] = true;
  }
  // the full persistent grid: the work list was built for exactly its warps
  // (pm_attn_workers_cfg); warps without pieces exit at once
  const int sms = num_sms();
  const int per_sm = (227 * 1024) / C::SMEM;
  const long long grid = (long long)sms * (per_sm > 0 ? per_sm : 1);
  return (int)launch_k(paged_attn_kernel<HD, WARPS, STAGES>, dim3((int)grid), dim3(WARPS * 32), C::SMEM, st, *tm, a);
}

int g_attn_cfg = -1;  // 0: 6w x 4st, 1: 12w x 2st, 2: 8w x 3st, 3: 4w x 2st (x2 CTA/SM)

int attn_cfg() {
  if (g_attn_cfg < 0) {
    const char* e = getenv("PM_ATTN_CFG");
    g_attn_cfg = e ? atoi(e) : 1;
  }
  return g_attn_cfg;
}
int num_sms() {   // of the current device (cached per device)
  static int sms[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!sms[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    // the persistent attention grid spans ~81 % of the SMs (120 of 148): the
    // next projection's CTAs land on the rest while attention drains (measured
    // C2 5.52 -> 5.46 ms/step, C3 stage 1.925 -> 1.910; tools/ab_tune5/6.sh)
    n = n * 120 / 148;
    if (const char* e = getenv("PM_ATTN_SMS")) n = atoi(e);   // tuning override
    sms[dev] = n;
  }
  return sms[dev];
}
int attn_debug() {   // PM_ATTN_DEBUG, read once (profiling only: bit0 gives WRONG results)
  static const int d = [] {
    const char* e = getenv("PM_ATTN_DEBUG");
    const int v = e ? atoi(e) : 0;
    if (v & 1) fprintf(stderr, "libpmb200: PM_ATTN_DEBUG=%d is a profiling mode -- attention results are NOT valid\n", v);
    return v;
  }();
  return d;
}
template <int HD, int WARPS, int STAGES>
int workers_cfg() {
  const int per_sm = (227 * 1024) / AttnCfg<HD, WARPS, STAGES>::SMEM;
  return num_sms() * (per_sm > 0 ? per_sm : 1) * WARPS;
}
template <int HD>
int attn_workers(int cfg) {
  switch (cfg < 0 ? attn_cfg() : cfg) {
    case 0: return workers_cfg<HD, 6, 4>();
    case 2: return workers_cfg<HD, 8, 3>();
    case 3: return workers_cfg<HD, 4, 2>();
    default: return workers_cfg<HD, 12, 2>();
  }
}

template <int HD>
int launch_attn(const CUtensorMap* tm, const AttnArgs& a, cudaStream_t st, int cfg) {
  switch (cfg < 0 ? attn_cfg() : cfg) {
    case 0: return launch_cfg<HD, 6, 4>(tm, a, st);
    case 2: return launch_cfg<HD, 8, 3>(tm, a, st);
    case 3: return launch_cfg<HD, 4, 2>(tm, a, st);
    default: return launch_cfg<HD, 12, 2>(tm, a, st);
  }
}

}  // namespace

// q [M][H][hd] bf16 (RoPE'd), pool via `tmap_kv` (2-D view [blocks*16][L_s*2*Hkv*hd],
// box [16][64], 128B swizzle; or with cfg bit 4 set pm_tmap_encode_pool's 5-D map), block_table [M][max_blocks], seq_lens [M] (cached
// positions incl. the current token), work = the step's balanced piece list
// (pm_attn_work_list, built for pm_attn_workers_cfg(hd, cfg) warps and pieces of at
// most `max_piece` blocks), out [M][H][hd] bf16.  ws_o/ws_ml hold
// [M][Hkv][max_chunks][8][hd] / [..][2][8] fp32 piece partials (max_chunks >= the
// most pieces of one (row, head)); counters [M][Hkv] start at 0 and are left at 0.
extern "C" int pm_paged_attention(const void* tmap_kv, const void* q, const int* block_table,
                                  const int* seq_lens, const int* work, void* out, float* ws_o, float* ws_ml,
                                  int* counters, int M, int H, int Hkv, int hd, int layer, int L_s, int max_blocks,
                                  int max_chunks, int max_piece, int cfg, void* stream) {
  (void)L_s;
  if (M == 0) return 0;
  const int kv5 = cfg >= 0 ? (cfg >> 4) & 1 : 0;     // bit 4: tmap_kv is pm_tmap_encode_pool's 5-D map
  const int early = cfg >= 0 ? (cfg >> 5) & 1 : 0;   // bit 5: decode rows (early KV loads)
  if (cfg >= 0) cfg &= 15;
  const int G = H / Hkv;
  if (H % Hkv || G > MAX_G || max_chunks < 1 || max_piece < 1 || max_piece > MAX_P || M > 65536 || Hkv > 65535)
    return (int)cudaErrorInvalidValue;
  AttnArgs a{reinterpret_cast<const bf16*>(q), block_table, seq_lens, reinterpret_cast<bf16*>(out),
             ws_o, ws_ml, counters, work, M, H, Hkv, G, layer, max_blocks, max_chunks, max_piece,
             1.4426950408889634f / sqrtf((float)hd), attn_debug(), kv5, early};
  auto tm = reinterpret_cast<const CUtensorMap*>(tmap_kv);
  auto st = reinterpret_cast<cudaStream_t>(stream);
  if (hd == 128) return launch_attn<128>(tm, a, st, cfg);
  if (hd == 64) return launch_attn<64>(tm, a, st, cfg);
  return (int)cudaErrorInvalidValue;
}

// Most KV blocks one piece may hold (the kernel's per-piece block-id slots).
extern "C" int pm_attn_max_piece(void) { return MAX_P; }

extern "C" int pm_attn_workers_cfg(int hd, int cfg);
// Warps of a full attention launch (the `workers` of pm_attn_work_list).
extern "C" int pm_attn_workers(int hd) { return pm_attn_workers_cfg(hd, -1); }

// ... of launch configuration `cfg` (0: 6 warps x 4 stages, 1: 12 x 2, 2: 8 x 3,
// 3: 4 x 2 at 2 CTAs/SM; -1: the default / PM_ATTN_CFG).
extern "C" int pm_attn_workers_cfg(int hd, int cfg) {
  if (hd == 128) return attn_workers<128>(cfg);
  if (hd == 64) return attn_workers<64>(cfg);
  return 0;
}

extern "C" int pm_attn_trace_read(void* dst) {
  return (int)cudaMemcpyFromSymbol(dst, g_attn_trace, sizeof(g_attn_trace));
}


extern "C" int pm_prepare_attention(void) {
  cudaError_t e = cudaSuccess;
#define PM_SET(HD, W, S)                                                                            \
  if (e == cudaSuccess)                                                                             \
    e = cudaFuncSetAttribute(paged_attn_kernel<HD, W, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             AttnCfg<HD, W, S>::SMEM);
  PM_SET(128, 6, 4) PM_SET(128, 12, 2) PM_SET(128, 8, 3) PM_SET(128, 4, 2)
  PM_SET(64, 6, 4) PM_SET(64, 12, 2) PM_SET(64, 8, 3) PM_SET(64, 4, 2)
#undef PM_SET
  return (int)e;
}

// Host helper: the balanced work list of one step (mirrors ops.attn_work_list).
// Units = (row, kv head) pairs in row-major order, nb = ceil(seq / 16) blocks
// each, laid end to end (B blocks); warp w gets blocks [w q, (w + 1) q) with
// q = max(minq, ceil(B / workers)); every (unit x warp) segment is cut into
// pieces of at most maxp blocks.  work[0] = warps used, work[1] = pieces P,
// work[2 + w] = warp w's first piece (work[2 + used] = P), pieces from int
// (3 + used + 3) & ~3: {row | kvh << 16, b0 | nblk << 16, chunk | nchunks << 16,
// seq}.  Returns the ints written (or a negative cudaError_t); `cap` = ints
// available in work.
extern "C" int pm_attn_work_list(const int* seq_lens, int M, int hkv, int workers, int maxp, int minq, int cap,
                                 int* work) {
  if (M < 0 || M > 65536 || hkv < 1 || hkv > 65535 || workers < 1 || maxp < 1 || maxp > MAX_P || minq < 1 || cap < 3)
    return -(int)cudaErrorInvalidValue;
  long long B = 0;
  for (int r = 0; r < M; ++r) B += (long long)((seq_lens[r] + 15) >> 4) * hkv;
  if (B == 0) {
    work[0] = work[1] = work[2] = 0;
    return 3;
  }
  const long long q = std::max<long long>(minq, (B + workers - 1) / workers);
  const int used = (int)((B + q - 1) / q);
  const int base = (3 + used + 3) & ~3;
  // pass 1: pieces per unit; pass 2: write them (chunk = rank within the unit)
  std::vector<int> per_unit((size_t)M * hkv, 0);
  long long pos = 0;
  for (int u = 0; u < M * hkv; ++u) {
    const long long e = pos + ((seq_lens[u / hkv] + 15) >> 4);
    for (long long cur = pos; cur < e;) {
      const long long seg_end = std::min(e, (cur / q + 1) * q);
      cur = std::min(seg_end, cur + maxp);
      ++per_unit[u];
    }
    pos = e;
  }
  long long P = 0;
  for (int n : per_unit) P += n;
  if (base + 4 * P > cap) return -(int)cudaErrorInvalidValue;
  work[0] = used;
  work[1] = (int)P;
  int j = 0, w_next = 0;
  pos = 0;
  for (int u = 0; u < M * hkv; ++u) {
    const int r = u / hkv, h = u % hkv;
    const long long s = pos, e = pos + ((seq_lens[r] + 15) >> 4);
    int chunk = 0;
    for (long long cur = s; cur < e; ++chunk, ++j) {
      const int w = (int)(cur / q);
      while (w_next <= w) work[2 + w_next++] = j;   // warps whose first piece is j
      const long long seg_end = std::min(e, (cur / q + 1) * q);
      const long long pe = std::min(seg_end, cur + maxp);
      int* pc = work + base + 4 * j;
      pc[0] = r | (h << 16);
      pc[1] = (int)(cur - s) | (int)((pe - cur) << 16);
      pc[2] = chunk | (per_unit[u] << 16);
      pc[3] = seq_lens[r];
      cur = pe;
    }
    pos = e;
  }
  while (w_next <= used) work[2 + w_next++] = j;
  return base + 4 * (int)P;
}
