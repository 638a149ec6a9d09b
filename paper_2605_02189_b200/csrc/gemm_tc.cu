// Decode projection GEMM on 5th-gen tensor cores (tcgen05 + TMEM), persistent
// stream-K, weights streamed as pre-packed contiguous chunks.
//
// Swap-AB: a 256-row weight unit is the MMA "A" operand and the micro-batch
// tokens are the MMA "N" (16..256), computed by a 2-CTA cluster (one 128-row
// UMMA tile per CTA; each CTA loads half of the activation tile and
// multicasts it to both, so activation traffic stays one tile per unit while
// every CTA's stream-K partial is 128 rows and there are 74 workers):
//     D^T[n_out, tok] = W[n_out, K] . X[tok, K]^T      (fp32 in TMEM)
// At decode batch sizes (M_tok <~ 255) the GEMM is weight-bandwidth bound, so
// the design goal is to keep all 148 SMs streaming weights from HBM at the
// copy rate every cycle of the kernel:
//   * weights are re-packed once at load time into [unit][k-block][2 x 128 x 64]
//     chunks that are already in the UMMA 128B-swizzled K-major smem image, so
//     each pipeline stage is ONE 32 KB contiguous bulk copy (cp.async.bulk);
//   * the activation tile [BN x 64] comes by 2-D TMA from L2 and is shared by
//     both 128-row halves of the unit (halves its SM ingress vs 128-row units);
//   * persistent grid = #SMs, stream-K: the (unit, k-block) sequence is cut
//     into #SMs equal contiguous ranges, so every SM streams the same bytes;
//     a unit split between CTAs leaves per-segment fp32 partials in L2 and a
//     second kernel (launched with PDL) sums them in segment order and applies
//     the epilogue -- fused with the consumer where one follows (residual add
//     + the next RMSNorm; q/k-norm + RoPE + paged KV append).  Boundaries
//     depend only on (N, K, #SMs), never on M_tok, so every token's result is
//     independent of its micro-batch mates (batch-invariant);
//   * warp roles: w0 bulk/TMA producer, w1 MMA issuer (+TMEM owner), w2..w5
//     epilogue; the TMEM accumulator is double-buffered (BN <= 128) so the
//     epilogue of one segment overlaps the mainloop of the next.
// Epilogues: bf16 store, fp32 residual add, SiLU(gate)*up over interleaved
// gate/up rows, fp32 logits + per-unit argmax partials.
#include <stdio.h>
#include <stdlib.h>

#include <type_traits>

#include "common.cuh"

namespace {

constexpr int UNIT_ROWS = 256;             // rows of W per work unit (2 UMMA tiles)
constexpr int BK = 64;                     // 64 bf16 = 128 B = one swizzle atom row
constexpr int SUB_BYTES = 128 * BK * 2;    // one 128x64 UMMA A tile (16 KB)
constexpr int A_BYTES = 2 * SUB_BYTES;     // 32 KB per stage, contiguous in global
constexpr int NUM_THREADS = 288;           // 9 warps: w0/w7 weights, w1 MMA, w2..w5 epilogue, w6/w8 activations
constexpr int EPI_WARP0 = 2;

enum Epilogue : int { EPI_STORE_BF16 = 0, EPI_RESID_ADD_F32 = 1, EPI_SILU_MUL = 2, EPI_LOGITS_ARGMAX = 3 };

struct GemmArgs {
  const uint8_t* w;   // packed weights
  int n_out;          // real output features (rows beyond are zero padding)
  int n_units;        // padded rows / 256
  int kb;             // K / 64
  int m_tok;
  int tok_tiles;
  int epilogue;
  void* out;
  int ld_out;
  float* ws;          // [units*tok_tiles][max_segs][BN][256] fp32 partials of split units
  int max_segs;
  float* amax_val;    // [units * 2 halves][m_cap]
  int* amax_idx;
  int m_cap;
  const uint8_t* pf;  // bytes the NEXT operation streams first: prefetched into L2 during this tail
  unsigned long long pf_bytes;
  unsigned long long pf_span;   // > 0: stripe c of pf_bytes / grid at pf + c * pf_span / grid
  unsigned int pf_ahead;        // bytes per CTA of its own range past the ring pulled into L2 once the ring is full
  long long total;    // units * tok_tiles * kb
  int debug;          // profiling only: bit0 skip epilogue math, bit2 skip partial stores, bit3 trace,
                      // bit4 skip the fixup/post kernel (bits 5/6/7: only reduce / resid-norm / qkv-rope)
  int fix_mode;       // FixMode: how split units are finished
  int post;           // Post: what the fixup applies (plain epilogue / residual + RMSNorm / q-k norm + RoPE)
  int* unit_cnt;      // FIX_FUSED / FIX_POLL: [units] segment arrivals, then [units] readers / finished tasks (zero at rest)
  int ctas_per_worker;   // 2 in pair mode (both halves arrive), else 1
  const int* fix_units;   // fused: the units with fixup tasks (split units; every unit for the QKV post)
  int n_fix;
};

enum Post : int { POST_NONE = 0, POST_RESID_NORM = 1, POST_QKV_ROPE = 2 };
// FIX_POST: the post kernel waits for the whole GEMM grid (griddepcontrol.wait),
// then finishes the split units.  FIX_POLL: the GEMM arrives per unit as its
// partials land (release) and each post-kernel CTA starts as soon as ITS unit
// is complete (acquire), overlapping the GEMM's tail; it still waits for the
// GEMM grid before it exits, so its completion implies the GEMM's (the next
// kernel's griddepcontrol.wait keeps its meaning).  Deadlock-free: the post
// kernel launches only after every GEMM CTA started, and GEMM CTAs never
// wait on it.  FIX_FUSED: the GEMM kernel finishes the units itself.
enum FixMode : int { FIX_POST = 0, FIX_FUSED = 1, FIX_POLL = 2 };

struct NormArgs {
  const bf16* w;      // [d] RMSNorm weight
  bf16* xn;           // [m_cap][d] normalised output (the next GEMM's TMA source)
  int* row_cnt;       // [m_cap] arrival counts, zero at rest
  int n_split;        // units of this launch with > 1 segment (all arrive once per row)
  float eps;
};

struct RopeArgs {
  bf16* q_out;              // [M][H][hd]
  bf16* pool;               // block-first KV pool
  const int* block_table;   // [M][max_blocks]
  const int* positions;     // [M]
  const float* rope;        // [pos][hd] cos | sin
  const bf16* qn_w;         // [hd] or null
  const bf16* kn_w;
  int H, Hkv, hd, layer, L_s, max_blocks;
  float eps;
};



// NH = 128-row halves of the 256-row unit one CTA computes: 2 (a CTA owns the
// unit) or 1 (a 2-CTA cluster owns it; the X tile is split and multicast).
template <int BN, int NH>
struct Cfg {
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE = NH * SUB_BYTES + B_BYTES;
  static constexpr int STAGES = (200 * 1024) / STAGE > 8 ? 8 : (200 * 1024) / STAGE;
  static constexpr int ACC_COLS = NH * BN;                       // one accumulator buffer
  static constexpr int ACC_BUFS = 2 * ACC_COLS <= 512 ? 2 : 1;
  static constexpr int TMEM_COLS = ACC_BUFS * ACC_COLS <= 32 ? 32 : (ACC_BUFS * ACC_COLS <= 64 ? 64 : (ACC_BUFS * ACC_COLS <= 128 ? 128 : (ACC_BUFS * ACC_COLS <= 256 ? 256 : 512)));
  static constexpr int SMEM = STAGES * STAGE + 1024 + 512 + 4 * BN * 8;
};

PM_DEV void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy) : "memory");
}
PM_DEV void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
PM_DEV float silu(float g) { return g / (1.0f + expf(-g)); }

// CTA c owns linear k-block indices [lo(c), lo(c+1)) with lo(c) = floor(c*T/G).
PM_DEV long long range_lo(long long c, long long T, long long G) { return (c * T) / G; }
// the CTA whose range holds index idx
PM_DEV long long owner_of(long long idx, long long T, long long G) { return ((idx + 1) * G + T - 1) / T - 1; }

struct Seg {
  int unit;     // (tok tile, weight unit) linear id
  int kb0, kb1; // k-block range inside the unit
  int seg;      // segment index within the unit
  int nseg;     // number of segments of the unit
};

// i-th segment of this CTA; returns false when past the end
PM_DEV bool get_seg(const GemmArgs& a, long long lo, long long hi, int i, Seg& s, long long G, long long wk) {
  long long pos = lo;
  const long long T = a.total;
  for (int j = 0; j <= i; ++j) {
    if (pos >= hi) return false;
    const long long u = pos / a.kb;
    const long long end = min(hi, (u + 1) * a.kb);
    if (j == i) {
      s.unit = (int)u;
      s.kb0 = (int)(pos - u * a.kb);
      s.kb1 = (int)(end - u * a.kb);
      const long long first = owner_of(u * a.kb, T, G);
      const long long last = owner_of((u + 1) * a.kb - 1, T, G);
      s.seg = (int)(wk - first);
      s.nseg = (int)(last - first + 1);
      return true;
    }
    pos = end;
  }
  return false;
}

// Epilogue of one output feature `n` (a row of D^T) over token columns
// c0..c0+15.  Rows held by one warp are 32 consecutive features, so the
// SiLU(gate)*up partner of row n (interleaved gate/up rows) is lane ^ 1.
template <int NC = 16>
PM_DEV void row_epilogue(const GemmArgs& a, int n, int tok_base, int tok_end, int c0, const float* v, int lane) {
  const bool row_ok = n < a.n_out;
  switch (a.epilogue) {
    case EPI_STORE_BF16: {
      bf16* o = reinterpret_cast<bf16*>(a.out);
#pragma unroll
      for (int j = 0; j < NC; ++j)
        if (c0 + j < tok_end && row_ok) o[(size_t)(tok_base + c0 + j) * a.ld_out + n] = __float2bfloat16(v[j]);
      break;
    }
    case EPI_RESID_ADD_F32: {
      float* o = reinterpret_cast<float*>(a.out);
      float r[NC];
#pragma unroll
      for (int j = 0; j < NC; ++j)
        r[j] = (c0 + j < tok_end && row_ok) ? o[(size_t)(tok_base + c0 + j) * a.ld_out + n] : 0.f;
#pragma unroll
      for (int j = 0; j < NC; ++j)
        if (c0 + j < tok_end && row_ok) o[(size_t)(tok_base + c0 + j) * a.ld_out + n] = r[j] + v[j];
      break;
    }
    case EPI_SILU_MUL: {
      bf16* o = reinterpret_cast<bf16*>(a.out);
#pragma unroll
      for (int j = 0; j < NC; ++j) {
        const float up = __shfl_xor_sync(0xffffffffu, v[j], 1);
        if ((lane & 1) == 0 && c0 + j < tok_end && row_ok)
          o[(size_t)(tok_base + c0 + j) * a.ld_out + (n >> 1)] = __float2bfloat16(silu(v[j]) * up);
      }
      break;
    }
    case EPI_LOGITS_ARGMAX: {
      if (a.out) {
        float* o = reinterpret_cast<float*>(a.out);
#pragma unroll
        for (int j = 0; j < NC; ++j)
          if (c0 + j < tok_end && row_ok) o[(size_t)(tok_base + c0 + j) * a.ld_out + n] = v[j];
      }
      break;
    }
  }
}

// Epilogue of rows n and n+128 over 16 token columns; the residual-add reads
// of both rows are issued before any store (one memory round trip).
PM_DEV void pair_epilogue(const GemmArgs& a, int n, int tok_base, int tok_end, int c0, const float* v0,
                          const float* v1, int lane) {
  if (a.epilogue == EPI_RESID_ADD_F32) {
    float* o = reinterpret_cast<float*>(a.out);
    const bool ok0 = n < a.n_out, ok1 = n + 128 < a.n_out;
    float r0[16], r1[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const size_t row = (size_t)(tok_base + c0 + j) * a.ld_out;
      r0[j] = (c0 + j < tok_end && ok0) ? o[row + n] : 0.f;
      r1[j] = (c0 + j < tok_end && ok1) ? o[row + n + 128] : 0.f;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const size_t row = (size_t)(tok_base + c0 + j) * a.ld_out;
      if (c0 + j < tok_end && ok0) o[row + n] = r0[j] + v0[j];
      if (c0 + j < tok_end && ok1) o[row + n + 128] = r1[j] + v1[j];
    }
    return;
  }
  row_epilogue<16>(a, n, tok_base, tok_end, c0, v0, lane);
  row_epilogue<16>(a, n + 128, tok_base, tok_end, c0, v1, lane);
}

// warp-level (max, lowest index) over the rows a lane holds; lane 0 gets the result
PM_DEV void warp_argmax(float& bv, int& bi) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
}

// profiling trace (PM_GEMM_DEBUG bit3): per CTA globaltimer stamps
__device__ unsigned long long g_gemm_trace[148 * 8];
PM_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PM_TRACE(slot)                                                              \
  do {                                                                              \
    if ((a.debug & 8) && blockIdx.x < 148) g_gemm_trace[blockIdx.x * 8 + (slot)] = gtimer(); \
  } while (0)

// ---------------------------------------------------------------- in-kernel split-K fixup (fused mode)
// Single-lane engines finish the units the stream-K partition splits inside
// the GEMM kernel instead of a post kernel.  Every split segment's CTA stores
// its fp32 partial and arrives on the unit's count (release); once its own
// segments are done, every CTA takes an equal, contiguous share of the fixup
// tasks (a task = one listed unit x FIX_COLS token columns), waits until the
// unit's segments have all arrived (acquire), sums the partials in segment
// order -- the post kernels' order, so results are bit-identical -- and
// applies the epilogue: bf16 store, SiLU*up, logits + argmax tiles, residual
// add (+ the next RMSNorm of every row whose 128-row tiles have all landed,
// by the CTA that lands the last one), or q/k RMSNorm + RoPE + paged KV append
// (QKV lists every unit; whole ones are read back from the stored bf16).
// The waits assume every CTA of the grid is resident: grid <= #SMs at one CTA
// per SM and nothing else on the SMs waits on this grid -- one stream of
// dependent kernels.  Two lanes interleave two persistent grids on the SMs, so
// only single-lane engines launch it (ops.Linear.fused).
constexpr int FIX_COLS = 8;   // token columns per task; 128 threads = 2 columns x 64 threads (4 rows each)

PM_DEV int useg(const GemmArgs& a, int unit, long long G) {
  const long long T = a.total;
  return (int)(owner_of((long long)(unit + 1) * a.kb - 1, T, G) - owner_of((long long)unit * a.kb, T, G) + 1);
}
PM_DEV void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
PM_DEV int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
PM_DEV int atom_add_acq_rel(int* p, int v) {
  int prev;
  asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], %2;" : "=r"(prev) : "l"(p), "r"(v) : "memory");
  return prev;
}

// RMSNorm of one fp32 row by the 128 epilogue threads with rmsnorm_kernel's
// arithmetic and reduction tree (thread tid plays its virtual threads tid and
// tid + 128): bit-identical to the unfused norm.  V4 = ceil(d / 1024).
template <int V4>
PM_DEV void norm_row128(const float* x, const bf16* w, bf16* y, int d, float eps, float* red, int tid) {
  const int n4 = d / 4, lane = tid & 31;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  float4 va[V4], vb[V4];
#pragma unroll
  for (int i = 0; i < V4; ++i) {
    const int ia = tid + i * 256, ib = tid + 128 + i * 256;
    va[i] = ia < n4 ? __ldcg(x4 + ia) : make_float4(0.f, 0.f, 0.f, 0.f);
    vb[i] = ib < n4 ? __ldcg(x4 + ib) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float sa = 0.f, sb = 0.f;
#pragma unroll
  for (int i = 0; i < V4; ++i) {
    sa += va[i].x * va[i].x + va[i].y * va[i].y + va[i].z * va[i].z + va[i].w * va[i].w;
    sb += vb[i].x * vb[i].x + vb[i].y * vb[i].y + vb[i].z * vb[i].z + vb[i].w * vb[i].w;
  }
  sa = warp_sum(sa);
  sb = warp_sum(sb);
  if (lane == 0) { red[tid >> 5] = sa; red[(tid >> 5) + 4] = sb; }
  epi_bar();
  float t = lane < 8 ? red[lane] : 0.f;
  t = warp_sum(t);
  epi_bar();   // red is reused by the next row
  const float r = rsqrtf(t / (float)d + eps);
  const uint2* wr = reinterpret_cast<const uint2*>(w);
  uint2* yr = reinterpret_cast<uint2*>(y);
#pragma unroll
  for (int i = 0; i < V4; ++i) {
    const int ia = tid + i * 256, ib = tid + 128 + i * 256;
    if (ia < n4) {
      const uint2 ww = wr[ia];
      yr[ia] = make_uint2(pack_bf16(va[i].x * r * bf16_lo(ww.x), va[i].y * r * bf16_hi(ww.x)),
                          pack_bf16(va[i].z * r * bf16_lo(ww.y), va[i].w * r * bf16_hi(ww.y)));
    }
    if (ib < n4) {
      const uint2 ww = wr[ib];
      yr[ib] = make_uint2(pack_bf16(vb[i].x * r * bf16_lo(ww.x), vb[i].y * r * bf16_hi(ww.x)),
                          pack_bf16(vb[i].z * r * bf16_lo(ww.y), vb[i].w * r * bf16_hi(ww.y)));
    }
  }
}
PM_DEV void norm_rows128(const GemmArgs& a, const NormArgs& na, const int* rows, int nrows, float* red, int tid) {
  const float* x = reinterpret_cast<const float*>(a.out);
  const int d = a.n_out;
  for (int j = 0; j < nrows; ++j) {
    const int m = rows[j];
    if (d <= 4096) norm_row128<4>(x + (size_t)m * a.ld_out, na.w, na.xn + (size_t)m * d, d, na.eps, red, tid);
    else if (d <= 5120) norm_row128<5>(x + (size_t)m * a.ld_out, na.w, na.xn + (size_t)m * d, d, na.eps, red, tid);
    else norm_row128<8>(x + (size_t)m * a.ld_out, na.w, na.xn + (size_t)m * d, d, na.eps, red, tid);
  }
}

// Residual tiles landed for token columns [c_lo, c_hi) of the tile (`add`
// 128-row tiles each): arrive on each row's count; the arrivals that complete
// a row (2 x n_units tiles) normalise it.  Called by all 128 epilogue threads
// after the tile's residual stores.
PM_DEV void resid_arrive(const GemmArgs& a, const NormArgs& na, int tok_base, int c_lo, int c_hi, int add,
                         int* list, float* red, int tid) {
  const int target = 2 * a.n_units;
  epi_bar();   // every thread's residual stores precede the releases below
  if (tid == 0) list[0] = 0;
  epi_bar();
  for (int c = c_lo + tid; c < c_hi; c += 128) {
    const int row = tok_base + c;
    if (atom_add_acq_rel(na.row_cnt + row, add) + add == target) {
      na.row_cnt[row] = 0;
      list[1 + atomicAdd(&list[0], 1)] = row;
    }
  }
  epi_bar();
  const int n = list[0];
  if (n) norm_rows128(a, na, list + 1, n, red, tid);
  epi_bar();   // list reused by the next call
}

// One column c of the QKV task (64 threads x 4 features; the v4 post kernel's
// lane layout), x = the column's 4 features as the unfused qkv buffer holds them.
template <int HD>
PM_DEV void qkv_rope_col(const GemmArgs& a, const RopeArgs& ra, int wunit, int m, int t, int lane, float (&x)[4]) {
  constexpr int HL = HD / 4;
  const int r = 4 * t, n = wunit * UNIT_ROWS + r;
  const bool row_ok = n < a.n_out;
  const int hg = n / HD, d = n % HD;
  const bool is_q = hg < ra.H, is_k = !is_q && hg < ra.H + ra.Hkv;
  const bf16* nw = is_q ? ra.qn_w : (is_k ? ra.kn_w : nullptr);
  const int pos = ra.positions[m];
  const int fi = (lane & (HL / 2 - 1)) * 4;
  float4 cs = make_float4(0.f, 0.f, 0.f, 0.f), sn = cs;
  if (is_q || is_k) {
    cs = *reinterpret_cast<const float4*>(ra.rope + (size_t)pos * HD + fi);
    sn = *reinterpret_cast<const float4*>(ra.rope + (size_t)pos * HD + HD / 2 + fi);
  }
  float w4[4] = {1.f, 1.f, 1.f, 1.f};
  if (nw) {
    const uint2 ww = *reinterpret_cast<const uint2*>(nw + d);
    w4[0] = bf16_lo(ww.x); w4[1] = bf16_hi(ww.x); w4[2] = bf16_lo(ww.y); w4[3] = bf16_hi(ww.y);
  }
  float ss = 0.f;
#pragma unroll
  for (int e = 0; e < 4; ++e) ss += x[e] * x[e];
#pragma unroll
  for (int o = HL / 2; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (nw) {
    const float rr = rsqrtf(ss / (float)HD + ra.eps);
#pragma unroll
    for (int e = 0; e < 4; ++e) x[e] = x[e] * rr * w4[e];
  }
  const bool lo_half = (lane & (HL - 1)) < HL / 2;
  const float c4[4] = {cs.x, cs.y, cs.z, cs.w}, s4[4] = {sn.x, sn.y, sn.z, sn.w};
  float y[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float partner = __shfl_xor_sync(0xffffffffu, x[e], HL / 2);
    y[e] = lo_half ? (x[e] * c4[e] - partner * s4[e]) : (x[e] * c4[e] + partner * s4[e]);
  }
  if (is_q || is_k) {
#pragma unroll
    for (int e = 0; e < 4; ++e) x[e] = y[e];
  }
  if (!row_ok) return;
  bf16* dst;
  if (is_q) {
    dst = ra.q_out + ((size_t)m * ra.H + hg) * HD + d;
  } else {
    const int kv = is_k ? 0 : 1;
    const int g = is_k ? hg - ra.H : hg - ra.H - ra.Hkv;
    const int slot_off = ra.block_table[(size_t)m * ra.max_blocks + pos / 16];
    const size_t tok_stride = (size_t)ra.L_s * 2 * ra.Hkv * HD;
    dst = ra.pool + ((size_t)slot_off * 16 + (pos & 15)) * tok_stride + (((size_t)ra.layer * 2 + kv) * ra.Hkv + g) * HD + d;
  }
  *reinterpret_cast<uint2*>(dst) = make_uint2(pack_bf16(x[0], x[1]), pack_bf16(x[2], x[3]));
}

// The fixup phase of one CTA (128 epilogue threads).  list/n_list: the
// launch's task units (a.fix_units), G = stream-K workers, NHW = CTAs per
// worker (2 in pair mode: both halves arrive).
template <int BN>
PM_DEV void fused_fixup(const GemmArgs& a, const NormArgs& na, const RopeArgs& ra, long long G, int NHW, int* slist,
                        float* red, int tid) {
  const int lane = tid & 31;
  const int groups = (a.m_tok + FIX_COLS - 1) / FIX_COLS;   // tok_tiles == 1 in fused mode
  const long long T = (long long)a.n_fix * groups;
  const long long t0 = (long long)blockIdx.x * T / gridDim.x, t1 = (long long)(blockIdx.x + 1) * T / gridDim.x;
  const int units = a.n_units;
  for (long long task = t0; task < t1; ++task) {
    const int unit = a.fix_units[task / groups];
    const int c0 = (int)(task % groups) * FIX_COLS;
    const int nseg = useg(a, unit, G);
    if (tid == 0) {
      const int want = nseg * NHW;
      int spins = 0;
      while (ld_acquire(a.unit_cnt + unit) < want) {
        if (++spins > 4) __nanosleep(64);
      }
    }
    epi_bar();
    const int cg = tid >> 6, t = tid & 63, r = 4 * t, n = unit * UNIT_ROWS + r;
    const bool whole_qkv = a.post == POST_QKV_ROPE && nseg == 1;
    // 4 columns per thread (c0 + cg + 2j): every segment's loads in flight, rounds of 4 segments
    float4 v[FIX_COLS / 2];
#pragma unroll
    for (int j = 0; j < FIX_COLS / 2; ++j) v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (!whole_qkv) {
      const float* part = a.ws + (size_t)unit * a.max_segs * BN * UNIT_ROWS + r;
      for (int s0 = 0; s0 < nseg; s0 += 4) {
        float4 y[4][FIX_COLS / 2];
#pragma unroll
        for (int s = 0; s < 4; ++s)
#pragma unroll
          for (int j = 0; j < FIX_COLS / 2; ++j) {
            const int c = c0 + cg + 2 * j;
            y[s][j] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (s0 + s < nseg && c < a.m_tok)
              asm volatile("ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];"
                           : "=f"(y[s][j].x), "=f"(y[s][j].y), "=f"(y[s][j].z), "=f"(y[s][j].w)
                           : "l"(part + ((size_t)(s0 + s) * BN + c) * UNIT_ROWS) : "memory");
          }
#pragma unroll
        for (int j = 0; j < FIX_COLS / 2; ++j)
#pragma unroll
          for (int s = 0; s < 4; ++s)
            if (s0 + s < nseg) { v[j].x += y[s][j].x; v[j].y += y[s][j].y; v[j].z += y[s][j].z; v[j].w += y[s][j].w; }
      }
    }
    const bool full4 = n + 3 < a.n_out;
#pragma unroll
    for (int j = 0; j < FIX_COLS / 2; ++j) {
      const int c = c0 + cg + 2 * j;           // warp-uniform
      const bool col_ok = c < a.m_tok;
      const size_t row = (size_t)c * a.ld_out;
      if (a.post == POST_QKV_ROPE) {
        if (!col_ok) continue;                  // warp-uniform: the shuffles stay convergent
        float x[4];
        if (!whole_qkv) {
          x[0] = __bfloat162float(__float2bfloat16(v[j].x));
          x[1] = __bfloat162float(__float2bfloat16(v[j].y));
          x[2] = __bfloat162float(__float2bfloat16(v[j].z));
          x[3] = __bfloat162float(__float2bfloat16(v[j].w));
        } else {
          uint2 q = make_uint2(0u, 0u);
          if (n < a.n_out) q = __ldcg(reinterpret_cast<const uint2*>(reinterpret_cast<const bf16*>(a.out) + row + n));
          x[0] = bf16_lo(q.x); x[1] = bf16_hi(q.x); x[2] = bf16_lo(q.y); x[3] = bf16_hi(q.y);
        }
        if (ra.hd == 128) qkv_rope_col<128>(a, ra, unit, c, t, lane, x);
        else qkv_rope_col<64>(a, ra, unit, c, t, lane, x);
        continue;
      }
      if (a.post == POST_RESID_NORM || a.epilogue == EPI_RESID_ADD_F32) {
        if (col_ok && n < a.n_out) {
          float* o = reinterpret_cast<float*>(a.out) + row + n;
          float4 rr = __ldcg(reinterpret_cast<const float4*>(o));
          rr.x += v[j].x; rr.y += v[j].y; rr.z += v[j].z; rr.w += v[j].w;
          __stcg(reinterpret_cast<float4*>(o), rr);
        }
        continue;
      }
      switch (a.epilogue) {
        case EPI_STORE_BF16: {
          bf16* o = reinterpret_cast<bf16*>(a.out) + row + n;
          if (col_ok && full4) {
            *reinterpret_cast<uint2*>(o) = make_uint2(pack_bf16(v[j].x, v[j].y), pack_bf16(v[j].z, v[j].w));
          } else if (col_ok) {
            const float e[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
            for (int i = 0; i < 4; ++i)
              if (n + i < a.n_out) o[i] = __float2bfloat16(e[i]);
          }
          break;
        }
        case EPI_SILU_MUL: {
          bf16* o = reinterpret_cast<bf16*>(a.out) + row + (n >> 1);
          if (col_ok && full4) {
            *reinterpret_cast<uint32_t*>(o) = pack_bf16(silu(v[j].x) * v[j].y, silu(v[j].z) * v[j].w);
          } else if (col_ok) {
            if (n + 1 < a.n_out) o[0] = __float2bfloat16(silu(v[j].x) * v[j].y);
            if (n + 3 < a.n_out) o[1] = __float2bfloat16(silu(v[j].z) * v[j].w);
          }
          break;
        }
        case EPI_LOGITS_ARGMAX: {
          if (!col_ok) break;                   // warp-uniform
          if (a.out) {
            float* o = reinterpret_cast<float*>(a.out) + row + n;
            if (full4) {
              *reinterpret_cast<float4*>(o) = v[j];
            } else {
              const float e[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
              for (int i = 0; i < 4; ++i)
                if (n + i < a.n_out) o[i] = e[i];
            }
          }
          const float e[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
          float bv = -INFINITY;
          int bi = n;
          for (int i = 0; i < 4; ++i)
            if (n + i < a.n_out && e[i] > bv) { bv = e[i]; bi = n + i; }
          warp_argmax(bv, bi);
          if (lane == 0) {
            const size_t tile = (size_t)(unit * 2 + (t >> 5)) * a.m_cap + c;
            a.amax_val[tile] = bv;
            a.amax_idx[tile] = bi;
          }
          break;
        }
      }
    }
    if (a.post == POST_RESID_NORM)
      resid_arrive(a, na, 0, c0, min(c0 + FIX_COLS, a.m_tok), 2, slist, red, tid);
    // task done: the last of the unit's tasks resets its counts for the next launch
    epi_bar();
    if (tid == 0 && atom_add_acq_rel(a.unit_cnt + units + unit, 1) + 1 == groups) {
      a.unit_cnt[unit] = 0;
      a.unit_cnt[units + unit] = 0;
    }
  }
}

#ifdef PM_GEMM_MAXNREG   // build-time A/B: leave register room for a co-resident fixup CTA
#define PM_GEMM_BOUNDS __maxnreg__(PM_GEMM_MAXNREG)
#else
#define PM_GEMM_BOUNDS __launch_bounds__(NUM_THREADS, 1)
#endif
template <int BN, int NH, bool FUSED>
__global__ void PM_GEMM_BOUNDS
gemm_stream_kernel(const __grid_constant__ CUtensorMap tmap_x, GemmArgs a, NormArgs na, RopeArgs ra) {
  using C = Cfg<BN, NH>;
  constexpr bool PAIR = NH == 1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;                                     // [STAGES][NH x 128 rows][64] weights
  uint8_t* sb = smem + C::STAGES * NH * SUB_BYTES;        // [STAGES][BN rows][64] X tile
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;      // [2]
  uint64_t* tempty = tfull + 2;             // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* red_val = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE + 512);   // [4][BN]
  int* red_idx = reinterpret_cast<int*>(red_val + 4 * BN);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = PAIR ? cluster_ctarank() : 0;   // which 128-row half (pair mode)
  const long long G = PAIR ? gridDim.x >> 1 : gridDim.x, wk = PAIR ? blockIdx.x >> 1 : blockIdx.x;
  const long long lo = range_lo(wk, a.total, G);
  const long long hi = range_lo(wk + 1, a.total, G);

  pdl_trigger();
  if (threadIdx.x == 0) PM_TRACE(0);
  if (threadIdx.x == 0 && (a.debug & 8) && blockIdx.x < 148) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_gemm_trace[blockIdx.x * 8 + 4] = smid;
  }
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmap_x);
    // full: own producer's arrive + tx (own weights, both X halves);
    // empty: both CTAs' MMA commits (the X multicast writes both CTAs' stage)
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], PAIR ? 2 : 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 4); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();             // partner's barriers initialised before any multicast
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 || warp == 7) {
    if (lane == 0) {
      // ---------------- weight producers: own 16 KB half-chunk (pair) or 32 KB unit chunk,
      // even / odd k-block steps from two threads.  Every copy is issued from its own
      // thread pool: one thread's bulk / TMA copies are served at ~3.6 M ops/s
      // (tools/sm_stream_probe.cu), which capped a CTA near 40-55 GB/s with one
      // producer issuing both operands of every k-block.
      const int par = warp == 0 ? 0 : 1;
      const uint64_t pol_w = policy_evict_first();
      auto wsrc = [&](int wunit, int kb) {
        return a.w + (((size_t)wunit * a.kb + kb) * 2 + crank) * SUB_BYTES;   // NH halves from here
      };
      // Weights do not depend on the previous kernel: they stream before (and
      // regardless of) the dependency wait the activation producer does.
      int it = 0;
      Seg sg;
      for (int i = 0; get_seg(a, lo, hi, i, sg, G, wk); ++i) {
        const int wunit = sg.unit % a.n_units;
        for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++it) {
          if ((it & 1) != par) continue;
          const int s = it % C::STAGES;
          if (it == C::STAGES && a.pf_ahead && a.tok_tiles == 1 && crank == 0) {
            // The ring is full and the MMA is about to wait on the activations (the
            // previous kernel): keep HBM busy by pulling the worker's next bytes into
            // L2.  Linear k-block j of the packed weight is bytes [j, j + 1) x 32 KB
            // (both 128-row halves: in pair mode CTA 0 fetches for both).
            const unsigned long long b0 = (unsigned long long)(lo + C::STAGES) * A_BYTES;
            const unsigned long long b1 =
                min((unsigned long long)hi * A_BYTES, b0 + (unsigned long long)a.pf_ahead * (PAIR ? 2 : 1));
            for (unsigned long long o = b0; o < b1; o += 32768)
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.w + o), "r"((uint32_t)min(32768ull, b1 - o))
                           : "memory");
          }
          // both CTAs released the stage (the X multicast overwrites both)
          if (it >= C::STAGES) mbar_wait(&empty[s], ((it / C::STAGES) - 1) & 1);
          mbar_arrive_expect_tx(&full[s], C::STAGE);
          bulk_load(sa + s * NH * SUB_BYTES, wsrc(wunit, kb), NH * SUB_BYTES, &full[s], pol_w);
        }
      }
      PM_TRACE(1);
      // Every load of this CTA is issued: queue this CTA's share of the next
      // operation's first bytes behind them, so HBM keeps streaming through
      // this kernel's drain/exit and the next kernel's ramp (it reads from L2).
      if (a.pf_bytes && par == 0) {
        pdl_wait();
        const unsigned long long share = ((a.pf_bytes / gridDim.x) + 15) & ~15ull;
        unsigned long long b0 = share * blockIdx.x;
        unsigned long long b1 = min(a.pf_bytes & ~15ull, b0 + share);
        if (a.pf_span) {   // stripes: the first bytes of each next-GEMM worker's range
          b0 = ((a.pf_span / gridDim.x) * blockIdx.x) & ~15ull;
          b1 = min(a.pf_span & ~15ull, b0 + share);
        }
        for (unsigned long long o = b0; o < b1; o += 65536) {
          const uint32_t len = (uint32_t)min(65536ull, b1 - o);
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.pf + o), "r"(len) : "memory");
        }
      }
    }
    __syncwarp();
  } else if (warp == 6 || warp == 8) {
    // ---------------- activation producers (even / odd k-block steps): the X tile (pair: half
    // of it, multicast to both CTAs)
    pdl_wait();
    if (lane == 0) {
      const int par = warp == 6 ? 0 : 1;
      const uint64_t pol_x = policy_evict_last();
      int it = 0;
      Seg sg;
      for (int i = 0; get_seg(a, lo, hi, i, sg, G, wk); ++i) {
        const int ttile = sg.unit / a.n_units;
        for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++it) {
          if ((it & 1) != par) continue;
          const int s = it % C::STAGES;
          if (it >= C::STAGES) mbar_wait(&empty[s], ((it / C::STAGES) - 1) & 1);
          if (PAIR)
            tma_load_2d_mc(sb + s * C::B_BYTES + crank * (BN / 2) * 128, &tmap_x, &full[s], kb * BK,
                           ttile * BN + crank * (BN / 2), (uint16_t)0x3, pol_x);
          else
            tma_load_2d(sb + s * C::B_BYTES, &tmap_x, &full[s], kb * BK, ttile * BN, pol_x);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    pdl_wait();
    if (lane == 0) {
      // ---------------- MMA issuer: D[128 rows of this half][BN tokens]
      constexpr uint32_t idesc = umma_idesc_bf16(128, BN);
      int it = 0;
      Seg sg;
      for (int i = 0; get_seg(a, lo, hi, i, sg, G, wk); ++i) {
        const int b = i % C::ACC_BUFS;
        if (i >= C::ACC_BUFS) mbar_wait(&tempty[b], ((i / C::ACC_BUFS) - 1) & 1);
        tc_fence_after();
        for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++it) {
          const int s = it % C::STAGES;
          mbar_wait(&full[s], (it / C::STAGES) & 1);
          tc_fence_after();
          const uint64_t db = umma_desc_sw128(smem_u32(sb + s * C::B_BYTES));
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            const uint64_t da = umma_desc_sw128(smem_u32(sa + (s * NH + h) * SUB_BYTES));
            const uint32_t acc = tmem + (uint32_t)((b * NH + h) * BN);
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk)
              tc_mma_bf16(acc, da + 2 * kk, db + 2 * kk, idesc, (kb > sg.kb0 || kk > 0) ? 1u : 0u);
          }
          if (PAIR)
            tc_commit_mc(&empty[s], (uint16_t)0x3);   // release the stage in both CTAs
          else
            tc_commit(&empty[s]);
        }
        tc_commit(&tfull[b]);
      }
      PM_TRACE(2);   // last MMA issued
    }
    __syncwarp();
  } else {
    // ---------------- epilogue warps 2..5: TMEM lane quarter q = warp % 4
    pdl_wait();
    const int q = warp & 3;
    const int wq = warp - EPI_WARP0;
    const int rh = (int)crank * 128 + q * 32 + lane;     // row of the 256-row unit
    Seg sg;
    for (int i = 0; get_seg(a, lo, hi, i, sg, G, wk); ++i) {
      const int b = i % C::ACC_BUFS;
      mbar_wait(&tfull[b], (i / C::ACC_BUFS) & 1);
      tc_fence_after();
      const int tok_tile = sg.unit / a.n_units, wunit = sg.unit % a.n_units;
      const int tok_base = tok_tile * BN;
      const int tok_end = min(BN, a.m_tok - tok_base);
      const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * NH * BN);
      const bool whole = sg.nseg == 1;
      const bool argmax = whole && a.epilogue == EPI_LOGITS_ARGMAX;
      if (!(a.debug & 1)) {
        if (whole) {
          const int n0 = wunit * UNIT_ROWS + rh;
          for (int c0 = 0; c0 < BN && c0 < tok_end; c0 += 16) {
            float v[NH][16];
#pragma unroll
            for (int h = 0; h < NH; ++h) tmem_ld16(trow + h * BN + c0, v[h]);
            if (NH == 2)
              pair_epilogue(a, n0, tok_base, tok_end, c0, v[0], v[NH - 1], lane);
            else
              row_epilogue<16>(a, n0, tok_base, tok_end, c0, v[0], lane);
            if (argmax) {
              // the thread's best over its NH rows, then one warp reduction
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                float bv = n0 < a.n_out ? v[0][j] : -INFINITY;
                int bi = n0;
                if (NH == 2 && n0 + 128 < a.n_out && v[NH - 1][j] > bv) { bv = v[NH - 1][j]; bi = n0 + 128; }
                warp_argmax(bv, bi);
                if (lane == 0) { red_val[wq * BN + c0 + j] = bv; red_idx[wq * BN + c0 + j] = bi; }
              }
            }
          }
        } else {
          // partial segment: fp32 [seg][col][256 rows] at L2; the post kernel finishes the unit
          float* dst = a.ws + ((size_t)sg.unit * a.max_segs + sg.seg) * (size_t)BN * UNIT_ROWS + rh;
          for (int c0 = 0; c0 < BN && c0 < tok_end && !(a.debug & 4); c0 += 16) {
            float v[NH][16];
#pragma unroll
            for (int h = 0; h < NH; ++h) tmem_ld16(trow + h * BN + c0, v[h]);
#pragma unroll
            for (int h = 0; h < NH; ++h)
#pragma unroll
              for (int j = 0; j < 16; ++j) __stcg(&dst[(size_t)(c0 + j) * UNIT_ROWS + h * 128], v[h][j]);
          }
        }
      }
      // accumulator drained -> the MMA warp may reuse this TMEM buffer
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
      if ((FUSED || a.fix_mode == FIX_POLL) && !(a.debug & 1)) {
        const int tid = threadIdx.x - EPI_WARP0 * 32;
        if (!whole || a.post == POST_QKV_ROPE) {
          // this CTA's part of the unit is stored (partial, or the whole unit's bf16 for the QKV post)
          epi_bar();
          if (tid == 0) red_release_add(a.unit_cnt + sg.unit, 1);
        } else if (FUSED && a.post == POST_RESID_NORM) {
          resid_arrive(a, na, tok_base, 0, tok_end, NH, red_idx, red_val, tid);
        }
      }
      if (argmax && !(a.debug & 1)) {
        epi_bar();
        // argmax tiles are 128-row halves: this CTA's rows go to tile 2u + crank
        // (pair) or, for a whole-unit CTA, the unit's best to tile 2u and an
        // empty entry to tile 2u + 1
        for (int c = threadIdx.x - EPI_WARP0 * 32; c < tok_end; c += 128) {
          float bv = red_val[c];
          int bi = red_idx[c];
          for (int w = 1; w < 4; ++w)
            if (red_val[w * BN + c] > bv || (red_val[w * BN + c] == bv && red_idx[w * BN + c] < bi)) {
              bv = red_val[w * BN + c];
              bi = red_idx[w * BN + c];
            }
          a.amax_val[(size_t)(wunit * 2 + crank) * a.m_cap + tok_base + c] = bv;
          a.amax_idx[(size_t)(wunit * 2 + crank) * a.m_cap + tok_base + c] = bi;
          if (NH == 2) {
            a.amax_val[(size_t)(wunit * 2 + 1) * a.m_cap + tok_base + c] = -INFINITY;
            a.amax_idx[(size_t)(wunit * 2 + 1) * a.m_cap + tok_base + c] = 0x7fffffff;
          }
        }
        epi_bar();
      }
    }
  }
  if (FUSED && !(a.debug & 1) && warp >= EPI_WARP0 && warp < EPI_WARP0 + 4)
    fused_fixup<BN>(a, na, ra, G, PAIR ? 2 : 1, red_idx, red_val, threadIdx.x - EPI_WARP0 * 32);
  if (threadIdx.x == EPI_WARP0 * 32) PM_TRACE(3);   // epilogue done
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();             // no CTA leaves while its partner may still signal it
  if (warp == 1) tmem_dealloc(tmem, C::TMEM_COLS);
}

// ---------------------------------------------------------------- post kernels
// FIX_POLL: block until every CTA of `unit`'s segments stored its part, then
// count this CTA as a reader; the last of the `readers` CTAs re-arms both counts.
PM_DEV void poll_unit(const GemmArgs& a, int unit, int nseg, int readers) {
  if (threadIdx.x == 0) {
    const int want = nseg * a.ctas_per_worker;
    int spins = 0;
    while (ld_acquire(a.unit_cnt + unit) < want)
      if (++spins > 8) __nanosleep(32);
    const int units = a.n_units * a.tok_tiles;
    if (atom_add_acq_rel(a.unit_cnt + units + unit, 1) + 1 == readers) {
      a.unit_cnt[unit] = 0;
      a.unit_cnt[units + unit] = 0;
    }
  }
  __syncthreads();
}

// One CTA per (unit, RC token columns), thread = row of the 256-row unit.
// RC is chosen per launch so the grid fits in about one wave (launch()).
// segment count of stream-K unit `unit` (mirrors get_seg / pm_gemm_max_segments)
PM_DEV int unit_segments(const GemmArgs& a, int unit, int grid) {
  const long long T = a.total, G = grid;
  const long long first = owner_of((long long)unit * a.kb, T, G);
  const long long last = owner_of((long long)(unit + 1) * a.kb - 1, T, G);
  return (int)(last - first + 1);
}

// v[j] = sum over the unit's segments (in segment order) of row r, column c0+j.
// Rounds of P segments; each round issues all its loads before the
// first add (volatile keeps them in flight).
template <int BN, int RC>
PM_DEV void sum_partials(const GemmArgs& a, int unit, int nseg, int c0, int r, float (&v)[RC]) {
  // segments per round: every decode shape's units fit in one round at RC 4
  constexpr int P = RC <= 4 ? 12 : (RC <= 8 ? 6 : 4);
  const float* part = a.ws + (size_t)unit * a.max_segs * BN * UNIT_ROWS + (size_t)c0 * UNIT_ROWS + r;
#pragma unroll
  for (int j = 0; j < RC; ++j) v[j] = 0.f;
  for (int s0 = 0; s0 < nseg; s0 += P) {
    float t[P][RC];
#pragma unroll
    for (int s = 0; s < P; ++s)
#pragma unroll
      for (int j = 0; j < RC; ++j) {
        float x = 0.f;
        if (s0 + s < nseg)
          asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(x) : "l"(part + ((size_t)(s0 + s) * BN + j) * UNIT_ROWS) : "memory");
        t[s][j] = x;
      }
#pragma unroll
    for (int s = 0; s < P; ++s)
#pragma unroll
      for (int j = 0; j < RC; ++j) asm volatile("" : "+f"(t[s][j]));
#pragma unroll
    for (int j = 0; j < RC; ++j)
#pragma unroll
      for (int s = 0; s < P; ++s) v[j] += t[s][j];
  }
}

// Finishes the units the stream-K partition split across CTAs and applies
// the epilogue.  One CTA per (split unit, RC-column chunk); thread = row.
template <int BN, int RC>
__global__ void __launch_bounds__(256) gemm_reduce_kernel(GemmArgs a, int grid) {
  pdl_trigger();
  pdl_wait();
  const int unit = blockIdx.x, c0 = blockIdx.y * RC;
  const int nseg = unit_segments(a, unit, grid);
  if (nseg == 1) return;
  const int tok_tile = unit / a.n_units, wunit = unit % a.n_units;
  const int tok_base = tok_tile * BN;
  const int tok_end = min(BN, a.m_tok - tok_base);
  if (c0 >= tok_end) return;
  const int r = threadIdx.x, lane = r & 31, warp = r >> 5;
  const int n = wunit * UNIT_ROWS + r;
  float v[RC];
  sum_partials<BN, RC>(a, unit, nseg, c0, r, v);
  row_epilogue<RC>(a, n, tok_base, tok_end, c0, v, lane);
  if (a.epilogue == EPI_LOGITS_ARGMAX) {
    __shared__ float sv[8][RC];
    __shared__ int si[8][RC];
#pragma unroll
    for (int j = 0; j < RC; ++j) {
      float bv = n < a.n_out ? v[j] : -INFINITY;
      int bi = n;
      warp_argmax(bv, bi);
      if (lane == 0) { sv[warp][j] = bv; si[warp][j] = bi; }
    }
    __syncthreads();
    // one argmax tile per 128-row half (warps 0-3 / 4-7), as the GEMM writes them
    if (r < 2 * RC && c0 + (r % RC) < tok_end) {
      const int j = r % RC, h = r / RC;
      float bv = sv[4 * h][j];
      int bi = si[4 * h][j];
      for (int w = 4 * h + 1; w < 4 * h + 4; ++w)
        if (sv[w][j] > bv || (sv[w][j] == bv && si[w][j] < bi)) { bv = sv[w][j]; bi = si[w][j]; }
      a.amax_val[(size_t)(wunit * 2 + h) * a.m_cap + tok_base + c0 + j] = bv;
      a.amax_idx[(size_t)(wunit * 2 + h) * a.m_cap + tok_base + c0 + j] = bi;
    }
  }
}

// Vectorised variant: a thread owns 4 consecutive rows (16-byte partial
// loads, 8/4/16-byte epilogue stores) of RC token columns; 64 threads cover
// the 256-row unit, so one CTA finishes 4 x RC columns.  Same summation order
// as sum_partials (bit-identical).  Needs n_out % 4 == 0 and ld_out % 4 == 0.
template <int BN, int RC>
PM_DEV void reduce_v4_body(const GemmArgs& a, int grid) {
  const int unit = blockIdx.x;
  const int nseg = unit_segments(a, unit, grid);
  if (nseg == 1) return;
  if (a.fix_mode == FIX_POLL) poll_unit(a, unit, nseg, gridDim.y);
  const int tok_tile = unit / a.n_units, wunit = unit % a.n_units;
  const int tok_base = tok_tile * BN;
  const int tok_end = min(BN, a.m_tok - tok_base);
  const int c0 = (blockIdx.y * 4 + (threadIdx.x >> 6)) * RC;   // warp-uniform
  if (c0 >= tok_end) return;
  const int t = threadIdx.x & 63, lane = threadIdx.x & 31;
  const int r = 4 * t, n = wunit * UNIT_ROWS + r;
  const float* part = a.ws + (size_t)unit * a.max_segs * BN * UNIT_ROWS + (size_t)c0 * UNIT_ROWS + r;
  constexpr int P = 4;
  float4 v[RC];
#pragma unroll
  for (int j = 0; j < RC; ++j) v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int s0 = 0; s0 < nseg; s0 += P) {
    float4 x[P][RC];
#pragma unroll
    for (int s = 0; s < P; ++s)
#pragma unroll
      for (int j = 0; j < RC; ++j) {
        float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
        if (s0 + s < nseg)
          asm volatile("ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(y.x), "=f"(y.y), "=f"(y.z), "=f"(y.w)
                       : "l"(part + ((size_t)(s0 + s) * BN + j) * UNIT_ROWS) : "memory");
        x[s][j] = y;
      }
#pragma unroll
    for (int j = 0; j < RC; ++j)
#pragma unroll
      for (int s = 0; s < P; ++s) {
        v[j].x += x[s][j].x;
        v[j].y += x[s][j].y;
        v[j].z += x[s][j].z;
        v[j].w += x[s][j].w;
      }
  }
  const bool full4 = n + 3 < a.n_out;
#pragma unroll
  for (int j = 0; j < RC; ++j) {
    const bool col_ok = c0 + j < tok_end;
    const size_t row = (size_t)(tok_base + c0 + j) * a.ld_out;
    switch (a.epilogue) {
      case EPI_STORE_BF16: {
        bf16* o = reinterpret_cast<bf16*>(a.out) + row + n;
        if (col_ok && full4) {
          *reinterpret_cast<uint2*>(o) = make_uint2(pack_bf16(v[j].x, v[j].y), pack_bf16(v[j].z, v[j].w));
        } else if (col_ok) {
          const float e[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
          for (int i = 0; i < 4; ++i)
            if (n + i < a.n_out) o[i] = __float2bfloat16(e[i]);
        }
        break;
      }
      case EPI_RESID_ADD_F32: {
        float* o = reinterpret_cast<float*>(a.out) + row + n;
        if (col_ok && full4) {
          float4 rr = __ldcg(reinterpret_cast<const float4*>(o));
          rr.x += v[j].x; rr.y += v[j].y; rr.z += v[j].z; rr.w += v[j].w;
          __stcg(reinterpret_cast<float4*>(o), rr);
        } else if (col_ok) {
          const float e[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
          for (int i = 0; i < 4; ++i)
            if (n + i < a.n_out) o[i] = o[i] + e[i];
        }
        break;
      }
      case EPI_SILU_MUL: {   // rows (gate, up, gate, up) -> outputs n/2, n/2 + 1
        bf16* o = reinterpret_cast<bf16*>(a.out) + row + (n >> 1);
        if (col_ok && full4) {
          *reinterpret_cast<uint32_t*>(o) = pack_bf16(silu(v[j].x) * v[j].y, silu(v[j].z) * v[j].w);
        } else if (col_ok) {
          if (n + 1 < a.n_out) o[0] = __float2bfloat16(silu(v[j].x) * v[j].y);
          if (n + 3 < a.n_out) o[1] = __float2bfloat16(silu(v[j].z) * v[j].w);
        }
        break;
      }
      case EPI_LOGITS_ARGMAX: {
        if (a.out && col_ok) {
          float* o = reinterpret_cast<float*>(a.out) + row + n;
          if (full4) {
            *reinterpret_cast<float4*>(o) = v[j];
          } else {
            const float e[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
            for (int i = 0; i < 4; ++i)
              if (n + i < a.n_out) o[i] = e[i];
          }
        }
        // one warp = one 128-row half of the unit (argmax tile 2u + half)
        const float e[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
        float bv = -INFINITY;
        int bi = n;
        for (int i = 0; i < 4; ++i)
          if (n + i < a.n_out && e[i] > bv) { bv = e[i]; bi = n + i; }
        warp_argmax(bv, bi);
        if (lane == 0 && col_ok) {
          const size_t tile = (size_t)(wunit * 2 + (t >> 5)) * a.m_cap + tok_base + c0 + j;
          a.amax_val[tile] = bv;
          a.amax_idx[tile] = bi;
        }
        break;
      }
    }
  }
}

template <int BN, int RC>
__global__ void __launch_bounds__(256) gemm_reduce_v4_kernel(GemmArgs a, int grid) {
  pdl_trigger();
  if (a.fix_mode != FIX_POLL) pdl_wait();
  reduce_v4_body<BN, RC>(a, grid);
  if (a.fix_mode == FIX_POLL) pdl_wait();   // complete only after the GEMM grid
}

// ---------------------------------------------------------------- fused post kernels
// (1) residual GEMM (O / down projection) -> resid += x W^T, then the NEXT
// RMSNorm of every finished row: the CTA that completes a token row last
// (per-row arrival count over the split units) normalises it into `xn`.
// No CTA ever waits, so there is no co-residency assumption.

// RMSNorm of rows x[rows[j]] (fp32, row stride ld) -> y (bf16, row stride
// d) by the whole CTA (256 threads), one row at a time held in registers:
// one pass over L2 per row (d <= 256 * 4 * NORM_V4).  Same reduction tree as
// rmsnorm_kernel, so the result is bit-identical to the unfused norm.
constexpr int NORM_V4 = 8;   // d <= 8192 (instantiated per width: 4, 5, 8 float4 per thread)
template <int V4>
PM_DEV void norm_load_row(const float* x, int d, float4 (&v)[V4]) {
#pragma unroll
  for (int i = 0; i < V4; ++i) {
    const int c = threadIdx.x + i * 256;
    v[i] = c < d / 4 ? __ldcg(reinterpret_cast<const float4*>(x) + c) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// Up to d = 5120 (V4 <= 5) the weight slice is loaded once for all rows and
// row j+1's loads are in flight while row j is reduced, so the rows cost
// about one L2 round trip; wider rows go one at a time (register budget:
// the kernel must keep 4 CTAs per SM to stay one wave).
template <int V4>
PM_DEV void block_rmsnorm_rows(const float* x, int ld, const int* rows, int nrows, const bf16* w, bf16* y, int d,
                               float eps) {
  constexpr bool PIPE = V4 <= 5;
  __shared__ float red[2][8];
  uint2 ww[V4];
  auto load_w = [&]() {
#pragma unroll
    for (int i = 0; i < V4; ++i) {
      const int c = threadIdx.x + i * 256;
      ww[i] = c < d / 4 ? reinterpret_cast<const uint2*>(w)[c] : make_uint2(0u, 0u);
    }
  };
  if (PIPE) load_w();
  float4 v[V4], nx[PIPE ? V4 : 1];
  norm_load_row(x + (size_t)rows[0] * ld, d, v);
#pragma unroll 1
  for (int j = 0; j < nrows; ++j) {
    if constexpr (PIPE) {
      if (j + 1 < nrows) norm_load_row(x + (size_t)rows[j + 1] * ld, d, nx);
    } else {
      if (j > 0) norm_load_row(x + (size_t)rows[j] * ld, d, v);
    }
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < V4; ++i) ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[j & 1][threadIdx.x >> 5] = ss;   // double-buffered: one barrier per row
    __syncthreads();
    float t = (threadIdx.x & 31) < 8 ? red[j & 1][threadIdx.x & 31] : 0.f;
    t = __shfl_sync(0xffffffffu, warp_sum(t), 0);
    const float r = rsqrtf(t / (float)d + eps);
    if (!PIPE) load_w();
#pragma unroll
    for (int i = 0; i < V4; ++i) {
      const int c = threadIdx.x + i * 256;
      if (c < d / 4) {
        uint2 o;
        o.x = pack_bf16(v[i].x * r * bf16_lo(ww[i].x), v[i].y * r * bf16_hi(ww[i].x));
        o.y = pack_bf16(v[i].z * r * bf16_lo(ww[i].y), v[i].w * r * bf16_hi(ww[i].y));
        reinterpret_cast<uint2*>(y + (size_t)rows[j] * d)[c] = o;
      }
    }
    if constexpr (PIPE) {
#pragma unroll
      for (int i = 0; i < V4; ++i) v[i] = nx[i];
    }
  }
}

template <int BN, int RC, int V4>
__global__ void __launch_bounds__(256, 4) gemm_resid_norm_kernel(GemmArgs a, int grid, NormArgs na) {
  pdl_trigger();
  pdl_wait();
  const int unit = blockIdx.x, c0 = blockIdx.y * RC;
  const int nseg = unit_segments(a, unit, grid);
  if (nseg == 1) return;  // whole units were added by the GEMM epilogue and do not count
  const int tok_tile = unit / a.n_units, wunit = unit % a.n_units;
  const int tok_base = tok_tile * BN;
  const int tok_end = min(BN, a.m_tok - tok_base);
  if (c0 >= tok_end) return;
  const int r = threadIdx.x;
  const int n = wunit * UNIT_ROWS + r;
  float* o = reinterpret_cast<float*>(a.out);
  // residual loads issued together with the partial loads (one round trip)
  float res[RC];
#pragma unroll
  for (int j = 0; j < RC; ++j)
    res[j] = (n < a.n_out && c0 + j < tok_end) ? __ldcg(o + (size_t)(tok_base + c0 + j) * a.ld_out + n) : 0.f;
  float v[RC];
  sum_partials<BN, RC>(a, unit, nseg, c0, r, v);
  if (n < a.n_out) {
#pragma unroll
    for (int j = 0; j < RC; ++j)
      if (c0 + j < tok_end) __stcg(o + (size_t)(tok_base + c0 + j) * a.ld_out + n, res[j] + v[j]);
  }
  // arrive on each finished row (the CTA's stores are ordered before the
  // release by the barrier); the last unit to arrive normalises the row
  __shared__ int last_rows[RC];
  __shared__ int n_last;
  if (r == 0) n_last = 0;
  __syncthreads();
  if (r < RC && c0 + r < tok_end) {
    int prev;
    asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], 1;" : "=r"(prev) : "l"(na.row_cnt + tok_base + c0 + r) : "memory");
    if (prev == na.n_split - 1) {
      na.row_cnt[tok_base + c0 + r] = 0;
      last_rows[atomicAdd(&n_last, 1)] = tok_base + c0 + r;
    }
  }
  __syncthreads();
  if (n_last) block_rmsnorm_rows<V4>(o, a.ld_out, last_rows, n_last, na.w, na.xn, a.n_out, na.eps);
}

// Vectorised variant: thread = 4 consecutive rows x 1 token column (16-byte
// partial and residual accesses); a CTA finishes 4 columns, like RC = 4.
template <int BN, int V4>
PM_DEV void resid_norm_v4_body(const GemmArgs& a, int grid, const NormArgs& na) {
  const int unit = blockIdx.x;
  const int nseg = unit_segments(a, unit, grid);
  if (nseg == 1) return;  // whole units were added by the GEMM epilogue and do not count
  if (a.fix_mode == FIX_POLL) poll_unit(a, unit, nseg, gridDim.y);
  const int tok_tile = unit / a.n_units, wunit = unit % a.n_units;
  const int tok_base = tok_tile * BN;
  const int tok_end = min(BN, a.m_tok - tok_base);
  const int cbase = blockIdx.y * 4;
  if (cbase >= tok_end) return;            // CTA-uniform
  const int cg = threadIdx.x >> 6, t = threadIdx.x & 63;
  const int c = cbase + cg;
  const bool col_ok = c < tok_end;
  const int r = 4 * t, n = wunit * UNIT_ROWS + r;
  float* o = reinterpret_cast<float*>(a.out);
  float* orow = o + (size_t)(tok_base + c) * a.ld_out + n;
  const bool ok = col_ok && n < a.n_out;   // n_out % 8 == 0: 4 rows all in or all out
  float4 res = make_float4(0.f, 0.f, 0.f, 0.f);
  if (ok) res = __ldcg(reinterpret_cast<const float4*>(orow));
  if (col_ok) {
    const float* part = a.ws + (size_t)unit * a.max_segs * BN * UNIT_ROWS + (size_t)c * UNIT_ROWS + r;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s0 = 0; s0 < nseg; s0 += 12) {
      float4 y[12];
#pragma unroll
      for (int s = 0; s < 12; ++s) {
        y[s] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (s0 + s < nseg)
          asm volatile("ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(y[s].x), "=f"(y[s].y), "=f"(y[s].z), "=f"(y[s].w)
                       : "l"(part + (size_t)(s0 + s) * BN * UNIT_ROWS) : "memory");
      }
#pragma unroll
      for (int s = 0; s < 12; ++s) { v.x += y[s].x; v.y += y[s].y; v.z += y[s].z; v.w += y[s].w; }
    }
    if (ok) {
      res.x += v.x; res.y += v.y; res.z += v.z; res.w += v.w;
      __stcg(reinterpret_cast<float4*>(orow), res);
    }
  }
  // arrive on each finished row; the last unit to arrive normalises it
  __shared__ int last_rows[4];
  __shared__ int n_last;
  if (threadIdx.x == 0) n_last = 0;
  __syncthreads();
  if (threadIdx.x < 4 && cbase + threadIdx.x < tok_end) {
    const int row = tok_base + cbase + threadIdx.x;
    int prev;
    asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], 1;" : "=r"(prev) : "l"(na.row_cnt + row) : "memory");
    if (prev == na.n_split - 1) {
      na.row_cnt[row] = 0;
      last_rows[atomicAdd(&n_last, 1)] = row;
    }
  }
  __syncthreads();
  // the row's whole units come from the GEMM epilogue: with polling, wait for the GEMM grid first
  if (n_last && a.fix_mode == FIX_POLL) pdl_wait();
  if (n_last) block_rmsnorm_rows<V4>(o, a.ld_out, last_rows, n_last, na.w, na.xn, a.n_out, na.eps);
}
template <int BN, int V4>
__global__ void __launch_bounds__(256, 4) gemm_resid_norm_v4_kernel(GemmArgs a, int grid, NormArgs na) {
  pdl_trigger();
  if (a.fix_mode != FIX_POLL) pdl_wait();
  resid_norm_v4_body<BN, V4>(a, grid, na);
  if (a.fix_mode == FIX_POLL) pdl_wait();   // complete only after the GEMM grid
}

// (2) fused QKV projection -> (Qwen3 q/k RMSNorm) + RoPE + paged KV append.
// One CTA per (unit = 256 output features = 256/hd whole heads, RC tokens);
// thread = feature.  Split units are summed from the partials, whole units
// read the bf16 the GEMM epilogue stored; either way the value is rounded to
// bf16 first (the same rounding the unfused qkv buffer applies).

template <int BN, int RC>
__global__ void __launch_bounds__(256) gemm_qkv_rope_kernel(GemmArgs a, int grid, RopeArgs ra) {
  pdl_trigger();
  const int unit = blockIdx.x, c0 = blockIdx.y * RC;
  const int tok_tile = unit / a.n_units, wunit = unit % a.n_units;
  const int tok_base = tok_tile * BN;
  const int tok_end = min(BN, a.m_tok - tok_base);
  if (c0 >= tok_end) return;
  const int nseg = unit_segments(a, unit, grid);
  const int r = threadIdx.x, lane = r & 31, warp = r >> 5;
  const int n = wunit * UNIT_ROWS + r;
  const bool row_ok = n < a.n_out;
  const int hd = ra.hd, hg = n / hd, d = n % hd, half = hd / 2;   // global head, dim
  const bool is_q = hg < ra.H, is_k = !is_q && hg < ra.H + ra.Hkv;
  const bf16* nw = is_q ? ra.qn_w : (is_k ? ra.kn_w : nullptr);
  // step metadata and tables (written before this step's kernel chain
  // started -- pm_meta_upload is not a dependent launch): load ahead of the wait
  int pos[RC];
  float cs[RC], sn[RC];
  int slot_off[RC];
  const float nwd = nw ? __bfloat162float(nw[d]) : 1.f;
#pragma unroll
  for (int j = 0; j < RC; ++j) pos[j] = c0 + j < tok_end ? ra.positions[tok_base + c0 + j] : 0;
#pragma unroll
  for (int j = 0; j < RC; ++j) {
    const int m = tok_base + c0 + j;
    const float* t = ra.rope + (size_t)pos[j] * hd + d % half;
    cs[j] = t[0];
    sn[j] = t[half];
    slot_off[j] = (!is_q && c0 + j < tok_end) ? ra.block_table[(size_t)m * ra.max_blocks + pos[j] / 16] : 0;
  }
  pdl_wait();
  float v[RC];
  if (nseg > 1) {
    sum_partials<BN, RC>(a, unit, nseg, c0, r, v);
#pragma unroll
    for (int j = 0; j < RC; ++j) v[j] = __bfloat162float(__float2bfloat16(v[j]));
  } else {
    const bf16* q = reinterpret_cast<const bf16*>(a.out);
#pragma unroll
    for (int j = 0; j < RC; ++j)
      v[j] = (row_ok && c0 + j < tok_end) ? __bfloat162float(q[(size_t)(tok_base + c0 + j) * a.ld_out + n]) : 0.f;
  }
  const int wph = hd / 32;                               // warps per head
  __shared__ float sx[RC][UNIT_ROWS];
  __shared__ float sss[RC][8];
  // per-head RMSNorm (q, k) over the head's hd features
  if (nw) {
#pragma unroll
    for (int j = 0; j < RC; ++j) {
      const float ss = warp_sum(v[j] * v[j]);
      if (lane == 0) sss[j][warp] = ss;
    }
  }
  __syncthreads();
  if (nw) {
    const int w0 = (warp / wph) * wph;
#pragma unroll
    for (int j = 0; j < RC; ++j) {
      float ss = 0.f;
      for (int w = 0; w < wph; ++w) ss += sss[j][w0 + w];
      v[j] = v[j] * rsqrtf(ss / (float)hd + ra.eps) * nwd;
    }
  }
  // rotate_half RoPE: partner of feature d is d +- hd/2 in the same head
#pragma unroll
  for (int j = 0; j < RC; ++j) sx[j][r] = v[j];
  __syncthreads();
  if (!row_ok) return;
#pragma unroll
  for (int j = 0; j < RC; ++j) {
    if (c0 + j >= tok_end) continue;
    const int m = tok_base + c0 + j;
    float x = v[j];
    if (is_q || is_k) {
      const float partner = sx[j][d < half ? r + half : r - half];
      x = d < half ? (x * cs[j] - partner * sn[j]) : (x * cs[j] + partner * sn[j]);
    }
    bf16* dst;
    if (is_q) {
      dst = ra.q_out + ((size_t)m * ra.H + hg) * hd + d;
    } else {
      const int kv = is_k ? 0 : 1;
      const int g = is_k ? hg - ra.H : hg - ra.H - ra.Hkv;
      const size_t tok_stride = (size_t)ra.L_s * 2 * ra.Hkv * hd;
      dst = ra.pool + ((size_t)slot_off[j] * 16 + (pos[j] & 15)) * tok_stride +
            (((size_t)ra.layer * 2 + kv) * ra.Hkv + g) * hd + d;
    }
    *dst = __float2bfloat16(x);
  }
}

// Vectorised variant: thread = 4 consecutive features of one head (the
// unfused qkv_rope_append_kernel's lane layout: feature = lane * 4 + e, so
// for hd = 128 the result is bit-identical to the unfused path) x 1 token
// column; 64 threads span the 256-row unit, a CTA finishes 4 columns.  The
// head's norm and the RoPE partner are shuffles within its HL = hd / 4 lanes.
template <int BN, int HD>
PM_DEV void qkv_rope_v4_body(const GemmArgs& a, int grid, const RopeArgs& ra) {
  constexpr int HL = HD / 4;                       // lanes per head (32 or 16)
  const int unit = blockIdx.x;
  const int tok_tile = unit / a.n_units, wunit = unit % a.n_units;
  const int tok_base = tok_tile * BN;
  const int tok_end = min(BN, a.m_tok - tok_base);
  const int nseg = unit_segments(a, unit, grid);
  // every unit arrives (whole ones after storing their bf16): wait for this one only
  if (a.fix_mode == FIX_POLL) poll_unit(a, unit, nseg, gridDim.y);
  const int c = blockIdx.y * 4 + (threadIdx.x >> 6);   // warp-uniform column
  if (c >= tok_end) return;
  const int t = threadIdx.x & 63, lane = threadIdx.x & 31;
  const int r = 4 * t, n = wunit * UNIT_ROWS + r;
  const bool row_ok = n < a.n_out;                 // n_out % hd == 0: a head is all in or all out
  const int hg = n / HD, d = n % HD;               // global head, first dim
  const bool is_q = hg < ra.H, is_k = !is_q && hg < ra.H + ra.Hkv;
  const bf16* nw = is_q ? ra.qn_w : (is_k ? ra.kn_w : nullptr);
  const int m = tok_base + c;
  // step metadata (written before the step's chain; not a dependent launch) ahead of the wait
  const int pos = ra.positions[m];
  const int fi = (lane & (HL / 2 - 1)) * 4;
  float4 cs = make_float4(0.f, 0.f, 0.f, 0.f), sn = cs;
  if (is_q || is_k) {
    cs = *reinterpret_cast<const float4*>(ra.rope + (size_t)pos * HD + fi);
    sn = *reinterpret_cast<const float4*>(ra.rope + (size_t)pos * HD + HD / 2 + fi);
  }
  const int slot_off = is_q ? 0 : ra.block_table[(size_t)m * ra.max_blocks + pos / 16];
  float w4[4] = {1.f, 1.f, 1.f, 1.f};
  if (nw) {
    const uint2 ww = *reinterpret_cast<const uint2*>(nw + d);
    w4[0] = bf16_lo(ww.x); w4[1] = bf16_hi(ww.x); w4[2] = bf16_lo(ww.y); w4[3] = bf16_hi(ww.y);
  }
  if (a.fix_mode != FIX_POLL) pdl_wait();
  float x[4];
  if (nseg > 1) {
    const float* part = a.ws + (size_t)unit * a.max_segs * BN * UNIT_ROWS + (size_t)c * UNIT_ROWS + r;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s0 = 0; s0 < nseg; s0 += 12) {
      float4 y[12];
#pragma unroll
      for (int s = 0; s < 12; ++s) {
        y[s] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (s0 + s < nseg)
          asm volatile("ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(y[s].x), "=f"(y[s].y), "=f"(y[s].z), "=f"(y[s].w)
                       : "l"(part + (size_t)(s0 + s) * BN * UNIT_ROWS) : "memory");
      }
#pragma unroll
      for (int s = 0; s < 12; ++s) { v.x += y[s].x; v.y += y[s].y; v.z += y[s].z; v.w += y[s].w; }
    }
    // the bf16 rounding the stored qkv applies
    x[0] = __bfloat162float(__float2bfloat16(v.x));
    x[1] = __bfloat162float(__float2bfloat16(v.y));
    x[2] = __bfloat162float(__float2bfloat16(v.z));
    x[3] = __bfloat162float(__float2bfloat16(v.w));
  } else {
    uint2 q = make_uint2(0u, 0u);
    if (row_ok) q = __ldcg(reinterpret_cast<const uint2*>(reinterpret_cast<const bf16*>(a.out) + (size_t)m * a.ld_out + n));
    x[0] = bf16_lo(q.x); x[1] = bf16_hi(q.x); x[2] = bf16_lo(q.y); x[3] = bf16_hi(q.y);
  }
  // shuffles run on every lane (a warp may hold heads of different kinds when hd = 64)
  {
    float ss = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) ss += x[e] * x[e];
#pragma unroll
    for (int o = HL / 2; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (nw) {   // Qwen3 per-head RMSNorm (before RoPE)
      const float rr = rsqrtf(ss / (float)HD + ra.eps);
#pragma unroll
      for (int e = 0; e < 4; ++e) x[e] = x[e] * rr * w4[e];
    }
    const bool lo_half = (lane & (HL - 1)) < HL / 2;
    const float c4[4] = {cs.x, cs.y, cs.z, cs.w}, s4[4] = {sn.x, sn.y, sn.z, sn.w};
    float y[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float partner = __shfl_xor_sync(0xffffffffu, x[e], HL / 2);
      y[e] = lo_half ? (x[e] * c4[e] - partner * s4[e]) : (x[e] * c4[e] + partner * s4[e]);
    }
    if (is_q || is_k) {
#pragma unroll
      for (int e = 0; e < 4; ++e) x[e] = y[e];
    }
  }
  if (!row_ok) return;
  bf16* dst;
  if (is_q) {
    dst = ra.q_out + ((size_t)m * ra.H + hg) * HD + d;
  } else {
    const int kv = is_k ? 0 : 1;
    const int g = is_k ? hg - ra.H : hg - ra.H - ra.Hkv;
    const size_t tok_stride = (size_t)ra.L_s * 2 * ra.Hkv * HD;
    dst = ra.pool + ((size_t)slot_off * 16 + (pos & 15)) * tok_stride + (((size_t)ra.layer * 2 + kv) * ra.Hkv + g) * HD + d;
  }
  *reinterpret_cast<uint2*>(dst) = make_uint2(pack_bf16(x[0], x[1]), pack_bf16(x[2], x[3]));
}

template <int BN, int HD>
__global__ void __launch_bounds__(256) gemm_qkv_rope_v4_kernel(GemmArgs a, int grid, RopeArgs ra) {
  pdl_trigger();
  qkv_rope_v4_body<BN, HD>(a, grid, ra);
  if (a.fix_mode == FIX_POLL) pdl_wait();   // complete only after the GEMM grid
}

bool getenv_flag(const char* name) {
  const char* v = getenv(name);
  return v && atoi(v);
}

// Profiling only (bench.py's per-launch roofline): an event recorded right
// after the next GEMM main kernel is launched, before its fixup kernel, so
// the two can be timed separately.  One-shot; null = off.
cudaEvent_t g_split_event = nullptr;

template <int BN, int NH>
int launch(const CUtensorMap* tx, GemmArgs a, int grid, cudaStream_t st, int post, const NormArgs* na,
           const RopeArgs* ra) {
  using C = Cfg<BN, NH>;
  static bool attr_set[64] = {false};   // per device (the attribute is per-context)
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(gemm_stream_kernel<BN, NH, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::SMEM);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(gemm_stream_kernel<BN, NH, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return (int)e;
    attr_set[dev] = true;
  }
  cudaError_t e;
  const NormArgs nav = na ? *na : NormArgs{};
  const RopeArgs rav = ra ? *ra : RopeArgs{};
  auto kern = a.fix_mode == FIX_FUSED ? gemm_stream_kernel<BN, NH, true> : gemm_stream_kernel<BN, NH, false>;
  if (NH == 1)   // grid = 2 x workers: each stream-K worker is a (2,1,1) cluster
    e = launch_k_cluster(kern, dim3(grid), dim3(NUM_THREADS), C::SMEM, st, 2, *tx, a, nav, rav);
  else
    e = launch_k(kern, dim3(grid), dim3(NUM_THREADS), C::SMEM, st, *tx, a, nav, rav);
  if (e != cudaSuccess) return (int)e;
  if (g_split_event) {
    cudaEventRecord(g_split_event, st);
    g_split_event = nullptr;
  }
  if (a.fix_mode == FIX_FUSED) return 0;   // the kernel finished every unit itself
  const int G = NH == 1 ? grid / 2 : grid;
  if ((a.debug & 16) || ((a.debug & 32) && post == POST_NONE) || ((a.debug & 64) && post == POST_RESID_NORM) ||
      ((a.debug & 128) && post == POST_QKV_ROPE))
    return 0;
  if (post == POST_NONE && (a.max_segs <= 1 || (a.debug & 1))) return 0;
  if (post == POST_RESID_NORM && (a.max_segs <= 1 || (a.debug & 1))) return 0;
  // columns per post CTA (4: measured best for the decode shapes)
  const long long units = (long long)a.n_units * a.tok_tiles;
  static int rc_env = -1;   // tuning override PM_POST_RC (2, 4, 8 or 16)
  if (rc_env < 0) rc_env = getenv("PM_POST_RC") ? atoi(getenv("PM_POST_RC")) : 4;
  const int rc = rc_env;
  auto go = [&](auto rcc) -> int {
    constexpr int R = decltype(rcc)::value;
    const dim3 pg((unsigned)units, BN / R);
    static const bool scalar_env = getenv_flag("PM_POST_SCALAR");   // A/B: thread-per-row kernels
    const bool scalar = scalar_env && a.fix_mode != FIX_POLL;         // polling exists in the v4 kernels only
    if (post == POST_QKV_ROPE) {   // every unit (whole ones read the stored bf16)
      if (!scalar && BN >= 4) {
        const dim3 g4((unsigned)units, BN / 4);
        if (ra->hd == 128) return (int)launch_k(gemm_qkv_rope_v4_kernel<BN, 128>, g4, dim3(256), 0, st, a, G, *ra);
        if (ra->hd == 64) return (int)launch_k(gemm_qkv_rope_v4_kernel<BN, 64>, g4, dim3(256), 0, st, a, G, *ra);
      }
      if (a.fix_mode == FIX_POLL) return (int)cudaErrorInvalidValue;
      return (int)launch_k(gemm_qkv_rope_kernel<BN, R>, pg, dim3(256), 0, st, a, G, *ra);
    }
    if (post == POST_RESID_NORM && !scalar && BN >= 4) {
      const dim3 g4((unsigned)units, BN / 4);
      if (a.n_out <= 1024 * 4) return (int)launch_k(gemm_resid_norm_v4_kernel<BN, 4>, g4, dim3(256), 0, st, a, G, *na);
      if (a.n_out <= 1024 * 5) return (int)launch_k(gemm_resid_norm_v4_kernel<BN, 5>, g4, dim3(256), 0, st, a, G, *na);
      return (int)launch_k(gemm_resid_norm_v4_kernel<BN, NORM_V4>, g4, dim3(256), 0, st, a, G, *na);
    }
    if (post == POST_RESID_NORM) {   // norm width: float4s per thread of the d-wide row
      if (a.n_out <= 1024 * 4) return (int)launch_k(gemm_resid_norm_kernel<BN, R, 4>, pg, dim3(256), 0, st, a, G, *na);
      if (a.n_out <= 1024 * 5) return (int)launch_k(gemm_resid_norm_kernel<BN, R, 5>, pg, dim3(256), 0, st, a, G, *na);
      return (int)launch_k(gemm_resid_norm_kernel<BN, R, NORM_V4>, pg, dim3(256), 0, st, a, G, *na);
    }
    if (BN >= 4 * R && a.n_out % 4 == 0 && a.ld_out % 4 == 0 && !scalar)
      return (int)launch_k(gemm_reduce_v4_kernel<BN, R>, dim3((unsigned)units, BN / (4 * R)), dim3(256), 0, st, a, G);
    if (a.fix_mode == FIX_POLL) return (int)cudaErrorInvalidValue;
    return (int)launch_k(gemm_reduce_kernel<BN, R>, pg, dim3(256), 0, st, a, G);
  };
  if (rc == 2) return go(std::integral_constant<int, 2>{});
  if (rc == 8 && BN >= 8) return go(std::integral_constant<int, 8>{});
  if (rc == 16 && BN >= 16) return go(std::integral_constant<int, 16>{});
  return go(std::integral_constant<int, 4>{});
}

template <int BN>
int launch_any(bool pair, const CUtensorMap* tx, GemmArgs a, int grid, cudaStream_t st, int post = POST_NONE,
               const NormArgs* na = nullptr, const RopeArgs* ra = nullptr) {
  return pair ? launch<BN, 1>(tx, a, grid, st, post, na, ra) : launch<BN, 2>(tx, a, grid, st, post, na, ra);
}

}  // namespace

// Profiling only: record `event` (a cudaEvent_t) between the next GEMM's
// main kernel and its fixup kernel.
extern "C" int pm_gemm_split_event(void* event) {
  g_split_event = reinterpret_cast<cudaEvent_t>(event);
  return 0;
}

// Profiling only: copy the last traced launch's stamps ([148][8] u64 ns).
extern "C" int pm_gemm_trace_read(void* dst) {
  return (int)cudaMemcpyFromSymbol(dst, g_gemm_trace, sizeof(g_gemm_trace));
}

// One-time kernel attributes (call before any CUDA-graph capture).
extern "C" int pm_prepare_gemm(void) {
  cudaError_t e = cudaSuccess;
#define PM_SET(BN, NH)                                                                                    \
  if (e == cudaSuccess)                                                                                   \
    e = cudaFuncSetAttribute(gemm_stream_kernel<BN, NH, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             Cfg<BN, NH>::SMEM);                                                          \
  if (e == cudaSuccess)                                                                                   \
    e = cudaFuncSetAttribute(gemm_stream_kernel<BN, NH, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             Cfg<BN, NH>::SMEM);
  PM_SET(16, 1) PM_SET(32, 1) PM_SET(64, 1) PM_SET(128, 1) PM_SET(256, 1)
  PM_SET(16, 2) PM_SET(32, 2) PM_SET(64, 2) PM_SET(128, 2) PM_SET(256, 2)
#undef PM_SET
  return (int)e;
}

// Segments a unit of `kb` k-blocks can be cut into by `grid` stream-K workers
// over `total` k-blocks (host helper for workspace sizing; mirrors owner_of()).
extern "C" int pm_gemm_max_segments(long long total, int kb, int grid) {
  int best = 1;
  for (long long u = 0; u * kb < total; ++u) {
    const long long first = ((u * kb + 1) * grid + total - 1) / total - 1;
    const long long last = (((u + 1) * kb) * grid + total - 1) / total - 1;
    const int n = (int)(last - first + 1);
    if (n > best) best = n;
  }
  return best;
}

// Units of a stream-K launch split across more than one CTA (host helper;
// the per-row arrival count of pm_gemm_resid_rmsnorm).
extern "C" int pm_gemm_split_units(long long total, int kb, int grid) {
  int n = 0;
  for (long long u = 0; u * kb < total; ++u) {
    const long long first = ((u * kb + 1) * grid + total - 1) / total - 1;
    const long long last = (((u + 1) * kb) * grid + total - 1) / total - 1;
    n += last > first;
  }
  return n;
}

// Profiling / tuning switches, read once per process (never per launch).
struct Knobs {
  int debug;            // PM_GEMM_DEBUG: profiling bits (most give WRONG numerics; warned once)
  int grid;             // PM_GEMM_GRID: CTA count override (experiments)
  unsigned pf_ahead;    // PM_PF_AHEAD_KB: L2 run-ahead per CTA (A/B, off)
};
static const Knobs& knobs() {
  static const Knobs k = [] {
    Knobs r{0, 0, 0u};
    if (const char* e = getenv("PM_GEMM_DEBUG")) r.debug = atoi(e);
    if (const char* e = getenv("PM_GEMM_GRID")) r.grid = atoi(e);
    if (const char* e = getenv("PM_PF_AHEAD_KB")) r.pf_ahead = 1024u * (unsigned)atoi(e);
    if (r.debug & ~8)
      fprintf(stderr, "libpmb200: PM_GEMM_DEBUG=%d is a profiling mode -- GEMM results are NOT valid\n", r.debug);
    return r;
  }();
  return k;
}

// The units a stream-K partition splits (ascending) into out[] (room for
// total / kb entries); returns the count (the fused fixup's task units).
extern "C" int pm_gemm_fix_units(long long total, int kb, int grid, int* out) {
  int n = 0;
  for (long long u = 0; u * kb < total; ++u) {
    const long long first = ((u * kb + 1) * grid + total - 1) / total - 1;
    const long long last = (((u + 1) * kb) * grid + total - 1) / total - 1;
    if (last > first) out[n++] = (int)u;
  }
  return n;
}

static int make_args(GemmArgs& a, int& grid, int pair, const void* w_packed, int n_out, int n_units, int k,
                     int m_tok, int bn, int epilogue, void* out, int ld_out, float* ws, int max_segs,
                     float* amax_val, int* amax_idx, int m_cap, const void* prefetch,
                     unsigned long long prefetch_bytes, unsigned long long prefetch_span, int fix_mode,
                     int* fix_counters, const int* fix_units, int n_fix) {
  if (k % BK || m_tok < 1 || m_tok > m_cap || grid < (pair ? 2 : 1)) return (int)cudaErrorInvalidValue;
  const int tok_tiles = (m_tok + bn - 1) / bn;
  a = GemmArgs{reinterpret_cast<const uint8_t*>(w_packed), n_out, n_units, k / BK, m_tok, tok_tiles, epilogue,
               out, ld_out, ws, max_segs, amax_val, amax_idx, m_cap,
               reinterpret_cast<const uint8_t*>(prefetch), prefetch ? prefetch_bytes : 0ull,
               prefetch ? prefetch_span : 0ull, 0u, (long long)n_units * tok_tiles * (k / BK), 0,
               fix_mode, POST_NONE, fix_counters, pair ? 2 : 1, fix_units, n_fix};
  // FIX_FUSED / FIX_POLL: per-unit counters, 16-byte row quads (the v4 epilogues' layout);
  // FIX_FUSED also one token tile and a task list
  if (fix_mode < FIX_POST || fix_mode > FIX_POLL || (fix_mode != FIX_POST && !fix_counters) ||
      (fix_mode != FIX_POST && (n_out % 4 || ld_out % 4)) ||
      (fix_mode == FIX_FUSED && (tok_tiles != 1 || n_fix < 0 || (n_fix && !fix_units))))
    return (int)cudaErrorInvalidValue;
  const Knobs& kn = knobs();
  a.debug = kn.debug;
  if (a.fix_mode == FIX_POLL && (a.debug & (1 | 16 | 32 | 64 | 128))) a.fix_mode = FIX_POST;   // profiling modes
  a.pf_ahead = kn.pf_ahead;
  if (kn.grid > 0) grid = kn.grid;   // tuning experiments only
  // grid = CTAs; a worker is one CTA, or a 2-CTA cluster in pair mode; at
  // most one worker per k-block
  long long workers = pair ? grid / 2 : grid;
  if (workers > a.total) workers = a.total;
  grid = (int)(pair ? 2 * workers : workers);
  return 0;
}

template <typename F>
static int dispatch_bn(int bn, F&& f) {
  switch (bn) {
    case 16: return f(std::integral_constant<int, 16>{});
    case 32: return f(std::integral_constant<int, 32>{});
    case 64: return f(std::integral_constant<int, 64>{});
    case 128: return f(std::integral_constant<int, 128>{});
    case 256: return f(std::integral_constant<int, 256>{});
    default: return (int)cudaErrorInvalidValue;
  }
}

// w_packed: [n_units][kb][2][128][64] bf16, each 128x64 tile in the 128B-
// swizzled K-major UMMA smem image (see ops.pack_weight).
extern "C" int pm_gemm(const void* w_packed, const void* tmap_x, int n_out, int n_units, int k, int m_tok,
                       int bn, int grid, int cta_pair, int epilogue, void* out, int ld_out, float* ws, int max_segs,
                       float* amax_val, int* amax_idx, int m_cap, const void* prefetch,
                       unsigned long long prefetch_bytes, unsigned long long prefetch_span, int fix_mode,
                       int* fix_counters, const int* fix_units, int n_fix, void* stream) {
  GemmArgs a;
  int rc = make_args(a, grid, cta_pair, w_packed, n_out, n_units, k, m_tok, bn, epilogue, out, ld_out, ws, max_segs,
                     amax_val, amax_idx, m_cap, prefetch, prefetch_bytes, prefetch_span, fix_mode, fix_counters,
                     fix_units, n_fix);
  if (rc) return rc;
  auto tx = reinterpret_cast<const CUtensorMap*>(tmap_x);
  auto st = reinterpret_cast<cudaStream_t>(stream);
  return dispatch_bn(bn, [&](auto c) { return launch_any<decltype(c)::value>(cta_pair, tx, a, grid, st); });
}

// Residual projection fused with the next RMSNorm: resid[m][0..n_out) +=
// X W^T (fp32), then xn[m] = RMSNorm(resid[m]) * norm_w (bf16) for every
// row.  row_counters: int[m_cap], zero at rest (left zero).  When the
// stream-K partition splits no unit the norm runs as a separate kernel.
extern "C" int pm_gemm_resid_rmsnorm(const void* w_packed, const void* tmap_x, int n_out, int n_units, int k,
                                     int m_tok, int bn, int grid, int cta_pair, float* resid, float* ws, int max_segs, int m_cap,
                                     const void* prefetch, unsigned long long prefetch_bytes,
                                     unsigned long long prefetch_span, const void* norm_w, void* xn, float eps,
                                     int* row_counters, int split_norm, int fix_mode, int* fix_counters,
                                     const int* fix_units, int n_fix, void* stream) {
  GemmArgs a;
  int rc = make_args(a, grid, cta_pair, w_packed, n_out, n_units, k, m_tok, bn, EPI_RESID_ADD_F32, resid, n_out, ws,
                     max_segs, nullptr, nullptr, m_cap, prefetch, prefetch_bytes, prefetch_span, fix_mode,
                     fix_counters, fix_units, n_fix);
  if (rc) return rc;
  if (n_out % 8 || n_out > 256 * 4 * NORM_V4) return (int)cudaErrorInvalidValue;
  NormArgs na{reinterpret_cast<const bf16*>(norm_w), reinterpret_cast<bf16*>(xn), row_counters,
              pm_gemm_split_units(a.total, a.kb, cta_pair ? grid / 2 : grid), eps};
  auto tx = reinterpret_cast<const CUtensorMap*>(tmap_x);
  auto st = reinterpret_cast<cudaStream_t>(stream);
  // split_norm: finish split units with the plain reduce kernel and normalise in
  // a separate row-parallel kernel (measured better when nothing overlaps the
  // arrival chain: one micro-batch in flight)
  if (a.fix_mode == FIX_FUSED) {   // residual add and the next norm happen inside the GEMM kernel
    a.post = POST_RESID_NORM;
    return dispatch_bn(bn, [&](auto c) {
      return launch_any<decltype(c)::value>(cta_pair, tx, a, grid, st, POST_RESID_NORM, &na);
    });
  }
  const int post = (na.n_split > 0 && !(a.debug & 1) && !split_norm) ? POST_RESID_NORM : POST_NONE;
  rc = dispatch_bn(bn, [&](auto c) { return launch_any<decltype(c)::value>(cta_pair, tx, a, grid, st, post, &na); });
  if (rc || post == POST_RESID_NORM || (a.debug & (16 | 256))) return rc;   // 256: profiling, skip the norm
  return launch_rmsnorm(resid, norm_w, xn, m_tok, n_out, eps, st);
}

// QKV projection fused with (Qwen3 q/k RMSNorm) + rotate-half RoPE + paged KV
// append: q_out[m][H][hd] and the pool slot of positions[m] in layer `layer`
// (same contract as pm_qkv_rope_append).  qkv_out [m_cap][n_out] bf16 is
// scratch for units the partition leaves whole.
extern "C" int pm_gemm_qkv_rope(const void* w_packed, const void* tmap_x, int n_out, int n_units, int k, int m_tok,
                                int bn, int grid, int cta_pair, void* qkv_out, float* ws, int max_segs, int m_cap,
                                const void* prefetch, unsigned long long prefetch_bytes,
                                unsigned long long prefetch_span, int fix_mode, int* fix_counters,
                                const int* fix_units, int n_fix, void* q_out, void* pool,
                                const int* block_table, const int* positions, const float* rope, const void* qn_w,
                                const void* kn_w, int H, int Hkv, int hd, int layer, int L_s, int max_blocks,
                                float eps, void* stream) {
  GemmArgs a;
  int rc = make_args(a, grid, cta_pair, w_packed, n_out, n_units, k, m_tok, bn, EPI_STORE_BF16, qkv_out, n_out, ws,
                     max_segs, nullptr, nullptr, m_cap, prefetch, prefetch_bytes, prefetch_span, fix_mode,
                     fix_counters, fix_units, n_fix);
  a.post = POST_QKV_ROPE;   // every unit arrives in FIX_POLL / FIX_FUSED
  if (rc) return rc;
  if (n_out != (H + 2 * Hkv) * hd || (hd != 64 && hd != 128) || UNIT_ROWS % hd) return (int)cudaErrorInvalidValue;
  RopeArgs ra{reinterpret_cast<bf16*>(q_out), reinterpret_cast<bf16*>(pool), block_table, positions, rope,
              reinterpret_cast<const bf16*>(qn_w), reinterpret_cast<const bf16*>(kn_w), H, Hkv, hd, layer, L_s,
              max_blocks, eps};
  auto tx = reinterpret_cast<const CUtensorMap*>(tmap_x);
  auto st = reinterpret_cast<cudaStream_t>(stream);
  return dispatch_bn(bn, [&](auto c) {
    return launch_any<decltype(c)::value>(cta_pair, tx, a, grid, st, POST_QKV_ROPE, nullptr, &ra);
  });
}
