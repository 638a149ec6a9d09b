// Decode projection GEMM with the split-K reduction and the whole epilogue
// INSIDE one kernel: cluster split-K over tcgen05/TMEM, synchronised with
// cluster-scope mbarriers.
//
// The stream-K kernel (gemm_tc.cu) balances weight bytes over every SM by
// cutting 256-row units into segments anywhere, and finishes split units in a
// second (fixup) kernel -- 145 extra launches per C2 step, ~17 % of the
// serialized step.  Here the cut is confined to a thread-block cluster:
//
//   * a cluster is 2 x S CTAs: rank = half + 2 * slice.  The two CTAs of a
//     slice ("pair") compute the two 128-row halves of a 256-row weight unit
//     over the same K range and share one multicast activation tile (each
//     loads half of it); the S slices split the unit's K range evenly;
//   * cluster c owns units [c*U/NC, (c+1)*U/NC); all its CTAs walk them in
//     order, so every CTA streams ~U/NC * kb/S weight chunks -- the planner
//     (ops.cl_plan) picks (S, NC) so that NC * 2S CTAs cover the SMs evenly;
//   * weights and activations have separate rings: a weight producer warp keeps
//     WS x 16 KB of weights in flight from HBM (it starts before the
//     programmatic-launch dependency wait -- weights never depend on the
//     previous kernel), an activation producer warp keeps XS activation tiles
//     in flight from L2.  Per-SM streaming rate is bytes-in-flight / latency,
//     so shared memory goes to the weight ring;
//   * after a unit's last MMA each CTA writes its fp32 partial (128 rows x BN
//     token columns, from TMEM) to an L2 scratch slot and signals the S CTAs of
//     its half (remote mbarrier arrive, release.cluster).  Every CTA owns BN/S
//     token columns: it sums the S partials of those columns in slice order
//     (deterministic, batch-invariant) and applies the epilogue.  No second
//     kernel; the partials never leave L2;
//   * the TMEM accumulator is double-buffered, so a unit's reduction and
//     epilogue overlap the next unit's MMAs while the producers stream on.
//
// Epilogues (one per projection kind, all fused):
//   STORE     bf16 store
//   SILU      SiLU(gate) * up over interleaved gate/up rows       (gate/up)
//   RESID     resid += acc (fp32); optionally xn = bf16(resid * w_next_norm)
//             and the per-(128-row tile, token) sum of squares of resid  (O, down)
//   LOGITS    fp32 logits (optional) + per-128-row argmax partials      (lm_head)
//   QKV_ROPE  bf16 round, Qwen3 per-head q/k RMSNorm, rotate-half RoPE, q out
//             and the paged KV append                                    (QKV)
// RMSNorm folding: RESID writes xn = bf16(x * w) UNNORMALISED plus sum-of-
// squares partials; the consumer GEMM (gate/up, the next QKV, lm_head) scales
// each token column of its accumulator by rsqrt(mean(x^2) + eps) -- RMSNorm is
// a per-token scale, so W (x*w/rms) = (W (x*w)) / rms.  The next norm costs
// no kernel and no extra pass.
#include <type_traits>

#include "common.cuh"

namespace {

constexpr int CL_THREADS = 288;            // w0/w7 weight producers, w1 MMA, w2..w5 epilogue, w6/w8 X producers
constexpr int CL_BK = 64;
constexpr int CL_WBYTES = 128 * CL_BK * 2; // one 128x64 bf16 weight tile (16 KB)
constexpr int CL_SMEM_MAX = 232448;        // opt-in dynamic smem per CTA (227 KB)

enum ClEpi : int { CL_STORE = 0, CL_SILU = 1, CL_RESID = 2, CL_LOGITS = 3, CL_QKV_ROPE = 4 };

struct ClRope {
  bf16* q_out;              // [m_cap][H][hd]
  bf16* pool;               // block-first KV pool [block][16][L_s][2][Hkv][hd]
  const int* block_table;   // [m_cap][max_blocks]
  const int* positions;     // [m_cap]
  const float* rope;        // [pos][hd]: cos | sin halves
  const bf16* qn_w;         // [hd] or null (Qwen3 q/k norm)
  const bf16* kn_w;
  int H, Hkv, hd, layer, L_s, max_blocks;
};

struct ClArgs {
  const uint8_t* w;         // packed weights [unit][kb][2][128][64] (ops.pack_weight)
  int n_out, n_units, kb, m_tok, m_cap;
  int S, n_clusters;        // slices per unit, clusters
  int epilogue;
  void* out;                // STORE/SILU: bf16 [m][ld_out]; LOGITS: fp32 [m][ld_out] or null
  int ld_out;
  // folded RMSNorm of the GEMM INPUT: rs[m] = rsqrt(sum_t ssq_in[t][m] / d_in + eps); null = none
  const float* ssq_in;
  int n_ht_in;
  float inv_d_in, eps;
  // RESID
  float* resid;             // [m_cap][n_out] fp32
  const bf16* norm_w;       // [n_out] next RMSNorm weight, or null (no xn / ssq)
  bf16* xn;                 // [m_cap][n_out]
  float* ssq_out;           // [n_out / 128][m_cap]
  float* part;              // [grid][BN][128] fp32 split-K partials (L2 scratch)
  int trace;                // profiling only: per-CTA %globaltimer stamps into g_cl_trace
  int debug;                // profiling only (PM_CL_DEBUG): bit0 no activation loads, bit1 no multicast,
                            // bit2 no MMA (wrong numerics)
  // LOGITS
  float* amax_val;          // [n_units * 2][m_cap]
  int* amax_idx;
  ClRope ra;
};

template <int BN>
struct ClCfg {
  static constexpr int X_BYTES = BN * CL_BK * 2;                  // one [BN x 64] activation tile
  static constexpr int XS = 4;                                    // activation ring (from L2)
  static constexpr int WAVAIL = CL_SMEM_MAX - 1024 - 1024 - XS * X_BYTES;
  static constexpr int WS = WAVAIL / CL_WBYTES > 14 ? 14 : WAVAIL / CL_WBYTES;   // weight ring (from HBM)
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;     // double-buffered accumulator
  static constexpr int SMEM = WS * CL_WBYTES + XS * X_BYTES + 1024 + 1024;
};

PM_DEV void cl_bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy) : "memory");
}
PM_DEV uint32_t cl_mapa(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
PM_DEV void cl_arrive_remote(uint64_t* bar, uint32_t rank) {
  const uint32_t ra = cl_mapa(smem_u32(bar), rank);
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
PM_DEV void cl_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr), "r"(parity) : "memory");
}
PM_DEV float cl_silu(float g) { return g / (1.0f + expf(-g)); }

PM_DEV void cl_warp_argmax(float& bv, int& bi) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
}

// Epilogue of one token column m for the 4 consecutive rows n..n+3 a lane
// owns (n = unit*256 + half*128 + 4*lane).  `v` is the slice-summed fp32
// accumulator.  Every lane of the warp calls it (warp reductions).
template <int HD>
PM_DEV void cl_qkv_rope(const ClArgs& a, int m, int n, float (&x)[4], int lane) {
  constexpr int HL = HD / 4;                        // lanes per head (32 or 16)
  const ClRope& ra = a.ra;
  const int hg = n / HD, d = n % HD;                // global head, first dim
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
  if (nw) {   // Qwen3 per-head RMSNorm (before RoPE)
    const float rr = rsqrtf(ss / (float)HD + a.eps);
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
  if (n >= a.n_out) return;
  bf16* dst;
  if (is_q) {
    dst = ra.q_out + ((size_t)m * ra.H + hg) * HD + d;
  } else {
    const int kv = is_k ? 0 : 1;
    const int g = is_k ? hg - ra.H : hg - ra.H - ra.Hkv;
    const int blk = ra.block_table[(size_t)m * ra.max_blocks + pos / 16];
    const size_t tok_stride = (size_t)ra.L_s * 2 * ra.Hkv * HD;
    dst = ra.pool + ((size_t)blk * 16 + (pos & 15)) * tok_stride + (((size_t)ra.layer * 2 + kv) * ra.Hkv + g) * HD + d;
  }
  *reinterpret_cast<uint2*>(dst) = make_uint2(pack_bf16(x[0], x[1]), pack_bf16(x[2], x[3]));
}

PM_DEV void cl_epilogue(const ClArgs& a, int m, int unit, int half, float4 acc, int lane) {
  const int n = unit * 256 + half * 128 + 4 * lane;
  const bool ok = n < a.n_out;   // n_out % 4 == 0: a lane's 4 rows are all in or all out
  float v[4] = {acc.x, acc.y, acc.z, acc.w};
  if (a.ssq_in) {
    // rs = rsqrt(mean(x^2) + eps) of the input row m (folded RMSNorm); the
    // lanes sum the tile partials in a fixed order
    float s = 0.f;
    for (int t = lane; t < a.n_ht_in; t += 32) s += a.ssq_in[(size_t)t * a.m_cap + m];
    s = warp_sum(s);
    const float rs = rsqrtf(s * a.inv_d_in + a.eps);
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] *= rs;
  }
  switch (a.epilogue) {
    case CL_STORE: {
      if (ok) {
        bf16* o = reinterpret_cast<bf16*>(a.out) + (size_t)m * a.ld_out + n;
        *reinterpret_cast<uint2*>(o) = make_uint2(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]));
      }
      break;
    }
    case CL_SILU: {   // rows (gate_i, up_i, gate_i+1, up_i+1) -> outputs n/2, n/2 + 1
      if (ok) {
        bf16* o = reinterpret_cast<bf16*>(a.out) + (size_t)m * a.ld_out + (n >> 1);
        *reinterpret_cast<uint32_t*>(o) = pack_bf16(cl_silu(v[0]) * v[1], cl_silu(v[2]) * v[3]);
      }
      break;
    }
    case CL_RESID: {
      float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
      float* rrow = a.resid + (size_t)m * a.n_out + n;
      if (ok) {
        x = __ldcg(reinterpret_cast<const float4*>(rrow));
        x.x += v[0]; x.y += v[1]; x.z += v[2]; x.w += v[3];
        __stcg(reinterpret_cast<float4*>(rrow), x);
      }
      if (a.norm_w) {
        if (ok) {
          const uint2 ww = *reinterpret_cast<const uint2*>(a.norm_w + n);
          *reinterpret_cast<uint2*>(a.xn + (size_t)m * a.n_out + n) =
              make_uint2(pack_bf16(x.x * bf16_lo(ww.x), x.y * bf16_hi(ww.x)),
                         pack_bf16(x.z * bf16_lo(ww.y), x.w * bf16_hi(ww.y)));
        }
        const float ss = warp_sum(x.x * x.x + x.y * x.y + x.z * x.z + x.w * x.w);
        if (lane == 0 && unit * 256 + half * 128 < a.n_out)
          a.ssq_out[(size_t)(unit * 2 + half) * a.m_cap + m] = ss;
      }
      break;
    }
    case CL_LOGITS: {
      if (ok && a.out)
        __stcg(reinterpret_cast<float4*>(reinterpret_cast<float*>(a.out) + (size_t)m * a.ld_out + n),
               make_float4(v[0], v[1], v[2], v[3]));
      float bv = -INFINITY;
      int bi = n;
      for (int e = 0; e < 4; ++e)
        if (n + e < a.n_out && v[e] > bv) { bv = v[e]; bi = n + e; }
      cl_warp_argmax(bv, bi);
      if (lane == 0) {
        a.amax_val[(size_t)(unit * 2 + half) * a.m_cap + m] = bv;
        a.amax_idx[(size_t)(unit * 2 + half) * a.m_cap + m] = bi;
      }
      break;
    }
    case CL_QKV_ROPE: {
      // the bf16 rounding the qkv projection's output applies
#pragma unroll
      for (int e = 0; e < 4; ++e) v[e] = __bfloat162float(__float2bfloat16(v[e]));
      if (a.ra.hd == 128)
        cl_qkv_rope<128>(a, m, n, v, lane);
      else
        cl_qkv_rope<64>(a, m, n, v, lane);
      break;
    }
  }
}

// profiling only (PM_CL_TRACE=1, read once): per-CTA globaltimer stamps of the
// last launch: 0 start, 1 after setup, 2 first weight chunk landed (MMA), 3 last
// MMA issued, 4 first partial written, 5 partials of the last unit ready,
// 6 epilogue done, 7 exit
__device__ unsigned long long g_cl_trace[160 * 8];
PM_DEV unsigned long long cl_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define CL_TRACE(slot) \
  do {                 \
    if (a.trace && blockIdx.x < 160) g_cl_trace[blockIdx.x * 8 + (slot)] = cl_gtimer(); \
  } while (0)

template <int BN>
__global__ void __launch_bounds__(CL_THREADS, 1) gemm_cluster_kernel(const __grid_constant__ CUtensorMap tmap_x,
                                                                     ClArgs a) {
  using C = ClCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sw = smem;                                     // [WS][128][64] weight ring
  uint8_t* sx = smem + C::WS * CL_WBYTES;                 // [XS][BN][64] activation ring
  uint64_t* wfull = reinterpret_cast<uint64_t*>(sx + C::XS * C::X_BYTES);
  uint64_t* wempty = wfull + C::WS;
  uint64_t* xfull = wempty + C::WS;
  uint64_t* xempty = xfull + C::XS;
  uint64_t* tfull = xempty + C::XS;         // [2]
  uint64_t* tempty = tfull + 2;             // [2]
  uint64_t* red_full = tempty + 2;          // all S partials of my half are in L2 (4S arrivals)
  uint64_t* red_free = red_full + 1;        // every reader is done with my partial (4S arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(red_free + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int S = a.S, CS = 2 * S;
  const int half = (int)(rank & 1), slice = (int)(rank >> 1);
  const int cl = blockIdx.x / CS;
  const int u0 = (int)(((long long)cl * a.n_units) / a.n_clusters);
  const int u1 = (int)(((long long)(cl + 1) * a.n_units) / a.n_clusters);
  const int k0 = (slice * a.kb) / S, k1 = ((slice + 1) * a.kb) / S;
  const int nk = k1 - k0;
  const long long total = (long long)(u1 - u0) * nk;
  const uint16_t pair_mask = (uint16_t)(3u << (2 * slice));

  pdl_trigger();
  if (threadIdx.x == 0) CL_TRACE(0);
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmap_x);
    for (int s = 0; s < C::WS; ++s) { mbar_init(&wfull[s], 1); mbar_init(&wempty[s], 1); }
    for (int s = 0; s < C::XS; ++s) { mbar_init(&xfull[s], 1); mbar_init(&xempty[s], 2); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 4); }
    mbar_init(red_full, 4 * S);
    mbar_init(red_free, 4 * S);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  cluster_sync();                           // every peer's barriers initialised before any remote signal
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) CL_TRACE(1);

  if (warp == 0 || warp == 7) {
    if (lane == 0) {
      // ---------------- weight producers: this half's 16 KB chunks, WS deep, issued by two
      // threads (even / odd chunks): one thread's bulk copies are served at ~3.6 M ops/s
      // (tools/sm_stream_probe.cu).  Weights do not depend on the previous kernel, so the
      // ring fills before the dependency wait.
      const uint64_t pol_w = policy_evict_first();
      for (long long it = warp == 0 ? 0 : 1; it < total; it += 2) {
        const int s = (int)(it % C::WS);
        if (it >= C::WS) mbar_wait(&wempty[s], (uint32_t)(((it / C::WS) - 1) & 1));
        mbar_arrive_expect_tx(&wfull[s], CL_WBYTES);
        const int u = u0 + (int)(it / nk), kb = k0 + (int)(it % nk);
        cl_bulk_load(sw + s * CL_WBYTES, a.w + (((size_t)u * a.kb + kb) * 2 + half) * CL_WBYTES, CL_WBYTES,
                     &wfull[s], pol_w);
      }
    }
    __syncwarp();
  } else if (warp == 6 || warp == 8) {
    // ---------------- activation producers (even / odd steps): half of each [BN x 64] tile,
    // multicast to the pair
    pdl_wait();
    if (lane == 0) {
      const uint64_t pol_x = policy_evict_last();
      for (long long it = warp == 6 ? 0 : 1; it < total; it += 2) {
        const int s = (int)(it % C::XS);
        // both CTAs of the pair released the stage (the multicast writes both)
        if (it >= C::XS) mbar_wait(&xempty[s], (uint32_t)(((it / C::XS) - 1) & 1));
        const int kb = k0 + (int)(it % nk);
        if (a.debug & 1) {
          mbar_arrive(&xfull[s]);
        } else if (a.debug & 2) {
          mbar_arrive_expect_tx(&xfull[s], C::X_BYTES);
          tma_load_2d(sx + s * C::X_BYTES, &tmap_x, &xfull[s], kb * CL_BK, 0, pol_x);
          tma_load_2d(sx + s * C::X_BYTES + (BN / 2) * 128, &tmap_x, &xfull[s], kb * CL_BK, BN / 2, pol_x);
        } else {
          mbar_arrive_expect_tx(&xfull[s], C::X_BYTES);
          tma_load_2d_mc(sx + s * C::X_BYTES + half * (BN / 2) * 128, &tmap_x, &xfull[s], kb * CL_BK,
                         half * (BN / 2), pair_mask, pol_x);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    pdl_wait();
    if (lane == 0) {
      // ---------------- MMA issuer: D[128 rows of this half][BN tokens], one unit per accumulator buffer
      constexpr uint32_t idesc = umma_idesc_bf16(128, BN);
      long long it = 0;
      for (int i = 0; i < u1 - u0; ++i) {
        const int b = i & 1;
        if (i >= 2) mbar_wait(&tempty[b], (uint32_t)(((i >> 1) - 1) & 1));
        tc_fence_after();
        const uint32_t acc = tmem + (uint32_t)(b * BN);
        for (int kk = 0; kk < nk; ++kk, ++it) {
          const int ws = (int)(it % C::WS), xs = (int)(it % C::XS);
          mbar_wait(&wfull[ws], (uint32_t)((it / C::WS) & 1));
          if (it == 0) CL_TRACE(2);
          mbar_wait(&xfull[xs], (uint32_t)((it / C::XS) & 1));
          tc_fence_after();
          const uint64_t da = umma_desc_sw128(smem_u32(sw + ws * CL_WBYTES));
          const uint64_t db = umma_desc_sw128(smem_u32(sx + xs * C::X_BYTES));
          if (!(a.debug & 4)) {
#pragma unroll
            for (int k = 0; k < CL_BK / 16; ++k)
              tc_mma_bf16(acc, da + 2 * k, db + 2 * k, idesc, (kk > 0 || k > 0) ? 1u : 0u);
          }
          tc_commit(&wempty[ws]);
          tc_commit_mc(&xempty[xs], pair_mask);   // release the activation stage in both CTAs of the pair
        }
        tc_commit(&tfull[b]);
      }
      CL_TRACE(3);
    }
    __syncwarp();
  } else {
    // ---------------- epilogue warps 2..5: TMEM lane quarter q = warp % 4
    pdl_wait();
    const int q = warp & 3, wq = warp - 2;
    const int row = q * 32 + lane;                       // row of this CTA's 128-row half
    // columns this CTA finishes: [cb, ce) of the BN token columns
    const int cb = (slice * BN) / S, ce = ((slice + 1) * BN) / S;
    const int mt = a.m_tok;
    // fp32 partials of the cluster's CTAs in L2: [grid][BN cols][128 rows]
    float* mine = a.part + (size_t)blockIdx.x * BN * 128;
    const float* peer[4];
    for (int s = 0; s < S; ++s) peer[s] = a.part + (size_t)(blockIdx.x - rank + half + 2 * s) * BN * 128;
    const int ncols = mt < BN ? ((mt + 15) & ~15) : BN;
    for (int i = 0; i < u1 - u0; ++i) {
      const int b = i & 1, unit = u0 + i;
      mbar_wait(&tfull[b], (uint32_t)((i >> 1) & 1));
      tc_fence_after();
      if (i > 0) cl_wait_cluster(red_free, (uint32_t)((i - 1) & 1));   // readers done with unit i-1
      const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * BN);
      for (int c0 = 0; c0 < ncols; c0 += 16) {
        float v[16];
        tmem_ld16(trow + c0, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) __stcg(mine + (c0 + j) * 128 + row, v[j]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0 && wq == 0 && i == 0) CL_TRACE(4);
      if (lane == 0) mbar_arrive(&tempty[b]);
      if (lane < S) cl_arrive_remote(red_full, (uint32_t)(half + 2 * lane));
      cl_wait_cluster(red_full, (uint32_t)(i & 1));
      if (lane == 0 && wq == 0 && i == u1 - u0 - 1) CL_TRACE(5);
      // owner phase: columns cb + wq, cb + wq + 4, ...; lane = rows 4*lane..4*lane+3
      for (int c = cb + wq; c < ce && c < mt; c += 4) {
        float4 p[4];
#pragma unroll
        for (int s = 0; s < 4; ++s)
          if (s < S) p[s] = __ldcg(reinterpret_cast<const float4*>(peer[s] + c * 128 + 4 * lane));
        float4 acc = p[0];
        for (int s = 1; s < S; ++s) { acc.x += p[s].x; acc.y += p[s].y; acc.z += p[s].z; acc.w += p[s].w; }
        cl_epilogue(a, c, unit, half, acc, lane);
      }
      __syncwarp();
      if (lane < S) cl_arrive_remote(red_free, (uint32_t)(half + 2 * lane));
    }
    if (lane == 0 && wq == 0) CL_TRACE(6);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();                           // no CTA leaves while a peer may still signal it
  if (threadIdx.x == 0) CL_TRACE(7);
  if (warp == 1) tmem_dealloc(tmem, C::TMEM_COLS);
}

template <int BN>
int cl_launch(const CUtensorMap* tx, const ClArgs& a, cudaStream_t st) {
  using C = ClCfg<BN>;
  const int cs = 2 * a.S;
  return (int)launch_k_cluster(gemm_cluster_kernel<BN>, dim3(a.n_clusters * cs), dim3(CL_THREADS), C::SMEM, st, cs,
                               *tx, a);
}

template <typename F>
int cl_dispatch(int bn, F&& f) {
  switch (bn) {
    case 16: return f(std::integral_constant<int, 16>{});
    case 32: return f(std::integral_constant<int, 32>{});
    case 64: return f(std::integral_constant<int, 64>{});
    case 128: return f(std::integral_constant<int, 128>{});
    default: return (int)cudaErrorInvalidValue;
  }
}

}  // namespace

// One-time kernel attributes (before any CUDA-graph capture).
extern "C" int pm_prepare_gemm_cl(void) {
  cudaError_t e = cudaSuccess;
#define PM_SET(BN)                                                                                              \
  if (e == cudaSuccess)                                                                                         \
    e = cudaFuncSetAttribute(gemm_cluster_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, ClCfg<BN>::SMEM);
  PM_SET(16) PM_SET(32) PM_SET(64) PM_SET(128)
#undef PM_SET
  return (int)e;
}

// Clusters of `cluster_size` CTAs of the BN instantiation that can be
// co-resident on this device (cudaOccupancyMaxActiveClusters); the planner
// never launches more, so every cluster of a launch runs in one wave.
extern "C" int pm_gemm_cl_max_clusters(int bn, int cluster_size, int* out) {
  return cl_dispatch(bn, [&](auto c) -> int {
    constexpr int BN = decltype(c)::value;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cluster_size * 64);
    cfg.blockDim = dim3(CL_THREADS);
    cfg.dynamicSmemBytes = ClCfg<BN>::SMEM;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cluster_size;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return (int)cudaOccupancyMaxActiveClusters(out, gemm_cluster_kernel<BN>, &cfg);
  });
}

// Profiling only: the last traced launch's stamps ([160][8] u64 ns, PM_CL_TRACE=1).
extern "C" int pm_gemm_cl_trace_read(void* dst) {
  return (int)cudaMemcpyFromSymbol(dst, g_cl_trace, sizeof(g_cl_trace));
}

// Pipeline depth of the BN instantiation (host introspection / tests).
extern "C" int pm_gemm_cl_stages(int bn) {
  return cl_dispatch(bn, [&](auto c) -> int { return ClCfg<decltype(c)::value>::WS; });
}

// The cluster split-K projection: Y = epilogue(X W^T) for m_tok <= bn <= 128
// token rows.  w_packed as ops.pack_weight; tmap_x: the activation buffer
// with a [bn/2 x 64] box.  `slices` S in 1..4 (cluster = 2S CTAs),
// `n_clusters` clusters (the caller's plan, ops.cl_plan).  Epilogue args as
// ClArgs (unused ones null).  ssq_in: folded RMSNorm of the input ([n_ht_in]
// [m_cap] sums of squares of the d_in-wide input rows), or null.  part: fp32
// scratch of n_clusters * 2 * slices * bn * 128 floats (the split-K partials).
extern "C" int pm_gemm_cl(const void* w_packed, const void* tmap_x, int n_out, int n_units, int k, int m_tok, int bn,
                          int m_cap, int slices, int n_clusters, int epilogue, void* out, int ld_out,
                          const float* ssq_in, int n_ht_in, int d_in, float eps, float* resid, const void* norm_w,
                          void* xn, float* ssq_out, float* amax_val, int* amax_idx, void* q_out, void* pool,
                          const int* block_table, const int* positions, const float* rope, const void* qn_w,
                          const void* kn_w, int H, int Hkv, int hd, int layer, int L_s, int max_blocks, float* part,
                          void* stream) {
  if (k % CL_BK || m_tok < 1 || m_tok > bn || m_tok > m_cap || slices < 1 || slices > 4 || n_clusters < 1 ||
      n_clusters > n_units || n_out % 8 || epilogue < 0 || epilogue > CL_QKV_ROPE)
    return (int)cudaErrorInvalidValue;
  if (epilogue == CL_QKV_ROPE && (n_out != (H + 2 * Hkv) * hd || (hd != 64 && hd != 128)))
    return (int)cudaErrorInvalidValue;
  ClArgs a{};
  a.w = reinterpret_cast<const uint8_t*>(w_packed);
  a.n_out = n_out;
  a.n_units = n_units;
  a.kb = k / CL_BK;
  a.m_tok = m_tok;
  a.m_cap = m_cap;
  a.S = slices;
  a.n_clusters = n_clusters;
  a.epilogue = epilogue;
  a.out = out;
  a.ld_out = ld_out;
  a.ssq_in = ssq_in;
  a.n_ht_in = n_ht_in;
  a.inv_d_in = d_in > 0 ? 1.0f / (float)d_in : 0.f;
  a.eps = eps;
  a.resid = resid;
  a.norm_w = reinterpret_cast<const bf16*>(norm_w);
  a.xn = reinterpret_cast<bf16*>(xn);
  a.ssq_out = ssq_out;
  a.amax_val = amax_val;
  a.amax_idx = amax_idx;
  a.part = part;
  static const int trace = getenv("PM_CL_TRACE") ? atoi(getenv("PM_CL_TRACE")) : 0;   // profiling only
  a.trace = trace;
  static const int dbg = getenv("PM_CL_DEBUG") ? atoi(getenv("PM_CL_DEBUG")) : 0;   // profiling only
  a.debug = dbg;

  a.ra = ClRope{reinterpret_cast<bf16*>(q_out), reinterpret_cast<bf16*>(pool), block_table, positions, rope,
                reinterpret_cast<const bf16*>(qn_w), reinterpret_cast<const bf16*>(kn_w), H, Hkv, hd, layer, L_s,
                max_blocks};
  if (a.kb < slices || !part) return (int)cudaErrorInvalidValue;
  auto tx = reinterpret_cast<const CUtensorMap*>(tmap_x);
  auto st = reinterpret_cast<cudaStream_t>(stream);
  return cl_dispatch(bn, [&](auto c) { return cl_launch<decltype(c)::value>(tx, a, st); });
}
