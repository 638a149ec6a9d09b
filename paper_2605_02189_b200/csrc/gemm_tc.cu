// Decode projection GEMM on 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// Swap-AB: the weight tile is the 128-row MMA "A" operand and the micro-batch
// tokens are the MMA "N" (16..256), so D^T[n_out, tok] = W[n_out, K] . X[tok, K]^T
// accumulates in TMEM.  At decode batch sizes the kernel streams each weight
// byte from HBM exactly once (weight-bandwidth bound for M_tok <~ 255).
//
// Roles (128 threads, 1 CTA / output tile x K-split):
//   warp0.lane0  TMA producer: W tile [128 x 64] and X tile [BN x 64] per stage,
//                both K-major with the 128-byte swizzle, weights evict-first.
//   warp1.lane0  MMA issuer: 4 x tcgen05.mma (K=16 each) per stage, commit frees
//                the stage, final commit signals the epilogue.
//   warps0-3     epilogue: tcgen05.ld rows 32w..32w+31 of the accumulator.
// Fixed K-split per (N, K) shape (chosen on the host, independent of M_tok)
// keeps every token's result independent of its micro-batch mates; the last
// CTA of a tile sums the fp32 partials in split order (deterministic).
#include "common.cuh"

namespace {

constexpr int BM = 128;
constexpr int BK = 64;           // 64 bf16 = 128 B rows -> SWIZZLE_128B
constexpr int A_BYTES = BM * BK * 2;

enum Epilogue : int {
  EPI_STORE_BF16 = 0,    // out_bf16[tok][n] = acc
  EPI_RESID_ADD_F32 = 1, // out_f32[tok][n] += acc          (residual stream)
  EPI_SILU_MUL = 2,      // rows interleaved gate/up: out_bf16[tok][n/2] = silu(g)*u
  EPI_LOGITS_ARGMAX = 3, // optional out_f32[tok][n] = acc; per-tile argmax partials
};

struct GemmArgs {
  int n_out, k, m_tok;
  int splits;
  int epilogue;
  void* out;
  int ld_out;
  float* ws;          // [splits][m_cap][n_out] fp32 partials (splits > 1)
  int m_cap;
  int* counters;      // [tok_tiles][n_tiles], zero at rest (self-resetting)
  float* amax_val;    // [n_tiles][m_cap]
  int* amax_idx;
};

template <int BN>
struct Cfg {
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (200 * 1024) / STAGE_BYTES > 8 ? 8 : (200 * 1024) / STAGE_BYTES;
  static constexpr int TMEM_COLS = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

__device__ __forceinline__ float silu(float g) { return g / (1.0f + expf(-g)); }

template <int BN>
__global__ void __launch_bounds__(128, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_x,
               GemmArgs a) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;                                  // STAGES x A tile
  uint8_t* sb = smem + C::STAGES * A_BYTES;             // STAGES x B tile
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* done = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  int* flag = reinterpret_cast<int*>(tmem_slot + 1);
  float* red_val = reinterpret_cast<float*>(flag + 1);   // [4] cross-warp argmax
  int* red_idx = reinterpret_cast<int*>(red_val + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x, split = blockIdx.y, ttile = blockIdx.z;
  const int kb_total = a.k / BK;
  const int kb0 = (int)((long long)kb_total * split / a.splits);
  const int kb1 = (int)((long long)kb_total * (split + 1) / a.splits);
  const int nkb = kb1 - kb0;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmap_w);
    tma_prefetch_desc(&tmap_x);
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    const uint64_t pol_w = policy_evict_first(), pol_x = policy_evict_last();
    for (int it = 0; it < nkb; ++it) {
      const int s = it % C::STAGES;
      if (it >= C::STAGES) mbar_wait(&empty[s], ((it / C::STAGES) - 1) & 1);
      mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
      const int kx = (kb0 + it) * BK;
      tma_load_2d(sa + s * A_BYTES, &tmap_w, &full[s], kx, tile * BM, pol_w);
      tma_load_2d(sb + s * C::B_BYTES, &tmap_x, &full[s], kx, ttile * BN, pol_x);
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer
    constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
    for (int it = 0; it < nkb; ++it) {
      const int s = it % C::STAGES;
      mbar_wait(&full[s], (it / C::STAGES) & 1);
      tc_fence_after();
      const uint64_t da = umma_desc_sw128(smem_u32(sa + s * A_BYTES));
      const uint64_t db = umma_desc_sw128(smem_u32(sb + s * C::B_BYTES));
#pragma unroll
      for (int kk = 0; kk < BK / 16; ++kk)  // +32 B per K=16 slice -> +2 in the >>4 field
        tc_mma_bf16(tmem, da + 2 * kk, db + 2 * kk, idesc, (it | kk) != 0);
      tc_commit(&empty[s]);
    }
    tc_commit(done);
  }
  __syncwarp();

  // ---------------- epilogue (all 4 warps)
  mbar_wait(done, 0);
  tc_fence_after();
  const int row = warp * 32 + lane;
  const int n = tile * BM + row;
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  const int tok_base = ttile * BN;
  const int tok_end = min(BN, a.m_tok - tok_base);

  bool last = true;
  if (a.splits > 1) {
    float* part = a.ws + (size_t)split * a.m_cap * a.n_out;
    for (int c0 = 0; c0 < BN; c0 += 16) {
      if (c0 >= tok_end) break;
      float v[16];
      tmem_ld16(trow + c0, v);
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (c0 + j < tok_end) part[(size_t)(tok_base + c0 + j) * a.n_out + n] = v[j];
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      int* ctr = a.counters + (size_t)ttile * gridDim.x + tile;
      const int prev = atomicAdd(ctr, 1);
      const int is_last = prev == a.splits - 1;
      if (is_last) *ctr = 0;  // self-reset for the next launch
      *flag = is_last;
    }
    __syncthreads();
    last = *flag != 0;
    if (last) __threadfence();
  }
  if (last) {
    for (int c0 = 0; c0 < BN; c0 += 16) {
      if (c0 >= tok_end) break;
      float v[16];
      if (a.splits > 1) {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = 0.f;
        for (int s = 0; s < a.splits; ++s) {
          const float* part = a.ws + (size_t)s * a.m_cap * a.n_out;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (c0 + j < tok_end) v[j] += __ldcg(&part[(size_t)(tok_base + c0 + j) * a.n_out + n]);
        }
      } else {
        tmem_ld16(trow + c0, v);
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int c = c0 + j;
        const int tok = tok_base + c;
        const bool valid = c < tok_end;
        const float acc = v[j];
        switch (a.epilogue) {
          case EPI_STORE_BF16:
            if (valid) reinterpret_cast<bf16*>(a.out)[(size_t)tok * a.ld_out + n] = __float2bfloat16(acc);
            break;
          case EPI_RESID_ADD_F32:
            if (valid) reinterpret_cast<float*>(a.out)[(size_t)tok * a.ld_out + n] += acc;
            break;
          case EPI_SILU_MUL: {
            const float up = __shfl_xor_sync(0xffffffffu, acc, 1);
            if (valid && (lane & 1) == 0)
              reinterpret_cast<bf16*>(a.out)[(size_t)tok * a.ld_out + (n >> 1)] =
                  __float2bfloat16(silu(acc) * up);
            break;
          }
          case EPI_LOGITS_ARGMAX: {
            if (valid && a.out) reinterpret_cast<float*>(a.out)[(size_t)tok * a.ld_out + n] = acc;
            float bv = (n < a.n_out) ? acc : -INFINITY;
            int bi = n;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
              const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
              if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
            }
            if (lane == 0) { red_val[warp] = bv; red_idx[warp] = bi; }
            __syncthreads();
            if (threadIdx.x == 0 && valid) {
              float best = red_val[0];
              int bidx = red_idx[0];
              for (int w = 1; w < 4; ++w)
                if (red_val[w] > best || (red_val[w] == best && red_idx[w] < bidx)) { best = red_val[w]; bidx = red_idx[w]; }
              a.amax_val[(size_t)tile * a.m_cap + tok] = best;
              a.amax_idx[(size_t)tile * a.m_cap + tok] = bidx;
            }
            __syncthreads();
            break;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, C::TMEM_COLS);
}

template <int BN>
int launch(const CUtensorMap* tw, const CUtensorMap* tx, const GemmArgs& a, cudaStream_t st) {
  using C = Cfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return (int)e;
    attr_set = true;
  }
  dim3 grid(a.n_out / BM, a.splits, (a.m_tok + BN - 1) / BN);
  gemm_tc_kernel<BN><<<grid, 128, C::SMEM, st>>>(*tw, *tx, a);
  return (int)cudaGetLastError();
}

}  // namespace

extern "C" int pm_gemm(const void* tmap_w, const void* tmap_x, int n_out, int k, int m_tok, int bn,
                       int splits, int epilogue, void* out, int ld_out, float* ws, int m_cap,
                       int* counters, float* amax_val, int* amax_idx, void* stream) {
  if (n_out % BM || k % BK || m_tok < 1 || splits < 1 || splits > k / BK) return (int)cudaErrorInvalidValue;
  if (m_tok > m_cap) return (int)cudaErrorInvalidValue;
  GemmArgs a{n_out, k, m_tok, splits, epilogue, out, ld_out, ws, m_cap, counters, amax_val, amax_idx};
  auto tw = reinterpret_cast<const CUtensorMap*>(tmap_w);
  auto tx = reinterpret_cast<const CUtensorMap*>(tmap_x);
  auto st = reinterpret_cast<cudaStream_t>(stream);
  switch (bn) {
    case 16: return launch<16>(tw, tx, a, st);
    case 32: return launch<32>(tw, tx, a, st);
    case 64: return launch<64>(tw, tx, a, st);
    case 128: return launch<128>(tw, tx, a, st);
    case 256: return launch<256>(tw, tx, a, st);
    default: return (int)cudaErrorInvalidValue;
  }
}
