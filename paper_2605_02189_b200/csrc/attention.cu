// Paged GQA decode attention over the block-first KV pool (one query token
// per request).  HBM-bound: every KV byte of the active micro-batch is read
// once per layer.
//
// CTA = (request row, kv head, split of 16 KV blocks); 4 warps, each warp
// owns every 4th block of the split and runs its own 2-stage TMA pipeline:
// one lane issues the 128B-swizzled TMA boxes of a [16 tok x hd] K tile and
// V tile, the warp consumes them with ldmatrix + mma.sync.m16n8k16 in the
// "transposed" arrangement
//     S^T[16 tok x 8 heads] = K[16 x hd] . Q^T[hd x 8]
//     O^T[hd x 8 heads]   += V^T[hd x 16] . P^T[16 x 8]
// so the 8 q-heads of a GQA group fill the MMA N=8 exactly (Qwen3-32B,
// Llama-70B; half-filled for group 4) and P^T goes from the S accumulator to
// the B fragment with one movmatrix.trans per 8x8.  Online softmax in fp32
// with warp shuffles; warps merge in shared memory; splits merge in the last
// CTA of a (request, kv head) in split order, so results depend only on the
// request's own length (batch-invariant).
#include "common.cuh"

namespace {

constexpr int BLOCKS_PER_SPLIT = 16;
constexpr int WARPS = 4;
constexpr int STAGES = 2;

PM_DEV void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
PM_DEV void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
PM_DEV uint32_t movmatrix_t(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
PM_DEV void mma16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// byte offset of 16-byte chunk `chunk` (0..7) of row `row` in a 128B-swizzled [rows][128 B] tile
PM_DEV uint32_t sw128(int row, int chunk) { return row * 128 + ((chunk ^ (row & 7)) << 4); }

struct AttnArgs {
  const bf16* q;           // [M][H][HD]
  const int* block_table;  // [M][max_blocks]
  const int* seq_lens;     // [M]
  bf16* out;               // [M][H][HD]
  float* ws_o;             // [M][H][max_splits][HD]
  float* ws_ml;            // [M][H][max_splits][2]
  int* counters;           // [M][Hkv] zero at rest
  int H, Hkv, G, layer, L_s, max_blocks, max_splits;
  float scale_log2;        // log2(e)/sqrt(hd)
};

template <int HD>
__global__ void __launch_bounds__(WARPS * 32)
paged_attn_kernel(const __grid_constant__ CUtensorMap tmap_kv, AttnArgs a) {
  constexpr int HALVES = HD / 64;             // 64-col TMA boxes per tile
  constexpr int TILE = 16 * HD * 2;           // bytes of one K (or V) tile
  constexpr int STAGE = 2 * TILE;             // K + V
  constexpr int KC = HD / 16;                 // k-chunks of QK, m-tiles of PV
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* wbuf = smem + warp * STAGES * STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + WARPS * STAGES * STAGE) + warp * STAGES;
  float* mrg = reinterpret_cast<float*>(smem);  // reused after the main loop: [WARPS][8][HD] + m,l
  __shared__ int s_last;

  const int r = blockIdx.x, kvh = blockIdx.y, split = blockIdx.z;
  const int seq = a.seq_lens[r];
  const int nblk = (seq + 15) >> 4;
  const int nsplit = (nblk + BLOCKS_PER_SPLIT - 1) / BLOCKS_PER_SPLIT;
  if (split >= nsplit) return;
  const int b_begin = split * BLOCKS_PER_SPLIT;
  const int b_end = min(nblk, b_begin + BLOCKS_PER_SPLIT);
  const int my_n = b_end - b_begin > warp ? (b_end - b_begin - warp + WARPS - 1) / WARPS : 0;
  const int* btab = a.block_table + (size_t)r * a.max_blocks;
  const int col_k = ((a.layer * 2 + 0) * a.Hkv + kvh) * HD;
  const int col_v = ((a.layer * 2 + 1) * a.Hkv + kvh) * HD;

  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
  }
  __syncwarp();
  auto issue = [&](int i) {  // lane 0 only
    const int s = i % STAGES;
    const int phys = btab[b_begin + warp + i * WARPS];
    const uint64_t pol = policy_evict_first();
    mbar_arrive_expect_tx(&bars[s], STAGE);
    uint8_t* dst = wbuf + s * STAGE;
#pragma unroll
    for (int hh = 0; hh < HALVES; ++hh) {
      tma_load_2d(dst + hh * 2048, &tmap_kv, &bars[s], col_k + hh * 64, phys * 16, pol);
      tma_load_2d(dst + TILE + hh * 2048, &tmap_kv, &bars[s], col_v + hh * 64, phys * 16, pol);
    }
  };
  if (lane == 0) {
    for (int i = 0; i < STAGES && i < my_n; ++i) issue(i);
  }

  // Q^T fragments (B operand): head n = lane/4 of the group, d pairs 2t, 2t+8
  const int g = lane >> 2, t = lane & 3;
  uint32_t qf[KC][2];
  {
    const bool live = g < a.G;
    const uint32_t* qrow = reinterpret_cast<const uint32_t*>(a.q + ((size_t)r * a.H + kvh * a.G + (live ? g : 0)) * HD);
#pragma unroll
    for (int kc = 0; kc < KC; ++kc) {
      qf[kc][0] = live ? qrow[(kc * 16 + 2 * t) >> 1] : 0u;
      qf[kc][1] = live ? qrow[(kc * 16 + 8 + 2 * t) >> 1] : 0u;
    }
  }
  float o[KC][4];
#pragma unroll
  for (int i = 0; i < KC; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float mrun[2] = {-INFINITY, -INFINITY}, lrun[2] = {0.f, 0.f};

  for (int i = 0; i < my_n; ++i) {
    const int s = i % STAGES;
    mbar_wait(&bars[s], (i / STAGES) & 1);
    const uint32_t kbase = smem_u32(wbuf + s * STAGE), vbase = kbase + TILE;
    // ---- S^T = K Q^T
    float sc[4] = {0.f, 0.f, 0.f, 0.f};
    {
      const int row = ((lane >> 3) & 1) * 8 + (lane & 7);
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) {
        const int d = kc * 16 + (lane >> 4) * 8;
        uint32_t a0, a1, a2, a3;
        ldsm_x4(kbase + (d >> 6) * 2048 + sw128(row, (d & 63) >> 3), a0, a1, a2, a3);
        mma16816(sc, a0, a1, a2, a3, qf[kc][0], qf[kc][1]);
      }
    }
    // ---- mask + online softmax (columns = heads 2t, 2t+1; rows = tokens g, g+8)
    const int tok0 = (b_begin + warp + i * WARPS) * 16;
    const bool v0 = tok0 + g < seq, v1 = tok0 + g + 8 < seq;
    float x0 = v0 ? sc[0] * a.scale_log2 : -INFINITY, x1 = v0 ? sc[1] * a.scale_log2 : -INFINITY;
    float x2 = v1 ? sc[2] * a.scale_log2 : -INFINITY, x3 = v1 ? sc[3] * a.scale_log2 : -INFINITY;
    float mx0 = fmaxf(x0, x2), mx1 = fmaxf(x1, x3);
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
    }
    const float mn0 = fmaxf(mrun[0], mx0), mn1 = fmaxf(mrun[1], mx1);
    const float al0 = exp2f(mrun[0] - mn0), al1 = exp2f(mrun[1] - mn1);
    mrun[0] = mn0; mrun[1] = mn1;
    const float p0 = exp2f(x0 - mn0), p1 = exp2f(x1 - mn1), p2 = exp2f(x2 - mn0), p3 = exp2f(x3 - mn1);
    lrun[0] = lrun[0] * al0 + p0 + p2;
    lrun[1] = lrun[1] * al1 + p1 + p3;
#pragma unroll
    for (int mt = 0; mt < KC; ++mt) { o[mt][0] *= al0; o[mt][1] *= al1; o[mt][2] *= al0; o[mt][3] *= al1; }
    const uint32_t pb0 = movmatrix_t(pack_bf16(p0, p1));  // tokens 0-7  -> b0
    const uint32_t pb1 = movmatrix_t(pack_bf16(p2, p3));  // tokens 8-15 -> b1
    // ---- O^T += V^T P^T
    {
      const int q4 = lane >> 3, ii = lane & 7;
      const int tok = (q4 >> 1) * 8 + ii;
#pragma unroll
      for (int mt = 0; mt < KC; ++mt) {
        const int d = mt * 16 + (q4 & 1) * 8;
        uint32_t a0, a1, a2, a3;
        ldsm_x4_t(vbase + (d >> 6) * 2048 + sw128(tok, (d & 63) >> 3), a0, a1, a2, a3);
        mma16816(o[mt], a0, a1, a2, a3, pb0, pb1);
      }
    }
    __syncwarp();
    if (lane == 0 && i + STAGES < my_n) {
      fence_proxy_async();
      issue(i + STAGES);
    }
  }
  // row sums: reduce the per-lane partial l over the 8 token-lanes of a column
#pragma unroll
  for (int off = 4; off < 32; off <<= 1) {
    lrun[0] += __shfl_xor_sync(0xffffffffu, lrun[0], off);
    lrun[1] += __shfl_xor_sync(0xffffffffu, lrun[1], off);
  }
  __syncthreads();  // all warps done with their stage buffers -> reuse as merge area
  // merge area: per warp [8 heads][HD] O + [8] m + [8] l
  float* wo = mrg + warp * (8 * HD + 16);
#pragma unroll
  for (int mt = 0; mt < KC; ++mt) {
    const int d = mt * 16 + g;
    wo[(2 * t) * HD + d] = o[mt][0];
    wo[(2 * t + 1) * HD + d] = o[mt][1];
    wo[(2 * t) * HD + d + 8] = o[mt][2];
    wo[(2 * t + 1) * HD + d + 8] = o[mt][3];
  }
  if (g == 0) {
    wo[8 * HD + 2 * t] = mrun[0]; wo[8 * HD + 2 * t + 1] = mrun[1];
    wo[8 * HD + 8 + 2 * t] = lrun[0]; wo[8 * HD + 8 + 2 * t + 1] = lrun[1];
  }
  __syncthreads();
  const int G = a.G;
  const bool single = nsplit == 1;
  // each thread handles (head, d) pairs
  for (int e = threadIdx.x; e < G * HD; e += blockDim.x) {
    const int h = e / HD, d = e % HD;
    float M = -INFINITY;
    for (int w = 0; w < WARPS; ++w) M = fmaxf(M, mrg[w * (8 * HD + 16) + 8 * HD + h]);
    float acc = 0.f, l = 0.f;
    for (int w = 0; w < WARPS; ++w) {
      const float* ww = mrg + w * (8 * HD + 16);
      const float f = ww[8 * HD + h] == -INFINITY ? 0.f : exp2f(ww[8 * HD + h] - M);
      acc += ww[h * HD + d] * f;
      l += ww[8 * HD + 8 + h] * f;
    }
    const int head = kvh * G + h;
    if (single) {
      a.out[((size_t)r * a.H + head) * HD + d] = __float2bfloat16(acc / l);
    } else {
      const size_t base = ((size_t)r * a.H + head) * a.max_splits + split;
      a.ws_o[base * HD + d] = acc;
      if (d == 0) { a.ws_ml[base * 2] = M; a.ws_ml[base * 2 + 1] = l; }
    }
  }
  if (single) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    int* ctr = a.counters + (size_t)r * a.Hkv + kvh;
    const int prev = atomicAdd(ctr, 1);
    s_last = prev == nsplit - 1;
    if (s_last) *ctr = 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int e = threadIdx.x; e < G * HD; e += blockDim.x) {
    const int h = e / HD, d = e % HD;
    const int head = kvh * G + h;
    const size_t base = ((size_t)r * a.H + head) * a.max_splits;
    float M = -INFINITY;
    for (int s = 0; s < nsplit; ++s) M = fmaxf(M, __ldcg(&a.ws_ml[(base + s) * 2]));
    float acc = 0.f, l = 0.f;
    for (int s = 0; s < nsplit; ++s) {
      const float f = exp2f(__ldcg(&a.ws_ml[(base + s) * 2]) - M);
      acc += __ldcg(&a.ws_o[(base + s) * HD + d]) * f;
      l += __ldcg(&a.ws_ml[(base + s) * 2 + 1]) * f;
    }
    a.out[((size_t)r * a.H + head) * HD + d] = __float2bfloat16(acc / l);
  }
}

template <int HD>
int launch_attn(const CUtensorMap* tm, const AttnArgs& a, int M, cudaStream_t st) {
  constexpr int SMEM = WARPS * STAGES * 2 * 16 * HD * 2 + WARPS * STAGES * 8 + 1024;
  static_assert(WARPS * (8 * HD + 16) * 4 <= WARPS * STAGES * 2 * 16 * HD * 2, "merge area must fit");
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(paged_attn_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return (int)e;
    attr = true;
  }
  dim3 grid(M, a.Hkv, a.max_splits);
  paged_attn_kernel<HD><<<grid, WARPS * 32, SMEM, st>>>(*tm, a);
  return (int)cudaGetLastError();
}

}  // namespace

// q [M][H][hd] bf16 (RoPE'd), pool via `tmap_kv` (2-D view [blocks*16][L_s*2*Hkv*hd],
// box [16][64], 128B swizzle), block_table [M][max_blocks], seq_lens [M] (cached
// positions incl. the current token), out [M][H][hd] bf16.
extern "C" int pm_paged_attention(const void* tmap_kv, const void* q, const int* block_table,
                                  const int* seq_lens, void* out, float* ws_o, float* ws_ml, int* counters,
                                  int M, int H, int Hkv, int hd, int layer, int L_s, int max_blocks,
                                  int max_splits, void* stream) {
  if (M == 0) return 0;
  const int G = H / Hkv;
  if (H % Hkv || G > 8 || max_splits < 1) return (int)cudaErrorInvalidValue;
  if (max_splits * BLOCKS_PER_SPLIT < max_blocks) return (int)cudaErrorInvalidValue;
  AttnArgs a{reinterpret_cast<const bf16*>(q), block_table, seq_lens, reinterpret_cast<bf16*>(out),
             ws_o, ws_ml, counters, H, Hkv, G, layer, L_s, max_blocks, max_splits,
             1.4426950408889634f / sqrtf((float)hd)};
  auto tm = reinterpret_cast<const CUtensorMap*>(tmap_kv);
  auto st = reinterpret_cast<cudaStream_t>(stream);
  if (hd == 128) return launch_attn<128>(tm, a, M, st);
  if (hd == 64) return launch_attn<64>(tm, a, M, st);
  return (int)cudaErrorInvalidValue;
}

extern "C" int pm_attn_blocks_per_split(void) { return BLOCKS_PER_SPLIT; }

extern "C" int pm_prepare_attention(void) {
  constexpr int S128 = WARPS * STAGES * 2 * 16 * 128 * 2 + WARPS * STAGES * 8 + 1024;
  constexpr int S64 = WARPS * STAGES * 2 * 16 * 64 * 2 + WARPS * STAGES * 8 + 1024;
  cudaError_t e = cudaFuncSetAttribute(paged_attn_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, S128);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(paged_attn_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, S64);
  return (int)e;
}
