// Bandwidth/latency-bound decode kernels around the GEMMs and attention:
//   pm_embed            token ids -> fp32 residual rows (stage 0)
//   pm_rmsnorm          fp32 residual -> bf16 normalised activations
//   pm_qkv_rope_append  (Qwen3 per-head q/k RMSNorm) + RoPE + paged KV append
//   pm_argmax_reduce    per-tile argmax partials -> greedy ids (last stage)
//
// KV pool layout (one per stage, block-first, token-major inside a block):
//   pool[block][slot 0..15][layer 0..L_s-1][k|v][kv_head][hd]  bf16
// so one token's whole-stage KV is one contiguous run (eager D2H offload is
// one copy per token) and one block is one contiguous run (prefetch H2D is
// one copy per block; the paper's block-first layout).
#include "common.cuh"

namespace {

__global__ void embed_kernel(const int* __restrict__ tok_table, const int* __restrict__ slots,
                             const bf16* __restrict__ table, float* __restrict__ resid, int d) {
  pdl_trigger();
  pdl_wait();
  const int m = blockIdx.x;
  const int id = tok_table[slots ? slots[m] : m];
  const uint4* src = reinterpret_cast<const uint4*>(table + (size_t)id * d);
  float4* dst = reinterpret_cast<float4*>(resid + (size_t)m * d);
  for (int i = threadIdx.x; i < d / 8; i += blockDim.x) {
    const uint4 v = src[i];
    dst[2 * i] = make_float4(bf16_lo(v.x), bf16_hi(v.x), bf16_lo(v.y), bf16_hi(v.y));
    dst[2 * i + 1] = make_float4(bf16_lo(v.z), bf16_hi(v.z), bf16_lo(v.w), bf16_hi(v.w));
  }
}

// one CTA per row; 256 threads; d % 8 == 0
__global__ void rmsnorm_kernel(const float* __restrict__ x, const bf16* __restrict__ w,
                               bf16* __restrict__ y, int d, float eps) {
  pdl_trigger();
  pdl_wait();
  const int m = blockIdx.x;
  const float4* xr = reinterpret_cast<const float4*>(x + (size_t)m * d);
  float ss = 0.f;
  for (int i = threadIdx.x; i < d / 4; i += blockDim.x) {
    const float4 v = xr[i];
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  __shared__ float red[32];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = rsqrtf(t / (float)d + eps);
  }
  __syncthreads();
  const float r = red[0];
  const uint2* wr = reinterpret_cast<const uint2*>(w);
  uint2* yr = reinterpret_cast<uint2*>(y + (size_t)m * d);
  for (int i = threadIdx.x; i < d / 4; i += blockDim.x) {
    const float4 v = xr[i];
    const uint2 ww = wr[i];
    uint2 o;
    o.x = pack_bf16(v.x * r * bf16_lo(ww.x), v.y * r * bf16_hi(ww.x));
    o.y = pack_bf16(v.z * r * bf16_lo(ww.y), v.w * r * bf16_hi(ww.y));
    yr[i] = o;
  }
}

// One warp per (token, head) over H q-heads, Hkv k-heads and Hkv v-heads.
// E = hd/32 contiguous elements per lane; lane l and lane l^16 hold the
// rotate_half partners (i, i + hd/2).
template <int E>
__global__ void qkv_rope_append_kernel(const bf16* __restrict__ qkv, bf16* __restrict__ q_out,
                                       bf16* __restrict__ pool, const int* __restrict__ block_table,
                                       const int* __restrict__ positions, const float* __restrict__ rope,
                                       const bf16* __restrict__ qn_w, const bf16* __restrict__ kn_w,
                                       int M, int H, int Hkv, int layer, int L_s, int max_blocks,
                                       float eps) {
  constexpr int HD = 32 * E;
  pdl_trigger();
  pdl_wait();
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int heads = H + 2 * Hkv;
  if (gw >= M * heads) return;
  const int m = gw / heads, h = gw % heads;
  const bf16* src = qkv + (size_t)m * heads * HD + (size_t)h * HD + lane * E;
  float x[E];
  if constexpr (E == 4) {
    const uint2 v = *reinterpret_cast<const uint2*>(src);
    x[0] = bf16_lo(v.x); x[1] = bf16_hi(v.x); x[2] = bf16_lo(v.y); x[3] = bf16_hi(v.y);
  } else {
    const uint32_t v = *reinterpret_cast<const uint32_t*>(src);
    x[0] = bf16_lo(v); x[1] = bf16_hi(v);
  }
  const int pos = positions[m];
  const bool is_q = h < H, is_k = !is_q && h < H + Hkv;
  if (is_q || is_k) {
    const bf16* nw = is_q ? qn_w : kn_w;
    if (nw) {  // Qwen3 per-head RMSNorm (before RoPE)
      float ss = 0.f;
#pragma unroll
      for (int e = 0; e < E; ++e) ss += x[e] * x[e];
      const float r = rsqrtf(warp_sum(ss) / (float)HD + eps);
#pragma unroll
      for (int e = 0; e < E; ++e) x[e] = x[e] * r * __bfloat162float(nw[lane * E + e]);
    }
    // rotate_half RoPE with the precomputed fp32 table rope[pos][0..HD/2) = cos, [HD/2..HD) = sin
    const float* cs = rope + (size_t)pos * HD;
    const bool lo_half = lane < 16;
    float y[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const float partner = __shfl_xor_sync(0xffffffffu, x[e], 16);
      const int fi = (lane & 15) * E + e;
      const float c = cs[fi], s = cs[HD / 2 + fi];
      y[e] = lo_half ? (x[e] * c - partner * s) : (x[e] * c + partner * s);
    }
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = y[e];
  }
  bf16* dst;
  if (is_q) {
    dst = q_out + ((size_t)m * H + h) * HD + lane * E;
  } else {
    const int kv = is_k ? 0 : 1;
    const int g = is_k ? h - H : h - H - Hkv;
    const int blk = block_table[(size_t)m * max_blocks + pos / 16];
    const size_t tok_stride = (size_t)L_s * 2 * Hkv * HD;
    dst = pool + ((size_t)blk * 16 + (pos & 15)) * tok_stride + (((size_t)layer * 2 + kv) * Hkv + g) * HD + lane * E;
  }
  if constexpr (E == 4) {
    uint2 o;
    o.x = pack_bf16(x[0], x[1]);
    o.y = pack_bf16(x[2], x[3]);
    *reinterpret_cast<uint2*>(dst) = o;
  } else {
    *reinterpret_cast<uint32_t*>(dst) = pack_bf16(x[0], x[1]);
  }
}

// argmax over n_tiles partials per token; ties -> lowest vocabulary index
__global__ void argmax_reduce_kernel(const float* __restrict__ val, const int* __restrict__ idx,
                                     int n_tiles, int m_cap, int* __restrict__ out_ids,
                                     int* __restrict__ tok_table, const int* __restrict__ slots) {
  pdl_trigger();
  pdl_wait();
  const int m = blockIdx.x;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
    const float v = val[(size_t)t * m_cap + m];
    const int i = idx[(size_t)t * m_cap + m];
    if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  __shared__ float sv[32];
  __shared__ int si[32];
  if ((threadIdx.x & 31) == 0) { sv[threadIdx.x >> 5] = bv; si[threadIdx.x >> 5] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (sv[w] > bv || (sv[w] == bv && si[w] < bi)) { bv = sv[w]; bi = si[w]; }
    if (out_ids) out_ids[m] = bi;
    if (tok_table) tok_table[slots ? slots[m] : m] = bi;
  }
}

// Inter-stage activation hop (pipeline.py): the fp32 residual rows travel as
// bf16 (half the NVLink bytes) -- pack before the send, unpack
// into the receiving stage's residual.  8 elements per thread (16-byte bf16).
__global__ void hop_pack_kernel(const float* __restrict__ x, bf16* __restrict__ y, long long n8) {
  pdl_trigger();
  pdl_wait();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n8; i += (long long)gridDim.x * blockDim.x) {
    const float4 a = reinterpret_cast<const float4*>(x)[2 * i], b = reinterpret_cast<const float4*>(x)[2 * i + 1];
    reinterpret_cast<uint4*>(y)[i] = make_uint4(pack_bf16(a.x, a.y), pack_bf16(a.z, a.w), pack_bf16(b.x, b.y),
                                                pack_bf16(b.z, b.w));
  }
}
__global__ void hop_unpack_kernel(const bf16* __restrict__ y, float* __restrict__ x, long long n8) {
  pdl_trigger();
  pdl_wait();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n8; i += (long long)gridDim.x * blockDim.x) {
    const uint4 v = reinterpret_cast<const uint4*>(y)[i];
    reinterpret_cast<float4*>(x)[2 * i] = make_float4(bf16_lo(v.x), bf16_hi(v.x), bf16_lo(v.y), bf16_hi(v.y));
    reinterpret_cast<float4*>(x)[2 * i + 1] = make_float4(bf16_lo(v.z), bf16_hi(v.z), bf16_lo(v.w), bf16_hi(v.w));
  }
}
// Stage 0: greedy ids returned by the last stage -> the token table by slot.
// `slots` may live in mapped pinned host memory (read over PCIe, no copy).
__global__ void scatter_tokens_kernel(const int* __restrict__ ids, const int* __restrict__ slots, int n,
                                      int* __restrict__ tok_table) {
  pdl_trigger();
  pdl_wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) tok_table[slots[i]] = ids[i];
}

}  // namespace

extern "C" int pm_hop_pack(const float* resid, void* out, long long n, void* stream) {
  if (n % 8) return (int)cudaErrorInvalidValue;
  if (n == 0) return 0;
  const long long n8 = n / 8;
  const int blocks = (int)((n8 + 255) / 256 < 592 ? (n8 + 255) / 256 : 592);
  cudaError_t e = launch_k(hop_pack_kernel, dim3(blocks), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), resid,
                           reinterpret_cast<bf16*>(out), n8);
  return e != cudaSuccess ? (int)e : (int)cudaGetLastError();
}

extern "C" int pm_hop_unpack(const void* in, float* resid, long long n, void* stream) {
  if (n % 8) return (int)cudaErrorInvalidValue;
  if (n == 0) return 0;
  const long long n8 = n / 8;
  const int blocks = (int)((n8 + 255) / 256 < 592 ? (n8 + 255) / 256 : 592);
  cudaError_t e = launch_k(hop_unpack_kernel, dim3(blocks), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream),
                           reinterpret_cast<const bf16*>(in), resid, n8);
  return e != cudaSuccess ? (int)e : (int)cudaGetLastError();
}

extern "C" int pm_scatter_tokens(const int* ids, const int* slots, int n, int* tok_table, void* stream) {
  if (n == 0) return 0;
  cudaError_t e = launch_k(scatter_tokens_kernel, dim3((n + 255) / 256), dim3(256), 0,
                           reinterpret_cast<cudaStream_t>(stream), ids, slots, n, tok_table);
  return e != cudaSuccess ? (int)e : (int)cudaGetLastError();
}

extern "C" int pm_embed(const int* tok_table, const int* slots, const void* table, float* resid, int M,
                        int d, void* stream) {
  if (d % 8) return (int)cudaErrorInvalidValue;
  if (M == 0) return 0;
  cudaError_t e = launch_k(embed_kernel, dim3(M), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), tok_table,
                           slots, reinterpret_cast<const bf16*>(table), resid, d);
  if (e != cudaSuccess) return (int)e;
  return (int)cudaGetLastError();
}

int launch_rmsnorm(const float* x, const void* w, void* y, int M, int d, float eps, cudaStream_t st) {
  if (d % 8) return (int)cudaErrorInvalidValue;
  if (M == 0) return 0;
  cudaError_t e = launch_k(rmsnorm_kernel, dim3(M), dim3(256), 0, st, x, reinterpret_cast<const bf16*>(w),
                           reinterpret_cast<bf16*>(y), d, eps);
  if (e != cudaSuccess) return (int)e;
  return (int)cudaGetLastError();
}

extern "C" int pm_rmsnorm(const float* x, const void* w, void* y, int M, int d, float eps, void* stream) {
  return launch_rmsnorm(x, w, y, M, d, eps, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int pm_qkv_rope_append(const void* qkv, void* q_out, void* pool, const int* block_table,
                                  const int* positions, const float* rope, const void* qn_w,
                                  const void* kn_w, int M, int H, int Hkv, int hd, int layer, int L_s,
                                  int max_blocks, float eps, void* stream) {
  if (M == 0) return 0;
  const int warps = M * (H + 2 * Hkv);
  const int threads = 256, blocks = (warps * 32 + threads - 1) / threads;
  auto st = reinterpret_cast<cudaStream_t>(stream);
  auto a = reinterpret_cast<const bf16*>(qkv);
  auto q = reinterpret_cast<bf16*>(q_out);
  auto p = reinterpret_cast<bf16*>(pool);
  auto qn = reinterpret_cast<const bf16*>(qn_w);
  auto kn = reinterpret_cast<const bf16*>(kn_w);
  cudaError_t e;
  if (hd == 128)
    e = launch_k(qkv_rope_append_kernel<4>, dim3(blocks), dim3(threads), 0, st, a, q, p, block_table, positions,
                 rope, qn, kn, M, H, Hkv, layer, L_s, max_blocks, eps);
  else if (hd == 64)
    e = launch_k(qkv_rope_append_kernel<2>, dim3(blocks), dim3(threads), 0, st, a, q, p, block_table, positions,
                 rope, qn, kn, M, H, Hkv, layer, L_s, max_blocks, eps);
  else
    return (int)cudaErrorInvalidValue;
  if (e != cudaSuccess) return (int)e;
  return (int)cudaGetLastError();
}

extern "C" int pm_argmax_reduce(const float* val, const int* idx, int n_tiles, int M, int m_cap, int* out_ids,
                                int* tok_table, const int* slots, void* stream) {
  if (M == 0) return 0;
  cudaError_t e = launch_k(argmax_reduce_kernel, dim3(M), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), val,
                           idx, n_tiles, m_cap, out_ids, tok_table, slots);
  if (e != cudaSuccess) return (int)e;
  return (int)cudaGetLastError();
}
