// Probe: 148 persistent CTAs x W warps; each warp streams 16-row x 128 B TMA
// boxes (2 KB) from a pool whose rows are `stride` bytes apart (token-major KV:
// stride = L_s*2*Hkv*hd*2), 4 boxes per "block", S stages per warp.
// Compare with 1-D bulk copies of contiguous 8 KB blocks (head-major layout).
#include <cstdio>
#include <cudaTypedefs.h>
#include "../paper_2605_02189_b200/csrc/common.cuh"

PM_DEV void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

template <int MODE, int W, int S>
__global__ void __launch_bounds__(W * 32) probe(const __grid_constant__ CUtensorMap tm, const uint8_t* base,
                                                int blocks_per_warp, int n_rows_blocks, long long cols) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  uint8_t* wb = smem + warp * S * 8192;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + W * S * 8192) + warp * S;
  if (lane == 0) { for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1); fence_barrier_init(); }
  __syncwarp();
  const int gw = blockIdx.x * W + warp;
  unsigned seed = gw * 2654435761u;
  auto issue = [&](int i) {
    int s = i % S;
    seed = seed * 1664525u + 1013904223u;
    int blk = seed % n_rows_blocks;
    int col = (seed >> 8) % (int)(cols / 128) * 128;  // a (layer, head) column group
    mbar_arrive_expect_tx(&bars[s], 8192);
    if (MODE == 0) {
      for (int h = 0; h < 4; ++h) tma_load_2d(wb + s * 8192 + h * 2048, &tm, &bars[s], col + (h & 1) * 64, blk * 16, policy_evict_first());
    } else {
      bulk_load(wb + s * 8192, base + ((long long)blk * (cols / 128) + col / 128) * 8192, 8192, &bars[s]);
    }
  };
  if (lane == 0) for (int i = 0; i < S && i < blocks_per_warp; ++i) issue(i);
  for (int i = 0; i < blocks_per_warp; ++i) {
    int s = i % S;
    mbar_wait(&bars[s], (i / S) & 1);
    __syncwarp();
    if (lane == 0 && i + S < blocks_per_warp) issue(i + S);
  }
}

template <int MODE, int W, int S>
void run(const CUtensorMap& tm, uint8_t* buf, int nrb, long long cols) {
  constexpr int smem = W * S * 8192 + 1024 + W * S * 8;
  cudaFuncSetAttribute(probe<MODE, W, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int per_sm = (227 * 1024) / smem;
  int grid = 148 * per_sm;
  int bpw = 400;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9;
  for (int it = 0; it < 4; ++it) {
    cudaEventRecord(a);
    probe<MODE, W, S><<<grid, W * 32, smem>>>(tm, buf, bpw, nrb, cols);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  double bytes = (double)grid * W * bpw * 8192;
  printf("%s W=%d S=%d ctas/sm=%d: %7.0f GB/s (%s)\n", MODE == 0 ? "tma 4x2KB strided" : "bulk 8KB contig ", W, S,
         per_sm, bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  // token-major pool: rows = token slots, row = L_s*2*Hkv*hd bf16 = 36*2*8*128*2 B = 147456 B
  const long long cols = 36LL * 2 * 8 * 128;  // elements per row
  const long long row_bytes = cols * 2;
  const int nrb = 8192;                        // blocks of 16 rows -> 19.3 GB
  size_t bytes = (size_t)nrb * 16 * row_bytes;
  uint8_t* buf;
  if (cudaMalloc(&buf, bytes) != cudaSuccess) { printf("oom\n"); return 1; }
  cudaMemset(buf, 1, bytes);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", (void**)&enc, 12000, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)nrb * 16};
  cuuint64_t str[1] = {(cuuint64_t)row_bytes};
  cuuint32_t box[2] = {64, 16}, es[2] = {1, 1};
  enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  run<0, 8, 2>(tm, buf, nrb, cols);
  run<0, 8, 3>(tm, buf, nrb, cols);
  run<0, 4, 4>(tm, buf, nrb, cols);
  run<0, 4, 2>(tm, buf, nrb, cols);
  run<1, 8, 2>(tm, buf, nrb, cols);
  run<1, 8, 3>(tm, buf, nrb, cols);
  run<1, 4, 4>(tm, buf, nrb, cols);
  run<1, 4, 2>(tm, buf, nrb, cols);
  return 0;
}
