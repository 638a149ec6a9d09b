// Probe: how fast can 148 persistent CTAs stream HBM into shared memory with
// (a) 1-D bulk copies of contiguous chunks, (b) 2-D TMA tiles [128 rows x 128 B]
// from a row-major matrix with an 8 KB row stride?  Consumer just releases.
#include <cstdio>
#include <vector>
#include <cudaTypedefs.h>
#include "../paper_2605_02189_b200/csrc/common.cuh"

PM_DEV void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(64, 1) probe(const __grid_constant__ CUtensorMap tm, const uint8_t* base,
                                              long long chunks_total, int chunk_bytes, int stages) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * chunk_bytes);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  long long per = chunks_total / gridDim.x;
  long long c0 = per * blockIdx.x;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0 && lane == 0) {
    for (long long i = 0; i < per; ++i) {
      int s = i % stages;
      if (i >= stages) mbar_wait(&empty[s], ((i / stages) - 1) & 1);
      mbar_arrive_expect_tx(&full[s], chunk_bytes);
      long long c = c0 + i;
      if (MODE == 0) {
        bulk_load(smem + s * chunk_bytes, base + c * chunk_bytes, chunk_bytes, &full[s]);
      } else {
        // chunk = [128 rows x 64 cols] tile(s); matrix [rows][4096] bf16
        int tiles = chunk_bytes / 16384;
        for (int t = 0; t < tiles; ++t) {
          long long ct = c * tiles + t;
          int kb = ct % 64, rt = ct / 64;
          tma_load_2d(smem + s * chunk_bytes + t * 16384, &tm, &full[s], kb * 64, rt * 128, policy_evict_first());
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    for (long long i = 0; i < per; ++i) {
      int s = i % stages;
      mbar_wait(&full[s], (i / stages) & 1);
      mbar_arrive(&empty[s]);
    }
  }
  __syncthreads();
}

int main(int argc, char** argv) {
  const size_t bytes = 2ull << 30;  // 2 GiB
  const int grid = argc > 1 ? atoi(argv[1]) : 148;  // CTAs (one per SM)
  uint8_t* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", (void**)&enc, 12000, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {4096, bytes / 8192};
  cuuint64_t str[1] = {8192};
  cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode < 1; ++mode) {
    for (int cb : {16384, 32768, 65536}) {
      for (int stages : {2, 3, 4, 6, 8, 12}) {
        if ((size_t)cb * stages > 200 * 1024) continue;
        int smem = cb * stages + 1024;
        auto k = mode == 0 ? probe<0> : probe<1>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        long long chunks = bytes / cb;
        float best = 1e9;
        for (int it = 0; it < 5; ++it) {
          cudaEventRecord(a);
          k<<<grid, 64, smem>>>(tm, buf, chunks, cb, stages);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (ms < best) best = ms;
        }
        long long moved = (chunks / grid) * grid * (long long)cb;
        printf("grid=%3d %s chunk=%6d stages=%2d  %7.0f GB/s  %6.1f GB/s/SM (%s)\n", grid,
               mode == 0 ? "bulk1d" : "tma2d ", cb, stages, moved / (best * 1e-3) / 1e9,
               moved / (best * 1e-3) / 1e9 / grid, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
