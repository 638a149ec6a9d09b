// Probe: per-SM HBM -> shared-memory streaming rate of one CTA per SM, as a
// function of the number of CTAs and the copy path:
//   mode 0: cp.async.bulk (TMA bulk) chunks of `chunk` bytes, `stages` deep
//   mode 1: cp.async (LDGSTS, 16 B per thread, 256 threads) into the same ring
//   mode 2: ld.global.nc.v4 by 256 threads into registers (no smem), 8 loads in flight per thread
// Each CTA streams a disjoint contiguous region; prints per-CTA and total GB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/sm_stream_probe tools/sm_stream_probe.cu
#include <cstdio>
#include <vector>

#include "../paper_2605_02189_b200/csrc/common.cuh"

PM_DEV void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(256, 1) probe_bulk(const uint8_t* base, long long bytes_per_cta, int chunk,
                                                     int stages, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * chunk);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  const uint8_t* src = base + bytes_per_cta * blockIdx.x;
  const long long n = bytes_per_cta / chunk;
  if (threadIdx.x == 0) {
    for (long long i = 0; i < n; ++i) {
      const int s = i % stages;
      if (i >= stages) mbar_wait(&empty[s], ((i / stages) - 1) & 1);
      mbar_arrive_expect_tx(&full[s], chunk);
      bulk_load(smem + s * chunk, src + i * chunk, chunk, &full[s]);
    }
  } else if (threadIdx.x == 32) {
    unsigned long long acc = 0;
    for (long long i = 0; i < n; ++i) {
      const int s = i % stages;
      mbar_wait(&full[s], (i / stages) & 1);
      acc += smem[s * chunk + (i & 1023)];
      mbar_arrive(&empty[s]);
    }
    sink[blockIdx.x] = acc;
  }
}

__global__ void __launch_bounds__(256, 1) probe_ldgsts(const uint8_t* base, long long bytes_per_cta, int chunk,
                                                       int stages, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint8_t* src = base + bytes_per_cta * blockIdx.x;
  const long long n = bytes_per_cta / chunk;
  const int per_thread = chunk / (256 * 16);
  unsigned long long acc = 0;
  // prologue: stages-1 chunks in flight
  for (long long i = 0; i < n + stages - 1; ++i) {
    if (i < n) {
      const int s = i % stages;
      for (int j = 0; j < per_thread; ++j) {
        const int off = (j * 256 + threadIdx.x) * 16;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem + s * chunk + off)),
                     "l"(src + i * chunk + off) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (i >= stages - 1) {
      asm volatile("cp.async.wait_group %0;" ::"n"(0) : "memory");   // conservative: drain (probe only)
      __syncthreads();
      acc += smem[((i - stages + 1) % stages) * chunk + threadIdx.x];
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) sink[blockIdx.x] = acc;
}

// mode 3: bulk chunks issued by P producer warps (warp w issues the stages s % P == w)
__global__ void __launch_bounds__(256, 1) probe_bulk_multi(const uint8_t* base, long long bytes_per_cta, int chunk,
                                                           int stages, int P, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * chunk);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  const uint8_t* src = base + bytes_per_cta * blockIdx.x;
  const long long n = bytes_per_cta / chunk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < P && lane == 0) {
    for (long long i = warp; i < n; i += P) {
      const int s = i % stages;
      if (i >= stages) mbar_wait(&empty[s], ((i / stages) - 1) & 1);
      mbar_arrive_expect_tx(&full[s], chunk);
      bulk_load(smem + s * chunk, src + i * chunk, chunk, &full[s]);
    }
  } else if (warp == 7 && lane == 0) {
    unsigned long long acc = 0;
    for (long long i = 0; i < n; ++i) {
      const int s = i % stages;
      mbar_wait(&full[s], (i / stages) & 1);
      acc += smem[s * chunk + (i & 1023)];
      mbar_arrive(&empty[s]);
    }
    sink[blockIdx.x] = acc;
  }
}

template <int DEPTH>
__global__ void __launch_bounds__(256, 1) probe_ldg(const uint8_t* base, long long bytes_per_cta,
                                                    unsigned long long* sink) {
  const uint4* src = reinterpret_cast<const uint4*>(base + bytes_per_cta * blockIdx.x);
  const long long n = bytes_per_cta / 16;
  unsigned acc = 0;
  for (long long i = threadIdx.x; i < n; i += 256 * DEPTH) {
    uint4 v[DEPTH];
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) {
      const long long k = i + (long long)d * 256;
      if (k < n) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                              : "=r"(v[d].x), "=r"(v[d].y), "=r"(v[d].z), "=r"(v[d].w) : "l"(src + k));
      else v[d] = make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) acc ^= v[d].x ^ v[d].w;
  }
  if (acc == 0x12345678) sink[blockIdx.x] = acc;
}

int main() {
  const size_t total = 4ull << 30;   // 4 GB region (> L2)
  uint8_t* buf;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  unsigned long long* sink;
  cudaMalloc(&sink, 4096 * 8);
  cudaFuncSetAttribute(probe_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(probe_ldgsts, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(probe_bulk_multi, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int grids[] = {8, 74, 148};
  struct Cfg { int mode, chunk, stages; };
  const Cfg cfgs[] = {{0, 4096, 16}, {0, 8192, 16}, {0, 16384, 12}, {0, 32768, 6}, {0, 65536, 3},
                      {0, 131072, 1}, {3, 16384, 12}, {4, 16384, 12}, {5, 8192, 16}, {6, 32768, 6}};
  for (const Cfg& c : cfgs) {
    for (int g : grids) {
      const long long per = (long long)(total / 2 / g) & ~((long long)65535);
      float best = 1e9f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        if (c.mode == 0)
          probe_bulk<<<g, 256, c.chunk * c.stages + 1024>>>(buf, per, c.chunk, c.stages, sink);
        else if (c.mode == 1)
          probe_ldgsts<<<g, 256, c.chunk * c.stages + 1024>>>(buf, per, c.chunk, c.stages, sink);
        else if (c.mode >= 3)   // 3: 2 producer warps, 4: 4 warps, 5: 4 warps (8 KB), 6: 2 warps (32 KB)
          probe_bulk_multi<<<g, 256, c.chunk * c.stages + 1024>>>(buf, per, c.chunk, c.stages,
                                                                  c.mode == 3 || c.mode == 6 ? 2 : 4, sink);
        else if (c.stages == 4)
          probe_ldg<4><<<g, 256>>>(buf, per, sink);
        else
          probe_ldg<8><<<g, 256>>>(buf, per, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
      }
      const cudaError_t e = cudaGetLastError();
      const double tot = (double)per * g / (best * 1e-3) / 1e9;
      printf("mode %d chunk %6d stages %2d grid %3d: per-CTA %6.1f GB/s  total %7.1f GB/s %s\n", c.mode, c.chunk,
             c.stages, g, tot / g, tot, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  return 0;
}
