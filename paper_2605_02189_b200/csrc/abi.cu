// C-ABI utilities: version, error strings, TMA descriptor encoding, pinned
// host memory, batched KV block copies for the offload engine.
#include <cudaTypedefs.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <thread>
#include <vector>

#include "common.cuh"

extern "C" int pm_abi_version(void) { return 1; }

extern "C" const char* pm_error_string(int code) {
  return cudaGetErrorString(static_cast<cudaError_t>(code));
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D bf16 tensor map over a row-major matrix [outer][inner] whose rows are
// `row_stride_bytes` apart; box = [box_outer][box_inner]; swizzle128 selects
// the 128-byte swizzle (box_inner*2 must then be 128).  Writes 128 bytes.
extern "C" int pm_tmap_encode_2d(void* tmap_out, const void* gaddr, unsigned long long inner,
                                 unsigned long long outer, unsigned long long row_stride_bytes,
                                 unsigned box_inner, unsigned box_outer, int swizzle128) {
  auto enc = get_encode();
  if (!enc) return (int)cudaErrorNotSupported;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(reinterpret_cast<CUtensorMap*>(tmap_out), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(gaddr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)cudaErrorInvalidValue;
}

// 5-D bf16 tensor map over the block-first KV pool [rows = block*16 + slot][L_s][k|v][Hkv][hd]
// whose box is one KV block's K and V of one (layer, kv head) -- 16 slots x hd, both halves of
// 64 dims, K and V -- in ONE copy: dims (innermost first) {64 dims, rows, hd/64 halves, k|v,
// L_s*2*Hkv head columns}, byte strides {row pitch, 128, Hkv*hd*2, hd*2}, box {64, 16, hd/64,
// 2, 1}, 128B swizzle.  The copy lands as [k|v][half][16 slots][128 B] -- the same shared
// image the four 2-D boxes of pm_tmap_encode_2d produce -- at coordinates
// (0, block*16, 0, 0, layer*2*Hkv + kv_head) (the k|v coordinate steps Hkv head columns).
extern "C" int pm_tmap_encode_pool(void* tmap_out, const void* pool, unsigned long long n_rows, int L_s, int Hkv,
                                   int hd) {
  auto enc = get_encode();
  if (!enc) return (int)cudaErrorNotSupported;
  if (hd % 64 || L_s < 1 || Hkv < 1) return (int)cudaErrorInvalidValue;
  const unsigned long long pitch = (unsigned long long)L_s * 2 * Hkv * hd * 2;
  cuuint64_t dims[5] = {64, n_rows, (cuuint64_t)(hd / 64), 2, (cuuint64_t)L_s * 2 * Hkv};
  cuuint64_t strides[4] = {pitch, 128, (cuuint64_t)Hkv * hd * 2, (cuuint64_t)hd * 2};
  cuuint32_t box[5] = {64, 16, (cuuint32_t)(hd / 64), 2, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(reinterpret_cast<CUtensorMap*>(tmap_out), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5,
                   const_cast<void*>(pool), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)cudaErrorInvalidValue;
}

// Pitched copy (cudaMemcpy2DAsync): `height` rows of `width` bytes, row
// strides dpitch / spitch -- one layer's K/V of a run of tokens between the
// pool and the host replica (token stride = the pitch).
// The pinned replica is registered in 1 GB pieces aligned to 1 GB (see
// pm_host_alloc_numa) and a single cudaMemcpy may not span two registrations,
// so host-side copies are cut at absolute 1 GB boundaries of either pointer
// (harmless for device pointers).
static constexpr unsigned long long PIN_CHUNK = 1ull << 30;
static inline unsigned long long to_piece_end(const void* p) {
  return PIN_CHUNK - (reinterpret_cast<unsigned long long>(p) & (PIN_CHUNK - 1));
}
static cudaError_t copy_1d(void* dst, const void* src, unsigned long long n, cudaStream_t st) {
  while (n) {
    const unsigned long long m = std::min(n, std::min(to_piece_end(dst), to_piece_end(src)));
    cudaError_t e = cudaMemcpyAsync(dst, src, m, cudaMemcpyDefault, st);
    if (e != cudaSuccess) return e;
    dst = static_cast<char*>(dst) + m;
    src = static_cast<const char*>(src) + m;
    n -= m;
  }
  return cudaSuccess;
}

extern "C" int pm_copy_2d(void* dst, unsigned long long dpitch, const void* src, unsigned long long spitch,
                          unsigned long long width, unsigned long long height, void* stream) {
  auto st = reinterpret_cast<cudaStream_t>(stream);
  unsigned long long r = 0;
  while (r < height) {
    char* d = static_cast<char*>(dst) + r * dpitch;
    const char* sp = static_cast<const char*>(src) + r * spitch;
    const unsigned long long ed = to_piece_end(d), es = to_piece_end(sp);
    cudaError_t e;
    if (width > ed || width > es) {   // this row straddles a piece boundary
      e = copy_1d(d, sp, width, st);
      r += 1;
    } else {   // rows that end before the next boundary on both sides
      unsigned long long k = height - r;
      k = std::min(k, (ed - width) / dpitch + 1);
      k = std::min(k, (es - width) / spitch + 1);
      e = cudaMemcpy2DAsync(d, dpitch, sp, spitch, width, k, cudaMemcpyDefault, st);
      r += k;
    }
    if (e != cudaSuccess) return (int)e;
  }
  return 0;
}

// Pinned, portable host memory for the KV host replica (the paper's "CPU KV
// pool").  The caller owns it and frees it with pm_host_free.
// Pinning large host ranges fails intermittently on some boxes with
// cudaErrorOperatingSystem (measured: 8-48 GB requests failing at random,
// tools/diag_pinned.sh), so pinned allocations retry, and the replica is pinned
// in 1 GB pieces (each retried) rather than as one multi-GB registration.
static cudaError_t host_alloc_retry(void** out, unsigned long long bytes) {
  cudaError_t e = cudaSuccess;
  for (int attempt = 0; attempt < 8; ++attempt) {
    e = cudaHostAlloc(out, bytes, cudaHostAllocPortable | cudaHostAllocMapped);
    if (e == cudaSuccess) return e;
    cudaGetLastError();
    usleep(20000 * (attempt + 1));
  }
  return e;
}

extern "C" int pm_host_alloc(unsigned long long bytes, void** out) {
  return (int)host_alloc_retry(out, bytes);
}
// NUMA node of a CUDA device's PCIe attachment (sysfs), -1 when unknown.
extern "C" int pm_device_numa_node(int device, int* node) {
  *node = -1;
  char bus[32];
  cudaError_t e = cudaDeviceGetPCIBusId(bus, sizeof(bus), device);
  if (e != cudaSuccess) return (int)e;
  for (char* c = bus; *c; ++c)
    if (*c >= 'A' && *c <= 'F') *c = (char)(*c - 'A' + 'a');
  char path[128];
  snprintf(path, sizeof(path), "/sys/bus/pci/devices/%s/numa_node", bus);
  FILE* f = fopen(path, "r");
  if (!f) return 0;
  int n = -1;
  if (fscanf(f, "%d", &n) != 1) n = -1;
  fclose(f);
  *node = n;
  return 0;
}

// Pinned, mapped host memory placed on NUMA node `numa_node` (the node the
// GPU's PCIe root hangs off, pm_device_numa_node): anonymous mmap, mbind
// (MPOL_BIND) before first touch, then cudaHostRegister (portable | mapped) in
// 1 GB pieces, each retried.  If a piece cannot be pinned the range falls back
// to cudaHostAlloc (no NUMA placement).  numa_node < 0: plain pm_host_alloc.
// The range is contiguous and fully pinned either way; its mapped device
// address (pm_host_device_ptr) covers the first piece only.  Free with
// pm_host_free_numa.
extern "C" int pm_host_alloc_numa(unsigned long long bytes, int numa_node, void** out) {
  if (numa_node < 0) return (int)host_alloc_retry(out, bytes);
  // reserve one piece more and trim, so the range starts on a 1 GB boundary
  const unsigned long long page = 4096, len = (bytes + page - 1) / page * page;
  void* raw = mmap(nullptr, len + PIN_CHUNK, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (raw == MAP_FAILED) return (int)host_alloc_retry(out, bytes);
  const unsigned long long r0 = reinterpret_cast<unsigned long long>(raw);
  const unsigned long long b0 = (r0 + PIN_CHUNK - 1) & ~(PIN_CHUNK - 1);
  if (b0 > r0) munmap(raw, b0 - r0);
  if (r0 + PIN_CHUNK > b0) munmap(reinterpret_cast<void*>(b0 + len), r0 + PIN_CHUNK - b0);
  void* p = reinterpret_cast<void*>(b0);
  unsigned long mask[16] = {0};
  if (numa_node < 16 * 64) {
    mask[numa_node / 64] = 1ul << (numa_node % 64);
    // MPOL_BIND = 2; a failure (no NUMA support in the kernel / container) leaves the default policy
    syscall(SYS_mbind, p, bytes, 2, mask, (unsigned long)(16 * 64), 0u);
  }
  unsigned long long done = 0;
  while (done < bytes) {
    const unsigned long long n = bytes - done < PIN_CHUNK ? bytes - done : PIN_CHUNK;
    cudaError_t e = cudaErrorUnknown;
    for (int attempt = 0; attempt < 8 && e != cudaSuccess; ++attempt) {
      e = cudaHostRegister(static_cast<char*>(p) + done, n, cudaHostRegisterPortable | cudaHostRegisterMapped);
      if (e != cudaSuccess) {
        cudaGetLastError();
        usleep(20000 * (attempt + 1));
      }
    }
    if (e != cudaSuccess) {   // give the range back and use the driver's allocation instead
      for (unsigned long long o = 0; o < done; o += PIN_CHUNK) cudaHostUnregister(static_cast<char*>(p) + o);
      munmap(p, len);
      return (int)host_alloc_retry(out, bytes);
    }
    done += n;
  }
  *out = p;
  return 0;
}
extern "C" int pm_host_free_numa(void* p, unsigned long long bytes, int numa_node) {
  if (numa_node < 0) return (int)cudaFreeHost(p);
  cudaError_t e = cudaHostUnregister(p);
  if (e != cudaSuccess) {   // the cudaHostAlloc fallback of pm_host_alloc_numa
    cudaGetLastError();
    return (int)cudaFreeHost(p);
  }
  for (unsigned long long o = PIN_CHUNK; o < bytes; o += PIN_CHUNK) cudaHostUnregister(static_cast<char*>(p) + o);
  munmap(p, (bytes + 4095) / 4096 * 4096);
  return 0;
}

// Device-side address of pinned host memory from pm_host_alloc (zero-copy reads).
extern "C" int pm_host_device_ptr(void* host, void** dev) {
  return (int)cudaHostGetDevicePointer(dev, host, 0);
}

namespace {
constexpr int MAX_META_SEGS = 8;
struct MetaSegs {
  int* dst[MAX_META_SEGS];
  const int* src[MAX_META_SEGS];   // device addresses of mapped pinned host memory
  int n[MAX_META_SEGS];
  int count;
};
// One CTA per segment streams it from pinned host memory over PCIe with
// 16-byte loads (the step's block tables / positions / work list).  A kernel,
// not cudaMemcpyAsync: the copy engines are busy with KV prefetch DMAs, and a
// small metadata copy queued behind a 100+ MB prefetch would stall the
// compute stream for milliseconds.
__global__ void __launch_bounds__(512) meta_upload_kernel(MetaSegs m) {
  const int s = blockIdx.x;
  if (s >= m.count) return;
  const int n = m.n[s];
  const int* src = m.src[s];
  int* dst = m.dst[s];
  const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  const int n4 = vec ? n / 4 : 0;
  for (int i = threadIdx.x; i < n4; i += blockDim.x)
    reinterpret_cast<int4*>(dst)[i] = __ldcv(reinterpret_cast<const int4*>(src) + i);  // no caching: host rewrites it
  for (int i = n4 * 4 + threadIdx.x; i < n; i += blockDim.x) dst[i] = __ldcv(src + i);
}
}  // namespace

// dst[i][0..n[i]) <- src[i][0..n[i]) (int32), src = device addresses of mapped
// pinned host memory (pm_host_device_ptr), on `stream` (<= 8 segments).
extern "C" int pm_meta_upload(int count, void* const* dst, const void* const* src, const int* n, void* stream) {
  if (count < 0 || count > MAX_META_SEGS) return (int)cudaErrorInvalidValue;
  if (count == 0) return 0;
  MetaSegs m{};
  for (int i = 0; i < count; ++i) {
    m.dst[i] = static_cast<int*>(dst[i]);
    m.src[i] = static_cast<const int*>(src[i]);
    m.n[i] = n[i];
  }
  m.count = count;
  // launched WITHOUT programmatic dependent launch: the step's kernels read
  // this metadata before their griddepcontrol.wait (attention, fused QKV), so
  // the dependent chain must start only after the upload has completed
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(count);
  cfg.blockDim = dim3(512);
  cfg.stream = reinterpret_cast<cudaStream_t>(stream);
  return (int)cudaLaunchKernelEx(&cfg, meta_upload_kernel, m);
}
extern "C" int pm_host_free(void* p) { return (int)cudaFreeHost(p); }

namespace {
// Eager decode offload (REF pipeline_sim.py:486-490): every row's new-token
// KV (one contiguous `bytes` run in the block-first pool) is written straight
// into its request's host-replica slot through the mapped pinned mapping --
// one kernel instead of one DMA per row (the per-copy DMA setup capped the
// copy engines near 10-14 GB/s on ~150 KB pieces).  offs[2i] = host offset,
// offs[2i+1] = pool offset (mapped pinned memory, read over PCIe).
__global__ void __launch_bounds__(256) offload_rows_kernel(uint8_t* __restrict__ host, const uint8_t* __restrict__ pool,
                                                           const long long* __restrict__ offs, int n,
                                                           unsigned long long bytes) {
  const unsigned long long chunks = (bytes + 4095) / 4096;   // 4 KB per CTA iteration (256 x 16 B)
  for (unsigned long long w = blockIdx.x; w < (unsigned long long)n * chunks; w += gridDim.x) {
    const int row = (int)(w / chunks);
    const unsigned long long c = (w % chunks) * 4096 + threadIdx.x * 16ull;
    if (c >= bytes) continue;
    const long long ho = __ldcv(offs + 2 * row), po = __ldcv(offs + 2 * row + 1);
    const uint4 v = __ldcg(reinterpret_cast<const uint4*>(pool + po + c));
    *reinterpret_cast<uint4*>(host + ho + c) = v;
  }
}
}  // namespace

// host_dev: device address of the mapped replica (pm_host_device_ptr); offs:
// device address of mapped pinned int64 pairs (host offset, pool offset);
// bytes % 16 == 0.  `ctas` CTAs (a few suffice for PCIe rate; they co-reside
// with the forward's kernels).
extern "C" int pm_offload_rows(void* host_dev, const void* pool, const void* offs, int n, unsigned long long bytes,
                               int ctas, void* stream) {
  if (bytes % 16 || n < 0) return (int)cudaErrorInvalidValue;
  if (n == 0) return 0;
  offload_rows_kernel<<<ctas > 0 ? ctas : 32, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      static_cast<uint8_t*>(host_dev), static_cast<const uint8_t*>(pool), static_cast<const long long*>(offs), n,
      bytes);
  return (int)cudaGetLastError();
}

// Decode offload in one DMA (REF pipeline_sim.py:486-490).  Each row's new-
// token KV is one contiguous `bytes` run of the block-first pool; the rows of
// a step land at scattered host-replica offsets.  Instead of one small DMA per
// row, a gather kernel packs the rows into a device staging slab, ONE
// cudaMemcpyAsync moves the slab to pinned host staging, and a host function
// enqueued behind it (cudaLaunchHostFunc, stream order) scatters the rows into
// the replica -- so an event recorded on `stream` afterwards means "replica
// complete", exactly like the per-row copies.  Offsets travel by value.
namespace {
constexpr int GATHER_MAX = 2048;
struct GatherRows {
  long long pool_off[GATHER_MAX];
};
__global__ void __launch_bounds__(256) gather_rows_kernel(uint8_t* __restrict__ stage, const uint8_t* __restrict__ pool,
                                                          const __grid_constant__ GatherRows g, int n,
                                                          unsigned long long bytes) {
  const unsigned long long per_row = bytes / 16, total = per_row * (unsigned long long)n;
  for (unsigned long long i = blockIdx.x * 256ull + threadIdx.x; i < total; i += gridDim.x * 256ull) {
    const int row = (int)(i / per_row);
    const unsigned long long c = (i - row * per_row) * 16;
    *reinterpret_cast<uint4*>(stage + row * bytes + c) = __ldcs(reinterpret_cast<const uint4*>(pool + g.pool_off[row] + c));
  }
}
struct ScatterCtx {
  uint8_t* replica;
  const uint8_t* stage;
  unsigned long long bytes;
  int n;
  long long rep_off[1];   // n entries
};
// Host scatter of the staged rows.  One host thread copies ~6-8 GB/s between
// pinned buffers, so large steps are split over a few threads (no CUDA calls
// inside a host function).
void CUDART_CB scatter_rows(void* p) {
  ScatterCtx* c = static_cast<ScatterCtx*>(p);
  const size_t total = (size_t)c->n * c->bytes;
  const int nt = total >= (8u << 20) ? 4 : (total >= (2u << 20) ? 2 : 1);
  auto part = [c, nt](int t) {
    for (int i = t; i < c->n; i += nt) memcpy(c->replica + c->rep_off[i], c->stage + (size_t)i * c->bytes, c->bytes);
  };
  std::vector<std::thread> th;
  for (int t = 1; t < nt; ++t) th.emplace_back(part, t);
  part(0);
  for (auto& x : th) x.join();
  free(c);
}
}  // namespace

// replica: host address of the pinned replica; rep_off/pool_off: host arrays
// of n byte offsets; dev_stage / host_stage: n * bytes of device memory /
// pinned host memory, not reused until this call's work on `stream` is done
// (stream order).  bytes % 16 == 0.
extern "C" int pm_offload_gather(void* replica, const void* pool, const long long* rep_off, const long long* pool_off,
                                 int n, unsigned long long bytes, void* dev_stage, void* host_stage, void* stream) {
  if (bytes % 16 || n < 0) return (int)cudaErrorInvalidValue;
  if (n == 0) return 0;
  auto st = reinterpret_cast<cudaStream_t>(stream);
  for (int r0 = 0; r0 < n; r0 += GATHER_MAX) {
    const int k = n - r0 < GATHER_MAX ? n - r0 : GATHER_MAX;
    GatherRows g;
    for (int i = 0; i < k; ++i) g.pool_off[i] = pool_off[r0 + i];
    const unsigned long long chunks = bytes / 16 * (unsigned long long)k;
    const int grid = (int)((chunks + 255) / 256 < 296 ? (chunks + 255) / 256 : 296);
    gather_rows_kernel<<<grid, 256, 0, st>>>(static_cast<uint8_t*>(dev_stage) + (size_t)r0 * bytes,
                                             static_cast<const uint8_t*>(pool), g, k, bytes);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return (int)e;
  }
  cudaError_t e = cudaMemcpyAsync(host_stage, dev_stage, (size_t)n * bytes, cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return (int)e;
  ScatterCtx* c = static_cast<ScatterCtx*>(malloc(sizeof(ScatterCtx) + sizeof(long long) * (size_t)n));
  if (!c) return (int)cudaErrorMemoryAllocation;
  c->replica = static_cast<uint8_t*>(replica);
  c->stage = static_cast<const uint8_t*>(host_stage);
  c->bytes = bytes;
  c->n = n;
  memcpy(c->rep_off, rep_off, sizeof(long long) * (size_t)n);
  e = cudaLaunchHostFunc(st, scatter_rows, c);
  if (e != cudaSuccess) free(c);
  return (int)e;
}

// Batched copies of equal-sized KV pieces between two base addresses:
// dst_base + dst_off[i] <- src_base + src_off[i], `bytes` each, in order, on
// `stream` (a copy-engine stream of the offload engine).  Adjacent pieces
// that are contiguous on both sides are merged into one transfer, so a run
// of consecutive blocks of one request moves as a single DMA.
extern "C" int pm_copy_pieces(void* dst_base, const void* src_base, const long long* dst_off,
                              const long long* src_off, int n, unsigned long long bytes, void* stream) {
  auto st = reinterpret_cast<cudaStream_t>(stream);
  std::vector<void*> dsts, srcs;
  std::vector<size_t> sizes;
  int i = 0;
  while (i < n) {
    int j = i + 1;
    while (j < n && dst_off[j] == dst_off[j - 1] + (long long)bytes &&
           src_off[j] == src_off[j - 1] + (long long)bytes)
      ++j;
    dsts.push_back(static_cast<char*>(dst_base) + dst_off[i]);
    srcs.push_back(const_cast<char*>(static_cast<const char*>(src_base)) + src_off[i]);
    sizes.push_back(bytes * (size_t)(j - i));
    i = j;
  }
  for (size_t k = 0; k < dsts.size(); ++k) {
    cudaError_t e = copy_1d(dsts[k], srcs[k], sizes[k], st);
    if (e != cudaSuccess) return (int)e;
  }
  return 0;
}
