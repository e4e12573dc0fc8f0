// How many DRAM bytes does one small random load cost?  Random 16-byte record
// loads (one per lane) and random 64-byte row loads (4 lanes x 16 B) over an
// 8 GiB table, with different load flavours and cudaLimitMaxL2FetchGranularity
// settings; reports accesses/s (timing) — run under ncu for dram__bytes_read.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fetchgran tools/fetchgran.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
template <int KIND>
__device__ __forceinline__ uint4 ld16(const uint4* p) {
  uint4 v;
  if (KIND == 0) v = __ldg(p);
  else if (KIND == 1) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else if (KIND == 2) asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else if (KIND == 3) asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else if (KIND == 4) asm volatile("ld.global.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else if (KIND == 5) asm volatile("ld.global.L2::128B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else if (KIND == 6) asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else asm volatile("ld.global.lu.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
// LANES = lanes sharing one random position (1: 16-byte records, 4: 64-byte rows, 8: 128-byte lines)
template <int KIND, int LANES>
__global__ void kern(const uint4* tab, int64_t slots, int64_t n, uint32_t* sink, uint64_t seed) {
  const int sub = threadIdx.x % LANES;
  uint32_t acc = 0;
  const int64_t stride = (gridDim.x * (int64_t)blockDim.x) / LANES;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / LANES; i < n; i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t j = i + u * stride;
      const int64_t r = mix(seed + j) % slots;
      v[u] = j < n ? ld16<KIND>(tab + r * LANES + sub) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += v[u].x ^ v[u].w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}
template <int KIND, int LANES>
void run(const char* name, const uint4* tab, int64_t bytes, uint32_t* sink, int bps) {
  const int64_t slots = bytes / (16 * LANES);
  const int64_t n = LANES == 1 ? (1 << 26) : (1 << 25);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(a);
    kern<KIND, LANES><<<148 * bps, 256>>>(tab, slots, n, sink, 1234 + rep);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep && ms < best) best = ms;
  }
  printf("  %-22s %3d B/access  blocks/SM %d: %7.3f ms  %.3g accesses/s  %.0f GB/s useful\n", name,
         16 * LANES, bps, best, n / (best * 1e-3), n * 16.0 * LANES / (best * 1e-3) / 1e9);
}
int main(int argc, char** argv) {
  if (argc > 1) {  // footprint sweep: fetchgran <GiB> [<GiB> ...] -- 16- and 64-byte loads only
    uint32_t* sink;
    cudaMalloc(&sink, 4);
    for (int i = 1; i < argc; ++i) {
      const int64_t bytes = static_cast<int64_t>(atof(argv[i]) * (1ll << 30)) / 4096 * 4096;
      uint4* tab;
      if (cudaMalloc(&tab, bytes) != cudaSuccess) { printf("cudaMalloc(%s GiB) failed\n", argv[i]); continue; }
      cudaMemset(tab, 1, bytes);
      printf("table %s GiB\n", argv[i]);
      run<0, 1>("ld.nc", tab, bytes, sink, 4);
      run<4, 1>("ld.L2::64B", tab, bytes, sink, 4);
      run<0, 4>("ld.nc", tab, bytes, sink, 4);
      run<0, 8>("ld.nc", tab, bytes, sink, 4);
      cudaFree(tab);
    }
    return 0;
  }
  const int64_t bytes = 8ll << 30;
  uint4* tab;
  uint32_t* sink;
  cudaMalloc(&tab, bytes);
  cudaMalloc(&sink, 4);
  cudaMemset(tab, 1, bytes);
  const int lims[] = {-1, 32, 64, 128};
  for (int li = 0; li < 4; ++li) {
    if (lims[li] > 0) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, lims[li]);
    size_t got = 0;
    cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
    printf("cudaLimitMaxL2FetchGranularity = %zu%s\n", got, lims[li] < 0 ? " (default)" : "");
    for (int bps = 4; bps <= 8; bps += 4) {
      run<0, 1>("ld.nc", tab, bytes, sink, bps);
      if (li == 0) {
        run<1, 1>("ld.nc.L1::no_allocate", tab, bytes, sink, bps);
        run<2, 1>("ld.cg", tab, bytes, sink, bps);
        run<3, 1>("ld.cv", tab, bytes, sink, bps);
        run<4, 1>("ld.L2::64B", tab, bytes, sink, bps);
        run<5, 1>("ld.L2::128B", tab, bytes, sink, bps);
        run<6, 1>("ld.cs", tab, bytes, sink, bps);
        run<7, 1>("ld.lu", tab, bytes, sink, bps);
      }
      run<0, 2>("ld.nc", tab, bytes, sink, bps);
      run<0, 4>("ld.nc", tab, bytes, sink, bps);
      run<0, 8>("ld.nc", tab, bytes, sink, bps);
    }
  }
  return 0;
}
