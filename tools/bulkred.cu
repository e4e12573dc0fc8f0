// Scatter-add microbenchmark for C2's gradient (800 rows x 64 B, 32 L2-resident
// replicas): is one TMA bulk reduction per 64-byte row (cp.reduce.async.bulk
// from shared memory) cheaper than four 16-byte red.global.add.v4.f32 lanes?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulkred tools/bulkred.cu && ./bulkred
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix32(uint32_t z) {
  z ^= z >> 16;
  z *= 0x7feb352dU;
  z ^= z >> 15;
  z *= 0x846ca68bU;
  return z ^ (z >> 16);
}

constexpr int ROWS = 800, RF = 16, REPS = 32;

// MODE 0: 4 lanes x red.global.add.v4.f32 per row (the engine today)
// MODE 1: every lane stages one whole row in shared memory, one bulk reduce per lane
// MODE 2: 4 lanes stage a row (one 16-byte chunk each), lane 0 of 4 issues the bulk reduce
// MODE 3: 4 lanes x 4 scalar atomicAdd (shared) into a per-block shared copy of
//         the whole gradient (51 KB, dynamic smem), flushed with red.global at the end
template <int MODE>
__global__ void __launch_bounds__(256) kern(float* G, int64_t n, uint32_t seed) {
  __shared__ __align__(128) float stage[MODE == 3 ? 1 : 2][MODE == 3 ? 1 : 256][RF];
  extern __shared__ float sg[];
  if (MODE == 3) {
    for (int e = threadIdx.x; e < ROWS * RF; e += blockDim.x) sg[e] = 0.f;
    __syncthreads();
  }
  const int lane4 = threadIdx.x & 3;
  float* Gb = G + (blockIdx.x % REPS) * ROWS * RF;
  int buf = 0;
  const int64_t step = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += step) {
    const float y = 1e-30f * static_cast<float>(i & 7);
    if (MODE == 0) {
      const uint32_t row = mix32(seed ^ static_cast<uint32_t>(i >> 2)) % ROWS;
      float* p = Gb + row * RF + lane4 * 4;
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(y), "f"(y), "f"(y),
                   "f"(y)
                   : "memory");
    } else if (MODE == 3) {
      const uint32_t row = mix32(seed ^ static_cast<uint32_t>(i >> 2)) % ROWS;
      float* p = sg + row * RF + lane4 * 4;
#pragma unroll
      for (int e = 0; e < 4; ++e) atomicAdd(p + ((e + lane4) & 3), y);
    } else if (MODE == 1) {
      const uint32_t row = mix32(seed ^ static_cast<uint32_t>(i)) % ROWS;
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      float* s = stage[buf][threadIdx.x];
#pragma unroll
      for (int c = 0; c < 4; ++c)
        *reinterpret_cast<float4*>(s + 4 * c) = make_float4(y, y, y, y);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(s));
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 64;" ::"l"(
                       Gb + row * RF),
                   "r"(sa)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      buf ^= 1;
    } else {
      const uint32_t row = mix32(seed ^ static_cast<uint32_t>(i >> 2)) % ROWS;
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncwarp();
      float* s = stage[buf][threadIdx.x & ~3];
      *reinterpret_cast<float4*>(s + 4 * lane4) = make_float4(y, y, y, y);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane4 == 0) {
        const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(s));
        asm volatile(
            "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 64;" ::"l"(
                Gb + row * RF),
            "r"(sa)
            : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      buf ^= 1;
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (MODE == 3) {
    __syncthreads();
    for (int e = threadIdx.x; e < ROWS * RF; e += blockDim.x) atomicAdd(Gb + e, sg[e]);
  }
}

template <int MODE>
void run(float* G, int64_t rows_total, int blocks_per_sm) {
  const int64_t n = MODE == 1 ? rows_total : rows_total * 4;  // threads-items
  const int grid = 148 * blocks_per_sm;
  const size_t smem = MODE == 3 ? ROWS * RF * sizeof(float) : 0;
  cudaFuncSetAttribute(kern<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  kern<MODE><<<grid, 256, smem>>>(G, n, 1);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int it = 0; it < 5; ++it) kern<MODE><<<grid, 256, smem>>>(G, n, 7 + it);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 5;
  printf("mode %d blocks/SM %d: %.3f ms  %.3g rows/s  (%s)\n", MODE, blocks_per_sm, ms,
         rows_total / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
}

int main() {
  float* G;
  cudaMalloc(&G, sizeof(float) * ROWS * RF * REPS);
  cudaMemset(G, 0, sizeof(float) * ROWS * RF * REPS);
  const int64_t rows_total = 64'000'000;  // C2: 1.6e7 samples x 4 modes
  for (int bps : {2, 4}) {
    if (bps > 0) {
      run<3>(G, rows_total, bps);
      continue;
    }
    run<0>(G, rows_total, bps);
    run<1>(G, rows_total, bps);
    run<2>(G, rows_total, bps);
    run<3>(G, rows_total, bps);
  }
  return 0;
}
