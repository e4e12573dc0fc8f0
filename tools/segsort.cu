// The MTTKRP scatter two ways, measured on C2's shapes (d = 4, n_k = 200,
// r = 16 fp32, 1.6e7 samples per step; factors and 32 gradient replicas
// L2/L1-resident) with the sampling and model evaluation left out:
//   atomic: per sample and mode, the leave-one-out row product and four
//           red.global.add.v4.f32 lanes (the engine's phase B scatter);
//   sorted: per block, chunks of 2048 samples counting-sorted by each mode's
//           row in shared memory (native integer smem atomics), then groups of
//           4 lanes walk 32 consecutive sorted samples accumulating in
//           registers and issue one vector reduction per run of equal rows.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o segsort tools/segsort.cu && ./segsort
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

constexpr int D = 4, N = 200, R = 16, REPS = 32, S = 2048, TPB = 256;

__device__ __forceinline__ void red4(float* p, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ float4 mul4(float4 a, float4 b) {
  return make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w);
}

// idx: 4 x u8 packed per sample; y: weight * loss derivative per sample
__global__ void __launch_bounds__(TPB) atomic_kernel(const float* __restrict__ A,
                                                     const uint32_t* __restrict__ idx,
                                                     const float* __restrict__ y, int64_t n,
                                                     float* G) {
  const int c = threadIdx.x & 3;
  float* Gb = G + (blockIdx.x % REPS) * D * N * R;
  for (int64_t s = (blockIdx.x * (int64_t)TPB + threadIdx.x) >> 2; s < n;
       s += ((int64_t)gridDim.x * TPB) >> 2) {
    const uint32_t p = __ldg(idx + s);
    const float ys = __ldg(y + s);
    float4 row[D];
#pragma unroll
    for (int k = 0; k < D; ++k)
      row[k] = __ldg(reinterpret_cast<const float4*>(A + (k * N + ((p >> (8 * k)) & 255)) * R) + c);
    float4 pre[D];
    pre[0] = make_float4(ys, ys, ys, ys);
#pragma unroll
    for (int k = 1; k < D; ++k) pre[k] = mul4(pre[k - 1], row[k - 1]);
    float4 suf = make_float4(1.f, 1.f, 1.f, 1.f);
#pragma unroll
    for (int k = D - 1; k >= 0; --k) {
      red4(Gb + (k * N + ((p >> (8 * k)) & 255)) * R + 4 * c, mul4(pre[k], suf));
      suf = mul4(suf, row[k]);
    }
  }
}

__global__ void __launch_bounds__(TPB) sorted_kernel(const float* __restrict__ A,
                                                     const uint32_t* __restrict__ idx,
                                                     const float* __restrict__ y, int64_t n,
                                                     float* G) {
  __shared__ uint32_t sidx[S];
  __shared__ float sy[S];
  __shared__ uint16_t perm[S];
  __shared__ uint16_t rnk[S];
  __shared__ int hist[N];
  const int c = threadIdx.x & 3;
  const int grp = threadIdx.x >> 2;  // 64 groups of 4 lanes, 32 sorted samples each
  float* Gb = G + (blockIdx.x % REPS) * D * N * R;
  const int64_t nchunks = (n + S - 1) / S;
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int64_t base = ch * S;
    const int cnt = (int)((n - base) < S ? (n - base) : S);
    for (int t = threadIdx.x; t < S; t += TPB) {
      sidx[t] = t < cnt ? __ldg(idx + base + t) : 0u;
      sy[t] = t < cnt ? __ldg(y + base + t) : 0.f;
    }
    for (int k = 0; k < D; ++k) {
      for (int t = threadIdx.x; t < N; t += TPB) hist[t] = 0;
      __syncthreads();
      for (int t = threadIdx.x; t < S; t += TPB)
        rnk[t] = (uint16_t)atomicAdd(&hist[(sidx[t] >> (8 * k)) & 255], 1);
      __syncthreads();
      if (threadIdx.x < 32) {  // exclusive scan of the N bucket counts by one warp
        constexpr int PER = (N + 31) / 32;
        int loc[PER], sum = 0;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
          const int b = threadIdx.x * PER + j;
          loc[j] = b < N ? hist[b] : 0;
          sum += loc[j];
        }
        int incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (threadIdx.x >= o) incl += v;
        }
        int run = incl - sum;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
          const int b = threadIdx.x * PER + j;
          if (b < N) hist[b] = run;
          run += loc[j];
        }
      }
      __syncthreads();
      for (int t = threadIdx.x; t < S; t += TPB)
        perm[hist[(sidx[t] >> (8 * k)) & 255] + rnk[t]] = (uint16_t)t;
      __syncthreads();
      // segmented walk: group grp owns sorted positions [32 grp, 32 grp + 32)
      int cur = -1;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int q = 0; q < S / (TPB / 4); ++q) {
        const int pos = grp * (S / (TPB / 4)) + q;
        if (pos >= cnt) break;
        const int s = perm[pos];
        const uint32_t p = sidx[s];
        const int rowk = (p >> (8 * k)) & 255;
        float4 prod = make_float4(sy[s], sy[s], sy[s], sy[s]);
#pragma unroll
        for (int kk = 0; kk < D; ++kk)
          if (kk != k)
            prod = mul4(prod, __ldg(reinterpret_cast<const float4*>(
                                        A + (kk * N + ((p >> (8 * kk)) & 255)) * R) + c));
        if (rowk != cur) {
          if (cur >= 0) red4(Gb + (k * N + cur) * R + 4 * c, acc);
          cur = rowk;
          acc = prod;
        } else {
          acc.x += prod.x, acc.y += prod.y, acc.z += prod.z, acc.w += prod.w;
        }
      }
      if (cur >= 0) red4(Gb + (k * N + cur) * R + 4 * c, acc);
      __syncthreads();
    }
  }
}

int main() {
  const int64_t n = 16'000'000;
  std::vector<uint32_t> hidx(n);
  std::vector<float> hy(n), hA(D * N * R);
  srand(1);
  for (int64_t s = 0; s < n; ++s) {
    uint32_t p = 0;
    for (int k = 0; k < D; ++k) p |= (uint32_t)(rand() % N) << (8 * k);
    hidx[s] = p;
    hy[s] = (rand() % 1000) * 1e-3f;  // positive: the comparison below is not dominated by cancellation
  }
  for (auto& a : hA) a = (rand() % 1000) * 1e-3f;
  float *A, *y, *G1, *G2;
  uint32_t* idx;
  cudaMalloc(&A, hA.size() * 4);
  cudaMalloc(&y, n * 4);
  cudaMalloc(&idx, n * 4);
  cudaMalloc(&G1, REPS * D * N * R * 4);
  cudaMalloc(&G2, REPS * D * N * R * 4);
  cudaMemcpy(A, hA.data(), hA.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(y, hy.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(idx, hidx.data(), n * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int variant = 0; variant < 2; ++variant) {
    float* G = variant ? G2 : G1;
    for (int bps : {2, 4, 8}) {
      const int grid = 148 * bps;
      cudaMemset(G, 0, REPS * D * N * R * 4);
      if (variant) sorted_kernel<<<grid, TPB>>>(A, idx, y, n, G);
      else atomic_kernel<<<grid, TPB>>>(A, idx, y, n, G);
      cudaEventRecord(a);
      for (int it = 0; it < 5; ++it) {
        if (variant) sorted_kernel<<<grid, TPB>>>(A, idx, y, n, G);
        else atomic_kernel<<<grid, TPB>>>(A, idx, y, n, G);
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, a, b);
      printf("%s blocks/SM %d: %.3f ms per 1.6e7 samples (%s)\n", variant ? "sorted" : "atomic",
             bps, ms / 5, cudaGetErrorString(cudaGetLastError()));
    }
  }
  // both variants summed the same samples 6 times (one warm-up + 5): compare
  std::vector<float> g1(REPS * D * N * R), g2(g1.size());
  cudaMemcpy(g1.data(), G1, g1.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(g2.data(), G2, g2.size() * 4, cudaMemcpyDeviceToHost);
  double num = 0, den = 0;
  for (int e = 0; e < D * N * R; ++e) {
    double s1 = 0, s2 = 0;
    for (int q = 0; q < REPS; ++q) s1 += g1[q * D * N * R + e], s2 += g2[q * D * N * R + e];
    num += (s1 - s2) * (s1 - s2);
    den += s1 * s1;
  }
  printf("relative difference of the summed gradients: %.3g\n", den > 0 ? sqrt(num / den) : 0.0);
  return 0;
}
