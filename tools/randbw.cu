// Random-access HBM microbenchmark: the practical roofline for C5's access
// pattern (64-byte rows at random positions of a 1 GiB table), for reads,
// for red.global.add.v4.f32 read-modify-writes, and for the mix the fused
// kernel issues (3 row gathers + 3 row reductions per sample).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o randbw tools/randbw.cu && ./randbw
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// mode 0: gather rows; 1: red rows; 2: 3 gathers + 3 reds per "sample";
// 3: as 2, but odd samples first gather a 16-byte nonzero record at a random
// position of a 4 GiB record table and take their rows from it (C5's
// semi-stratified mix: half nonzero picks, half unrestricted draws);
// 4/5: as 2/3 with factor row and gradient row of one table row interleaved
// in one 128-byte line ([A row | G row], pitch 128 B), so a row's gather and
// its reduction hit the same DRAM burst; 6: random 128-byte row gathers.
template <int MODE>
__global__ void kern(float* tab, int64_t rows, int64_t n, float* sink, uint64_t seed,
                     const uint4* rec = nullptr, int64_t nrec = 0) {
  const int lane = threadIdx.x & 3;  // 4 lanes x 16 B = one 64-byte row
  float acc = 0.f;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 2; i < n;
       i += (gridDim.x * (int64_t)blockDim.x) >> 2) {
    if (MODE == 6) {
      const int64_t r = mix(seed + i) % (rows / 2);
      const float4 v = __ldg(reinterpret_cast<const float4*>(tab + r * 32) + lane);
      const float4 u = __ldg(reinterpret_cast<const float4*>(tab + r * 32 + 16) + lane);
      acc += v.x + v.y + v.z + v.w + u.x + u.y + u.z + u.w;
    } else if (MODE >= 4) {
      float4 v[3];
      int64_t r[3];
      uint4 q = make_uint4(0, 0, 0, 0);
      if (MODE == 5 && (i & 1)) q = __ldg(rec + mix(seed ^ i) % nrec);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        r[k] = (mix(seed + i * 3 + k) + (k == 0 ? q.x : (k == 1 ? q.y : q.z))) % (rows / 2);
        v[k] = __ldg(reinterpret_cast<const float4*>(tab + r[k] * 32) + lane);
      }
      const float y = v[0].x * v[1].y * v[2].z + 1e-30f;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        float* p = tab + r[k] * 32 + 16 + lane * 4;
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(y), "f"(y),
                     "f"(y), "f"(y) : "memory");
      }
    } else if (MODE >= 2) {
      float4 v[3];
      int64_t r[3];
      uint4 q = make_uint4(0, 0, 0, 0);
      if (MODE == 3 && (i & 1)) q = __ldg(rec + mix(seed ^ i) % nrec);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        r[k] = (mix(seed + i * 3 + k) + (k == 0 ? q.x : (k == 1 ? q.y : q.z))) % rows;
        v[k] = __ldg(reinterpret_cast<const float4*>(tab + r[k] * 16) + lane);
      }
      const float y = v[0].x * v[1].y * v[2].z + 1e-30f;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        // the gradient is a separate table (as in the engine): its lines
        // are not the ones the gathers just brought into L2
        float* p = tab + ((r[k] + rows / 2) % rows) * 16 + lane * 4;
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(y), "f"(y),
                     "f"(y), "f"(y) : "memory");
      }
    } else {
      const int64_t r = mix(seed + i) % rows;
      if (MODE == 0) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(tab + r * 16) + lane);
        acc += v.x + v.y + v.z + v.w;
      } else {
        float* p = tab + r * 16 + lane * 4;
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1e-30f),
                     "f"(1e-30f), "f"(1e-30f), "f"(1e-30f) : "memory");
      }
    }
  }
  if (acc == 123.f) sink[0] = acc;
}

int main() {
  const int64_t bytes = (getenv("TABMB") ? int64_t(atoi(getenv("TABMB"))) << 20 : int64_t(1) << 30),
                rows = bytes / 64;
  float* tab;
  float* sink;
  cudaMalloc(&tab, bytes);
  cudaMalloc(&sink, 64);
  cudaMemset(tab, 0, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int64_t n = 64 << 20;  // rows (or samples) per launch
  const int64_t recbytes = int64_t(getenv("RECGB") ? atoi(getenv("RECGB")) : 4) << 30, nrec = recbytes / 16;
  uint4* rec;
  cudaMalloc(&rec, recbytes);
  cudaMemset(rec, 0, recbytes);
  for (int mode = 0; mode < 7; ++mode) {
    for (int bps : {1, 2, 4}) {
      const int grid = sms * bps;  // 512-thread blocks: 16 warps each
      float best = 1e30f;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(a);
        if (mode == 0) kern<0><<<grid, 512>>>(tab, rows, n, sink, rep);
        if (mode == 1) kern<1><<<grid, 512>>>(tab, rows, n, sink, rep);
        if (mode == 2) kern<2><<<grid, 512>>>(tab, rows, n, sink, rep);
        if (mode == 3) kern<3><<<grid, 512>>>(tab, rows, n, sink, rep, rec, nrec);
        if (mode == 4) kern<4><<<grid, 512>>>(tab, rows, n, sink, rep);
        if (mode == 5) kern<5><<<grid, 512>>>(tab, rows, n, sink, rep, rec, nrec);
        if (mode == 6) kern<6><<<grid, 512>>>(tab, rows, n, sink, rep);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep > 0 && ms < best) best = ms;
      }
      // algorithmic bytes: 64 B per row access (x6 for the mixed sample)
      const double alg = (mode == 6 ? 2.0 : (mode >= 2 ? 6.0 : 1.0)) * 64.0 * n;
      const char* names[7] = {"gather     ", "red        ", "3g+3red    ", "rec+3g+3red",
                              "3g+3red  il", "rec+3g+3r il", "gather128  "};
      printf("mode %s warps/SM %2d: %.3f ms  %.0f GB/s (64 B row accesses)  %.3g units/s\n",
             names[mode], bps * 16, best,
             alg / best / 1e6, n / (best / 1e3));
    }
  }
  return 0;
}
