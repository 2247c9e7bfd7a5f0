// Microbenchmark: does the column template's tile layout (128-column tiles, rows
// 4 KB apart, 512 B per row segment) cost DRAM efficiency when the kernel also
// writes a full-size root (C3b's db group: reads dy, x; writes dx; sums columns)?
// K_tile: 8 column tiles x 37 stripes (the template's layout); K_row: 296 stripes
// of full 1024-column rows (4 KB contiguous per row per CTA).  Both: 256 threads,
// 2 CTAs/SM, 16 rows in flight per thread, fp64 column accumulators, streaming
// stores.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o col_layout col_layout.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float4 lds(const float* p) {
  float4 v;
  asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void sts(float* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
constexpr int N = 65536, C = 1024, UR = 16;

template <bool WRITE>
__global__ void __launch_bounds__(256, 2) k_tile(const float* dy, const float* x, float* dx, double* part) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c0 = blockIdx.x * 128 + lane * 4;
  const int RS = (N + 36) / 37;
  const int rb = blockIdx.y * RS, re = min(N, rb + RS);
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  int r = rb + warp;
  for (; r + (UR - 1) * 8 < re; r += UR * 8) {
#pragma unroll
    for (int u = 0; u < UR; ++u) {
      const long long i = (long long)(r + u * 8) * C + c0;
      float4 d = lds(dy + i), q = lds(x + i);
      float4 o = make_float4(q.x > 0 ? d.x : 0.f, q.y > 0 ? d.y : 0.f, q.z > 0 ? d.z : 0.f, q.w > 0 ? d.w : 0.f);
      a0 += o.x; a1 += o.y; a2 += o.z; a3 += o.w;
      if (WRITE) sts(dx + i, o);
    }
  }
  for (; r < re; r += 8) {
    const long long i = (long long)r * C + c0;
    float4 d = lds(dy + i), q = lds(x + i);
    float4 o = make_float4(q.x > 0 ? d.x : 0.f, q.y > 0 ? d.y : 0.f, q.z > 0 ? d.z : 0.f, q.w > 0 ? d.w : 0.f);
    a0 += o.x; a1 += o.y; a2 += o.z; a3 += o.w;
    if (WRITE) sts(dx + i, o);
  }
  double* p = part + ((long long)blockIdx.y * 8 + warp) * C + c0;
  p[0] = a0; p[1] = a1; p[2] = a2; p[3] = a3;
}

template <bool WRITE>
__global__ void __launch_bounds__(256, 2) k_row(const float* dy, const float* x, float* dx, double* part) {
  const int c0 = threadIdx.x * 4;
  const int RS = (N + 295) / 296;
  const int rb = blockIdx.x * RS, re = min(N, rb + RS);
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  int r = rb;
  for (; r + UR - 1 < re; r += UR) {
#pragma unroll
    for (int u = 0; u < UR; ++u) {
      const long long i = (long long)(r + u) * C + c0;
      float4 d = lds(dy + i), q = lds(x + i);
      float4 o = make_float4(q.x > 0 ? d.x : 0.f, q.y > 0 ? d.y : 0.f, q.z > 0 ? d.z : 0.f, q.w > 0 ? d.w : 0.f);
      a0 += o.x; a1 += o.y; a2 += o.z; a3 += o.w;
      if (WRITE) sts(dx + i, o);
    }
  }
  for (; r < re; ++r) {
    const long long i = (long long)r * C + c0;
    float4 d = lds(dy + i), q = lds(x + i);
    float4 o = make_float4(q.x > 0 ? d.x : 0.f, q.y > 0 ? d.y : 0.f, q.z > 0 ? d.z : 0.f, q.w > 0 ? d.w : 0.f);
    a0 += o.x; a1 += o.y; a2 += o.z; a3 += o.w;
    if (WRITE) sts(dx + i, o);
  }
  double* p = part + (long long)blockIdx.x * C + c0;
  p[0] = a0; p[1] = a1; p[2] = a2; p[3] = a3;
}

template <typename F>
float time_it(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f(i);
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f(i);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / reps;
}

int main() {
  const size_t bytes = (size_t)N * C * 4;
  const int SETS = 2;
  float *dy[SETS], *x[SETS], *dx[SETS];
  double* part;
  for (int s = 0; s < SETS; ++s) {
    cudaMalloc(&dy[s], bytes);
    cudaMalloc(&x[s], bytes);
    cudaMalloc(&dx[s], bytes);
    cudaMemset(dy[s], 0x3f, bytes);
    cudaMemset(x[s], 0x3f, bytes);
  }
  cudaMalloc(&part, (size_t)296 * 8 * C * 8);
  const int reps = 30;
  for (int round = 0; round < 2; ++round) {
    float t1 = time_it([&](int i) { k_tile<true><<<dim3(8, 37), 256>>>(dy[i % SETS], x[i % SETS], dx[i % SETS], part); }, reps);
    float t2 = time_it([&](int i) { k_row<true><<<296, 256>>>(dy[i % SETS], x[i % SETS], dx[i % SETS], part); }, reps);
    float t3 = time_it([&](int i) { k_tile<false><<<dim3(8, 37), 256>>>(dy[i % SETS], x[i % SETS], dx[i % SETS], part); }, reps);
    float t4 = time_it([&](int i) { k_row<false><<<296, 256>>>(dy[i % SETS], x[i % SETS], dx[i % SETS], part); }, reps);
    printf("{\"tile_write_us\": %.1f, \"row_write_us\": %.1f, \"tile_read_us\": %.1f, \"row_read_us\": %.1f, "
           "\"tile_write_gbs\": %.0f, \"row_write_gbs\": %.0f, \"tile_read_gbs\": %.0f, \"row_read_gbs\": %.0f}\n",
           t1, t2, t3, t4, 3 * bytes / t1 / 1e3, 3 * bytes / t2 / 1e3, 2 * bytes / t3 / 1e3, 2 * bytes / t4 / 1e3);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
