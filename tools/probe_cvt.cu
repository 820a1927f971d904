// Microbenchmark: throughput of the fp32<->fp64 conversions and fp64 floor used by the sampler.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_f2f(float* o, int it) {
  float a = threadIdx.x * 1e-3f, b = a + 1, c = a + 2, d = a + 3;
  double s = 0;
  for (int i = 0; i < it; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { s += (double)a; s += (double)b; s += (double)c; s += (double)d; a += 1e-7f; }
  }
  o[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
}
__global__ void k_dadd(float* o, int it) {
  double a = threadIdx.x * 1e-3, b = a + 1, c = a + 2, d = a + 3, s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  for (int i = 0; i < it; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { s0 += a; s1 += b; s2 += c; s3 += d; s0 += b; s1 += c; s2 += d; s3 += a; }
  }
  o[blockIdx.x * blockDim.x + threadIdx.x] = (float)(s0 + s1 + s2 + s3);
}
__global__ void k_floor_f2i(float* o, int it) {
  double a = threadIdx.x * 1.37;
  int acc = 0;
  for (int i = 0; i < it; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { double f = floor(a); acc += (int)f; a += 0.731; }
  }
  o[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
}
__global__ void k_f2i_floor(float* o, int it) {
  double a = threadIdx.x * 1.37;
  int acc = 0;
  for (int i = 0; i < it; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { acc += __double2int_rd(a); a += 0.731; }
  }
  o[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
}
__global__ void k_d2f(float* o, int it) {
  double a = threadIdx.x * 1.37;
  float acc = 0;
  for (int i = 0; i < it; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { acc += (float)a; a += 0.731; }
  }
  o[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  int blocks = 148 * 8, threads = 256, it = 2048;
  float* o; cudaMalloc(&o, blocks * threads * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  double per = (double)blocks * threads * it;
  for (int rep = 0; rep < 2; ++rep) {
#define T(kern, ops, name) cudaEventRecord(e0); kern<<<blocks, threads>>>(o, it); cudaEventRecord(e1); cudaEventSynchronize(e1); \
    cudaEventElapsedTime(&ms, e0, e1); printf("%-28s %.2f lanes-op/clk/SM\n", name, per * ops / (ms * 1e-3) / 148 / 1.965e9);
    T(k_f2f, 32, "F2F f32->f64 (+DADD)")
    T(k_dadd, 64, "DADD")
    T(k_floor_f2i, 8, "floor(f64)+F2I (+DADD)")
    T(k_f2i_floor, 8, "F2I.floor f64 (+DADD)")
    T(k_d2f, 8, "F2F f64->f32 (+FADD,DADD)")
  }
  return 0;
}
