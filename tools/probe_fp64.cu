// Microbenchmark: FP32 vs FP64 FMA issue throughput and cvt.rmi.f64 on this part.
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void fma_loop(T* out, int iters, T a, T b) {
  T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
      x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void floor_loop(double* out, int iters, double a) {
  double x0 = threadIdx.x * 0.37, x1 = x0 + 1.3, x2 = x0 + 2.7, x3 = x0 + 3.1;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x0 = floor(x0 + a); x1 = floor(x1 + a); x2 = floor(x2 + a); x3 = floor(x3 + a);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("%s SMs=%d cc=%d.%d clock=%d kHz smem/SM=%zu L2=%d\n", p.name, p.multiProcessorCount, p.major, p.minor, p.clockRate, p.sharedMemPerMultiprocessor, p.l2CacheSize);
  int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4096;
  float* of; double* od; cudaMalloc(&of, blocks*threads*8); cudaMalloc(&od, blocks*threads*8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); fma_loop<float><<<blocks, threads>>>(of, iters, 0.999f, 0.001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * blocks * threads * (double)iters * 64;
    printf("fp32 FMA: %.1f TFLOP/s\n", flops / ms / 1e9);
    cudaEventRecord(e0); fma_loop<double><<<blocks, threads>>>(od, iters, 0.999, 0.001); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("fp64 FMA: %.1f TFLOP/s\n", flops / ms / 1e9);
    cudaEventRecord(e0); floor_loop<<<blocks, threads>>>(od, iters, 0.3); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("fp64 add+floor: %.1f Gop/s (pairs)\n", (double)blocks * threads * iters * 32 / ms / 1e6);
  }
  return 0;
}
