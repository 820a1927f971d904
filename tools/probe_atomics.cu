// Microbenchmark: shared-memory float atomics (spread / clustered / same address) and
// global float4 vector reductions, as candidate MI joint-histogram accumulation paths.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void smem_atom(float* out, int iters, int mode) {
  __shared__ float h[1088 * 4];
  for (int i = threadIdx.x; i < 1088 * 4; i += blockDim.x) h[i] = 0;
  __syncthreads();
  unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned s = threadIdx.x * 2654435761u + blockIdx.x;
  float v = 1.0f;
  for (int i = 0; i < iters; ++i) {
    s = s * 1664525u + 1013904223u;
    int base;
    if (mode == 0) base = (w * 32 + lane) % 1024;               // distinct per lane
    else if (mode == 1) base = ((s >> 16) & 1023);             // random
    else if (mode == 2) base = (w * 32) % 1024 + (lane >> 3);  // 4 distinct per warp (clustered)
    else base = 0;                                              // same address
#pragma unroll
    for (int k = 0; k < 16; ++k) atomicAdd(&h[(base + k * 33) & 4095], v);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 1088; i += blockDim.x) atomicAdd(&out[i], h[i]);
}
template <typename U>
__global__ void smem_atom_int(float* out, int iters, int mode) {
  __shared__ U h[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) h[i] = 0;
  __syncthreads();
  unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned s = threadIdx.x * 2654435761u + blockIdx.x;
  U v = 12345;
  for (int i = 0; i < iters; ++i) {
    s = s * 1664525u + 1013904223u;
    int base;
    if (mode == 0) base = (w * 32 + lane) % 1024;
    else if (mode == 1) base = ((s >> 16) & 1023);
    else if (mode == 2) base = (w * 32) % 1024 + (lane >> 3);
    else base = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) atomicAdd(&h[(base + k * 33) & 4095], v);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 1088; i += blockDim.x) atomicAdd(&out[i], (float)h[i]);
}
__global__ void gred_v4(float* hist, int iters) {
  unsigned s = threadIdx.x * 2654435761u + blockIdx.x;
  float* my = hist + (blockIdx.x % 148) * 4096;
  for (int i = 0; i < iters; ++i) {
    s = s * 1664525u + 1013904223u;
    int base = ((s >> 16) & 1023) * 4;
    float4 v = make_float4(1, 2, 3, 4);
#pragma unroll
    for (int k = 0; k < 4; ++k) atomicAdd(reinterpret_cast<float4*>(my + ((base + k * 132) & 4095 & ~3)), v);
  }
}
int main() {
  int blocks = 148 * 4, threads = 256, iters = 256;
  float* out; cudaMalloc(&out, 148 * 4096 * 4); cudaMemset(out, 0, 148*4096*4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  const char* names[] = {"distinct", "random", "clustered4", "same"};
  for (int rep = 0; rep < 2; ++rep) {
    for (int mode = 0; mode < 4; ++mode) {
      cudaEventRecord(e0); smem_atom<<<blocks, threads>>>(out, iters, mode); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)blocks * threads * iters * 16;
      printf("smem atomicAdd f32 %-10s: %.1f Gatom/s  (%.2f cyc per warp-atom per SM @1.9GHz)\n", names[mode], ops / ms / 1e6,
             (ms * 1e-3 * 1.9e9 * 148) / (ops / 32));
    }
    for (int mode = 0; mode < 4; ++mode) {
      cudaEventRecord(e0); smem_atom_int<unsigned><<<blocks, threads>>>(out, iters, mode); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)blocks * threads * iters * 16;
      printf("smem atomicAdd u32 %-10s: %.1f Gatom/s  (%.2f cyc per warp-atom per SM)\n", names[mode], ops / ms / 1e6, (ms * 1e-3 * 1.9e9 * 148) / (ops / 32));
      cudaEventRecord(e0); smem_atom_int<unsigned long long><<<blocks, threads>>>(out, iters, mode); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("smem atomicAdd u64 %-10s: %.1f Gatom/s  (%.2f cyc per warp-atom per SM)\n", names[mode], ops / ms / 1e6, (ms * 1e-3 * 1.9e9 * 148) / (ops / 32));
    }
    cudaEventRecord(e0); gred_v4<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * iters * 4;
    printf("global red.v4.f32 random (148 private copies): %.1f Gred/s\n", ops / ms / 1e6);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
