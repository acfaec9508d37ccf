// Microbenchmark: FP64 DFMA vs DMMA (mma.sync m8n8k4 f64) throughput on sm_100a,
// plus a plain HBM copy.  Used to pick the fp64 contraction strategy.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CH>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int CH>
__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double d0[CH], d1[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { d0[c] = 0; d1[c] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d0[c]), "+d"(d1[c]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d0[c] + d1[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) b[i] = a[i];
}

int main() {
  int dev = 0; cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, dev));
  printf("device %s SMs %d smemOptin %zu clock %d kHz\n", pr.name, pr.multiProcessorCount, pr.sharedMemPerBlockOptin, pr.clockRate);
  double* out; CK(cudaMalloc(&out, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = pr.multiProcessorCount;
  for (int occ : {4, 8, 16}) {
    int blocks = sms * occ, threads = 256, iters = 20000;
    dfma_kernel<8><<<blocks, threads>>>(out, 100, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_kernel<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * (double)blocks * threads;
    printf("DFMA occ=%d: %.2f TFLOP/s (%.3f ms)\n", occ, flops / ms / 1e9, ms);
  }
  for (int occ : {2, 4, 8, 16}) {
    int blocks = sms * occ, threads = 128, iters = 20000;
    dmma_kernel<4><<<blocks, threads>>>(out, 100);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dmma_kernel<4><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 4 * iters * (double)blocks * (threads / 32);
    printf("DMMA occ=%d: %.2f TFLOP/s (%.3f ms)\n", occ, flops / ms / 1e9, ms);
  }
  size_t n = (size_t)1 << 28;  // 2^28 double2 = 4 GiB each
  double2 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
  cudaMemset(a, 0, n * 16);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    copy_kernel<<<sms * 8, 512>>>(a, b, n);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy: %.1f GB/s\n", 2.0 * n * 16 / ms / 1e6);
  }
  return 0;
}
