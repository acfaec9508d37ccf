// Do DFMA and DMMA share a pipe on sm_100a?  Also: DMMA dependent-chain latency.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int NMMA, int NFMA>
__global__ void mix(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double d0[4] = {0, 0, 0, 0}, d1[4] = {0, 0, 0, 0};
  double f[8];
  for (int c = 0; c < 8; ++c) f[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < NMMA; ++c) dmma(d0[c & 3], d1[c & 3], a, b);
#pragma unroll
    for (int c = 0; c < NFMA; ++c) f[c & 7] = fma(f[c & 7], 1.0000001, 1e-9);
  }
  double s = 0;
  for (int c = 0; c < 4; ++c) s += d0[c] + d1[c];
  for (int c = 0; c < 8; ++c) s += f[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}
__global__ void lat(double* out, int iters, long long* cyc) {
  double a = 1.0, b = 1.0, d0 = 0, d1 = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) dmma(d0, d1, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  if (d0 == 12345.678) out[0] = d1;
}
template <int NMMA, int NFMA>
void run(const char* name, double* out, int sms) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = sms * 4, threads = 256, iters = 4000;
  mix<NMMA, NFMA><<<blocks, threads>>>(out, 10);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  mix<NMMA, NFMA><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double warps = (double)blocks * threads / 32;
  double mma_fl = 2.0 * 256 * NMMA * iters * warps, fma_fl = 2.0 * 32 * NFMA * iters * warps;
  printf("%-22s %.3f ms  DMMA %.2f TF  DFMA %.2f TF  total %.2f TF\n", name, ms, mma_fl / ms / 1e9, fma_fl / ms / 1e9, (mma_fl + fma_fl) / ms / 1e9);
}
int main() {
  double* out; cudaMalloc(&out, 1 << 20);
  long long* cyc; cudaMalloc(&cyc, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<4, 0>("dmma only", out, sms);
  run<0, 32>("dfma only", out, sms);
  run<4, 32>("dmma4 + dfma32", out, sms);
  run<4, 16>("dmma4 + dfma16", out, sms);
  run<4, 64>("dmma4 + dfma64", out, sms);
  lat<<<1, 32>>>(out, 1000, cyc);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DMMA dependent latency: %.1f cycles\n", c / 1000.0);
  return 0;
}
