// Is the fp64 tensor pipe (DMMA) per SMSP or shared by the SM?
// Active warps issue independent DMMA chains; idle warps exit at once.
// Warp w runs on SMSP w % 4, so "mask" picks which SMSPs carry the work.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__global__ void k(int iters, unsigned long long active_mask, double* out) {
  const int w = threadIdx.x >> 5;
  if (!((active_mask >> w) & 1ull)) return;
  double c[8][2];
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  struct C { const char* name; int warps; unsigned long long mask; } cs[] = {
      {"1 warp  (SMSP0)", 1, 0x1ull},
      {"4 warps (SMSP0,1,2,3)", 4, 0xFull},
      {"4 warps (all on SMSP0)", 16, 0x1111ull},
      {"8 warps (2 per SMSP)", 8, 0xFFull},
      {"8 warps (all on SMSP0,1)", 16, 0x3333ull},
      {"12 warps (3 per SMSP)", 12, 0xFFFull},
      {"10 warps (3,3,2,2)", 10, 0x3FFull},
      {"16 warps (4 per SMSP)", 16, 0xFFFFull},
  };
  const int iters = 4096;
  for (auto& c : cs) {
    k<<<sms, 32 * c.warps>>>(16, c.mask, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<sms, 32 * c.warps>>>(iters, c.mask, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int nact = __builtin_popcountll(c.mask);
    double dmmas = (double)sms * nact * iters * 8;
    double tf = dmmas * 512 / (ms * 1e-3) / 1e12;
    double per_sm_clk = dmmas / sms / (ms * 1e-3 * 1965e6);
    printf("%-28s %8.3f ms  %6.2f TF/s  %5.3f DMMA/clk/SM  (%.1f clk per DMMA per SM)\n", c.name, ms, tf,
           per_sm_clk, 1.0 / per_sm_clk);
  }
  return 0;
}
