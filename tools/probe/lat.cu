// Dependent-chain latency of the march's fp64 / fp32 / conversion ops on this
// GPU (one warp, clock64).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 lat.cu -o lat
#include <cstdio>
#include <cuda_runtime.h>
constexpr int N = 4096;
__global__ void k(double *od, float *of, long long *cyc, double a, float b) {
  double x = a; float y = b; int z = (int)b;
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) x = __dadd_rn(x, a);
  long long t1 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) x = __dmul_rn(x, a);
  long long t2 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) x = __fma_rn(x, a, a);
  long long t3 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) y = __fadd_rn(y, b);
  long long t4 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) y = __fmaf_rn(y, b, b);
  long long t5 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) x = (double)(float)x;     // F2F pair
  long long t6 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) z = __double2loint(__dadd_rd((double)z, 4503599627370496.0));   // I2F + DADD.RD + mov
  long long t7 = clock64();
  od[threadIdx.x] = x; of[threadIdx.x] = y + z;
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0); cyc[1] = (t2 - t1); cyc[2] = (t3 - t2); cyc[3] = (t4 - t3); cyc[4] = (t5 - t4);
    cyc[5] = (t6 - t5); cyc[6] = (t7 - t6);
  }
}
int main() {
  double *od; float *of; long long *c, h[7];
  cudaMalloc(&od, 1024); cudaMalloc(&of, 1024); cudaMalloc(&c, 64);
  for (int rep = 0; rep < 2; ++rep) k<<<1, 32>>>(od, of, c, 1.0000001, 1.0000001f);
  cudaMemcpy(h, c, 56, cudaMemcpyDeviceToHost);
  const char *nm[7] = {"DADD", "DMUL", "DFMA", "FADD", "FFMA", "F2F.F32.F64+F2F.F64.F32", "I2F.F64+DADD.RD+mov"};
  for (int i = 0; i < 7; ++i) printf("%-26s %.2f cyc/op\n", nm[i], (double)h[i] / N);
  return 0;
}
