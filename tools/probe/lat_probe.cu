// Dependent-chain latencies on this GPU (one warp): DFMA, DMUL, double rsqrt, shfl of a double, LDS.64, BAR.SYNC
// (512 threads). nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat_probe lat_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b) {
  __shared__ double sm[1024];
  const int tid = threadIdx.x;
  sm[tid] = tid;
  sm[tid + 512] = 0;
  __syncthreads();
  double x = a + tid;
  long long t0 = clock64();
  for (int i = 0; i < 1000; ++i) x = fma(x, b, a);
  long long t1 = clock64();
  for (int i = 0; i < 1000; ++i) x = x * b;
  long long t2 = clock64();
  for (int i = 0; i < 200; ++i) x = rsqrt(x + 2.0);
  long long t3 = clock64();
  for (int i = 0; i < 1000; ++i) x = __shfl_sync(0xffffffffu, x, (tid + 1) & 31);
  long long t4 = clock64();
  int idx = tid & 31;
  for (int i = 0; i < 1000; ++i) idx = (int)sm[idx] & 511;
  long long t5 = clock64();
  for (int i = 0; i < 1000; ++i) __syncthreads();
  long long t6 = clock64();
  out[tid] = x + idx;
  if (tid == 0) {
    cyc[0] = (t1 - t0) / 1000; cyc[1] = (t2 - t1) / 1000; cyc[2] = (t3 - t2) / 200; cyc[3] = (t4 - t3) / 1000;
    cyc[4] = (t5 - t4) / 1000; cyc[5] = (t6 - t5) / 1000;
  }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 4096); cudaMallocManaged(&c, 64);
  for (int rep = 0; rep < 2; ++rep) k<<<1, 512>>>(o, c, 1.0000001, 0.9999999);
  cudaDeviceSynchronize();
  printf("cycles per dependent op: DFMA %lld DMUL %lld rsqrt(double) %lld shfl(double) %lld LDS.64 %lld bar.sync(512) %lld\n",
         c[0], c[1], c[2], c[3], c[4], c[5]);
  return 0;
}
