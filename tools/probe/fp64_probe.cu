// FP64 throughput probe for sm_100a: DFMA vs DMMA (mma.sync .f64) shapes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template<int CH>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template<int NACC>
__global__ void mma_m8n8k4(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template<int NACC>
__global__ void mma_m16n8k4(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 - threadIdx.x * 1e-4;
  double c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template<int NACC>
__global__ void mma_m16n8k8(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = 1.0 - threadIdx.x * 1e-4, b1 = b0 + 1;
  double c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template<int NACC>
__global__ void mma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
  for (int j = 0; j < 4; ++j) b[j] = 1.0 - threadIdx.x * 1e-4 + j;
  double c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template<typename F>
float time_it(F f, int reps) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"device\":\"%s\",\"sms\":%d,\"cc\":\"%d.%d\",\"clock_khz\":%d,\"l2_bytes\":%d,\"smem_optin\":%zu}\n",
         p.name, p.multiProcessorCount, p.major, p.minor, clk, p.l2CacheSize, p.sharedMemPerBlockOptin);
  double* out; CK(cudaMalloc(&out, 1 << 20));
  int sms = p.multiProcessorCount;
  const int iters = 4096;
  for (int bpsm : {1, 2, 4}) for (int threads : {128, 256, 512}) {
    int blocks = sms * bpsm;
    float ms = time_it([&]{ dfma_kernel<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); }, 5);
    double fl = 2.0 * 8 * iters * (double)blocks * threads;
    printf("{\"kernel\":\"dfma\",\"blocks\":%d,\"threads\":%d,\"tflops\":%.3f}\n", blocks, threads, fl / ms / 1e9);
  }
  for (int bpsm : {1, 2, 4}) for (int threads : {128, 256}) {
    int blocks = sms * bpsm;
    float ms = time_it([&]{ mma_m8n8k4<8><<<blocks, threads>>>(out, iters); }, 5);
    double fl = 2.0 * 8 * 8 * 4 * 8 * (double)iters * blocks * (threads / 32);
    printf("{\"kernel\":\"mma_m8n8k4\",\"blocks\":%d,\"threads\":%d,\"tflops\":%.3f}\n", blocks, threads, fl / ms / 1e9);
    ms = time_it([&]{ mma_m16n8k4<8><<<blocks, threads>>>(out, iters); }, 5);
    fl = 2.0 * 16 * 8 * 4 * 8 * (double)iters * blocks * (threads / 32);
    printf("{\"kernel\":\"mma_m16n8k4\",\"blocks\":%d,\"threads\":%d,\"tflops\":%.3f}\n", blocks, threads, fl / ms / 1e9);
    ms = time_it([&]{ mma_m16n8k8<8><<<blocks, threads>>>(out, iters / 2); }, 5);
    fl = 2.0 * 16 * 8 * 8 * 8 * (double)(iters / 2) * blocks * (threads / 32);
    printf("{\"kernel\":\"mma_m16n8k8\",\"blocks\":%d,\"threads\":%d,\"tflops\":%.3f}\n", blocks, threads, fl / ms / 1e9);
    ms = time_it([&]{ mma_m16n8k16<8><<<blocks, threads>>>(out, iters / 4); }, 5);
    fl = 2.0 * 16 * 8 * 16 * 8 * (double)(iters / 4) * blocks * (threads / 32);
    printf("{\"kernel\":\"mma_m16n8k16\",\"blocks\":%d,\"threads\":%d,\"tflops\":%.3f}\n", blocks, threads, fl / ms / 1e9);
  }
  // latency: single warp, dependent chain
  {
    float ms = time_it([&]{ mma_m16n8k4<1><<<1, 32>>>(out, iters); }, 3);
    printf("{\"kernel\":\"mma_m16n8k4_latency\",\"cycles_per_mma\":%.1f}\n", ms * 1e-3 * clk * 1e3 / iters);
    ms = time_it([&]{ mma_m16n8k16<1><<<1, 32>>>(out, iters / 4); }, 3);
    printf("{\"kernel\":\"mma_m16n8k16_latency\",\"cycles_per_mma\":%.1f}\n", ms * 1e-3 * clk * 1e3 / (iters / 4));
    ms = time_it([&]{ dfma_kernel<1><<<1, 32>>>(out, iters, 1.0000001, 1e-9); }, 3);
    printf("{\"kernel\":\"dfma_latency\",\"cycles_per_op\":%.1f}\n", ms * 1e-3 * clk * 1e3 / iters);
  }
  return 0;
}
