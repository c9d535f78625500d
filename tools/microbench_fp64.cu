// FP64 pipe microbenchmark for B200 (sm_100a): DMMA.8x8x4 (mma.sync f64) vs
// DFMA issue throughput, register-resident, to fix the roofline denominator
// for the chord kernel. Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters) {
  double acc[CHAINS][2];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) { acc[c][0] = 0; acc[c][1] = 0; }
  double a = 1e-3 * threadIdx.x, b = 2e-3 * threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c][0] + acc[c][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * c;
  double a = 1.0000001, b = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
static double time_kernel(K kern, int blocks, int threads, double* out, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(out, iters);  // warm
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best * 1e-3;
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * 148 * 64 * 1024);
  const int iters = 4096;
  printf("{\"sms\": %d", sms);
  for (int wpb : {4, 8, 16}) {
    int threads = 32 * wpb, blocks = sms * 2;
    double t = time_kernel(dmma_loop<8>, blocks, threads, out, iters);
    double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (blocks * wpb);
    printf(", \"dmma_w%d_tflops\": %.3f", wpb, flops / t / 1e12);
  }
  for (int wpb : {4, 8, 16}) {
    int threads = 32 * wpb, blocks = sms * 2;
    double t = time_kernel(dfma_loop<8>, blocks, threads, out, iters);
    double flops = 2.0 * 8.0 * iters * (double)blocks * threads;
    printf(", \"dfma_w%d_tflops\": %.3f", wpb, flops / t / 1e12);
  }
  printf("}\n");
  return 0;
}
