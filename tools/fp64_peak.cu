// FP64 peak microbenchmarks for the roofline denominator (run on the B200 box).
// DMMA: mma.sync.aligned.m8n8k4.row.col.f64 register-only; DFMA: fma.rn.f64 chains.
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
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
  if (s == 12345.0) out[0] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}

template <typename K>
void run(const char* name, K kern, int threads, int blocks_per_sm, int iters, double flop_per_thread_iter) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 8);
  int grid = sms * blocks_per_sm;
  kern<<<grid, threads>>>(out, 10);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kern<<<grid, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double flops = (double)grid * threads * iters * flop_per_thread_iter;
  printf("{\"kernel\": \"%s\", \"threads\": %d, \"blocks_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n",
         name, threads, blocks_per_sm, best, flops / best / 1e9);
  cudaError_t err = cudaGetLastError(); if (err) printf("err %s\n", cudaGetErrorString(err));
  cudaFree(out);
}

int main() {
  // DMMA m8n8k4: 8*8*4 FMA = 512 flop per warp instruction = 16 flop/thread
  for (int bps : {1, 2, 4}) {
    run("dmma_acc4", dmma_loop<4>, 256, bps, 20000, 4 * 16.0);
    run("dmma_acc8", dmma_loop<8>, 256, bps, 10000, 8 * 16.0);
  }
  run("dmma_acc8_128t", dmma_loop<8>, 128, 4, 10000, 8 * 16.0);
  run("dmma_acc16", dmma_loop<16>, 256, 2, 5000, 16 * 16.0);
  for (int bps : {1, 2, 4}) {
    run("dfma_acc8", dfma_loop<8>, 256, bps, 40000, 8 * 2.0);
    run("dfma_acc16", dfma_loop<16>, 256, bps, 20000, 16 * 2.0);
  }
  return 0;
}
