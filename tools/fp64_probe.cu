// fp64_probe.cu — measures the B200's FP64 add latency (one warp, one dependent chain)
// and the FP64 add / FP32 fma instruction throughput (all SMs, many independent chains),
// plus the 32-bit shuffle latency: the compute roofline of the fused (temporally blocked)
// kernels, which are arithmetic-bound.  bench.py runs it and reports the rates.
//   make build/fp64_probe   (nvcc -O3 -gencode arch=compute_100a,code=sm_100a)
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_dadd(double* out, double a, int iters, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = __dadd_rn(x, a);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  out[threadIdx.x] = x;
}

__global__ void lat_shfl(float* out, float a, int iters, long long* cyc) {
  float x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = __shfl_up_sync(0xffffffffu, x, 1) + 1.0f;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  out[threadIdx.x] = x;
}

template <int CH>
__global__ void thr_ffma(float* out, float a, int iters) {
  float x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = a * (c + 1 + threadIdx.x);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = __fmaf_rn(x[c], a, 0.5f);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CH>
__global__ void thr_dadd(double* out, double a, int iters) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = a * (c + 1 + threadIdx.x);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = __dadd_rn(x[c], a);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 26);
  cudaMalloc(&cyc, 8);
  int iters = 4096;
  lat_dadd<<<1, 32>>>(out, 1e-3, iters, cyc);
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("{\"dadd_latency_cycles\": %.2f, ", double(c) / (iters * 16.0));
  lat_shfl<<<1, 32>>>(reinterpret_cast<float*>(out), 1.0f, iters, cyc);
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("\"shfl_plus_fadd_latency_cycles\": %.2f, ", double(c) / (iters * 16.0));
  int nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 16, 32}) {
    const int blocks = nsm * warps / 4, threads = 128, it = 20000;
    thr_dadd<8><<<blocks, threads>>>(out, 1e-3, 10);
    cudaEventRecord(e0);
    thr_dadd<8><<<blocks, threads>>>(out, 1e-3, it);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = double(blocks) * threads * it * 8;
    printf("\"dadd_rate_%dwarps_per_sm_Gops\": %.1f, ", warps, ops / (ms * 1e-3) / 1e9);
  }
  {
    const int blocks = nsm * 8, threads = 256, it = 20000;
    thr_ffma<8><<<blocks, threads>>>(reinterpret_cast<float*>(out), 1.0001f, 10);
    cudaEventRecord(e0);
    thr_ffma<8><<<blocks, threads>>>(reinterpret_cast<float*>(out), 1.0001f, it);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = double(blocks) * threads * it * 8;
    printf("\"ffma_rate_Gops\": %.1f, ", ops / (ms * 1e-3) / 1e9);
  }
  printf("\"nsm\": %d, \"clock_khz\": %d}\n", nsm, clk);
  return 0;
}
