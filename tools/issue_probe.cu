// Issue-slot probe: does an FP64 warp instruction hold a sub-partition's issue port for two
// cycles, or can other instructions issue in its shadow?  Each warp runs NCH independent
// DADD chains with K independent integer (or shuffle) instructions interleaved per DADD;
// printed: DADD lanes per clock per SM for K = 0..3 at 8 and 16 warps per SM.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/issue_probe tools/issue_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int K, int KIND>
__global__ void mix(double* out, double a, int* iout, int iters) {
  constexpr int NCH = 8;
  double x[NCH];
  int y[NCH];
#pragma unroll
  for (int i = 0; i < NCH; ++i) {
    x[i] = a * (threadIdx.x + i);
    y[i] = threadIdx.x + i;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(x[i]) : "d"(a));
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (KIND == 0)
          asm volatile("add.s32 %0, %0, %1;" : "+r"(y[(i + k) % NCH]) : "r"(it));
        else if (KIND == 1)
          asm volatile("shfl.sync.up.b32 %0, %0, 1, 0, 0xffffffff;" : "+r"(y[(i + k) % NCH]));
        else
          asm volatile("fma.rn.f32 %0, %0, %1, %1;"
                       : "+f"(reinterpret_cast<float&>(y[(i + k) % NCH]))
                       : "f"(1.0001f));
      }
    }
  }
  double s = 0;
  int t = 0;
#pragma unroll
  for (int i = 0; i < NCH; ++i) {
    s += x[i];
    t += y[i];
  }
  if (s == 123.456) out[0] = s;
  if (t == 123456789) iout[0] = t;
}

template <int K, int KIND>
void run(int warps, int nsm, int clk_khz, const char* kind) {
  double* d;
  int* di;
  cudaMalloc(&d, 8);
  cudaMalloc(&di, 4);
  const int iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mix<K, KIND><<<nsm, warps * 32>>>(d, 1.0, di, 100);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  mix<K, KIND><<<nsm, warps * 32>>>(d, 1.0, di, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double dadd = double(nsm) * warps * 32.0 * iters * 8;
  const double cycles = ms * 1e-3 * clk_khz * 1e3;
  printf("{\"kind\": \"%s\", \"k_per_dadd\": %d, \"warps_per_sm\": %d, \"dadd_lanes_per_clk_per_sm\": %.1f, "
         "\"issue_cycles_per_dadd_plus_k\": %.2f}\n",
         kind, K, warps, dadd / cycles / nsm, cycles * 4.0 / (double(warps) * iters * 8));
  cudaFree(d);
  cudaFree(di);
}

int main() {
  cudaDeviceProp pr;
  cudaGetDeviceProperties(&pr, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int w : {8, 16}) {
    run<0, 0>(w, pr.multiProcessorCount, clk, "int");
    run<1, 0>(w, pr.multiProcessorCount, clk, "int");
    run<2, 0>(w, pr.multiProcessorCount, clk, "int");
    run<3, 0>(w, pr.multiProcessorCount, clk, "int");
    run<1, 1>(w, pr.multiProcessorCount, clk, "shfl");
    run<2, 1>(w, pr.multiProcessorCount, clk, "shfl");
    run<1, 2>(w, pr.multiProcessorCount, clk, "ffma");
    run<2, 2>(w, pr.multiProcessorCount, clk, "ffma");
  }
  return 0;
}
