// FP32 / FP64 peak microbenchmark for the roofline denominator (SURVEY §8(d):
// "confirm both with an FMA microbenchmark on the box").  Independent FMA
// chains per thread, grid = 148 SMs x 8 blocks x 256 threads; reports
// TFLOP/s (2 flops per FMA lane) for scalar FFMA, packed FFMA2 (fma.rn.f32x2)
// and DFMA.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fma_peak fma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void ffma_kernel(float* out, float a, float b) {
  float x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = fmaf(x[c], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.f) out[0] = s;
}

__device__ __forceinline__ unsigned long long ffma2(unsigned long long x, unsigned long long a,
                                                    unsigned long long b) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(x), "l"(a), "l"(b));
  return r;
}

__global__ void ffma2_kernel(float* out, float a, float b) {
  unsigned long long x[kChains];
  float2 av = make_float2(a, a), bv = make_float2(b, b);
  const unsigned long long A = *reinterpret_cast<unsigned long long*>(&av);
  const unsigned long long B = *reinterpret_cast<unsigned long long*>(&bv);
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    float2 v = make_float2(threadIdx.x * 1e-3f + c, c + 0.5f);
    x[c] = *reinterpret_cast<unsigned long long*>(&v);
  }
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = ffma2(x[c], A, B);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    float2 v = *reinterpret_cast<float2*>(&x[c]);
    s += v.x + v.y;
  }
  if (s == 12345.f) out[0] = s;
}

__global__ void dfma_kernel(double* out, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < kIters / 4; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0.;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  float* dout;
  cudaMalloc(&dout, 64);
  const int threads = 256, blocks = sms * 8;
  const double lanes = (double)threads * blocks;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto time = [&](auto launch, double flops) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    return flops / (best * 1e-3) / 1e12;
  };
  const double f1 = lanes * kChains * kIters * 2.0;
  double t1 = time([&] { ffma_kernel<<<blocks, threads>>>(dout, 0.999f, 1e-3f); }, f1);
  double t2 = time([&] { ffma2_kernel<<<blocks, threads>>>(dout, 0.999f, 1e-3f); }, 2.0 * f1);
  double t3 = time([&] { dfma_kernel<<<blocks, threads>>>((double*)dout, 0.999, 1e-3); }, f1 / 4.0);
  printf("{\"sms\": %d, \"clock_mhz_attr\": %.0f, \"ffma_tflops\": %.2f, \"ffma2_tflops\": %.2f, "
         "\"dfma_tflops\": %.2f, \"error\": \"%s\"}\n",
         sms, clk_khz / 1e3, t1, t2, t3, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
