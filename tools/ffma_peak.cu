// ffma_peak.cu — measure the FP32 / FP64 FMA-pipe peak of this GPU (roofline denominator for
// the ALU-bound unit kernel; MEASURED_PEAKS.json has only HBM and bf16 peaks).
// Three forms: register-register FFMA, FFMA with a constant-bank operand, DFMA.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;

__constant__ float cf[kChains];

__global__ void ffma_reg(float* out, float a, float b) {
  float x[kChains];
  for (int i = 0; i < kChains; ++i) x[i] = threadIdx.x + i;
  float y = a, z = b;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) x[i] = fmaf(x[i], y, z);
  }
  float s = 0;
  for (int i = 0; i < kChains; ++i) s += x[i];
  if (s == 1.2345f) out[0] = s;
}

__global__ void ffma_const(float* out) {
  float x[kChains];
  for (int i = 0; i < kChains; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) x[i] = fmaf(cf[i], x[i], x[(i + 1) % kChains]);
  }
  float s = 0;
  for (int i = 0; i < kChains; ++i) s += x[i];
  if (s == 1.2345f) out[0] = s;
}

__global__ void dfma_reg(double* out, double a, double b) {
  double x[kChains];
  for (int i = 0; i < kChains; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < kChains; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float hc[kChains];
  for (int i = 0; i < kChains; ++i) hc[i] = 0.999f + 1e-4f * i;
  cudaMemcpyToSymbol(cf, hc, sizeof(hc));
  float* of;
  double* od;
  cudaMalloc(&of, 64);
  cudaMalloc(&od, 64);
  const int grid = nsm * 8, block = 256;
  const double flops = 2.0 * kChains * kIters * double(grid) * block;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    ffma_reg<<<grid, block>>>(of, 0.999f, 0.001f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (rep) printf("{\"ffma_reg_tflops\": %.2f, ", flops / ms / 1e9);
    cudaEventRecord(a);
    ffma_const<<<grid, block>>>(of);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (rep) printf("\"ffma_const_tflops\": %.2f, ", flops / ms / 1e9);
    cudaEventRecord(a);
    dfma_reg<<<grid, block>>>(od, 0.999, 0.001);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (rep) printf("\"dfma_tflops\": %.2f, \"sms\": %d}\n", flops / ms / 1e9, nsm);
  }
  return 0;
}
