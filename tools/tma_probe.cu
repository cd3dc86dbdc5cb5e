// Standalone TMA probe: 3-D tiled box loads from a (m, n, n) fp32 tensor, compared with direct reads.
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_2005_09870_b200/csrc tools/tma_probe.cu -lcuda -o tools/tma_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include "tma.h"

using namespace pcwd;

__global__ void probe(const __grid_constant__ CUtensorMap map, const float* v, int n, int bx, int by, int nbox, int x, int y,
                      int k, int* bad) {
  extern __shared__ __align__(128) float sm[];
  __shared__ unsigned long long bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, unsigned(4 * bx * by * nbox));
    for (int j = 0; j < nbox; ++j) tma_load_3d(sm + j * bx * by, &map, x + j * bx, y, k, &bar);
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < bx * by * nbox; i += blockDim.x) {
    const int j = i / (bx * by), r = (i / bx) % by, c = i % bx;
    const int gx = x + j * bx + c, gy = y + r;
    const float ref = (gx < n && gy < n) ? v[(size_t(k) * n + gy) * n + gx] : 0.f;
    if (sm[i] != ref) atomicAdd(bad, 1);
  }
}

int main(int argc, char** argv) {
  const int n = 1024, m = 10;
  const int bx = argc > 1 ? atoi(argv[1]) : 144, by = argc > 2 ? atoi(argv[2]) : 16, nbox = argc > 3 ? atoi(argv[3]) : 2;
  float* v;
  cudaMalloc(&v, size_t(m) * n * n * 4);
  float* h = (float*)malloc(size_t(m) * n * n * 4);
  for (size_t i = 0; i < size_t(m) * n * n; ++i) h[i] = float(i % 1000003);
  cudaMemcpy(v, h, size_t(m) * n * n * 4, cudaMemcpyHostToDevice);
  CUtensorMap map;
  const cuuint64_t dims[3] = {cuuint64_t(n), cuuint64_t(n), cuuint64_t(m)};
  const cuuint64_t strides[2] = {cuuint64_t(n) * 4, cuuint64_t(n) * n * 4};
  const cuuint32_t box[3] = {cuuint32_t(bx), cuuint32_t(by), 1u};
  const cuuint32_t es[3] = {1u, 1u, 1u};
  CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, v, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d (box %d x %d, %d boxes)\n", int(r), bx, by, nbox);
  int* bad;
  cudaMalloc(&bad, 4);
  const size_t smem = size_t(bx) * by * nbox * 4;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  const int xs[] = {0, 100, 700, 880, 1000}, ys[] = {0, 500, 1008};
  for (int x : xs)
    for (int y : ys)
      for (int k : {0, 9}) {
        cudaMemset(bad, 0, 4);
        probe<<<1, 256, smem>>>(map, v, n, bx, by, nbox, x, y, k, bad);
        cudaError_t e = cudaDeviceSynchronize();
        int b = -1;
        cudaMemcpy(&b, bad, 4, cudaMemcpyDeviceToHost);
        printf("x %4d y %4d k %d: %s bad %d\n", x, y, k, cudaGetErrorString(e), b);
        if (e != cudaSuccess) return 1;
      }
  return 0;
}
