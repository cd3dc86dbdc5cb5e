// sort.cu — the library's own scan and CSR transpose (no CUB device-wide primitives):
//   * exclusive_scan_i64: three-phase block scan (tile sums, a scan of the tile sums, tile rescans).
//   * csr_transpose: Θᵀ as a CSR over the columns, the entries of each column in increasing row order — a stable
//     LSD radix sort of the (row-ordered) entries by column, 8-bit digits, one histogram / scan / scatter per digit.
//     Stability (rank of an item among equal digits = its position order within the tile) keeps the row order, so
//     Θᵀ x is a gather with the same summation order every time (deterministic, no atomics in the product).
#include <algorithm>
#include <cstdint>

#include "kernels.cuh"

namespace pcwd {
namespace {

constexpr int kST = 256;          // threads per CTA
constexpr int kItems = 16;        // items per thread per tile
constexpr int kTile = kST * kItems;

// ---- exclusive scan of int64 --------------------------------------------------------------------------------
__device__ int64_t block_excl_scan(int64_t x, int64_t* sh, int64_t* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t v = x;
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  if (lane == 31) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    int64_t s = lane < kST / 32 ? sh[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < kST / 32) sh[lane] = s;
  }
  __syncthreads();
  const int64_t before = (w > 0 ? sh[w - 1] : 0) + v - x;
  *total = sh[kST / 32 - 1];
  __syncthreads();
  return before;
}

__global__ void scan_tiles(const int64_t* __restrict__ in, int64_t n, int64_t* __restrict__ sums) {
  __shared__ int64_t sh[kST / 32];
  const int64_t base = int64_t(blockIdx.x) * kTile + int64_t(threadIdx.x) * kItems;
  int64_t s = 0;
  for (int i = 0; i < kItems; ++i) s += base + i < n ? in[base + i] : 0;
  int64_t tot;
  block_excl_scan(s, sh, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void scan_sums(int64_t* sums, int64_t nt) {   // one CTA, in place, exclusive
  __shared__ int64_t sh[kST / 32];
  int64_t carry = 0;
  for (int64_t b = 0; b < nt; b += kST) {
    const int64_t i = b + threadIdx.x;
    const int64_t x = i < nt ? sums[i] : 0;
    int64_t tot;
    const int64_t e = block_excl_scan(x, sh, &tot);
    if (i < nt) sums[i] = carry + e;
    carry += tot;
  }
}

__global__ void scan_apply(const int64_t* __restrict__ in, int64_t n, const int64_t* __restrict__ sums,
                           int64_t* __restrict__ out) {
  __shared__ int64_t sh[kST / 32];
  const int64_t base = int64_t(blockIdx.x) * kTile + int64_t(threadIdx.x) * kItems;
  int64_t v[kItems];
  int64_t s = 0;
  for (int i = 0; i < kItems; ++i) {
    v[i] = base + i < n ? in[base + i] : 0;
    s += v[i];
  }
  int64_t tot;
  int64_t run = block_excl_scan(s, sh, &tot) + sums[blockIdx.x];
  for (int i = 0; i < kItems; ++i) {
    if (base + i < n) out[base + i] = run;
    run += v[i];
  }
}

// ---- stable LSD radix sort of the entries by column ----------------------------------------------------------
__global__ void expand_rows(const int64_t* __restrict__ rp, int64_t rows, int32_t* __restrict__ row) {
  const int64_t warp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  for (int64_t j = rp[warp] + lane; j < rp[warp + 1]; j += 32) row[j] = int32_t(warp);
}

__global__ void digit_hist(const int32_t* __restrict__ key, int64_t nnz, int shift, int64_t ntiles,
                           int64_t* __restrict__ cnt) {
  __shared__ int h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = int64_t(blockIdx.x) * kTile;
  for (int i = 0; i < kItems; ++i) {
    const int64_t j = base + int64_t(i) * kST + threadIdx.x;
    if (j < nnz) atomicAdd(&h[(key[j] >> shift) & 255], 1);
  }
  __syncthreads();
  cnt[int64_t(threadIdx.x) * ntiles + blockIdx.x] = h[threadIdx.x];   // digit-major: [digit][tile]
}

template <typename T>
__global__ void digit_scatter(const int32_t* __restrict__ key, const int32_t* __restrict__ row, const T* __restrict__ val,
                              int64_t nnz, int shift, int64_t ntiles, const int64_t* __restrict__ off,
                              int32_t* __restrict__ key2, int32_t* __restrict__ row2, T* __restrict__ val2) {
  __shared__ int64_t running[256];
  __shared__ int wcnt[kST / 32][257];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  running[threadIdx.x] = off[int64_t(threadIdx.x) * ntiles + blockIdx.x];
  for (int q = 0; q < kST / 32; ++q) wcnt[q][threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = int64_t(blockIdx.x) * kTile;
  for (int r = 0; r < kItems; ++r) {   // rounds in item order: earlier rounds, then lower warps, then lower lanes
    const int64_t j = base + int64_t(r) * kST + threadIdx.x;
    const bool ok = j < nnz;
    const int d = ok ? (key[j] >> shift) & 255 : 256;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    if (ok && rank == 0) wcnt[w][d] = __popc(peers);
    __syncthreads();
    if (ok) {
      int64_t pos = running[d] + rank;
      for (int q = 0; q < w; ++q) pos += wcnt[q][d];
      key2[pos] = key[j];
      row2[pos] = row[j];
      val2[pos] = val[j];
    }
    __syncthreads();
    int add = 0;
    for (int q = 0; q < kST / 32; ++q) { add += wcnt[q][threadIdx.x]; wcnt[q][threadIdx.x] = 0; }
    running[threadIdx.x] += add;
    __syncthreads();
  }
}

__global__ void col_bounds(const int32_t* __restrict__ key, int64_t nnz, int64_t ncols, int64_t* __restrict__ rpT) {
  // rpT[c] = first position whose key ≥ c (keys sorted): boundaries where the key changes
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j <= nnz; j += int64_t(gridDim.x) * blockDim.x) {
    const int64_t lo = j == 0 ? 0 : int64_t(key[j - 1]) + 1;
    const int64_t hi = j == nnz ? ncols : int64_t(key[j]);
    for (int64_t c = lo; c <= hi; ++c) rpT[c] = j;
  }
}

int grid_of(int64_t n, int per) { return int(std::max<int64_t>(1, std::min<int64_t>((n + per - 1) / per, 148 * 32))); }

}  // namespace

cudaError_t exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, void* tmp, size_t* tmp_bytes,
                               cudaStream_t st) {
  const int64_t nt = (n + kTile - 1) / kTile;
  if (!tmp) {
    *tmp_bytes = size_t(std::max<int64_t>(nt, 1)) * sizeof(int64_t);
    return cudaSuccess;
  }
  if (n == 0) return cudaSuccess;
  int64_t* sums = static_cast<int64_t*>(tmp);
  scan_tiles<<<int(nt), kST, 0, st>>>(in, n, sums);
  scan_sums<<<1, kST, 0, st>>>(sums, nt);
  scan_apply<<<int(nt), kST, 0, st>>>(in, n, sums, out);
  return cudaGetLastError();
}

size_t csr_transpose_bytes(int64_t nnz, int64_t ncols, int vbytes) {
  const int64_t ntiles = (nnz + kTile - 1) / kTile;
  const int64_t cnts = 256 * std::max<int64_t>(ntiles, 1);
  size_t scan_tmp = 0;
  exclusive_scan_i64(nullptr, nullptr, cnts, nullptr, &scan_tmp, nullptr);
  (void)ncols;
  return size_t(cnts) * 8 * 2 + scan_tmp + size_t(nnz) * (4 + 4 + vbytes + 4) + 4096;   // + 7 × 256 B alignment
}

// work: ≥ csr_transpose_bytes + (ncols + 1)·8 + nnz·(4 + vbytes) (the caller's historical layout; only
// csr_transpose_bytes is used).  Outputs rpT (ncols + 1), rowT (nnz, shard-local rows), valT (nnz).
cudaError_t csr_transpose(const int64_t* rp, const int32_t* col, const void* val, int64_t rows, int64_t nnz,
                          int64_t ncols, int vbytes, int64_t* rpT, int32_t* rowT, void* valT, void* work,
                          size_t work_bytes, cudaStream_t st) {
  (void)work_bytes;
  const int64_t ntiles = std::max<int64_t>((nnz + kTile - 1) / kTile, 1);
  const int64_t cnts = 256 * ntiles;
  char* w = static_cast<char*>(work);
  auto take = [&](size_t b) { char* p = w; w += (b + 255) & ~size_t(255); return p; };
  int64_t* cnt = reinterpret_cast<int64_t*>(take(cnts * 8));
  int64_t* off = reinterpret_cast<int64_t*>(take(cnts * 8));
  size_t scan_tmp = 0;
  exclusive_scan_i64(nullptr, nullptr, cnts, nullptr, &scan_tmp, st);
  void* stmp = take(scan_tmp);
  int32_t* keyA = reinterpret_cast<int32_t*>(take(size_t(nnz) * 4));
  int32_t* rowA = reinterpret_cast<int32_t*>(take(size_t(nnz) * 4));
  char* valA = take(size_t(nnz) * vbytes);
  // ping-pong: (keyA,rowA,valA) ↔ (keyB = col copy target, rowT, valT)
  cudaError_t e;
  if (nnz == 0) {
    if ((e = cudaMemsetAsync(rpT, 0, (ncols + 1) * 8, st))) return e;
    return cudaSuccess;
  }
  if ((e = cudaMemcpyAsync(keyA, col, size_t(nnz) * 4, cudaMemcpyDeviceToDevice, st))) return e;
  if ((e = cudaMemcpyAsync(valA, val, size_t(nnz) * vbytes, cudaMemcpyDeviceToDevice, st))) return e;
  expand_rows<<<int((rows * 32 + kST - 1) / kST), kST, 0, st>>>(rp, rows, rowA);
  int bits = 1;
  while ((int64_t(1) << bits) < ncols) ++bits;
  const int passes = (bits + 7) / 8;
  // the last pass must land in (rowT, valT): with an odd pass count A → T directly, else via a scratch second buffer
  int32_t* keyB = reinterpret_cast<int32_t*>(take(size_t(nnz) * 4));
  char* rowBuf[2] = {reinterpret_cast<char*>(rowA), reinterpret_cast<char*>(rowT)};
  char* valBuf[2] = {valA, static_cast<char*>(valT)};
  int32_t* keyBuf[2] = {keyA, keyB};
  int cur = 0;
  if (passes % 2 == 0) {   // start the ping-pong so that the final pass writes buffer 1
    if ((e = cudaMemcpyAsync(rowT, rowA, size_t(nnz) * 4, cudaMemcpyDeviceToDevice, st))) return e;
    if ((e = cudaMemcpyAsync(valT, valA, size_t(nnz) * vbytes, cudaMemcpyDeviceToDevice, st))) return e;
    if ((e = cudaMemcpyAsync(keyB, keyA, size_t(nnz) * 4, cudaMemcpyDeviceToDevice, st))) return e;
    cur = 1;
  }
  for (int p = 0; p < passes; ++p) {
    const int shift = 8 * p;
    digit_hist<<<int(ntiles), kST, 0, st>>>(keyBuf[cur], nnz, shift, ntiles, cnt);
    if ((e = exclusive_scan_i64(cnt, off, cnts, stmp, &scan_tmp, st))) return e;
    const int nx = cur ^ 1;
    if (vbytes == 8)
      digit_scatter<double><<<int(ntiles), kST, 0, st>>>(
          keyBuf[cur], reinterpret_cast<int32_t*>(rowBuf[cur]), reinterpret_cast<double*>(valBuf[cur]), nnz, shift,
          ntiles, off, keyBuf[nx], reinterpret_cast<int32_t*>(rowBuf[nx]), reinterpret_cast<double*>(valBuf[nx]));
    else
      digit_scatter<float><<<int(ntiles), kST, 0, st>>>(
          keyBuf[cur], reinterpret_cast<int32_t*>(rowBuf[cur]), reinterpret_cast<float*>(valBuf[cur]), nnz, shift,
          ntiles, off, keyBuf[nx], reinterpret_cast<int32_t*>(rowBuf[nx]), reinterpret_cast<float*>(valBuf[nx]));
    cur = nx;
  }
  // cur == 1: (keyB, rowT, valT) hold the entries sorted by column, rows increasing within a column
  col_bounds<<<grid_of(nnz + 1, kST), kST, 0, st>>>(keyBuf[cur], nnz, ncols, rpT);
  return cudaGetLastError();
}

}  // namespace pcwd
