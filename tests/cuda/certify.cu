// TEST INFRASTRUCTURE ONLY -- a brute-force skyline certificate on the GPU.
//
// Independent of the product kernels (paper_2107_09993_b200/csrc): it shares
// no code with them and implements only the definition the reference's own
// brute-force oracle uses, brute_force_skyline (/root/reference/proj/src/
// baseline.cpp:32-58) with point_dominates (proj/include/skycell/
// dataset.hpp:55-62): q dominates p iff q <= p in every dimension and q < p
// in at least one.
//
// found[j] = 1 iff some row of the whole data set dominates query row j.
// Checked by tests/test_gpu_certificate.py on configurations the CPU
// reference cannot finish ("Oracle limits"): sampled
// reported ids must have found = 0, sampled unreported ids found = 1.
//
// Plain data-parallel layout: each thread owns data rows (grid-stride), each
// CTA stages a tile of query rows in shared memory, every thread tests its
// row against every query of the tile.  n * m tests, no early exit: at
// n = 1e8 and m = 2e4 about 2e12 tests, well under a second on a B200.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

constexpr int kTile = 1024;

template <int D>
__global__ void k_certify(const float* __restrict__ data, unsigned long long n, const float* __restrict__ q,
                          int m, uint8_t* __restrict__ found) {
  __shared__ float qs[kTile * D];
  __shared__ int hit[kTile];
  for (int t0 = 0; t0 < m; t0 += kTile) {
    const int tn = min(kTile, m - t0);
    __syncthreads();
    for (int i = threadIdx.x; i < tn * D; i += blockDim.x) qs[i] = q[(size_t)t0 * D + i];
    for (int i = threadIdx.x; i < tn; i += blockDim.x) hit[i] = 0;
    __syncthreads();
    for (unsigned long long r = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; r < n;
         r += (unsigned long long)gridDim.x * blockDim.x) {
      float v[D];
#pragma unroll
      for (int k = 0; k < D; ++k) v[k] = data[r * D + k];
      for (int j = 0; j < tn; ++j) {
        bool le = true, lt = false;
#pragma unroll
        for (int k = 0; k < D; ++k) {
          const float w = qs[j * D + k];
          le &= v[k] <= w;
          lt |= v[k] < w;
        }
        if (le && lt) hit[j] = 1;
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < tn; i += blockDim.x)
      if (hit[i]) found[t0 + i] = 1;
  }
}

}  // namespace

extern "C" int certify_dominated(const float* data, unsigned long long n, int d, const float* queries, int m,
                                 uint8_t* found, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(found, 0, (size_t)m, s) != cudaSuccess) return 1;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)sms * 4;
#define CERT_CASE(DD) \
  case DD: k_certify<DD><<<grid, 256, 0, s>>>(data, n, queries, m, found); break;
  switch (d) {
    CERT_CASE(2) CERT_CASE(3) CERT_CASE(4) CERT_CASE(5) CERT_CASE(6) CERT_CASE(7) CERT_CASE(8)
    default: return 2;
  }
#undef CERT_CASE
  if (cudaGetLastError() != cudaSuccess) return 3;
  return cudaStreamSynchronize(s) == cudaSuccess ? 0 : 4;
}
