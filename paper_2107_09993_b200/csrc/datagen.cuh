// On-device synthetic data, same streams as the reference generator
// (proj/src/datagen.cpp:22-87, proj/include/skycell/datagen.hpp:22-60):
// splitmix64-seeded xoshiro256++ per 65,536-point block, uniforms as
// (next >> 11) * 2^-53, normals by Box-Muller.  One thread per block stream.
//
// Independent data is bit-identical to the host generator (integer ops and an
// exact conversion).  Correlated / anti-correlated data go through CUDA's
// log/cos (sqrt is correctly rounded), which may differ from glibc by an ulp;
// after the 2^-24 quantisation that changes a coordinate with probability
// ~2^-29.  Parity tests therefore always feed the *same bytes* to the GPU path
// and to the oracle; the generator only has to reproduce the distributions.
#pragma once

#include "common.cuh"

namespace sk {

struct Xo {
  u64 s[4];
  __device__ __forceinline__ static u64 rotl(u64 x, int k) { return (x << k) | (x >> (64 - k)); }
  __device__ __forceinline__ u64 next() {
    const u64 result = rotl(s[0] + s[3], 23) + s[0];
    const u64 t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
  }
  __device__ __forceinline__ double uniform() { return __dmul_rn((double)(next() >> 11), 0x1.0p-53); }
  __device__ __forceinline__ double normal(double mean, double stddev) {
    const double u1 = __dmul_rn((double)((next() >> 11) + 1), 0x1.0p-53);
    const double u2 = uniform();
    const double mag = sqrt(__dmul_rn(-2.0, log(u1)));
    return __dadd_rn(mean, __dmul_rn(__dmul_rn(stddev, mag), cos(__dmul_rn(2.0 * 3.141592653589793, u2))));
  }
};

__device__ __forceinline__ u64 splitmix(u64& st) {
  u64 z = (st += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double clamp_unit(double v) {
  return v < 0.0 ? 0.0 : (kUnitUpperBound < v ? kUnitUpperBound : v);
}

// kind 0: raw f64; kind 1: f32 quantised to the 2^-24 grid.
// Writes records [rbegin, rbegin + rcount) of the n-record dataset to out
// (record rbegin at out[0]): a shard generates only its own index range.
template <int D>
__global__ void k_generate(int dist, u64 n, u64 seed, int kind, u64 rbegin, u64 rcount, void* out) {
  pdl_enter();
  const u64 b0 = rbegin / 65536, b1 = (rbegin + rcount + 65535) / 65536;
  for (u64 b = b0 + blockIdx.x * (u64)blockDim.x + threadIdx.x; b < b1; b += (u64)gridDim.x * blockDim.x) {
    Xo rng;
    u64 st = seed ^ ((b + 1) * 0x9e3779b97f4a7c15ull);
    for (int i = 0; i < 4; ++i) rng.s[i] = splitmix(st);
    const u64 begin = b * 65536;
    const u64 count = (n - begin < 65536) ? n - begin : 65536;
    const u64 rend = rbegin + rcount;
    for (u64 p = 0; p < count; ++p) {
      const u64 rec = begin + p;
      if (rec >= rend) break;
      double row[D];
      if (dist == 0) {
#pragma unroll
        for (int k = 0; k < D; ++k) row[k] = rng.uniform();
      } else if (dist == 1) {
        const double t = rng.uniform();
#pragma unroll
        for (int k = 0; k < D; ++k) row[k] = clamp_unit(__dadd_rn(t, rng.normal(0.0, 0.05)));
      } else {
        double sum = 0;
#pragma unroll
        for (int k = 0; k < D; ++k) {
          row[k] = rng.uniform();
          sum = __dadd_rn(sum, row[k]);
        }
        const double shift = __ddiv_rn(__dsub_rn(D / 2.0, sum), (double)D);
#pragma unroll
        for (int k = 0; k < D; ++k) row[k] = clamp_unit(__dadd_rn(__dadd_rn(row[k], shift), rng.normal(0.0, 0.05)));
      }
      if (rec < rbegin) continue;  // the stream still advances
      const u64 o = (rec - rbegin) * D;
      if (kind == 0) {
#pragma unroll
        for (int k = 0; k < D; ++k) static_cast<double*>(out)[o + k] = row[k];
      } else {
#pragma unroll
        for (int k = 0; k < D; ++k)
          static_cast<float*>(out)[o + k] = (float)__dmul_rn(floor(__dmul_rn(row[k], 16777216.0)), 1.0 / 16777216.0);
      }
    }
  }
}

}  // namespace sk
