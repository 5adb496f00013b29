// Counter-based byte generator G(seed, j) -- CUDA twin of inputs/gen.py.
//
// Bench / test input plumbing only: it holds no base64 arithmetic and is not
// part of the product library (paper_1704_00605_b200/libb64gpu.so).
// byte j = little-endian byte (j mod 8) of SplitMix64 output floor(j/8),
// stream started at state `seed`.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint64_t splitmix_out(uint64_t seed, uint64_t k) {
  uint64_t z = seed + (k + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// One thread per generator word k; words fully inside [begin, begin+n) whose
// destination is 8-byte aligned are stored as one u64, the rest byte-wise.
__global__ void fill_kernel(uint8_t* __restrict__ d, int64_t n, uint64_t seed,
                            int64_t begin, int64_t k0, int64_t nwords) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwords; w += stride) {
    const int64_t k = k0 + w;
    const uint64_t z = splitmix_out(seed, (uint64_t)k);
    const int64_t g0 = 8 * k;          // global byte index of the word's byte 0
    const int64_t lo = g0 - begin;     // local index
    uint8_t* p = d + lo;
    if (lo >= 0 && lo + 8 <= n && (((uintptr_t)p) & 7) == 0) {
      *reinterpret_cast<uint64_t*>(p) = z;
    } else {
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const int64_t i = lo + b;
        if (i >= 0 && i < n) d[i] = (uint8_t)(z >> (8 * b));
      }
    }
  }
}

}  // namespace

extern "C" int b64gen_fill(uint8_t* d, int64_t n, uint64_t seed, int64_t begin,
                           cudaStream_t stream) {
  if (n < 0 || begin < 0 || (n > 0 && d == nullptr)) return -1;
  if (n == 0) return 0;
  const int64_t k0 = begin / 8;
  const int64_t k1 = (begin + n + 7) / 8;
  const int64_t nwords = k1 - k0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = (nwords + 255) / 256;
  if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
  fill_kernel<<<(unsigned)blocks, 256, 0, stream>>>(d, n, seed, begin, k0, nwords);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}
