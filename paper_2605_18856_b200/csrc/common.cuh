// Shared device/host helpers for libsphkv_b200 (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>
#include <string>

#include "../../include/sphkv_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libsphkv_b200 is built for sm_100a only"
#endif

namespace sphkv {

// ---- error reporting (thread-local, surfaced by sphkv_last_error) ---------
void set_error(const char* fmt, ...);
int fail(int code, const char* fmt, ...);

#define SPHKV_CUDA_TRY(expr)                                                   \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess)                                                     \
      return ::sphkv::fail(SPHKV_E_CUDA, "%s failed: %s (%s:%d)", #expr,       \
                           cudaGetErrorString(_e), __FILE__, __LINE__);        \
  } while (0)

#define SPHKV_LAUNCH_CHECK()                                                   \
  do {                                                                         \
    cudaError_t _e = cudaGetLastError();                                       \
    if (_e != cudaSuccess)                                                     \
      return ::sphkv::fail(SPHKV_E_CUDA, "launch failed: %s (%s:%d)",          \
                           cudaGetErrorString(_e), __FILE__, __LINE__);        \
  } while (0)

constexpr double kTwoPi = 6.283185307179586;   // 2.0 * math.pi
constexpr double kPi = 3.141592653589793;      // math.pi
constexpr double kNormEps = 1e-12;             // codec.py:218
constexpr int SM_COUNT = 148;

// A tier table passed BY VALUE as a kernel parameter (512 bytes): no device
// copy, hence no hidden allocation and capture-safe in CUDA graphs.
struct TierSet {
  sphkv_tier_t t[SPHKV_MAX_TIERS];
};
inline TierSet make_tierset(const sphkv_tier_t* host, int n) {
  TierSet ts{};
  for (int i = 0; i < n && i < SPHKV_MAX_TIERS; ++i) ts.t[i] = host[i];
  return ts;
}

__host__ __device__ inline int64_t div_up(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Device angle-code layout of a page: "word-interleaved, item-major" (WI).
// Item i's d-1 angle codes form one LSB-first bit string (code j at bits
// [j*b, j*b+b)), padded to W words, W = ceil((d-1)*b/32) rounded up to a
// multiple of 4.  Items are grouped in granules of 32 and the string is cut
// into 16-byte quads; quad w4 of item i lives at quad index
//   ((i / 32) * (W / 4) + w4) * 32 + (i % 32)
// so lane l of a warp loading quad w4 of items 32t..32t+31 issues one fully
// coalesced 512-byte LDG.128, and each lane ends up holding its own item's
// whole code string in registers.  The radius codes follow as one LSB-first
// row of P*rb bits (the reference radius stream, store.py:205-211).  Export
// (sphkv_export_streams) converts back to the reference's coordinate-major
// SoA stream bit for bit.
__host__ __device__ constexpr int item_words(int d, int abits) {
  return ((((d - 1) * abits + 31) / 32) + 3) / 4 * 4;
}
__host__ __device__ inline uint64_t angle_part_bytes(int d, int P, int abits) {
  return (uint64_t)((P + 31) / 32) * item_words(d, abits) * 128;
}
__host__ __device__ inline uint64_t code_block_bytes(int d, int P, int abits, int rbits) {
  const uint64_t rbytes = ((uint64_t)P * rbits + 7) / 8;
  return angle_part_bytes(d, P, abits) + ((rbytes + 15) & ~uint64_t(15));
}
// Bytes per dimension row of the decode kernels' shared q table: GP packed
// (q_2g, q_2g+1) float2 pairs, padded to 32 B when GP = 3 so every row start
// stays 16-byte aligned for the paired 128-bit loads.
__host__ __device__ constexpr uint32_t q_row_bytes(int GP) { return (GP == 3 ? 4u : (uint32_t)GP) * 8u; }
// word index (uint32 units from the block start) of string word w of item i
__host__ __device__ inline uint64_t wi_word(int i, int w, int W) {
  return (((uint64_t)(i >> 5) * (W >> 2) + (w >> 2)) * 32 + (i & 31)) * 4 + (w & 3);
}

// Value-pool element offset (in fp16 elements) of (item i, column e) inside a
// page: 16-byte chunks XOR-swizzled by (i & 7) -- see sphkv_b200.h.
__host__ __device__ inline int vswz(int i, int e, int d_v) {
  const int nchunks = d_v >> 3;  // d_v is padded to a multiple of 16
  const int mask = (nchunks < 8 ? nchunks : 8) - 1;
  int chunk = (e >> 3) ^ (i & mask);
  return i * d_v + chunk * 8 + (e & 7);
}

// ---- numpy-exact fp64 helpers (compiled with --fmad=false where used) ----

template <typename T>
__device__ inline double load_as_double(const T* p) { return (double)(*p); }
template <>
__device__ inline double load_as_double<__nv_bfloat16>(const __nv_bfloat16* p) {
  return (double)__bfloat162float(*p);
}
template <>
__device__ inline double load_as_double<__half>(const __half* p) {
  return (double)__half2float(*p);
}

// numpy pairwise_sum (loops_utils.h) of n doubles produced by f(i).
template <typename F>
__device__ double np_pairwise_sum(F f, int lo, int n) {
  // iterative emulation of the recursion via an explicit stack of blocks
  // (n <= 4096 in practice; recursion depth log2(n/128)).
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, f(lo + i));
    return res;
  } else if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = f(lo + j);
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], f(lo + i + j));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, f(lo + i));
    return res;
  } else {
    int n2 = n / 2;
    n2 -= n2 % 8;
    double a = np_pairwise_sum(f, lo, n2);
    double b = np_pairwise_sum(f, lo + n2, n - n2);
    return __dadd_rn(a, b);
  }
}

// Quantizers (codec.py:318-340): division by the step constants, rint.
__device__ inline double polar_step(int bits) {
  return __ddiv_rn(kPi, (double)((1ull << bits) - 1ull));
}
__device__ inline double circular_step(int bits) {
  return __ddiv_rn(kTwoPi, (double)(1ull << bits));
}
__device__ inline uint32_t quant_polar(double a, double step, int bits) {
  double c = rint(__ddiv_rn(a, step));
  double top = (double)((1ull << bits) - 1ull);
  c = fmin(fmax(c, 0.0), top);  // np.clip
  return (uint32_t)c;
}
__device__ inline uint32_t quant_circ(double a, double cstep, int bits) {
  long long c = (long long)rint(__ddiv_rn(a, cstep));
  long long m = (long long)(1ull << bits);
  c %= m;
  if (c < 0) c += m;  // np.mod with positive divisor
  return (uint32_t)c;
}

}  // namespace sphkv
