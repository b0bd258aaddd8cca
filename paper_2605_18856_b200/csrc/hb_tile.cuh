// 2-bit tier logits from per-query "h-byte" tables (G <= 4 query heads).
//
// Same function as the generic recurrence (decode.py:123-192; features
// f_j = (prod_{l<j} sin a_l) cos a_j, codec.py:459-477), specialised to
// angle width 2, where the polar step is pi/3 and a code c in {0..3} has
//   cos = {1, 1/2, -1/2, -1},  sin = {0, s, s, ~0}   (s = sin(pi/3)).
// While no code is 0 or 3 ("alive"), the running sine product is exactly
// s^j, so the feature row is s^j (1/2 - h_j) with h_j the code's high bit,
// and the dot with the query is LINEAR in the bits:
//   feat . q = sum_j (1/2 - h_j) q'_j,   q'_j = s^j q_j.
// Per decode unit the kernel folds q' into tables indexed by the 8 high bits
// of 8 consecutive rows (one 16-bit half of a code word):
//   T[p][idx] = -sum_{i<8} h_i(idx) q'_{8p+i}
// so one LDS.128 + two FADD2 replace 8 rows x (lookup, sine product,
// 2 FFMA2) of the generic recurrence.  A code 0 or 3 ("death" at row D)
// ends the sum: the feature there is s^D cos(c) and every later one is 0
// (exactly 0 for c = 0; ~1e-16 s^D for c = 3, below fp32).  Each item finds
// its first death D from the code bits (none: D = d-2), zeroes the codes at
// and after D (zero codes add nothing to T) and adds one entry of
//   E[D][c] = 1/2 sum_{j<D} q'_j + s^D cos(c) q_D          (death, c = 0 / 3)
//   E[d-2][phi] = 1/2 sum_{j<d-2} q'_j + s^(d-2) (cos phi q_{d-2} + sin phi q_{d-1})
// (no death: the circular row's pair, phi = circular code * pi/2).  Deaths
// concentrate in the last 32 rows (the polar angle of row j sits at pi/2
// with spread ~1/sqrt(d-j)); an item dead earlier takes a short divergent
// branch, nothing else changes.
// Tables are built in fp64 from the fp32 query and rounded once.
#pragma once
#include "ada_tile.cuh"

namespace sphkv {

template <int D>
struct HBGeom {
  static constexpr int W = item_words(D, 2);  // code words per item (8 / 4)
  static constexpr int NPOS = 2 * W;          // 8-row positions (16-bit halves)
  static constexpr int NP = D - 2;            // polar rows; row NP = circular
  static constexpr int NE = NP + 1;           // death rows 0..NP (NP = none)
  static constexpr uint32_t T_BYTES = NPOS * 256 * 16;
  static constexpr uint32_t E_BYTES = NE * 4 * 16;
  static constexpr uint32_t BYTES = T_BYTES + E_BYTES;
  // circular row NP and the padding row are codes 14, 15 of the last word
  static_assert(W >= 4 && NP == 16 * (W - 1) + 14, "h-byte geometry");
};

__host__ __device__ inline bool hb_supported(int d) { return d == 128 || d == 64; }
__host__ __device__ inline uint32_t hb_bytes(int d) {
  return d == 128 ? HBGeom<128>::BYTES : (d == 64 ? HBGeom<64>::BYTES : 0u);
}

// s^j in fp64 by binary exponentiation (<= 14 multiplies, ~1e-15 relative)
__device__ __forceinline__ double hb_ipow(double s, int j) {
  double r = 1.0, b = s;
  for (; j > 0; j >>= 1, b *= b)
    if (j & 1) r *= b;
  return r;
}

// Build T and E for one query group (all threads of the block).  qg: fp32
// query rows [G][D]; scratch: >= (D + NE) * 4 doubles of free shared
// memory.  Ends with __syncthreads().
template <int D>
__device__ __noinline__ void hb_build(uint8_t* tab, double* scratch, const float* __restrict__ qg,
                                      int G, double qscale) {
  using C = HBGeom<D>;
  const double s = sin(kPi / 3.0);  // sin of the 2-bit polar step (codec.py:318-321)
  double* pre = scratch + D * 4;    // [NE][4]: 1/2 sum_{j<D} q'_j
  for (int i = threadIdx.x; i < D * 4; i += blockDim.x) {
    const int j = i >> 2, g = i & 3;
    scratch[i] = (g < G && j < C::NP) ? (double)qg[g * D + j] * qscale * hb_ipow(s, j) : 0.0;
  }
  __syncthreads();
  if (threadIdx.x < 4) {  // prefix sums over the polar rows, one thread per head
    double acc = 0.0;
    for (int j = 0; j <= C::NP; ++j) {
      pre[j * 4 + threadIdx.x] = 0.5 * acc;
      acc += scratch[j * 4 + threadIdx.x];
    }
  }
  float4* T = reinterpret_cast<float4*>(tab);
  for (int e = threadIdx.x; e < C::NPOS * 256; e += blockDim.x) {
    const int p = e >> 8, idx = e & 255;
    double a[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      // idx bit 2m = high bit of row 8p+m, bit 2m+1 = high bit of row 8p+4+m
      const int h = (i < 4) ? (idx >> (2 * i)) & 1 : (idx >> (2 * (i - 4) + 1)) & 1;
      if (h)
#pragma unroll
        for (int g = 0; g < 4; ++g) a[g] -= scratch[(8 * p + i) * 4 + g];
    }
    T[e] = make_float4((float)a[0], (float)a[1], (float)a[2], (float)a[3]);
  }
  __syncthreads();
  float4* E = reinterpret_cast<float4*>(tab + C::T_BYTES);
  const double sNP = hb_ipow(s, C::NP) * qscale;
  for (int e = threadIdx.x; e < C::NE * 4; e += blockDim.x) {
    const int Dd = e >> 2, c = e & 3;
    double a[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      double acc = pre[Dd * 4 + g];
      if (Dd < C::NP) {  // death at row Dd with code c (0 -> cos 1, 3 -> cos -1)
        acc += (c == 0 ? 1.0 : (c == 3 ? -1.0 : 0.0)) * scratch[Dd * 4 + g];
      } else if (g < G) {  // alive through every polar row: circular pair, phi = c pi/2
        const double cs = (c == 0) ? 1.0 : (c == 2 ? -1.0 : 0.0);
        const double sn = (c == 1) ? 1.0 : (c == 3 ? -1.0 : 0.0);
        acc += sNP * (cs * (double)qg[g * D + C::NP] + sn * (double)qg[g * D + C::NP + 1]);
      }
      a[g] = acc;
    }
    E[e] = make_float4((float)a[0], (float)a[1], (float)a[2], (float)a[3]);
  }
  __syncthreads();
}

// (not volatile: the tables are read-only while tiles run, so the loads may
// be scheduled freely; they are only issued after the build's barrier)
__device__ __forceinline__ void lds_f4(uint32_t addr, ptx::f2& a, ptx::f2& b) {
  asm("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(a.v), "=l"(b.v) : "r"(addr));
}
__device__ __forceinline__ void f2_add_acc(ptx::f2& acc, ptx::f2 b) {
  asm("add.rn.f32x2 %0, %0, %1;" : "+l"(acc.v) : "l"(b.v));
}

// Logits (base 2) of a 128-item tile of 2-bit pages.  hb: shared-memory
// address of T (E follows it).
template <int D, int GP>
__device__ __noinline__ void ada_tile_hb(const uint8_t* __restrict__ blkb, int sub, int lane,
                                         uint32_t hb, uint32_t rbit0, int rb, float rscale,
                                         float lg[TK][2 * GP]) {
  static_assert(GP <= 2, "h-byte tables hold 4 heads");
  using C = HBGeom<D>;
  constexpr int W = C::W;
  const uint4* blk4 = reinterpret_cast<const uint4*>(blkb);
  uint32_t w[TK][W];
#pragma unroll
  for (int k = 0; k < TK; ++k) load_item<W>(w[k], blk4, sub * TK + k, lane);
  ptx::f2 acc[TK][2];
#pragma unroll
  for (int k = 0; k < TK; ++k) {
    // a code 0 or 3 (equal bits) before the last two words?
    uint32_t e = 0;
#pragma unroll
    for (int i = 0; i < W - 2; ++i) e |= ~(w[k][i] ^ (w[k][i] >> 1));
    int dr;       // death row (NP: none)
    uint32_t c;   // its code (none: the circular code)
    if ((e & 0x55555555u) == 0u) {
      // common case: the first death, if any, is in the last two words
      const uint64_t ab = (uint64_t)w[k][W - 2] | ((uint64_t)w[k][W - 1] << 32);
      const uint64_t dead = ~(ab ^ (ab >> 1)) & 0x0555555555555555ull;  // polar codes only
      const int pos = __ffsll((long long)dead) - 1;                      // -1: none
      dr = pos < 0 ? C::NP : 16 * (W - 2) + (pos >> 1);
      const int cp = pos < 0 ? 60 : pos;  // code 30 of the pair = circular row NP
      c = (uint32_t)(ab >> cp) & 3u;
      const uint64_t keep = (1ull << cp) - 1ull;  // zero the codes from the death on
      w[k][W - 2] = (uint32_t)(ab & keep);
      w[k][W - 1] = (uint32_t)((ab & keep) >> 32);
    } else {
      // rare: an earlier death -- find it, zero everything from there on
      dr = C::NP;
      c = 0u;
#pragma unroll
      for (int i = 0; i < W; ++i) {
        const uint32_t dd = ~(w[k][i] ^ (w[k][i] >> 1)) & 0x55555555u;
        if (dr == C::NP && dd != 0u) {
          const int pos = __ffs(dd) - 1;
          dr = 16 * i + (pos >> 1);
          c = (w[k][i] >> pos) & 3u;
          w[k][i] &= (1u << pos) - 1u;
        } else if (dr != C::NP) {
          w[k][i] = 0u;
        }
      }
    }
    lds_f4(hb + C::T_BYTES + (uint32_t)(dr * 4 + (int)c) * 16u, acc[k][0], acc[k][1]);
  }
#pragma unroll
  for (int p = 0; p < C::NPOS; ++p) {
#pragma unroll
    for (int k = 0; k < TK; ++k) {
      const uint32_t x = w[k][p >> 1];
      // idx * 16: high bits of rows 8p..8p+3 -> idx bits 0,2,4,6 and of rows
      // 8p+4..8p+7 -> bits 1,3,5,7
      const uint32_t s1 = (p & 1) ? (x >> 13) : (x << 3);
      const uint32_t s2 = (p & 1) ? (x >> 20) : (x >> 4);
      const uint32_t off = (s1 & 0x550u) | (s2 & 0xAA0u);
      ptx::f2 t0, t1;
      lds_f4(hb + (uint32_t)p * 4096u + off, t0, t1);
      f2_add_acc(acc[k][0], t0);
      f2_add_acc(acc[k][1], t1);
    }
  }
  const uint32_t* blk = reinterpret_cast<const uint32_t*>(blkb);
#pragma unroll
  for (int k = 0; k < TK; ++k) {
    const uint32_t rc = read_bits_g(blk, rbit0 + (uint64_t)(sub * TTI + 32 * k + lane) * rb, rb);
    const float rr = (float)rc * rscale;
    const float v[4] = {ptx::f2_lo(acc[k][0]), ptx::f2_hi(acc[k][0]), ptx::f2_lo(acc[k][1]),
                        ptx::f2_hi(acc[k][1])};
#pragma unroll
    for (int g = 0; g < 2 * GP; ++g) lg[k][g] = rr * v[g];
  }
}

}  // namespace sphkv
