// ADA logit tile: logits of 4 consecutive page items per lane, straight from
// the angle/radius codes (decode.py:123-192: l = (r_q/sqrt d) r~ (feat.qfeat)).
//
// The feature row of an item is the recurrence f_j = (prod_{l<j} sin a_l) cos a_j
// (codec.py:459-477); the kernel never forms it in memory: per code row it
// looks (cos, sin) up in a shared-memory table, updates the running sine
// product and accumulates f_j * q_j for all G query heads with packed FFMA2
// (q is pre-scaled by log2(e)/sqrt(d), so logits come out in base-2 units).
#pragma once
#include "common.cuh"
#include "ptx.cuh"

#ifndef SPHKV_RING
#define SPHKV_RING 1
#endif

namespace sphkv {

constexpr int LUT_MAX_BITS = 12;
#ifndef SPHKV_LUT_KB
#define SPHKV_LUT_KB 90
#endif
constexpr int LUT_BUDGET_BYTES = SPHKV_LUT_KB * 1024;

// Polar (cos, sin) tables in shared memory, one per tier with B <= 12.
//  * B <= 4: "pair" tables indexed by two consecutive items' codes (2B bits);
//    an entry (cos a, cos b, sin a, sin b) is one LDS.128 feeding packed FMUL2.
//  * 5 <= B <= 12: single-code tables, entry (cos, sin) = one LDS.64.
// Random gathers from a small table bank-conflict heavily, so when the budget
// allows a table is stored REP times interleaved: entry e of copy r lives at
// (e * REP + r) * entry_bytes and lane L reads copy L % REP.  REP = 8 for
// 16-byte entries (8 lanes per LDS.128 phase) and 16 for 8-byte entries
// (16 lanes per LDS.64 phase), so every phase hits distinct banks and the
// entry stride is 128 bytes either way.
__host__ __device__ constexpr int lut_group(int B) { return B <= 4 ? 2 : 1; }
__host__ __device__ constexpr int lut_entry_bytes(int B) { return 8 * lut_group(B); }
__host__ __device__ constexpr int lut_rep(int B) { return lut_group(B) == 2 ? 8 : 16; }
__host__ __device__ constexpr int lut_bytes(int B, bool repl) {
  return (1 << (lut_group(B) * B)) * lut_entry_bytes(B) * (repl ? lut_rep(B) : 1);
}

// Encoded per-tier table descriptor: (byte offset << 1) | replicated, or -1.
__host__ __device__ inline int lut_layout_tiers(const sphkv_tier_t* tiers, int n_tiers,
                                                int off[SPHKV_MAX_TIERS]) {
  for (int t = 0; t < SPHKV_MAX_TIERS; ++t) off[t] = -1;
  int minimal = 0;
  for (int t = 1; t < n_tiers; ++t) {
    const int b = tiers[t].angle_bits;
    if (b <= LUT_MAX_BITS && minimal + lut_bytes(b, false) <= LUT_BUDGET_BYTES) {
      minimal += lut_bytes(b, false);
      off[t] = 0;  // has a table; placed below
    }
  }
  bool repl[SPHKV_MAX_TIERS] = {};
  int total = minimal;
  for (int pass_b = 1; pass_b <= LUT_MAX_BITS; ++pass_b)  // narrow tiers first
    for (int t = 1; t < n_tiers; ++t)
      if (off[t] == 0 && tiers[t].angle_bits == pass_b) {
        const int extra = lut_bytes(pass_b, true) - lut_bytes(pass_b, false);
        if (total + extra <= LUT_BUDGET_BYTES) {
          repl[t] = true;
          total += extra;
        }
      }
  int used = 0;  // every table size is a multiple of 16 bytes
  for (int t = 1; t < n_tiers; ++t)
    if (off[t] == 0) {
      off[t] = (used << 1) | (repl[t] ? 1 : 0);
      used += lut_bytes(tiers[t].angle_bits, repl[t]);
    }
  return used;
}

// Fill byte range [i*16, i*16+16) ... one entry copy per call: tier bits B,
// entry e, copy r of a table starting at `dst`.
__device__ inline void lut_write_entry(uint8_t* dst, int B, bool repl, int e, int r) {
  const double step = kPi / (double)((1u << B) - 1u);
  const int R = repl ? lut_rep(B) : 1;
  float* out = reinterpret_cast<float*>(dst + ((size_t)e * R + r) * lut_entry_bytes(B));
  if (lut_group(B) == 1) {
    double sn, cs;
    sincos((double)e * step, &sn, &cs);
    out[0] = (float)cs;
    out[1] = (float)sn;
  } else {
    const uint32_t M = (1u << B) - 1u;
    double sa, ca, sb, cb;
    sincos((double)(e & M) * step, &sa, &ca);
    sincos((double)((e >> B) & M) * step, &sb, &cb);
    out[0] = (float)ca;
    out[1] = (float)cb;
    out[2] = (float)sa;
    out[3] = (float)sb;
  }
}

// all (entry, copy) pairs of every tier's table, strided over `nthreads`
__device__ inline void lut_fill(uint8_t* lut, const sphkv_tier_t* tiers, int n_tiers,
                                const int* enc, int tid, int nthreads) {
  for (int t = 1; t < n_tiers; ++t) {
    if (enc[t] < 0) continue;
    const int B = tiers[t].angle_bits;
    const bool repl = enc[t] & 1;
    const int R = repl ? lut_rep(B) : 1;
    const int n = (1 << (lut_group(B) * B)) * R;
    for (int i = tid; i < n; i += nthreads)
      lut_write_entry(lut + (enc[t] >> 1), B, repl, i / R, i % R);
  }
}

template <int B>
struct CodeWin {
  // max over lanes of the in-word shift of a lane's 4 codes (4 * lane * B mod 32)
  static constexpr int MAXSH = (B % 2) ? 28 : ((B % 4) ? 24 : ((B % 8) ? 16 : 0));
  static constexpr int WORDS = (4 * B <= 32 && MAXSH + 4 * B <= 32) ? 1
                             : (MAXSH + 4 * B <= 64 ? 2 : 3);
};

// 64-bit window of a lane's 4 codes starting at bit `sh` of its first word
template <int B>
__device__ __forceinline__ uint64_t code_window(const uint32_t (&r)[CodeWin<B>::WORDS], int sh) {
  if constexpr (CodeWin<B>::WORDS == 1) {
    return (uint64_t)(r[0] >> sh);
  } else if constexpr (CodeWin<B>::WORDS == 2) {
    const uint32_t a = __funnelshift_r(r[0], r[1], sh);
    return ((uint64_t)(r[1] >> sh) << 32) | a;
  } else {
    const uint32_t a = __funnelshift_r(r[0], r[1], sh);
    const uint32_t b = __funnelshift_r(r[1], r[2], sh);
    return ((uint64_t)b << 32) | a;
  }
}

template <int B>
__device__ __forceinline__ uint32_t code_at(uint64_t y, int k) {
  return (uint32_t)(y >> (k * B)) & ((1u << B) - 1u);
}

// Shared-memory reads are plain C++ loads through pointers into the kernel's
// extern __shared__ buffer (the compiler emits LDS and, unlike non-volatile
// asm, keeps them ordered after the barriers that publish the data).
__device__ __forceinline__ float2 lds_f2(const uint8_t* sm, uint32_t off) {
  return *reinterpret_cast<const float2*>(sm + off);
}
__device__ __forceinline__ void lds_pair2(const uint8_t* sm, uint32_t off, ptx::f2& a,
                                          ptx::f2& b) {
  const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(sm + off);
  a.v = v.x;
  b.v = v.y;
}

template <int GP>
__device__ __forceinline__ void load_q(const uint8_t* sm, uint32_t qrow, ptx::f2 (&qv)[GP]) {
#pragma unroll
  for (int g = 0; g + 1 < GP; g += 2) lds_pair2(sm, qrow + 8 * g, qv[g], qv[g + 1]);
  if constexpr (GP % 2)
    qv[GP - 1].v = *reinterpret_cast<const unsigned long long*>(sm + qrow + 8 * (GP - 1));
}

__device__ __forceinline__ uint32_t read_bits_g(const uint32_t* __restrict__ words, uint64_t bit,
                                                int nbits) {
  const uint64_t w = bit >> 5;
  const int sh = (int)(bit & 31);
  const uint32_t lo = __ldg(words + w);
  const uint32_t hi = (sh + nbits > 32) ? __ldg(words + w + 1) : 0u;
  const uint32_t v = __funnelshift_r(lo, hi, sh);
  return nbits >= 32 ? v : (v & ((1u << nbits) - 1u));
}

template <int B>
__device__ __forceinline__ void load_words(uint32_t (&w)[CodeWin<B>::WORDS],
                                           const uint32_t* __restrict__ row) {
#pragma unroll
  for (int i = 0; i < CodeWin<B>::WORDS; ++i) w[i] = __ldg(row + i);
}

// One code row of the recurrence for the lane's 4 items (prod kept as two
// packed pairs: items {0,1} and {2,3}).
template <int B, int GP, bool LUT, bool REPL>
__device__ __forceinline__ void chain_row(const uint8_t* sm, const uint32_t (&w)[CodeWin<B>::WORDS],
                                          int sh, uint32_t qrow, uint32_t lut_s, float pstep,
                                          ptx::f2 (&prod)[2], ptx::f2 (&acc)[4][GP]) {
  ptx::f2 qv[GP];
  load_q<GP>(sm, qrow, qv);
  if constexpr (LUT && lut_group(B) > 1) {
    // two pair lookups: items {0,1} and {2,3}; lut_s is this lane's copy base
    constexpr uint32_t STRIDE = REPL ? 128u : 16u;
    const uint32_t x = (uint32_t)code_window<B>(w, sh);
    constexpr uint32_t M2 = (1u << (2 * B)) - 1u;
    uint32_t i0, i1;
    if constexpr (B == 4) {
      const uint32_t b0 = (uint32_t)(sh >> 3);
      i0 = __byte_perm(w[0], 0u, 0x4440u | b0);
      i1 = __byte_perm(w[0], 0u, 0x4440u | (b0 + 1));
    } else {
      i0 = x & M2;
      i1 = (x >> (2 * B)) & M2;
    }
    ptx::f2 cp[2], sp[2];
    lds_pair2(sm, lut_s + i0 * STRIDE, cp[0], sp[0]);
    lds_pair2(sm, lut_s + i1 * STRIDE, cp[1], sp[1]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const ptx::f2 f = ptx::f2_mul(prod[h], cp[h]);
      ptx::f2_mul_acc(prod[h], sp[h]);
#pragma unroll
      for (int g = 0; g < GP; ++g) {
        ptx::f2_fma_s_acc(ptx::f2_lo(f), qv[g], acc[2 * h][g]);
        ptx::f2_fma_s_acc(ptx::f2_hi(f), qv[g], acc[2 * h + 1][g]);
      }
    }
  } else {
    const uint64_t y = code_window<B>(w, sh);
    float pr[4] = {ptx::f2_lo(prod[0]), ptx::f2_hi(prod[0]), ptx::f2_lo(prod[1]),
                   ptx::f2_hi(prod[1])};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t c = code_at<B>(y, k);
      float cs, sn;
      if constexpr (LUT) {
        const float2 t = lds_f2(sm, lut_s + c * (REPL ? 128u : 8u));
        cs = t.x;
        sn = t.y;
      } else {
        sincospif((float)c * pstep, &sn, &cs);
      }
      const float f = pr[k] * cs;
#pragma unroll
      for (int g = 0; g < GP; ++g) ptx::f2_fma_s_acc(f, qv[g], acc[k][g]);
      pr[k] *= sn;
    }
    prod[0] = ptx::f2_make(pr[0], pr[1]);
    prod[1] = ptx::f2_make(pr[2], pr[3]);
  }
}

// Logits (base 2) of items sub*TI + 4*lane + k, k < 4, for G heads.
//   codes : page code block (coordinate-major rows of P*B bits, radius row last)
//   sm    : the kernel's shared buffer; qs_s / lut_s: byte offsets of the q pairs
//           [d][GP] (float2) and of this tier's table
// Code words are requested LA rows ahead of use through a ring of register
// buffers (no moves of in-flight loads); the look-ahead may read a few rows
// past the block, which the code pool's tail slack absorbs.
template <int B, int GP, bool LUT, bool REPL, int PT>
__device__ __forceinline__ void ada_logit_tile(const uint8_t* __restrict__ codes, int d, int P_rt,
                                               int TI, const sphkv_page_t& pg, int sub, int lane,
                                               const uint8_t* sm, uint32_t qs_s, uint32_t lut_s,
                                               float lg[4][2 * GP]) {
  constexpr int NW = CodeWin<B>::WORDS;
  const int P = PT ? PT : P_rt;  // PT != 0: page size known at compile time (row stride immediates)
  const int item0 = sub * TI + 4 * lane;
  const uint32_t* base = reinterpret_cast<const uint32_t*>(codes + pg.code_off);
  const int row_words = P * B / 32;
  const uint32_t obit = (uint32_t)item0 * B;
  const uint32_t* lane_row = base + (obit >> 5);
  const int sh = (int)(obit & 31);
  const uint32_t qstride = GP * 8;
  const float pstep = (float)(1.0 / (double)((1u << B) - 1u));

  ptx::f2 prod[2] = {ptx::f2_make(1.f, 1.f), ptx::f2_make(1.f, 1.f)};
  ptx::f2 acc[4][GP];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int g = 0; g < GP; ++g) acc[k][g] = ptx::f2_make(0.f, 0.f);

#if SPHKV_RING
  // ring of LA+1 word buffers: row j+LA is requested while row j is consumed;
  // the unroll by LA+1 makes every buffer index a compile-time constant.
#ifndef SPHKV_LA
#define SPHKV_LA 6
#endif
  constexpr int LA = SPHKV_LA;
  uint32_t wb[LA + 1][NW];
#pragma unroll
  for (int u = 0; u < LA; ++u) load_words<B>(wb[u], lane_row + u * row_words);
  const int nrow = d - 2;
  const uint32_t* next = lane_row + LA * row_words;
  uint32_t qrow = qs_s;
  int j = 0;
  for (; j + (LA + 1) <= nrow; j += LA + 1) {
#pragma unroll
    for (int u = 0; u <= LA; ++u) {
      load_words<B>(wb[(u + LA) % (LA + 1)], next + u * row_words);  // may run past row d-1: pool has slack
      chain_row<B, GP, LUT, REPL>(sm, wb[u], sh, qrow + u * qstride, lut_s, pstep, prod, acc);
    }
    next += (LA + 1) * row_words;
    qrow += (LA + 1) * qstride;
  }
  // tail: wb[u] holds row j+u for u < LA; r = nrow - j < LA+1 polar rows remain
  const int r = nrow - j;
  if (r == LA) load_words<B>(wb[LA], next);
#pragma unroll
  for (int u = 0; u < LA; ++u)
    if (u < r) chain_row<B, GP, LUT, REPL>(sm, wb[u], sh, qrow + u * qstride, lut_s, pstep, prod, acc);
  uint32_t w0[NW];
#pragma unroll
  for (int u = 0; u <= LA; ++u) {
    if (u == r) {
#pragma unroll
      for (int i = 0; i < NW; ++i) w0[i] = wb[u][i];
    }
  }
#else
  uint32_t w0[NW], w1[NW], w2[NW];
  load_words<B>(w0, lane_row);
  load_words<B>(w1, lane_row + row_words);
  const int nrow = d - 2;
  const uint32_t* next = lane_row + 2 * row_words;
  uint32_t qrow = qs_s;
  int j = 0;
  for (; j + 3 <= nrow; j += 3) {
    load_words<B>(w2, next);
    chain_row<B, GP, LUT, REPL>(sm, w0, sh, qrow, lut_s, pstep, prod, acc);
    load_words<B>(w0, next + row_words);
    chain_row<B, GP, LUT, REPL>(sm, w1, sh, qrow + qstride, lut_s, pstep, prod, acc);
    load_words<B>(w1, next + 2 * row_words);
    chain_row<B, GP, LUT, REPL>(sm, w2, sh, qrow + 2 * qstride, lut_s, pstep, prod, acc);
    next += 3 * row_words;
    qrow += 3 * qstride;
  }
  const int rem = nrow - j;
  if (rem >= 1) {
    chain_row<B, GP, LUT, REPL>(sm, w0, sh, qrow, lut_s, pstep, prod, acc);
    qrow += qstride;
    if (rem == 2) {
      load_words<B>(w2, next);
      chain_row<B, GP, LUT, REPL>(sm, w1, sh, qrow, lut_s, pstep, prod, acc);
#pragma unroll
      for (int i = 0; i < NW; ++i) w0[i] = w2[i];
    } else {
#pragma unroll
      for (int i = 0; i < NW; ++i) w0[i] = w1[i];
    }
  }
#endif
  // circular last angle (row d-2, now in w0): step 2*pi/2^B -> sincospi(code * 2^(1-B))
  const float pf[4] = {ptx::f2_lo(prod[0]), ptx::f2_hi(prod[0]), ptx::f2_lo(prod[1]),
                       ptx::f2_hi(prod[1])};
  {
    const uint64_t y = code_window<B>(w0, sh);
    ptx::f2 qa[GP], qb[GP];
    load_q<GP>(sm, qs_s + (d - 2) * qstride, qa);
    load_q<GP>(sm, qs_s + (d - 1) * qstride, qb);
    const float cstep = ldexpf(1.0f, 1 - B);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float sn, cs;
      sincospif((float)code_at<B>(y, k) * cstep, &sn, &cs);
      const float f0 = pf[k] * cs, f1 = pf[k] * sn;
#pragma unroll
      for (int g = 0; g < GP; ++g) {
        acc[k][g] = ptx::f2_fma_s(f0, qa[g], acc[k][g]);
        acc[k][g] = ptx::f2_fma_s(f1, qb[g], acc[k][g]);
      }
    }
  }
  // decoded radii r~ = code * (scale / levels)  (row d-1 holds the radius stream)
  const uint64_t rbit0 = (uint64_t)(d - 1) * P * B;
  const int rb = pg.rbits;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t rc = read_bits_g(base, rbit0 + (uint64_t)(item0 + k) * rb, rb);
    const float rr = (float)rc * pg.rscale;
#pragma unroll
    for (int g = 0; g < GP; ++g) {
      lg[k][2 * g] = rr * ptx::f2_lo(acc[k][g]);
      lg[k][2 * g + 1] = rr * ptx::f2_hi(acc[k][g]);
    }
  }
}

template <int GP>
__device__ void ada_logit_dispatch(int B, const uint8_t* codes, int d, int P, int TI,
                                   const sphkv_page_t& pg, int sub, int lane, const uint8_t* sm,
                                   uint32_t qs_s, int lut_enc, float lg[4][2 * GP]) {
  // lut_enc: (byte offset << 1) | replicated, or -1 (no table: sincospi)
  const bool has = lut_enc >= 0;
  const bool repl = has && (lut_enc & 1);
  const uint32_t base = has ? (uint32_t)(lut_enc >> 1) : 0u;
  switch (B) {
#define SPHKV_TILE(b, L, R, PP)                                                              \
  ada_logit_tile<b, GP, L, R, PP>(codes, d, P, TI, pg, sub, lane, sm, qs_s,                 \
                                  base + (R ? (uint32_t)(lane % lut_rep(b)) * lut_entry_bytes(b) \
                                            : 0u), lg)
#define SPHKV_CASE(b)                                                                        \
  case b:                                                                                    \
    if (b <= LUT_MAX_BITS && has) {                                                          \
      if (repl) {                                                                            \
        if (P == 256) SPHKV_TILE(b, (b <= LUT_MAX_BITS), true, 256);                         \
        else SPHKV_TILE(b, (b <= LUT_MAX_BITS), true, 0);                                    \
      } else {                                                                               \
        if (P == 256) SPHKV_TILE(b, (b <= LUT_MAX_BITS), false, 256);                        \
        else SPHKV_TILE(b, (b <= LUT_MAX_BITS), false, 0);                                   \
      }                                                                                      \
    } else {                                                                                 \
      SPHKV_TILE(b, false, false, 0);                                                        \
    }                                                                                        \
    break;
    SPHKV_CASE(1) SPHKV_CASE(2) SPHKV_CASE(3) SPHKV_CASE(4) SPHKV_CASE(5) SPHKV_CASE(6)
    SPHKV_CASE(7) SPHKV_CASE(8) SPHKV_CASE(9) SPHKV_CASE(10) SPHKV_CASE(11) SPHKV_CASE(12)
    SPHKV_CASE(13) SPHKV_CASE(14) SPHKV_CASE(15) SPHKV_CASE(16)
#undef SPHKV_CASE
#undef SPHKV_TILE
    default: break;
  }
}

}  // namespace sphkv
