// ADA logit tile: logits of a 128-item tile (lane l owns items l, l+32, l+64,
// l+96), straight from the angle/radius codes (decode.py:123-192:
// l = (r_q/sqrt d) r~ (feat . qfeat)).
//
// The feature row of an item is the recurrence f_j = (prod_{l<j} sin a_l) cos a_j
// (codec.py:459-477); the kernel never forms it in memory: per code row it
// looks (cos, sin) up in a shared-memory table, updates the running sine
// product and accumulates f_j * q_j for all G query heads with packed FFMA2
// (q is pre-scaled by log2(e)/sqrt(d), so logits come out in base-2 units).
#pragma once
#include "common.cuh"
#include "ptx.cuh"

#include <utility>

namespace sphkv {

#ifdef SPHKV_MUFU12  // 12-bit tier on MUFU sin/cos: no table for it
constexpr int LUT_MAX_BITS = 11;
#else
constexpr int LUT_MAX_BITS = 12;
#endif
#ifndef SPHKV_LUT_KB
#define SPHKV_LUT_KB 124
#endif
constexpr int LUT_BUDGET_BYTES = SPHKV_LUT_KB * 1024;

// Polar (cos, sin) tables in shared memory, one per tier with B <= 12.
//  * B <= 2: "quad-row" tables indexed by the codes of four consecutive rows
//    (j..j+3) of one item (4B contiguous bits of its code string): part A,
//    16-byte entries (c0, s0 c1, s0 s1 c2, s0 s1 s2 c3), replicated 8x, and
//    part B, 4-byte entries s0 s1 s2 s3 (the running sine product's factor),
//    replicated 16x; products taken in fp64 and rounded once.  One LDS.128 +
//    one LDS.32 advance the feature recurrence by four rows.  Looking part A
//    up with the top two codes zero gives (c0, s0 c1, s0 s1, 0) -- a row pair.
//  * 3 <= B <= 4: "row-pair" tables: entry (c_j, s_j c_j+1, s_j s_j+1, 0),
//    one LDS.128 per two rows.
//  * 5 <= B <= 12: single-code tables, entry (cos, sin) = one LDS.64.
// Random gathers from a small table bank-conflict heavily, so a table may be
// stored REP times interleaved: entry e of copy r lives at (e * REP + r) *
// entry_bytes and lane L reads copy L % REP.  REP = 8 for 16-byte entries (8
// lanes per LDS.128 phase), 16 for 8-byte entries (16 lanes per LDS.64
// phase), so every phase hits distinct banks and the entry stride is 128
// bytes either way.  Quad tables are always replicated (the 2-bit tier holds
// most items); the others as the budget allows, narrow tiers first.
__host__ __device__ constexpr int lut_group(int B) { return B <= 2 ? 4 : (B <= 4 ? 2 : 1); }
__host__ __device__ constexpr int lut_entry_bytes(int B) { return lut_group(B) == 1 ? 8 : 16; }
__host__ __device__ constexpr int lut_rep(int B) { return lut_group(B) == 1 ? 16 : 8; }
__host__ __device__ constexpr int lut_quad_b_rep() { return 16; }
__host__ __device__ constexpr int lut_bytes(int B, int copies) {
  return lut_group(B) == 4
             ? (1 << (4 * B)) * (16 * 8 + 4 * lut_quad_b_rep())  // parts A + B, replicated
             : (1 << (lut_group(B) * B)) * lut_entry_bytes(B) * copies;
}
// table mode (low 2 bits of the encoded descriptor): 0 = one copy, 1 = full
// replication (lut_rep), 2 = two interleaved copies (single-code tables)
__host__ __device__ constexpr int lut_copies(int B, int mode) {
  return mode == 1 ? (lut_group(B) == 4 ? 8 : lut_rep(B)) : (mode == 2 ? 2 : 1);
}
__host__ __device__ constexpr int ilog2c(int x) { return x <= 1 ? 0 : 1 + ilog2c(x / 2); }

// Encoded per-tier table descriptor: (byte offset << 2) | mode, or -1.
// With item counts (`items`, per tier index; all zero = unknown) tiers
// without items get no table and replication goes to the most used tiers
// first; without them the fixed priority below applies.  Quad tables are
// always replicated; single-code tiers of 8..12 bits fall back to two copies
// when full replication (16 copies) does not fit.
// hb != 0: the 2-bit tier decodes from per-query h-byte tables (hb_tile.cuh)
// and gets no shared-memory table here.  budget: LUT bytes (0 = default).
__host__ __device__ inline int lut_layout_tiers(const sphkv_tier_t* tiers, int n_tiers,
                                                int off[SPHKV_MAX_TIERS],
                                                const int64_t* items = nullptr, int hb = 0,
                                                int budget = 0) {
  const int LUT_BUDGET = budget > 0 ? budget : LUT_BUDGET_BYTES;
  int mode[SPHKV_MAX_TIERS];
  bool known = false;
  if (items != nullptr)
    for (int t = 1; t < n_tiers; ++t) known = known || items[t] > 0;
  for (int t = 0; t < SPHKV_MAX_TIERS; ++t) {
    off[t] = -1;
    mode[t] = 0;
  }
  int total = 0;
  for (int t = 1; t < n_tiers; ++t) {
    const int b = tiers[t].angle_bits;
    const bool quad = lut_group(b) == 4;
    if (known && items[t] == 0) continue;
    if (hb && b == 2) continue;
    if (b <= LUT_MAX_BITS && total + lut_bytes(b, quad ? 8 : 1) <= LUT_BUDGET) {
      total += lut_bytes(b, quad ? 8 : 1);
      off[t] = 0;  // has a table; placed below
      mode[t] = quad ? 1 : 0;
    }
  }
  auto upgrade = [&](int t) {
    const int b = tiers[t].angle_bits;
    if (off[t] != 0 || mode[t] != 0) return;
    const int extra = lut_bytes(b, lut_copies(b, 1)) - lut_bytes(b, 1);
    if (total + extra <= LUT_BUDGET) {
      mode[t] = 1;
      total += extra;
    } else if (b >= 8) {
      const int extra2 = lut_bytes(b, 2) - lut_bytes(b, 1);
      if (total + extra2 <= LUT_BUDGET) {
        mode[t] = 2;
        total += extra2;
      }
    }
  };
  if (known) {  // most items first
    bool done[SPHKV_MAX_TIERS] = {};
    for (int k = 1; k < n_tiers; ++k) {
      int best = -1;
      for (int t = 1; t < n_tiers; ++t)
        if (!done[t] && off[t] == 0 && (best < 0 || items[t] > items[best])) best = t;
      if (best < 0) break;
      done[best] = true;
      upgrade(best);
    }
  } else {  // fixed priority: single-code 5..7 bits, row-pair 3..4, wide 8..12
    const int lo[3] = {5, 3, 8}, hi[3] = {7, 4, LUT_MAX_BITS};
    for (int r = 0; r < 3; ++r)
      for (int b = lo[r]; b <= hi[r]; ++b)
        for (int t = 1; t < n_tiers; ++t)
          if (tiers[t].angle_bits == b) upgrade(t);
  }
  int used = 0;  // every table size is a multiple of 16 bytes
  for (int t = 1; t < n_tiers; ++t)
    if (off[t] == 0) {
      off[t] = (used << 2) | mode[t];
      used += lut_bytes(tiers[t].angle_bits, lut_copies(tiers[t].angle_bits, mode[t]));
    }
  return used;
}

// Fill one (entry, copy) of a table: tier bits B, entry e, copy r.  Quad
// tables: copies r < 8 are part A, 8 <= r < 24 part B (copy r - 8).
__device__ inline void lut_write_entry(uint8_t* dst, int B, int copies, int e, int r) {
  const double step = kPi / (double)((1u << B) - 1u);
  if (lut_group(B) == 4) {
    const uint32_t M = (1u << B) - 1u;
    double sn[4], cs[4];
    for (int k = 0; k < 4; ++k) sincos((double)((e >> (k * B)) & M) * step, &sn[k], &cs[k]);
    const int nA = (1 << (4 * B)) * 128;
    if (r < 8) {
      float* out = reinterpret_cast<float*>(dst + ((size_t)e * 8 + r) * 16);
      out[0] = (float)cs[0];
      out[1] = (float)(sn[0] * cs[1]);
      out[2] = (float)(sn[0] * sn[1] * cs[2]);
      out[3] = (float)(sn[0] * sn[1] * sn[2] * cs[3]);
    } else {
      float* out = reinterpret_cast<float*>(dst + nA + ((size_t)e * lut_quad_b_rep() + (r - 8)) * 4);
      out[0] = (float)(sn[0] * sn[1] * sn[2] * sn[3]);
    }
    return;
  }
  const int R = copies;
  float* out = reinterpret_cast<float*>(dst + ((size_t)e * R + r) * lut_entry_bytes(B));
  if (lut_group(B) == 1) {
    double sn, cs;
    sincos((double)e * step, &sn, &cs);
    out[0] = (float)cs;
    out[1] = (float)sn;
  } else {
    const uint32_t M = (1u << B) - 1u;
    double sa, ca, sb, cb;
    sincos((double)(e & M) * step, &sa, &ca);          // row j   (low B bits)
    sincos((double)((e >> B) & M) * step, &sb, &cb);   // row j+1 (high B bits)
    out[0] = (float)ca;
    out[1] = (float)(sa * cb);
    out[2] = (float)(sa * sb);
    out[3] = 0.f;
  }
}

// all (entry, copy) pairs of every tier's table, strided over `nthreads`
__device__ inline void lut_fill(uint8_t* lut, const sphkv_tier_t* tiers, int n_tiers,
                                const int* enc, int tid, int nthreads) {
  for (int t = 1; t < n_tiers; ++t) {
    if (enc[t] < 0) continue;
    const int B = tiers[t].angle_bits;
    const int copies = lut_copies(B, enc[t] & 3);
    const int R = lut_group(B) == 4 ? 8 + lut_quad_b_rep() : copies;
    const int n = (1 << (lut_group(B) * B)) * R;
    for (int i = tid; i < n; i += nthreads)
      lut_write_entry(lut + (enc[t] >> 2), B, copies, i / R, i % R);
  }
}

template <int GP>
__device__ __forceinline__ void load_q(const uint8_t* sm, uint32_t qrow, ptx::f2 (&qv)[GP]) {
#pragma unroll
  for (int g = 0; g + 1 < GP; g += 2) {
    const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(sm + qrow + 8 * g);
    qv[g].v = v.x;
    qv[g + 1].v = v.y;
  }
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

// compile-time loop: f(std::integral_constant<int, i>) for i < N
template <typename F, int... I>
__device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, I...>) {
  (f(std::integral_constant<int, I>{}), ...);
}
template <int N, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  static_for_impl(f, std::make_integer_sequence<int, N>{});
}

// N-bit field at compile-time bit offset S of a register-resident string
template <int N, int S, int W>
__device__ __forceinline__ uint32_t field(const uint32_t (&w)[W]) {
  constexpr int wi = S / 32, sh = S % 32;
  constexpr uint32_t M = (N >= 32) ? 0xffffffffu : ((1u << N) - 1u);
  if constexpr (sh + N <= 32) {
    return (w[wi] >> sh) & M;
  } else {
    return __funnelshift_r(w[wi], w[wi + 1], sh) & M;
  }
}
// the same field pre-scaled by 2^L (a table byte offset): one shift + one
// LOP3 that also ORs in the lane's replica offset `orv` (< 2^L)
template <int N, int S, int L, int W>
__device__ __forceinline__ uint32_t field_addr(const uint32_t (&w)[W], uint32_t orv) {
  constexpr int wi = S / 32, sh = S % 32;
  constexpr uint32_t M = ((1u << N) - 1u) << L;
  uint32_t x;
  if constexpr (sh + N > 32) {
    x = __funnelshift_r(w[wi], w[wi + 1], sh) << L;
  } else if constexpr (sh >= L) {
    x = w[wi] >> (sh - L);
  } else {
    x = w[wi] << (L - sh);
  }
  return (x & M) | orv;
}

// code string of one item: W words from the WI layout (quad loads)
template <int W>
__device__ __forceinline__ void load_item(uint32_t (&w)[W], const uint4* __restrict__ blk4,
                                          int granule, int lane) {
#pragma unroll
  for (int q = 0; q < W / 4; ++q) {
    const uint4 v = __ldg(blk4 + ((size_t)granule * (W / 4) + q) * 32 + lane);
    w[4 * q] = v.x;
    w[4 * q + 1] = v.y;
    w[4 * q + 2] = v.z;
    w[4 * q + 3] = v.w;
  }
}

// Items per lane of a decode tile (a tile is TTI = 32 * TK items: lane l owns
// items l + 32 k, k < TK).
#ifndef SPHKV_K
#define SPHKV_K 4
#endif
constexpr int TK = SPHKV_K;
constexpr int TTI = 32 * TK;

// Rows per "period": the smallest row count whose codes fill whole 32-bit
// words, so every code's bit offset inside a period is a compile-time
// constant.  WP = words per period.
template <int B>
struct Period {
  static constexpr int R = (B == 1) ? 32 : (B == 2) ? 16 : (B == 4) ? 8 : (B == 8) ? 4
                         : (B == 16) ? 2 : (B % 4 == 0) ? 8 : (B % 2 == 0) ? 16 : 32;
  static constexpr int WP = R * B / 32;
};

// word w (runtime) of tile item k (lane + 32 k): one LDG.32 (L1-resident:
// the tile's granules are one contiguous block)
template <int W>
__device__ __forceinline__ uint32_t item_word(const uint32_t* __restrict__ blk, int sub, int k,
                                              int lane, int w) {
  return __ldg(blk + wi_word(sub * TTI + 32 * k + lane, w, W));
}

// One period (R rows starting at row r0 = per * R) of the feature recurrence
// for the lane's 4 items, codes in cw[k][0..WP).  MODE 2: row-pair table,
// 1: single-code table, 0: sincospif.
template <int B, int GP, int MODE, int STR, int RR = Period<B>::R>
__device__ __forceinline__ void period_rows(const uint32_t (&cw)[TK][Period<B>::WP],
                                            const uint8_t* sm, uint32_t qrow0, uint32_t tb,
                                            uint32_t orv, float (&prod)[TK],
                                            ptx::f2 (&acc)[TK][GP], uint32_t qb_off = 0) {
  constexpr int R = Period<B>::R, WP = Period<B>::WP;
  constexpr uint32_t QR = q_row_bytes(GP);
  if constexpr (MODE == 4) {
    // quad-row table: part A at tb, part B at tb + qb_off (4-byte entries, 16
    // copies, 64-byte stride); a trailing row pair uses part A alone
    static_assert(RR % 2 == 0, "row pairs");
    constexpr int NQ = RR / 4;
    const uint32_t orv_b = (uint32_t)(threadIdx.x & 15) * 4u;
    static_for<NQ>([&](auto pc) {
      constexpr int p = decltype(pc)::value;
      ptx::f2 q0[GP], q1[GP], q2[GP], q3[GP];
      load_q<GP>(sm, qrow0 + (4 * p) * QR, q0);
      load_q<GP>(sm, qrow0 + (4 * p + 1) * QR, q1);
      load_q<GP>(sm, qrow0 + (4 * p + 2) * QR, q2);
      load_q<GP>(sm, qrow0 + (4 * p + 3) * QR, q3);
#pragma unroll
      for (int k = 0; k < TK; ++k) {
        const uint32_t aa = field_addr<4 * B, 4 * p * B, 7, WP>(cw[k], orv);
        const uint32_t ab = field_addr<4 * B, 4 * p * B, 6, WP>(cw[k], orv_b);
        const float4 e = *reinterpret_cast<const float4*>(sm + tb + aa);
        const float sp = *reinterpret_cast<const float*>(sm + tb + qb_off + ab);
        const ptx::f2 pp = ptx::f2_make(prod[k], prod[k]);
        const ptx::f2 f01 = ptx::f2_mul(pp, ptx::f2_make(e.x, e.y));
        const ptx::f2 f23 = ptx::f2_mul(pp, ptx::f2_make(e.z, e.w));
        prod[k] *= sp;
#pragma unroll
        for (int g = 0; g < GP; ++g) {
          ptx::f2_fma_s_acc(ptx::f2_lo(f01), q0[g], acc[k][g]);
          ptx::f2_fma_s_acc(ptx::f2_hi(f01), q1[g], acc[k][g]);
          ptx::f2_fma_s_acc(ptx::f2_lo(f23), q2[g], acc[k][g]);
          ptx::f2_fma_s_acc(ptx::f2_hi(f23), q3[g], acc[k][g]);
        }
      }
    });
    if constexpr (RR % 4 == 2) {  // trailing pair: top two codes of the index zero
      constexpr int j0 = 4 * NQ;
      ptx::f2 qa[GP], qb[GP];
      load_q<GP>(sm, qrow0 + j0 * QR, qa);
      load_q<GP>(sm, qrow0 + (j0 + 1) * QR, qb);
#pragma unroll
      for (int k = 0; k < TK; ++k) {
        const uint32_t a = field_addr<2 * B, j0 * B, 7, WP>(cw[k], orv);
        const float4 e = *reinterpret_cast<const float4*>(sm + tb + a);
        const ptx::f2 f = ptx::f2_mul(ptx::f2_make(prod[k], prod[k]), ptx::f2_make(e.x, e.y));
        prod[k] *= e.z;
#pragma unroll
        for (int g = 0; g < GP; ++g) {
          ptx::f2_fma_s_acc(ptx::f2_lo(f), qa[g], acc[k][g]);
          ptx::f2_fma_s_acc(ptx::f2_hi(f), qb[g], acc[k][g]);
        }
      }
    }
  } else if constexpr (MODE == 2) {
    static_assert(RR % 2 == 0, "row pairs");
    static_for<RR / 2>([&](auto pc) {
      constexpr int p = decltype(pc)::value;
      ptx::f2 qa[GP], qb[GP];
      load_q<GP>(sm, qrow0 + (2 * p) * QR, qa);
      load_q<GP>(sm, qrow0 + (2 * p + 1) * QR, qb);
#pragma unroll
      for (int k = 0; k < TK; ++k) {
        const uint32_t a = field_addr<2 * B, 2 * p * B, STR, WP>(cw[k], orv);
        const float4 e = *reinterpret_cast<const float4*>(sm + tb + a);
        const ptx::f2 f = ptx::f2_mul(ptx::f2_make(prod[k], prod[k]), ptx::f2_make(e.x, e.y));
        prod[k] *= e.z;
#pragma unroll
        for (int g = 0; g < GP; ++g) {
          ptx::f2_fma_s_acc(ptx::f2_lo(f), qa[g], acc[k][g]);
          ptx::f2_fma_s_acc(ptx::f2_hi(f), qb[g], acc[k][g]);
        }
      }
    });
  } else {
    const float pstep = (float)(1.0 / (double)((1u << B) - 1u));
    const float pang = (float)(kPi / (double)((1u << B) - 1u));
    static_for<RR>([&](auto jc) {
      constexpr int j = decltype(jc)::value;
      ptx::f2 qa[GP];
      load_q<GP>(sm, qrow0 + j * QR, qa);
#pragma unroll
      for (int k = 0; k < TK; ++k) {
        float cs, sn;
        if constexpr (MODE == 1) {
          const uint32_t a = field_addr<B, j * B, STR, WP>(cw[k], orv);
          const float2 t = *reinterpret_cast<const float2*>(sm + tb + a);
          cs = t.x;
          sn = t.y;
        } else if constexpr (MODE == 3) {
          // MUFU sin/cos (no shared-memory traffic): code -> float exactly via
          // the 2^23 magic, angle = code * step in fp32 (abs err ~2e-7)
          const float x = __uint_as_float(0x4B000000u | field<B, j * B, WP>(cw[k])) - 8388608.f;
          __sincosf(x * pang, &sn, &cs);
        } else {
          sincospif((float)field<B, j * B, WP>(cw[k]) * pstep, &sn, &cs);
        }
        const float f = prod[k] * cs;
        prod[k] *= sn;
#pragma unroll
        for (int g = 0; g < GP; ++g) ptx::f2_fma_s_acc(f, qa[g], acc[k][g]);
      }
    });
  }
}

// Specialised tile (B, D known).  A runtime loop over whole periods (codes
// of the next period requested while the current one is computed), then the
// remaining polar rows and the circular row with runtime extraction.
template <int B, int D, int GP, int MODE, int REP>
__device__ __noinline__ void ada_tile_wi(const uint8_t* __restrict__ blkb, int sub, int lane,
                                         const uint8_t* sm, uint32_t qs, uint32_t tb,
                                         uint32_t rbit0, int rb, float rscale,
                                         float lg[TK][2 * GP]) {
  constexpr int W = item_words(D, B);
  constexpr int R = Period<B>::R, WP = Period<B>::WP;
  constexpr int NP = D - 2;      // polar rows
  constexpr int NFULL = NP / R;  // whole periods of polar rows
  constexpr int EB = (MODE == 2 || MODE == 4) ? 16 : 8;
  constexpr int STR = ilog2c(REP * EB);  // log2 of the entry stride (REP copies)
  const uint32_t qb_off = (MODE == 4) ? (uint32_t)((1 << (4 * B)) * 128) : 0u;
  constexpr uint32_t QR = q_row_bytes(GP);
  const uint32_t orv = (uint32_t)(lane % REP) * EB;
  const uint32_t* blk = reinterpret_cast<const uint32_t*>(blkb);
  float prod[TK];
  ptx::f2 acc[TK][GP];
#pragma unroll
  for (int k = 0; k < TK; ++k) {
    prod[k] = 1.f;
#pragma unroll
    for (int g = 0; g < GP; ++g) acc[k][g] = ptx::f2_make(0.f, 0.f);
  }
  uint32_t cw[TK][WP];
#pragma unroll
  for (int k = 0; k < TK; ++k)
#pragma unroll
    for (int i = 0; i < WP; ++i) cw[k][i] = item_word<W>(blk, sub, k, lane, i);
#pragma unroll 1
  for (int per = 0; per < NFULL; ++per) {
    uint32_t nw[TK][WP];
    const int wn = (per + 1) * WP;  // next period's first word (< W: a tail follows)
#pragma unroll
    for (int k = 0; k < TK; ++k)
#pragma unroll
      for (int i = 0; i < WP; ++i) nw[k][i] = item_word<W>(blk, sub, k, lane, min(wn + i, W - 1));
    period_rows<B, GP, MODE, STR>(cw, sm, qs + per * R * QR, tb, orv, prod, acc, qb_off);
#pragma unroll
    for (int k = 0; k < TK; ++k)
#pragma unroll
      for (int i = 0; i < WP; ++i) cw[k][i] = nw[k][i];
  }
  // last partial period (compile-time row count), then the circular row
  // NP = D-2, whose code lies in the same period window
  constexpr int RR = NP - NFULL * R;
  if constexpr (RR > 0)
    period_rows<B, GP, MODE, STR, RR>(cw, sm, qs + NFULL * R * QR, tb, orv, prod, acc, qb_off);
  {
    ptx::f2 qa[GP], qb[GP];
    load_q<GP>(sm, qs + NP * QR, qa);
    load_q<GP>(sm, qs + (NP + 1) * QR, qb);
#pragma unroll
    for (int k = 0; k < TK; ++k) {
      float sn, cs;
      sincospif((float)field<B, RR * B, WP>(cw[k]) * (1.0f / (float)(1u << (B - 1))), &sn, &cs);
      const float f0 = prod[k] * cs, f1 = prod[k] * sn;
#pragma unroll
      for (int g = 0; g < GP; ++g) {
        ptx::f2_fma_s_acc(f0, qa[g], acc[k][g]);
        ptx::f2_fma_s_acc(f1, qb[g], acc[k][g]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < TK; ++k) {
    const uint32_t rc = read_bits_g(blk, rbit0 + (uint64_t)(sub * TTI + 32 * k + lane) * rb, rb);
    const float rr = (float)rc * rscale;
#pragma unroll
    for (int g = 0; g < GP; ++g) {
      lg[k][2 * g] = rr * ptx::f2_lo(acc[k][g]);
      lg[k][2 * g + 1] = rr * ptx::f2_hi(acc[k][g]);
    }
  }
}

// Generic tile (any B <= 16, any d): runtime loops, words fetched per row
// from global memory; same math (row-pair table rows in pairs, single table,
// or sincospif).
template <int GP>
__device__ __noinline__ void ada_tile_generic(const uint8_t* __restrict__ blk, int B, int d,
                                              int P, int sub, int lane, const uint8_t* sm, uint32_t qs,
                                              int lut_enc, uint32_t rbit0, int rb, float rscale,
                                              float lg[TK][2 * GP]) {
  const int W = item_words(d, B);
  const uint32_t* words = reinterpret_cast<const uint32_t*>(blk);
  const bool has = lut_enc >= 0;
  const int copies = has ? lut_copies(B, lut_enc & 3) : 1;
  const int grp = lut_group(B), eb = lut_entry_bytes(B);
  const uint32_t tbase = has ? (uint32_t)(lut_enc >> 2) + (lane % copies) * eb : 0;
  const uint32_t stride = (uint32_t)(copies * eb);
  const uint32_t QR = q_row_bytes(GP);
  const float pstep = (float)(1.0 / (double)((1u << B) - 1u));
  for (int kk = 0; kk < TK; ++kk) {
    const int item = sub * TTI + 32 * kk + lane;
    if (item >= P) {  // beyond a narrow page: masked by the caller
      for (int g = 0; g < 2 * GP; ++g) lg[kk][g] = 0.f;
      continue;
    }
    auto code = [&](int bit, int n) -> uint32_t {
      const int w0 = bit >> 5, sh = bit & 31;
      const uint32_t lo = __ldg(words + wi_word(item, w0, W));
      const uint32_t hi = (sh + n > 32) ? __ldg(words + wi_word(item, w0 + 1, W)) : 0u;
      return __funnelshift_r(lo, hi, sh) & ((1u << n) - 1u);
    };
    float prod = 1.f;
    ptx::f2 acc[GP];
    for (int g = 0; g < GP; ++g) acc[g] = ptx::f2_make(0.f, 0.f);
    int j = 0;
    if (has && grp == 2) {
      for (; j + 1 < d - 2; j += 2) {
        const float4 e = *reinterpret_cast<const float4*>(sm + tbase + code(j * B, 2 * B) * stride);
        ptx::f2 qa[GP], qb[GP];
        load_q<GP>(sm, qs + j * QR, qa);
        load_q<GP>(sm, qs + (j + 1) * QR, qb);
        const float f0 = prod * e.x, f1 = prod * e.y;
        prod *= e.z;
        for (int g = 0; g < GP; ++g) {
          ptx::f2_fma_s_acc(f0, qa[g], acc[g]);
          ptx::f2_fma_s_acc(f1, qb[g], acc[g]);
        }
      }
    }
    for (; j < d - 2; ++j) {
      float cs, sn;
      const uint32_t c = code(j * B, B);
      if (has && grp == 1) {
        const float2 t = *reinterpret_cast<const float2*>(sm + tbase + c * stride);
        cs = t.x;
        sn = t.y;
      } else {
        sincospif((float)c * pstep, &sn, &cs);
      }
      ptx::f2 qa[GP];
      load_q<GP>(sm, qs + j * QR, qa);
      const float f = prod * cs;
      prod *= sn;
      for (int g = 0; g < GP; ++g) ptx::f2_fma_s_acc(f, qa[g], acc[g]);
    }
    {
      float sn, cs;
      sincospif((float)code((d - 2) * B, B) * (1.0f / (float)(1u << (B - 1))), &sn, &cs);
      ptx::f2 qa[GP], qb[GP];
      load_q<GP>(sm, qs + (d - 2) * QR, qa);
      load_q<GP>(sm, qs + (d - 1) * QR, qb);
      const float f0 = prod * cs, f1 = prod * sn;
      for (int g = 0; g < GP; ++g) {
        ptx::f2_fma_s_acc(f0, qa[g], acc[g]);
        ptx::f2_fma_s_acc(f1, qb[g], acc[g]);
      }
    }
    const uint32_t rc = read_bits_g(words, rbit0 + (uint64_t)item * rb, rb);
    const float rr = (float)rc * rscale;
    for (int g = 0; g < GP; ++g) {
      lg[kk][2 * g] = rr * ptx::f2_lo(acc[g]);
      lg[kk][2 * g + 1] = rr * ptx::f2_hi(acc[g]);
    }
  }
}

// Logits (base 2) of the tile's items sub*128 + 32 k + lane, k < 4, G heads.
// lut_enc: (table byte offset << 2) | mode, or -1 (no table).
template <int D, int GP>
__device__ __noinline__ void ada_tile_hb(const uint8_t* __restrict__ blkb, int sub, int lane,
                                         uint32_t hb, uint32_t rbit0, int rb, float rscale,
                                         float lg[TK][2 * GP]);

// hb_off: byte offset of the per-query 2-bit h-byte tables in `sm` (0: none).
// DK: the head dimension the kernel instantiation is specialised for (128,
// 64), 0 (any d: generic tiles only) or -1 (runtime d, both sets).
template <int GP, int DK>
__device__ __forceinline__ void ada_logit_dispatch(int B, const uint8_t* codes, int d, int P,
                                                   const sphkv_page_t& pg, int sub, int lane,
                                                   const uint8_t* sm, uint32_t qs, int lut_enc,
                                                   float lg[TK][2 * GP], uint32_t hb_off = 0) {
  const uint8_t* blk = codes + pg.code_off;
  const uint32_t rbit0 = (uint32_t)(angle_part_bytes(d, P, B) * 8);
  const int rb = pg.rbits;
  const float rs = pg.rscale;
  const bool has = lut_enc >= 0;
  const int mode = has ? (lut_enc & 3) : -1;
  const uint32_t tb = has ? (uint32_t)(lut_enc >> 2) : 0u;
#define SPHKV_WI(b, dd, mode, rp) \
  ada_tile_wi<b, dd, GP, mode, rp>(blk, sub, lane, sm, qs, tb, rbit0, rb, rs, lg)
#ifndef SPHKV_NO_HB
  if constexpr (GP <= 2 && DK > 0) {
    if (B == 2 && hb_off != 0 && P % TTI == 0) {
      ada_tile_hb<DK, GP>(blk, sub, lane, ptx::smem_u32(sm) + hb_off, rbit0, rb, rs, lg);
      return;
    }
  }
#endif
  if (P % TTI != 0) {
    // pages narrower than a tile: generic path (guards items >= P)
  } else if (DK == 128 || (DK < 0 && d == 128)) {
   if constexpr (DK == 128 || DK < 0) {
    if (B == 2 && mode == 1) { SPHKV_WI(2, 128, 4, 8); return; }
    if (B == 4 && mode == 1) { SPHKV_WI(4, 128, 2, 8); return; }
    if (B == 4 && mode == 0) { SPHKV_WI(4, 128, 2, 1); return; }
    if (B == 6 && mode == 1) { SPHKV_WI(6, 128, 1, 16); return; }
    if (B == 6 && mode == 0) { SPHKV_WI(6, 128, 1, 1); return; }
    if (B == 7 && mode == 1) { SPHKV_WI(7, 128, 1, 16); return; }
    if (B == 7 && mode == 0) { SPHKV_WI(7, 128, 1, 1); return; }
#ifdef SPHKV_MUFU12
    if (B == 12) { SPHKV_WI(12, 128, 3, 1); return; }
#endif
    if (B == 12 && mode == 2) { SPHKV_WI(12, 128, 1, 2); return; }
    if (B == 12 && mode == 0) { SPHKV_WI(12, 128, 1, 1); return; }
    // 13..16 bits have no table: MUFU sin/cos of the fp32 angle (abs error
    // ~5e-7 per row) -- the reference's max tier, which protected heads append
    // at during decode; sincospif cost ~4x as much per row
    if (B == 15 && !has) { SPHKV_WI(15, 128, 3, 1); return; }
   }
  } else if (DK == 64 || (DK < 0 && d == 64)) {
   if constexpr (DK == 64 || DK < 0) {
    if (B == 2 && mode == 1) { SPHKV_WI(2, 64, 4, 8); return; }
    if (B == 4 && mode == 1) { SPHKV_WI(4, 64, 2, 8); return; }
    if (B == 6 && mode == 1) { SPHKV_WI(6, 64, 1, 16); return; }
    if (B == 7 && mode == 1) { SPHKV_WI(7, 64, 1, 16); return; }
    if (B == 12 && mode == 2) { SPHKV_WI(12, 64, 1, 2); return; }
    if (B == 12 && mode == 0) { SPHKV_WI(12, 64, 1, 1); return; }
    if (B == 15 && !has) { SPHKV_WI(15, 64, 3, 1); return; }
   }
  }
#undef SPHKV_WI
  ada_tile_generic<GP>(blk, B, d, P, sub, lane, sm, qs, lut_enc, rbit0, rb, rs, lg);
}

}  // namespace sphkv
