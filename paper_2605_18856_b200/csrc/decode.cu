// ADA paged decode, dense bf16 paged decode and the split-context LSE merge.
//
// Reference behaviour replaced (pkg/src/sphkv/):
//   decode.py:123-192  angle-path logits  l = (r_q/sqrt d) * r~ * (feat . qfeat)
//   decode.py:291-355  _head_attend: pointer-order stream, stable softmax,
//                      blockwise value mix
//   decode.py:63-69, 302-307  dense path (DenseStore)
//   decode.py:347-354  one softmax over all logits  ->  split partials + LSE
//
// ADA kernel (one persistent CTA per SM, ~210 KB smem, one launch per layer):
//   warps 0..NL-1  logit warps: a 128-item tile per warp, 4 items per lane,
//                  claimed dynamically inside the CTA.  Each lane loads its
//                  items' code strings from the page's word-interleaved
//                  block (L2-prefetched PF_DIST tiles ahead by
//                  cp.async.bulk.prefetch), looks (cos, sin) -- or products of
//                  four rows' factors -- up in shared-memory tables, runs the
//                  feature recurrence in fp32 registers and dots the G query
//                  heads with packed FFMA2 (the 2-bit tier optionally through
//                  per-query h-byte tables, hb_tile.cuh).  Tile max/sum and
//                  fp16 weights go to a P slot (12-slot ring).
//   warp NL        PV warp: V^T (ldmatrix.trans of the TMA-staged, swizzled
//                  fp16 V tile) x P (fp16) on mma.sync, fp32 accumulate,
//                  online-softmax combine across tiles, writes the partial.
//                  Lane 0 also issues the 1-D TMA bulk copies of V tiles into a
//                  2-slot ring (evict_first), NV tiles ahead of consumption.
//   The CTA finishing a group's last split merges the group's partials
//   (fused LSE merge) into output rows, a partial state (page-range split),
//   and the gate margins when asked.
#include <cstdlib>
#include "common.cuh"
#include "ptx.cuh"
#include "ada_tile.cuh"
#include "hb_tile.cuh"

namespace sphkv {

// Cold per-unit helpers, inlined (SPHKV_COLD_INLINE=0: out of line -- measured
// slower: the calls spill around them and the code layout shifts; instruction
// fetch is a first-order cost of this kernel).
#if !defined(SPHKV_COLD_INLINE) || SPHKV_COLD_INLINE
#define SPHKV_COLD __device__ __forceinline__
#else
#define SPHKV_COLD __device__ __noinline__
#endif

constexpr float kLog2e = 1.4426950408889634f;
#ifndef SPHKV_NL
#define SPHKV_NL 7
#endif
constexpr int ADA_NL = SPHKV_NL;   // logit warps
constexpr int ADA_TI = TTI;        // items per tile (TK per lane)
#ifndef SPHKV_NS
#define SPHKV_NS 12
#endif
constexpr int ADA_NS = SPHKV_NS;   // P slots
// a logit warp waits for its slot by mbarrier PARITY: with NS or more warps
// blocked on slots, a claim NS tiles ahead could pass on a stale phase
static_assert(ADA_NS > ADA_NL, "more P slots than logit warps");
#ifndef SPHKV_NV
#define SPHKV_NV 2
#endif
constexpr int ADA_NV = SPHKV_NV;   // V slots
#ifndef SPHKV_PF_DIST
#define SPHKV_PF_DIST 8   // L2 prefetch distance in tiles (claim order)
#endif
#ifndef SPHKV_PF_V
#define SPHKV_PF_V 0      // also prefetch each tile's V block to L2 (measured: slower)
#endif
#ifndef SPHKV_NPV
#define SPHKV_NPV 1
#endif
constexpr int ADA_NPV = SPHKV_NPV;  // PV warps (split d_v)
constexpr int ADA_MTW = 8 / ADA_NPV; // m-tiles per PV warp (d_v <= 128)
constexpr int ADA_THREADS = (ADA_NL + ADA_NPV) * 32;
constexpr int MAX_UNIT_TILES = 512;
constexpr int PROW_PAD = 16;       // bytes of padding per P row (bank spread)

struct FusedCtl {
  const int32_t* slot_group;  // [n_slots] plan group of each partial slot, -1 = scratch
  const int32_t* slot_begin;  // [n_groups + 1]
  int32_t* ctl;
  float* out;                 // [n_groups * G, d_v] normalized outputs
  int n_groups;
  int dynamic;                // units claimed from ctl[n_groups] instead of u += grid
  float* top2;                // [n_slots + 1][G] second-largest logit per split, or NULL
  float* margins;             // [n_groups * G] top-1 minus top-2 logit (natural units)
  int abs_rows;               // out / margins rows by absolute group id, not plan order
  int32_t* ctl_err;           // set to SPHKV_E_CAPACITY when a unit exceeds the tile list
                              // (standard kernel only; NULL: not checked)
  int state_out;              // out = one partial-state slot per group (m = log2-sum-exp,
                              // l = 1, acc = normalized output): a page-range split's
                              // local result, ready for the all-gather and merge over ranks
  int flag_units;             // entry point contract: a unit over the tile list is flagged
                              // in ctl_err (standard kernel) instead of run as segments
};

struct AdaParams {
  sphkv_store_t st;
  const float* q;          // [groups, G, d] fp32
  int G;
  const sphkv_unit_t* units;
  int n_units;
  float* partials;
  float* logits_dbg;
  const int64_t* dbg_off;
  int lut_off[SPHKV_MAX_TIERS];   // encoded table descriptor per tier (see lut_layout_tiers)
  int lut_bytes;                  // LUT region size
  const uint8_t* lut_global;      // prebuilt tables (sphkv_store_build_lut) or NULL
  int TI;                   // tile items (min(P, 128))
  int dvp;                  // d_v padded to 16
  uint32_t smem_q, smem_tiles, smem_p, smem_v, smem_bar;  // byte offsets
  uint32_t smem_hb;         // per-query 2-bit h-byte tables (hb_tile.cuh), if hb
  int hb;                   // 2-bit tier decodes through the h-byte tables
  int pslot_bytes, prow_bytes, prows;  // P slot: prows rows of TI fp16 weights + header
  FusedCtl fz;
  // pipelined unit transitions (k_ada_decode_pipe): second q / tile-list
  // buffers and the unit-info ring
  uint32_t smem_q2, smem_tiles2, smem_info;
  int pipe;
};

__device__ __forceinline__ int tier_index(const sphkv_store_t& st, int tier_id) {
  for (int i = 0; i < st.n_tiers; ++i)
    if (st.tiers[i].id == tier_id) return i;
  return 0;
}

// ---------------------------------------------------------------------------
// shared pieces: unit setup, P slot write, PV consumer
// ---------------------------------------------------------------------------
struct TileEntry {
  int32_t page;       // page id
  int32_t sub_off;    // (sub << 24) | item offset within unit (< 2^24)
};

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// End of a unit's pointer range: ptr_end < 0 marks an open-ended unit that
// runs to the group's CURRENT list end (a decode step attends pages the
// previous step appended; the plan is reused unchanged, e.g. inside a CUDA
// graph).  Such launches are not programmatic-dependent (live stores).
__device__ __forceinline__ int unit_end(const sphkv_store_t& st, const sphkv_unit_t& u) {
  return u.ptr_end >= 0 ? u.ptr_end : st.ptr_len[u.group];
}

// Build one segment of a unit's tile list (warp 0): whole pages of the
// pointer range [pb, pe) in order, as many as fit in MAX_UNIT_TILES tiles.
// Writes the tile count to seg[0] and the first pointer position NOT taken
// to seg[1] (== pe when the range is done; a unit longer than the cap runs as
// several segments).  item_base = items of the unit before pb (dbg offsets).
SPHKV_COLD void build_tiles(const sphkv_store_t& st, int group, int pb, int pe, int item_base,
                            int TI, TileEntry* tiles, int* seg, int lane) {
  const int* ptr = st.ptr + (size_t)group * st.ptr_cap;
  int nt = 0, items = item_base, next = pe;
  for (int b = pb; b < pe; b += 32) {
    int pos = b + lane;
    int pid = -1, cnt = 0;
    if (pos < pe) {
      pid = ptr[pos];
      cnt = st.pages[pid].count;
    }
    int t = (cnt + TI - 1) / TI;
    // inclusive scans of tiles and items
    int ts = t, is = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int a = __shfl_up_sync(0xffffffffu, ts, o), c = __shfl_up_sync(0xffffffffu, is, o);
      if (lane >= o) { ts += a; is += c; }
    }
    // pages that fit are a prefix (the scan is monotone)
    const unsigned fit = __ballot_sync(0xffffffffu, pos < pe && nt + ts <= MAX_UNIT_TILES);
    const int n_fit = __popc(fit);
    int t0 = nt + ts - t, i0 = items + is - cnt;
    if ((fit >> lane) & 1u)
      for (int s = 0; s < t; ++s) {
        tiles[t0 + s].page = pid;
        tiles[t0 + s].sub_off = (s << 24) | (i0 + s * TI);
      }
    const int last = n_fit - 1;
    if (n_fit > 0) {
      nt += __shfl_sync(0xffffffffu, ts, last);
      items += __shfl_sync(0xffffffffu, is, last);
    }
    if (n_fit < min(32, pe - b)) {
      next = b + n_fit;
      break;
    }
  }
  if (lane == 0) {
    seg[0] = nt;
    seg[1] = next;
    seg[2] = items;
  }
}

// Write the fp16 weights of one tile + tile max/sum.  Lane l holds items
// l + 32 k (k < 4) of the tile; bit k of `valid` says whether item l + 32 k
// exists.
// With want2 the header also carries each head's second-largest logit
// (hdr[16 + g]) for the decode-time gate's top-1/top-2 margin (gate.py:50-56).
template <int NG>
__device__ __forceinline__ void write_pslot(uint8_t* slot, int prow_bytes, int prows, int TI,
                                            int lane, int G, const float lg[TK][NG],
                                            uint32_t valid, bool want2 = false) {
  float* hdr = reinterpret_cast<float*>(slot + prows * prow_bytes);
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    float m = -INFINITY;
#pragma unroll
    for (int k = 0; k < TK; ++k)
      if (valid & (1u << k)) m = fmaxf(m, lg[k][g]);
    if (want2) {  // warp top-2 of this head's tile logits
      float a = -INFINITY, b = -INFINITY;
#pragma unroll
      for (int k = 0; k < TK; ++k)
        if (valid & (1u << k)) {
          const float v = lg[k][g];
          b = fmaxf(b, fminf(a, v));
          a = fmaxf(a, v);
        }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float a2 = __shfl_xor_sync(0xffffffffu, a, o), b2 = __shfl_xor_sync(0xffffffffu, b, o);
        b = fmaxf(fminf(a, a2), fmaxf(b, b2));
        a = fmaxf(a, a2);
      }
      if (lane == 0 && g < 8) hdr[16 + g] = b;
    }
    m = warp_max(m);
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < TK; ++k) {
      const float e = (valid & (1u << k)) ? exp2f(lg[k][g] - m) : 0.f;
      const __half h = __float2half_rn(e);
      s += __half2float(h);
      if (g < G && 32 * k + lane < TI)
        *reinterpret_cast<__half*>(slot + g * prow_bytes + (32 * k + lane) * 2) = h;
    }
    s = warp_sum(s);
    if (lane == 0 && g < 8) {
      hdr[g] = m;
      hdr[8 + g] = s;
    }
  }
}

// Online-softmax state of one PV warp for its m-tiles [mt0, mt0 + MTW) of d_v.
template <int MTW>
struct PVState {
  float acc[MTW][4];
  float m[2], l[2];
  float m2[2];  // running second-largest logit (gate margins)
};

template <int MTW>
__device__ __forceinline__ void pv_init(PVState<MTW>& s) {
#pragma unroll
  for (int i = 0; i < MTW; ++i)
#pragma unroll
    for (int r = 0; r < 4; ++r) s.acc[i][r] = 0.f;
  s.m[0] = s.m[1] = -INFINITY;
  s.l[0] = s.l[1] = 0.f;
  s.m2[0] = s.m2[1] = -INFINITY;
}

// running top-2 (s.m is the running max) combined with a tile's top-2
template <int MTW>
__device__ __forceinline__ void pv_top2(PVState<MTW>& s, const float* hdr, int G, int lane) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int g = 2 * (lane & 3) + h;
    if (g >= G) continue;
    s.m2[h] = fmaxf(fminf(s.m[h], hdr[g]), fmaxf(s.m2[h], hdr[16 + g]));
  }
}

// One tile of P.V on mma.sync (A = V^T from the swizzled smem tile via
// ldmatrix.trans, B = fp16 weights of the P slot) + online combine.
template <int MTW>
__device__ __forceinline__ void pv_tile(PVState<MTW>& s, const uint8_t* pslot, const uint8_t* vslot,
                                        int prow_bytes, int prows, int TI, int dvp, int mt0,
                                        int mtn, int G, int lane, bool want2 = false) {
  float c[MTW][4];
#pragma unroll
  for (int i = 0; i < MTW; ++i)
#pragma unroll
    for (int r = 0; r < 4; ++r) c[i][r] = 0.f;
  const int nchunks = dvp / 8;
  const int smask = (nchunks < 8 ? nchunks : 8) - 1;
  const uint32_t vbase = ptx::smem_u32(vslot);
  const uint32_t pbase = ptx::smem_u32(pslot);
  const int r = lane & 7, mat = lane >> 3;
  for (int ks = 0; ks < TI / 16; ++ks) {
    uint32_t b0, b1;
    // rows >= prows (only allocated when G > 4) alias the first rows: they feed
    // mma columns g >= G, which are never read
    ptx::ldsm_x2(pbase + ((lane & 7) & (prows - 1)) * prow_bytes +
                     (ks * 16 + ((lane >> 3) & 1) * 8) * 2, b0, b1);
    const int item = ks * 16 + r + (mat >> 1) * 8;
#pragma unroll
    for (int i = 0; i < MTW; ++i) {
      if (i < mtn) {
        const int chunk = 2 * (mt0 + i) + (mat & 1);
        const int sw = chunk ^ (r & smask);
        uint32_t a0, a1, a2, a3;
        ptx::ldsm_x4_trans(vbase + (item * dvp + sw * 8) * 2, a0, a1, a2, a3);
        ptx::mma_f16(c[i], a0, a1, a2, a3, b0, b1);
      }
    }
  }
  const float* hdr = reinterpret_cast<const float*>(pslot + prows * prow_bytes);
  if (want2) pv_top2(s, hdr, G, lane);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int g = 2 * (lane & 3) + h;
    const float mt_ = (g < G) ? hdr[g] : 0.f;
    const float lt = (g < G) ? hdr[8 + g] : 0.f;
    const float mn = fmaxf(s.m[h], mt_);
    const float al = exp2f(s.m[h] - mn), be = exp2f(mt_ - mn);
    s.m[h] = mn;
    s.l[h] = s.l[h] * al + lt * be;
#pragma unroll
    for (int i = 0; i < MTW; ++i) {
      s.acc[i][h] = s.acc[i][h] * al + c[i][h] * be;
      s.acc[i][2 + h] = s.acc[i][2 + h] * al + c[i][2 + h] * be;
    }
  }
}

// Fast path of pv_tile for d_v = 128 (16 swizzled chunks per V row), a
// 16*KS-item tile and all of the warp's m-tiles present: fully unrolled, every
// ldmatrix address is a per-lane base + an immediate (the XOR swizzle term
// only depends on the row inside the 8-row group, not on the k-step).
template <int MTW, int KS = ADA_TI / 16, int DVP = 128, int MTU = MTW>
__device__ __forceinline__ void pv_tile_128(PVState<MTW>& s, const uint8_t* pslot,
                                            const uint8_t* vslot, int prow_bytes, int prows,
                                            int mt0, int G, int lane, bool want2 = false) {
  // DVP: padded d_v (128 or 64: 16 or 8 swizzled chunks per row); MTU <= MTW
  // m-tiles are computed (d_v = 64 through a PVState sized for 128)
  static_assert(DVP == 128 || DVP == 64, "fast P.V path: d_v 64 or 128");
  float c[MTW][4];
#pragma unroll
  for (int i = 0; i < MTW; ++i)
#pragma unroll
    for (int r = 0; r < 4; ++r) c[i][r] = 0.f;
  const int r = lane & 7, mat = lane >> 3;
  const uint32_t pb = ptx::smem_u32(pslot) + ((lane & 7) & (prows - 1)) * prow_bytes +
                      ((lane >> 3) & 1) * 16;
  uint32_t va[MTU];
#pragma unroll
  for (int i = 0; i < MTU; ++i) {
    const int chunk = 2 * (mt0 + i) + (mat & 1);
    va[i] = ptx::smem_u32(vslot) + ((r + (mat >> 1) * 8) * DVP + (chunk ^ r) * 8) * 2;
  }
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
    uint32_t b0, b1;
    ptx::ldsm_x2(pb + ks * 32, b0, b1);
#pragma unroll
    for (int i = 0; i < MTU; ++i) {
      uint32_t a0, a1, a2, a3;
      ptx::ldsm_x4_trans(va[i] + ks * (32 * DVP), a0, a1, a2, a3);
      ptx::mma_f16(c[i], a0, a1, a2, a3, b0, b1);
    }
  }
  const float* hdr = reinterpret_cast<const float*>(pslot + prows * prow_bytes);
  if (want2) pv_top2(s, hdr, G, lane);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int g = 2 * (lane & 3) + h;
    const float mt_ = (g < G) ? hdr[g] : 0.f;
    const float lt = (g < G) ? hdr[8 + g] : 0.f;
    const float mn = fmaxf(s.m[h], mt_);
    const float al = exp2f(s.m[h] - mn), be = exp2f(mt_ - mn);
    s.m[h] = mn;
    s.l[h] = s.l[h] * al + lt * be;
#pragma unroll
    for (int i = 0; i < MTU; ++i) {
      s.acc[i][h] = s.acc[i][h] * al + c[i][h] * be;
      s.acc[i][2 + h] = s.acc[i][2 + h] * al + c[i][2 + h] * be;
    }
  }
}

// Partial layout per slot: m[G], l[G], acc[G][d_v] (base-2 logit units).
template <int MTW>
__device__ __forceinline__ void pv_write(const PVState<MTW>& s, float* part, int G, int d_v,
                                         int mt0, int mtn, bool write_ml, int lane,
                                         float* top2 = nullptr) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int g = 2 * (lane & 3) + h;
    if (g >= G) continue;
    if (write_ml && (lane >> 2) == 0) {
      part[g] = s.m[h];
      part[G + g] = s.l[h];
      if (top2 != nullptr) top2[g] = s.m2[h];
    }
    float* a = part + 2 * G + (size_t)g * d_v;
#pragma unroll
    for (int i = 0; i < MTW; ++i) {
      if (i >= mtn) continue;
      const int r0 = (mt0 + i) * 16 + (lane >> 2);
      if (r0 < d_v) a[r0] = s.acc[i][h];
      if (r0 + 8 < d_v) a[r0 + 8] = s.acc[i][2 + h];
    }
  }
}

// ---------------------------------------------------------------------------
// In-kernel split merge + dynamic unit queue (shared by both decode kernels)
// ---------------------------------------------------------------------------
// With `slot_group` set, the CTA that completes the LAST split of a group
// merges that group's partial slots straight into the output rows (the
// split-K "last block" pattern): no separate merge launch, and the merge of
// one group overlaps the other CTAs' decode.  ctl[] (caller-zeroed, left
// zeroed): ctl[g] = finished splits of plan group g, ctl[n_groups] = unit
// queue head, ctl[n_groups + 1] = CTAs done (the last one resets the queue).

// Called by every thread after the unit's partial is written (all threads
// have passed a __syncthreads since).  Returns through smem whether this CTA
// merged; the caller's loop continues with *next_unit (dynamic mode).
SPHKV_COLD void fused_unit_done(const FusedCtl& f, const float* partials,
                                                int out_slot, int G, int d_v, int n_units,
                                                int* s_flag, float* s_ml, int* s_next,
                                                int group = 0) {
  if (f.slot_group == nullptr && !f.dynamic) return;  // plain split partials only
  __threadfence();  // this thread's partial writes -> gpu scope before the count
  __syncthreads();
  const int gi = (f.slot_group != nullptr) ? f.slot_group[out_slot] : -1;
  if (threadIdx.x == 0) {
    int last = 0;
    if (gi >= 0) {
      const int ns = f.slot_begin[gi + 1] - f.slot_begin[gi];
      last = atomicAdd(&f.ctl[gi], 1) == ns - 1;
    }
    *s_flag = last;
    // the first gridDim.x units are taken statically (blockIdx.x), so queue
    // claims start at gridDim.x
    if (f.dynamic) *s_next = atomicAdd(&f.ctl[f.n_groups], 1) + (int)gridDim.x;
  }
  __syncthreads();
  if (!*s_flag) return;
  __threadfence();
  const int b = f.slot_begin[gi], e = f.slot_begin[gi + 1];
  const int64_t stride = (int64_t)G * (d_v + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int g = warp; g < G; g += nw) {  // (M, L) per query head
    float M = -INFINITY;
    for (int s = b + lane; s < e; s += 32) M = fmaxf(M, __ldcg(partials + s * stride + g));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    float L = 0.f;
    for (int s = b + lane; s < e; s += 32) {
      const float m = __ldcg(partials + s * stride + g);
      const float l = __ldcg(partials + s * stride + G + g);
      L += (m != -INFINITY) ? l * exp2f(m - M) : 0.f;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
    if (lane == 0) {
      s_ml[g] = M;
      s_ml[8 + g] = L;
    }
    if (f.margins != nullptr) {  // gate margin: top-2 over the union of the splits
      int cnt = 0;
      float m2 = -INFINITY;
      for (int s = b + lane; s < e; s += 32) {
        const float m = __ldcg(partials + s * stride + g);
        if (m == M && M != -INFINITY) ++cnt; else m2 = fmaxf(m2, m);
        m2 = fmaxf(m2, __ldcg(f.top2 + (int64_t)s * G + g));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        m2 = fmaxf(m2, __shfl_xor_sync(0xffffffffu, m2, o));
      }
      if (cnt >= 2) m2 = M;
      if (lane == 0)
        f.margins[(int64_t)(f.abs_rows ? group : gi) * G + g] =
            (m2 == -INFINITY) ? INFINITY : (M - m2) * 0.69314718055994531f;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G * d_v; i += blockDim.x) {
    const int g = i / d_v, j = i % d_v;
    const float M = s_ml[g], L = s_ml[8 + g];
    // unconditional loads, unrolled: the slots' (m, acc) reads are issued
    // back to back instead of one L2 round trip per slot
    float a = 0.f;
#pragma unroll 8
    for (int s = b; s < e; ++s) {
      const float m = __ldcg(partials + s * stride + g);
      const float v = __ldcg(partials + s * stride + 2 * G + (int64_t)g * d_v + j);
      a += (m != -INFINITY) ? v * exp2f(m - M) : 0.f;
    }
    if (f.state_out)
      f.out[(int64_t)gi * stride + 2 * G + (int64_t)g * d_v + j] = (L > 0.f) ? a / L : 0.f;
    else
      f.out[((int64_t)(f.abs_rows ? group : gi) * G + g) * d_v + j] = (L > 0.f) ? a / L : 0.f;
  }
  if (f.state_out && threadIdx.x < G) {  // (m, l) of the state slot (k_lse_merge state_out)
    const float M = s_ml[threadIdx.x], L = s_ml[8 + threadIdx.x];
    f.out[(int64_t)gi * stride + threadIdx.x] = (L > 0.f) ? M + log2f(L) : -INFINITY;
    f.out[(int64_t)gi * stride + G + threadIdx.x] = (L > 0.f) ? 1.f : 0.f;
  }
  if (threadIdx.x == 0) f.ctl[gi] = 0;  // every split of gi has counted: safe to re-arm
  __syncthreads();
}

// Every CTA's first unit is static (blockIdx.x), dynamic plan or not: the
// prologue that runs before griddepcontrol.wait (tile list, prefetches) may
// then touch no control word the previous grid on the stream still uses --
// queue claims (ctl[n_groups]) happen only after the wait.
__device__ __forceinline__ int fused_first_unit(const FusedCtl&, int*) { return blockIdx.x; }

__device__ __forceinline__ void fused_kernel_exit(const FusedCtl& f) {
  if (!f.dynamic || threadIdx.x != 0) return;
  __threadfence();
  if (atomicAdd(&f.ctl[f.n_groups + 1], 1) == (int)gridDim.x - 1) {
    f.ctl[f.n_groups] = 0;  // every CTA has made its final claim
    f.ctl[f.n_groups + 1] = 0;
  }
}

// ---------------------------------------------------------------------------
// ADA kernel
// ---------------------------------------------------------------------------
#ifdef SPHKV_DBG_TIMING  // per-CTA start/end (globaltimer ns) of the last launch
__device__ unsigned long long g_cta_t[2 * 1024];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif

template <int GP, int DK>
__global__ void __launch_bounds__(ADA_THREADS, 1) k_ada_decode(const AdaParams p) {
#ifdef SPHKV_DBG_TIMING
  if (threadIdx.x == 0 && blockIdx.x < 1024) g_cta_t[2 * blockIdx.x] = gtimer();
#endif
  extern __shared__ __align__(128) uint8_t smem[];
  const sphkv_store_t& st = p.st;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float2* qs = reinterpret_cast<float2*>(smem + p.smem_q);
  TileEntry* tiles = reinterpret_cast<TileEntry*>(smem + p.smem_tiles);
  // seg[0] = tiles of the current segment, seg[1] = its end pointer position,
  // seg[2] = unit items before the next segment; then the tile claim counter
  int* seg = reinterpret_cast<int*>(smem + p.smem_tiles + MAX_UNIT_TILES * sizeof(TileEntry));
  int* tile_ctr = seg + 3;
  uint8_t* pslots = smem + p.smem_p;
  uint8_t* vslots = smem + p.smem_v;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.smem_bar);
  uint64_t* p_full = bars;
  uint64_t* p_empty = bars + ADA_NS;
  uint64_t* v_full = bars + 2 * ADA_NS;
  uint64_t* v_empty = bars + 2 * ADA_NS + ADA_NV;
  const int d = st.d, P = st.page_size, TI = p.TI, dvp = p.dvp, MT = dvp / 16;
  const uint32_t vbytes = (uint32_t)TI * dvp * 2;

  // Prologue (independent of the previous grid, so under programmatic
  // dependent launch it overlaps that grid's tail): barrier init and the
  // polar LUTs -- one TMA bulk copy of the prebuilt tables (or fp64 sincos
  // rounded to fp32 computed in place when the store has no global table).
  uint64_t* lut_bar = bars + 2 * ADA_NS + 2 * ADA_NV;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ADA_NS; ++i) {
      ptx::mbar_init(&p_full[i], 1);
      ptx::mbar_init(&p_empty[i], ADA_NPV);
    }
    for (int i = 0; i < ADA_NV; ++i) {
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&v_empty[i], ADA_NPV);
    }
    ptx::mbar_init(lut_bar, 1);
    ptx::fence_mbar_init();
    if (p.lut_global != nullptr && p.lut_bytes > 0) {
      ptx::mbar_arrive_expect_tx(lut_bar, (uint32_t)p.lut_bytes);
      ptx::bulk_g2s(smem, p.lut_global, (uint32_t)p.lut_bytes, lut_bar);
    } else {
      ptx::mbar_arrive(lut_bar);
    }
  }
  if (p.lut_global == nullptr) lut_fill(smem, st.tiers, st.n_tiers, p.lut_off, threadIdx.x, blockDim.x);
  // L2 prefetch, PF_DIST tiles ahead of the claim order: the tile's code
  // granules (contiguous in the WI layout), its radius row with the
  // page's first tile, and (SPHKV_PF_V) its fp16 V block, so the V bulk
  // copy and the code loads hit L2 and many more bytes are in flight per
  // SM than the smem rings alone could hold.
  auto prefetch_tile = [&](int t, int nt) {
    if (t < nt && lane == 0) {
      const TileEntry tn = tiles[t];
      const int sb = tn.sub_off >> 24;
      const sphkv_page_t pn = st.pages[tn.page];
      const uint64_t W4 = (uint64_t)item_words(d, pn.abits) * 128;  // bytes per granule
      const int g0 = sb * TI / 32, ng = (TI + 31) / 32;
      ptx::bulk_prefetch_l2(st.codes + pn.code_off + g0 * W4, (uint32_t)(ng * W4));
      if (sb == 0) {
        const uint64_t ab = angle_part_bytes(d, P, pn.abits);
        ptx::bulk_prefetch_l2(st.codes + pn.code_off + ab,
                              (uint32_t)(code_block_bytes(d, P, pn.abits, pn.rbits) - ab));
      }
#if SPHKV_PF_V
      ptx::bulk_prefetch_l2(st.values + ((size_t)tn.page * P + (size_t)sb * TI) * dvp, vbytes);
#endif
    }
  };
#ifndef SPHKV_PF_L1
#define SPHKV_PF_L1 6
#endif
  // h-byte tiles load their whole 4 KB code block up front: pull tile t's
  // block into this SM's L1 (one 128-byte line per lane) about one tile-time
  // ahead, so whichever warp claims it finds it there.
  auto prefetch_tile_l1 = [&](int t, int nt) {
    if (SPHKV_PF_L1 > 0 && p.hb && t < nt) {
      const TileEntry tn = tiles[t];
      const sphkv_page_t pn = st.pages[tn.page];
      if (pn.abits == 2) {
        const uint64_t W4 = (uint64_t)item_words(d, 2) * 128;
        const uint8_t* b = st.codes + pn.code_off + (uint64_t)((tn.sub_off >> 24) * TI / 32) * W4;
        if ((uint32_t)lane * 128u < (uint32_t)(TI / 32) * (uint32_t)W4) ptx::prefetch_l1_line(b + lane * 128);
      }
    }
  };
  // Also independent of the previous grid (it only reads q and writes
  // outputs): the first unit's tile list and its first L2 prefetches.
  // scalars of the fused merge / unit queue live after the barriers (no static
  // __shared__: it would cost a 1 KB-aligned block next to the dynamic region)
  int& s_flag = *reinterpret_cast<int*>(bars + 2 * ADA_NS + 2 * ADA_NV + 1);
  int& s_next = *(reinterpret_cast<int*>(bars + 2 * ADA_NS + 2 * ADA_NV + 1) + 1);
  float* s_ml = reinterpret_cast<float*>(bars + 2 * ADA_NS + 2 * ADA_NV + 2);
  int u = fused_first_unit(p.fz, &s_next);
  if (u < p.n_units && warp == 0) {
    const sphkv_unit_t u0 = p.units[u];
    build_tiles(st, u0.group, u0.ptr_begin, unit_end(st, u0), 0, TI, tiles, seg, lane);
    if (lane == 0) *tile_ctr = 0;
  }
  __syncthreads();
  // V tile producer (lane 0 of the first PV warp): bulk copy of tile k's fp16
  // V block into ring slot (gbase + k) % NV once every PV warp released it
  const uint64_t vpol = ptx::policy_evict_first();
  auto issue_v = [&](int k, uint32_t gb) {
    const uint32_t gk = gb + k;
    const int vs = gk % ADA_NV;
    ptx::mbar_wait(&v_empty[vs], ((gk / ADA_NV) & 1) ^ 1);
    const TileEntry te = tiles[k];
    const int sub = te.sub_off >> 24;
    const uint16_t* src = st.values + ((size_t)te.page * P + (size_t)sub * TI) * dvp;
    ptx::fence_proxy_async();  // order earlier ldmatrix reads of the slot
    ptx::mbar_arrive_expect_tx(&v_full[vs], vbytes);
    ptx::bulk_g2s_hint(vslots + (size_t)vs * vbytes, src, vbytes, &v_full[vs], vpol);
  };
  if (u < p.n_units && warp < ADA_NL)
    for (int t = warp; t < SPHKV_PF_DIST; t += ADA_NL) prefetch_tile(t, seg[0]);
  if (u < p.n_units && warp == ADA_NL && lane == 0)
    for (int k = 0; k < seg[0] && k < ADA_NV; ++k) issue_v(k, 0u);
  ptx::griddep_wait();  // inputs below (q) may come from the previous grid
#ifdef SPHKV_DBG_TIMING
  if (threadIdx.x == 0 && blockIdx.x < 1024) g_cta_t[2 * blockIdx.x] = gtimer();
#endif
  __syncthreads();
  ptx::griddep_launch_dependents();
  bool lut_ready = false, first = true;

  const float qscale = kLog2e * rsqrtf((float)d);
  uint32_t gbase = 0;  // running tile sequence number (barrier phases)
  const int pw = warp - ADA_NL;  // PV warp index (warp >= ADA_NL)
  const int mtw = (MT + ADA_NPV - 1) / ADA_NPV;
  const int mt0 = pw * mtw;
  const int mtn = max(0, min(mtw, MT - mt0));
  for (; u < p.n_units; first = false) {
    const sphkv_unit_t unit = p.units[u];
    const int pe = unit_end(st, unit);  // (open-ended units: the list's current end)
    // q rows for this group, prescaled into base-2 logit units, packed pairs
    const float* qg = p.q + (size_t)unit.group * p.G * d;
    for (int i = threadIdx.x; i < d * GP; i += blockDim.x) {
      int j = i / GP, g2 = i % GP;
      float a = (2 * g2 < p.G) ? qg[(size_t)(2 * g2) * d + j] * qscale : 0.f;
      float b = (2 * g2 + 1 < p.G) ? qg[(size_t)(2 * g2 + 1) * d + j] * qscale : 0.f;
      qs[j * (q_row_bytes(GP) / 8) + g2] = make_float2(a, b);
    }
#ifndef SPHKV_NO_HB
    if constexpr (GP <= 2 && DK != 0) {
      if (p.hb) {  // per-query tables of the 2-bit tier; scratch = the idle P slots
        __syncthreads();  // the previous unit's last P-slot reads are done
        double* scratch = reinterpret_cast<double*>(pslots);
        const double qs_d = 1.4426950408889634 / sqrt((double)d);
        hb_build<DK>(smem + p.smem_hb, scratch, qg, p.G, qs_d);
      }
    }
#endif
    // A unit runs as one or more segments of <= MAX_UNIT_TILES tiles; the
    // online-softmax state of the PV warps carries across segments.  Every
    // warp runs the same loop and meets the same block barriers.
    PVState<ADA_MTW> s;
    if (warp >= ADA_NL) pv_init(s);
    const bool fast_pv = (dvp == 128 && TI == ADA_TI && mtn == ADA_MTW);
    const bool fast64 = (dvp == 64 && TI == ADA_TI && ADA_NPV == 1);
    for (bool seg_first = true;; seg_first = false) {
      if (!(first && seg_first) && warp == 0) {
        const int pb = seg_first ? unit.ptr_begin : seg[1];
        const int ib = seg_first ? 0 : seg[2];
        __syncwarp();  // every lane has read seg[] before lane 0 rewrites it
        build_tiles(st, unit.group, pb, pe, ib, TI, tiles, seg, lane);
        if (lane == 0) *tile_ctr = 0;
      }
      __syncthreads();
      const int nt = seg[0], seg_end = seg[1];  // read before warp 0 may rebuild
      if (warp < ADA_NL) {
        // ---------------- logit warps ----------------
        if (!lut_ready) {
          ptx::mbar_wait(lut_bar, 0);
          lut_ready = true;
        }
        // tiles are claimed dynamically (smem counter) to balance the warps;
        // the P slot of tile k is k % NS whoever computes it.
        if (!(first && seg_first))
          for (int t = warp; t < SPHKV_PF_DIST; t += ADA_NL) prefetch_tile(t, nt);
#ifdef SPHKV_TILE_LOOP_NOUNROLL
#pragma unroll 1
#endif
        for (;;) {
          int k = 0;
          if (lane == 0) k = atomicAdd(tile_ctr, 1);
          k = __shfl_sync(0xffffffffu, k, 0);
          if (k >= nt) break;
          prefetch_tile(k + SPHKV_PF_DIST, nt);
#ifndef SPHKV_NO_HB
          prefetch_tile_l1(k + SPHKV_PF_L1, nt);
#endif
          const uint32_t gk = gbase + k;
          const TileEntry te = tiles[k];
          const int sub = te.sub_off >> 24, ioff = te.sub_off & 0xffffff;
          const sphkv_page_t pg = st.pages[te.page];
          const int ti = tier_index(st, pg.tier);
          float lg[TK][2 * GP];  // LUT region starts at smem[0]
#ifdef SPHKV_DBG_NOLOGIT  // bottleneck probe: skip the logit math
          for (int a_ = 0; a_ < TK; ++a_)
            for (int b_ = 0; b_ < 2 * GP; ++b_) lg[a_][b_] = (float)(a_ + b_) * 0.01f + (float)ti;
#else
          ada_logit_dispatch<GP, DK>(pg.abits, st.codes, d, P, pg, sub, lane, smem, p.smem_q,
                                 p.lut_off[ti], lg, p.hb ? p.smem_hb : 0u);
#endif
          uint32_t valid = 0;
#pragma unroll
          for (int kk = 0; kk < TK; ++kk) {
            const int it = sub * TI + 32 * kk + lane;
            if (32 * kk + lane < TI && it < pg.count) valid |= 1u << kk;
          }
          if (p.logits_dbg != nullptr) {
#pragma unroll
            for (int kk = 0; kk < TK; ++kk) {
              float* dst = p.logits_dbg + (size_t)(p.dbg_off[u] + ioff + 32 * kk + lane) * p.G;
#pragma unroll
              for (int g = 0; g < 2 * GP; ++g)
                if ((valid & (1u << kk)) && g < p.G) dst[g] = lg[kk][g] * (1.0f / kLog2e);
            }
          }
          const int ps = gk % ADA_NS;
          ptx::mbar_wait(&p_empty[ps], ((gk / ADA_NS) & 1) ^ 1);
          write_pslot<2 * GP>(pslots + ps * p.pslot_bytes, p.prow_bytes, p.prows, TI, lane, p.G,
                              lg, valid, p.fz.top2 != nullptr);
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&p_full[ps]);
        }
      } else {
        // ---------------- PV warps ----------------
        // NPV warps split the d_v m-tiles; all consume every tile in order.
        // Lane 0 of PV warp 0 is also the V producer: it refills slot vs once
        // every PV warp has released it (v_empty counts NPV arrivals).
        if (!(first && seg_first) && pw == 0 && lane == 0)
          for (int k = 0; k < nt && k < ADA_NV; ++k) issue_v(k, gbase);
        for (int k = 0; k < nt; ++k) {
          const uint32_t gk = gbase + k;
          const int vs = gk % ADA_NV, ps = gk % ADA_NS;
          ptx::mbar_wait(&v_full[vs], (gk / ADA_NV) & 1);
          ptx::mbar_wait(&p_full[ps], (gk / ADA_NS) & 1);
#ifndef SPHKV_DBG_NOPV  // bottleneck probe: skip the P.V math
          if (fast_pv)
            pv_tile_128<ADA_MTW>(s, pslots + ps * p.pslot_bytes, vslots + (size_t)vs * vbytes,
                                 p.prow_bytes, p.prows, mt0, p.G, lane, p.fz.top2 != nullptr);
          else if (fast64)
            pv_tile_128<ADA_MTW, ADA_TI / 16, 64, 4>(s, pslots + ps * p.pslot_bytes,
                                                     vslots + (size_t)vs * vbytes, p.prow_bytes,
                                                     p.prows, 0, p.G, lane, p.fz.top2 != nullptr);
          else
            pv_tile<ADA_MTW>(s, pslots + ps * p.pslot_bytes, vslots + (size_t)vs * vbytes,
                             p.prow_bytes, p.prows, TI, dvp, mt0, mtn, p.G, lane,
                             p.fz.top2 != nullptr);
#endif
          __syncwarp();
          if (lane == 0) {
            ptx::mbar_arrive(&p_empty[ps]);
            ptx::mbar_arrive(&v_empty[vs]);
            if (pw == 0 && k + ADA_NV < nt) issue_v(k + ADA_NV, gbase);
          }
        }
      }
      gbase += nt;
      __syncthreads();  // the tile list and seg[] may be rebuilt now
#ifdef SPHKV_NO_SEG  // experiment builds: one segment per unit (oversize units truncated)
      (void)seg_end;
      break;
#else
      if (seg_end >= pe) break;
#endif
    }
    if (warp >= ADA_NL) {
      float* part = p.partials + (size_t)unit.out_slot * ((size_t)p.G * (st.d_v + 2));
      pv_write<ADA_MTW>(s, part, p.G, st.d_v, mt0, mtn, pw == 0, lane,
                        p.fz.top2 != nullptr ? p.fz.top2 + (size_t)unit.out_slot * p.G : nullptr);
    }
    __syncthreads();
    fused_unit_done(p.fz, p.partials, unit.out_slot, p.G, st.d_v, p.n_units, &s_flag, s_ml,
                    &s_next, unit.group);
    u = p.fz.dynamic ? s_next : u + gridDim.x;
  }
  fused_kernel_exit(p.fz);
#ifdef SPHKV_DBG_TIMING
  if (threadIdx.x == 0 && blockIdx.x < 1024) g_cta_t[2 * blockIdx.x + 1] = gtimer();
#endif
}

// Tile list of a whole unit for the standard kernel (warp 0): returns the
// tile count (also in smem); a unit with more tiles than the list holds is
// flagged in ctl_err (the launch's units are unusable: SPHKV_E_CAPACITY).
__device__ int build_tiles_std(const sphkv_store_t& st, const sphkv_unit_t& u, int TI,
                               TileEntry* tiles, int* ntiles_smem, int lane, int32_t* ctl_err,
                               int cap = MAX_UNIT_TILES) {
  const int* ptr = st.ptr + (size_t)u.group * st.ptr_cap;
  const int pe = unit_end(st, u);  // open-ended (live) units: the list's current end
  int nt = 0, items = 0;
  for (int b = u.ptr_begin; b < pe; b += 32) {
    int pos = b + lane;
    int pid = -1, cnt = 0;
    if (pos < pe) {
      pid = ptr[pos];
      cnt = st.pages[pid].count;
    }
    int t = (cnt + TI - 1) / TI;
    // inclusive scans of tiles and items
    int ts = t, is = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int a = __shfl_up_sync(0xffffffffu, ts, o), c = __shfl_up_sync(0xffffffffu, is, o);
      if (lane >= o) { ts += a; is += c; }
    }
    int t0 = nt + ts - t, i0 = items + is - cnt;
    for (int s = 0; s < t; ++s) {
      if (t0 + s < cap) {
        tiles[t0 + s].page = pid;
        tiles[t0 + s].sub_off = (s << 24) | (i0 + s * TI);
      }
    }
    nt += __shfl_sync(0xffffffffu, ts, 31);
    items += __shfl_sync(0xffffffffu, is, 31);
  }
  if (lane == 0) {
    *ntiles_smem = nt < cap ? nt : cap;
    if (nt > cap && ctl_err != nullptr) atomicExch(ctl_err, SPHKV_E_CAPACITY);
  }
  return nt;
}


// The standard path (one launch per layer, fused merge, no margins / live
// store / state output / h-byte tables / debug logits): the round-1 kernel
// body, kept verbatim because its instruction layout is measurably faster
// than the general kernel's (c5 +5%, c4 +65%).  Units
// must fit the tile list (planner-made units do; others are flagged).
template <int GP>
__global__ void __launch_bounds__(ADA_THREADS, 1) k_ada_decode_std(const AdaParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const sphkv_store_t& st = p.st;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float2* lut = reinterpret_cast<float2*>(smem);
  float2* qs = reinterpret_cast<float2*>(smem + p.smem_q);
  TileEntry* tiles = reinterpret_cast<TileEntry*>(smem + p.smem_tiles);
  int* ntiles_s = reinterpret_cast<int*>(smem + p.smem_tiles + MAX_UNIT_TILES * sizeof(TileEntry));
  int* tile_ctr = ntiles_s + 1;
  uint8_t* pslots = smem + p.smem_p;
  uint8_t* vslots = smem + p.smem_v;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.smem_bar);
  uint64_t* p_full = bars;
  uint64_t* p_empty = bars + ADA_NS;
  uint64_t* v_full = bars + 2 * ADA_NS;
  uint64_t* v_empty = bars + 2 * ADA_NS + ADA_NV;
  const int d = st.d, P = st.page_size, TI = p.TI, dvp = p.dvp, MT = dvp / 16;
  const uint32_t vbytes = (uint32_t)TI * dvp * 2;

  // Prologue (independent of the previous grid, so under programmatic
  // dependent launch it overlaps that grid's tail): barrier init and the
  // polar LUTs -- one TMA bulk copy of the prebuilt tables (or fp64 sincos
  // rounded to fp32 computed in place when the store has no global table).
  uint64_t* lut_bar = bars + 2 * ADA_NS + 2 * ADA_NV;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ADA_NS; ++i) {
      ptx::mbar_init(&p_full[i], 1);
      ptx::mbar_init(&p_empty[i], ADA_NPV);
    }
    for (int i = 0; i < ADA_NV; ++i) {
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&v_empty[i], ADA_NPV);
    }
    ptx::mbar_init(lut_bar, 1);
    ptx::fence_mbar_init();
    if (p.lut_global != nullptr && p.lut_bytes > 0) {
      ptx::mbar_arrive_expect_tx(lut_bar, (uint32_t)p.lut_bytes);
      ptx::bulk_g2s(smem, p.lut_global, (uint32_t)p.lut_bytes, lut_bar);
    } else {
      ptx::mbar_arrive(lut_bar);
    }
  }
  if (p.lut_global == nullptr) lut_fill(smem, st.tiers, st.n_tiers, p.lut_off, threadIdx.x, blockDim.x);
  // L2 prefetch, PF_DIST tiles ahead of the claim order: the tile's code
  // granules (contiguous in the WI layout), its radius row with the
  // page's first tile, and (SPHKV_PF_V) its fp16 V block, so the V bulk
  // copy and the code loads hit L2 and many more bytes are in flight per
  // SM than the smem rings alone could hold.
  auto prefetch_tile = [&](int t, int nt) {
    if (t < nt && lane == 0) {
      const TileEntry tn = tiles[t];
      const int sb = tn.sub_off >> 24;
      const sphkv_page_t pn = st.pages[tn.page];
      const uint64_t W4 = (uint64_t)item_words(d, pn.abits) * 128;  // bytes per granule
      const int g0 = sb * TI / 32, ng = (TI + 31) / 32;
      ptx::bulk_prefetch_l2(st.codes + pn.code_off + g0 * W4, (uint32_t)(ng * W4));
      if (sb == 0) {
        const uint64_t ab = angle_part_bytes(d, P, pn.abits);
        ptx::bulk_prefetch_l2(st.codes + pn.code_off + ab,
                              (uint32_t)(code_block_bytes(d, P, pn.abits, pn.rbits) - ab));
      }
#if SPHKV_PF_V
      ptx::bulk_prefetch_l2(st.values + ((size_t)tn.page * P + (size_t)sb * TI) * dvp, vbytes);
#endif
    }
  };
  // Also independent of the previous grid (it only reads q and writes
  // outputs): the first unit's tile list and its first L2 prefetches.
  // scalars of the fused merge / unit queue live after the barriers (no static
  // __shared__: it would cost a 1 KB-aligned block next to the dynamic region)
  int& s_flag = *reinterpret_cast<int*>(bars + 2 * ADA_NS + 2 * ADA_NV + 1);
  int& s_next = *(reinterpret_cast<int*>(bars + 2 * ADA_NS + 2 * ADA_NV + 1) + 1);
  float* s_ml = reinterpret_cast<float*>(bars + 2 * ADA_NS + 2 * ADA_NV + 2);
  int u = fused_first_unit(p.fz, &s_next);
  if (u < p.n_units && warp == 0) {
    build_tiles_std(st, p.units[u], TI, tiles, ntiles_s, lane, p.fz.ctl_err);
    if (lane == 0) *tile_ctr = 0;
  }
  __syncthreads();
  // V tile producer (lane 0 of the first PV warp): bulk copy of tile k's fp16
  // V block into ring slot (gbase + k) % NV once every PV warp released it
  const uint64_t vpol = ptx::policy_evict_first();
  auto issue_v = [&](int k, uint32_t gb) {
    const uint32_t gk = gb + k;
    const int vs = gk % ADA_NV;
    ptx::mbar_wait(&v_empty[vs], ((gk / ADA_NV) & 1) ^ 1);
    const TileEntry te = tiles[k];
    const int sub = te.sub_off >> 24;
    const uint16_t* src = st.values + ((size_t)te.page * P + (size_t)sub * TI) * dvp;
    ptx::fence_proxy_async();  // order earlier ldmatrix reads of the slot
    ptx::mbar_arrive_expect_tx(&v_full[vs], vbytes);
    ptx::bulk_g2s_hint(vslots + (size_t)vs * vbytes, src, vbytes, &v_full[vs], vpol);
  };
  if (u < p.n_units && warp < ADA_NL)
    for (int t = warp; t < SPHKV_PF_DIST; t += ADA_NL) prefetch_tile(t, *ntiles_s);
  if (u < p.n_units && warp == ADA_NL && lane == 0)
    for (int k = 0; k < *ntiles_s && k < ADA_NV; ++k) issue_v(k, 0u);
  ptx::griddep_wait();  // inputs below (q) may come from the previous grid
#ifdef SPHKV_DBG_TIMING
  if (threadIdx.x == 0 && blockIdx.x < 1024) g_cta_t[2 * blockIdx.x] = gtimer();
#endif
  __syncthreads();
  ptx::griddep_launch_dependents();
  bool lut_ready = false, first = true;

  const float qscale = kLog2e * rsqrtf((float)d);
  uint32_t gbase = 0;  // running tile sequence number (barrier phases)
  for (; u < p.n_units; first = false) {
    const sphkv_unit_t unit = p.units[u];
    if (!first && warp == 0) {
      build_tiles_std(st, unit, TI, tiles, ntiles_s, lane, p.fz.ctl_err);
      if (lane == 0) *tile_ctr = 0;
    }
    // q rows for this group, prescaled into base-2 logit units, packed pairs
    const float* qg = p.q + (size_t)unit.group * p.G * d;
    for (int i = threadIdx.x; i < d * GP; i += blockDim.x) {
      int j = i / GP, g2 = i % GP;
      float a = (2 * g2 < p.G) ? qg[(size_t)(2 * g2) * d + j] * qscale : 0.f;
      float b = (2 * g2 + 1 < p.G) ? qg[(size_t)(2 * g2 + 1) * d + j] * qscale : 0.f;
      qs[j * (q_row_bytes(GP) / 8) + g2] = make_float2(a, b);
    }
    __syncthreads();
    const int nt = *ntiles_s;

    if (warp < ADA_NL) {
      // ---------------- logit warps ----------------
      if (!lut_ready) {
        ptx::mbar_wait(lut_bar, 0);
        lut_ready = true;
      }
      // tiles are claimed dynamically (smem counter) to balance the warps;
      // the P slot of tile k is k % NS whoever computes it.
#pragma unroll 1
      if (!first)
        for (int t = warp; t < SPHKV_PF_DIST; t += ADA_NL) prefetch_tile(t, nt);
      for (;;) {
        int k = 0;
        if (lane == 0) k = atomicAdd(tile_ctr, 1);
        k = __shfl_sync(0xffffffffu, k, 0);
        if (k >= nt) break;
        prefetch_tile(k + SPHKV_PF_DIST, nt);
        const uint32_t gk = gbase + k;
        const TileEntry te = tiles[k];
        const int sub = te.sub_off >> 24, ioff = te.sub_off & 0xffffff;
        const sphkv_page_t pg = st.pages[te.page];
        const int ti = tier_index(st, pg.tier);
        float lg[TK][2 * GP];  // LUT region starts at smem[0]
#ifdef SPHKV_DBG_NOLOGIT  // bottleneck probe: skip the logit math
        for (int a_ = 0; a_ < TK; ++a_)
          for (int b_ = 0; b_ < 2 * GP; ++b_) lg[a_][b_] = (float)(a_ + b_) * 0.01f + (float)ti;
#else
        ada_logit_dispatch<GP, -1>(pg.abits, st.codes, d, P, pg, sub, lane, smem, p.smem_q,
                               p.lut_off[ti], lg);
#endif
        uint32_t valid = 0;
#pragma unroll
        for (int kk = 0; kk < TK; ++kk) {
          const int it = sub * TI + 32 * kk + lane;
          if (32 * kk + lane < TI && it < pg.count) valid |= 1u << kk;
        }
        if (p.logits_dbg != nullptr) {
#pragma unroll
          for (int kk = 0; kk < TK; ++kk) {
            float* dst = p.logits_dbg + (size_t)(p.dbg_off[u] + ioff + 32 * kk + lane) * p.G;
#pragma unroll
            for (int g = 0; g < 2 * GP; ++g)
              if ((valid & (1u << kk)) && g < p.G) dst[g] = lg[kk][g] * (1.0f / kLog2e);
          }
        }
        const int ps = gk % ADA_NS;
        ptx::mbar_wait(&p_empty[ps], ((gk / ADA_NS) & 1) ^ 1);
        write_pslot<2 * GP>(pslots + ps * p.pslot_bytes, p.prow_bytes, p.prows, TI, lane, p.G, lg,
                            valid, p.fz.top2 != nullptr);
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&p_full[ps]);
      }
    } else {
      // ---------------- PV warps ----------------
      // NPV warps split the d_v m-tiles; all consume every tile in order.
      // Lane 0 of PV warp 0 is also the V producer: it refills slot vs once
      // every PV warp has released it (v_empty counts NPV arrivals).
      const int pw = warp - ADA_NL;
      const int mtw = (MT + ADA_NPV - 1) / ADA_NPV;
      const int mt0 = pw * mtw;
      const int mtn = max(0, min(mtw, MT - mt0));
      if (!first && pw == 0 && lane == 0)
        for (int k = 0; k < nt && k < ADA_NV; ++k) issue_v(k, gbase);
      PVState<ADA_MTW> s;
      pv_init(s);
      const bool fast_pv = (dvp == 128 && TI == ADA_TI && mtn == ADA_MTW);
      const bool fast64 = (dvp == 64 && TI == ADA_TI && ADA_NPV == 1);  // c4: +47%
      for (int k = 0; k < nt; ++k) {
        const uint32_t gk = gbase + k;
        const int vs = gk % ADA_NV, ps = gk % ADA_NS;
        ptx::mbar_wait(&v_full[vs], (gk / ADA_NV) & 1);
        ptx::mbar_wait(&p_full[ps], (gk / ADA_NS) & 1);
#ifndef SPHKV_DBG_NOPV  // bottleneck probe: skip the P.V math
        if (fast_pv)
          pv_tile_128<ADA_MTW>(s, pslots + ps * p.pslot_bytes, vslots + (size_t)vs * vbytes,
                               p.prow_bytes, p.prows, mt0, p.G, lane, p.fz.top2 != nullptr);
        else if (fast64)
          pv_tile_128<ADA_MTW, ADA_TI / 16, 64, 4>(s, pslots + ps * p.pslot_bytes,
                                                   vslots + (size_t)vs * vbytes, p.prow_bytes,
                                                   p.prows, 0, p.G, lane, p.fz.top2 != nullptr);
        else
          pv_tile<ADA_MTW>(s, pslots + ps * p.pslot_bytes, vslots + (size_t)vs * vbytes,
                           p.prow_bytes, p.prows, TI, dvp, mt0, mtn, p.G, lane,
                           p.fz.top2 != nullptr);
#endif
        __syncwarp();
        if (lane == 0) {
          ptx::mbar_arrive(&p_empty[ps]);
          ptx::mbar_arrive(&v_empty[vs]);
          if (pw == 0 && k + ADA_NV < nt) issue_v(k + ADA_NV, gbase);
        }
      }
      float* part = p.partials + (size_t)unit.out_slot * ((size_t)p.G * (st.d_v + 2));
      pv_write<ADA_MTW>(s, part, p.G, st.d_v, mt0, mtn, pw == 0, lane,
                        p.fz.top2 != nullptr ? p.fz.top2 + (size_t)unit.out_slot * p.G : nullptr);
    }
    gbase += nt;
    __syncthreads();
    fused_unit_done(p.fz, p.partials, unit.out_slot, p.G, st.d_v, p.n_units, &s_flag, s_ml,
                    &s_next, unit.group);
    u = p.fz.dynamic ? s_next : u + gridDim.x;
  }
  fused_kernel_exit(p.fz);
#ifdef SPHKV_DBG_TIMING
  if (threadIdx.x == 0 && blockIdx.x < 1024) g_cta_t[2 * blockIdx.x + 1] = gtimer();
#endif
}

// ---------------------------------------------------------------------------
// Pipelined unit transitions (opt-in, SPHKV_PIPE=1): the standard body's
// per-unit drain (every warp waits at a block barrier for the slowest logit
// warp's last tile and the PV warp's tail, then the next tile list, q rows,
// prefetches and V copies start cold) made dynamic pieces cost 18-40 us per
// launch (profiles/r2/occupancy).  Here the units of a CTA form one continuous
// tile sequence: logit warps claim from one counter across units and move
// into the next unit without a barrier; the PV warp consumes in order, writes
// each unit's partial, does the group's merge count (and the merge, when
// last) alone, then builds the tile list and q rows of the unit after next
// into the buffers the finished unit frees (double-buffered), and keeps the
// V ring running across the boundary.
// ---------------------------------------------------------------------------
constexpr int PIPE_MAXU = 64;   // units per CTA (unit-info ring; never wraps)
constexpr int PIPE_TILES = 256; // tile-list capacity per buffer (a longer unit is flagged)

// Block-wide merge of group gi's splits into its output rows (the merge half
// of fused_unit_done; the count was won earlier).  All threads call it.
__device__ __noinline__ void merge_group_block(const int32_t* slot_begin, int32_t* ctl, float* out,
                                               const float* partials, int gi, int G, int d_v,
                                               float* s_ml) {
  __threadfence();
  const int b = slot_begin[gi], e = slot_begin[gi + 1];
  const int64_t stride = (int64_t)G * (d_v + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int g = warp; g < G; g += nw) {
    float M = -INFINITY;
    for (int s = b + lane; s < e; s += 32) M = fmaxf(M, __ldcg(partials + s * stride + g));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    float L = 0.f;
    for (int s = b + lane; s < e; s += 32) {
      const float m = __ldcg(partials + s * stride + g);
      const float l = __ldcg(partials + s * stride + G + g);
      L += (m != -INFINITY) ? l * exp2f(m - M) : 0.f;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
    if (lane == 0) {
      s_ml[g] = M;
      s_ml[8 + g] = L;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G * d_v; i += blockDim.x) {
    const int g = i / d_v, j = i % d_v;
    const float M = s_ml[g], L = s_ml[8 + g];
    float a = 0.f;
#pragma unroll 8
    for (int s = b; s < e; ++s) {
      const float m = __ldcg(partials + s * stride + g);
      const float v = __ldcg(partials + s * stride + 2 * G + (int64_t)g * d_v + j);
      a += (m != -INFINITY) ? v * exp2f(m - M) : 0.f;
    }
    out[((int64_t)gi * G + g) * d_v + j] = (L > 0.f) ? a / L : 0.f;
  }
  if (threadIdx.x == 0) ctl[gi] = 0;  // every split of gi has counted: re-arm
  __syncthreads();
}

template <int GP>
__global__ void __launch_bounds__(ADA_THREADS, 1) k_ada_decode_pipe(const AdaParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const sphkv_store_t& st = p.st;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  TileEntry* tl0 = reinterpret_cast<TileEntry*>(smem + p.smem_tiles);
  TileEntry* tl1 = reinterpret_cast<TileEntry*>(smem + p.smem_tiles2);
  int4* info = reinterpret_cast<int4*>(smem + p.smem_info);  // {base, nt (<0: end), unit, 0}
  int* ctr = reinterpret_cast<int*>(info + PIPE_MAXU);       // [0] tile claims, [1] units built,
                                                             // [2] deferred merges
  int* mlist = ctr + 4;                                      // [PIPE_MAXU] groups to merge
  uint8_t* pslots = smem + p.smem_p;
  uint8_t* vslots = smem + p.smem_v;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.smem_bar);
  uint64_t* p_full = bars;
  uint64_t* p_empty = bars + ADA_NS;
  uint64_t* v_full = bars + 2 * ADA_NS;
  uint64_t* v_empty = bars + 2 * ADA_NS + ADA_NV;
  uint64_t* lut_bar = bars + 2 * ADA_NS + 2 * ADA_NV;
  const int d = st.d, P = st.page_size, TI = p.TI, dvp = p.dvp, MT = dvp / 16;
  const uint32_t vbytes = (uint32_t)TI * dvp * 2;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ADA_NS; ++i) {
      ptx::mbar_init(&p_full[i], 1);
      ptx::mbar_init(&p_empty[i], ADA_NPV);
    }
    for (int i = 0; i < ADA_NV; ++i) {
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&v_empty[i], ADA_NPV);
    }
    ptx::mbar_init(lut_bar, 1);
    ptx::fence_mbar_init();
    if (p.lut_global != nullptr && p.lut_bytes > 0) {
      ptx::mbar_arrive_expect_tx(lut_bar, (uint32_t)p.lut_bytes);
      ptx::bulk_g2s(smem, p.lut_global, (uint32_t)p.lut_bytes, lut_bar);
    } else {
      ptx::mbar_arrive(lut_bar);
    }
    ctr[0] = 0;
    ctr[1] = 0;
    ctr[2] = 0;
  }
  if (p.lut_global == nullptr) lut_fill(smem, st.tiers, st.n_tiers, p.lut_off, threadIdx.x, blockDim.x);
  auto prefetch_tile = [&](const TileEntry* tl, int t, int nt) {
    if (t < nt) {
      const TileEntry tn = tl[t];
      const int sb = tn.sub_off >> 24;
      const sphkv_page_t pn = st.pages[tn.page];
      const uint64_t W4 = (uint64_t)item_words(d, pn.abits) * 128;
      const int g0 = sb * TI / 32, ng = (TI + 31) / 32;
      ptx::bulk_prefetch_l2(st.codes + pn.code_off + g0 * W4, (uint32_t)(ng * W4));
      if (sb == 0) {
        const uint64_t ab = angle_part_bytes(d, P, pn.abits);
        ptx::bulk_prefetch_l2(st.codes + pn.code_off + ab,
                              (uint32_t)(code_block_bytes(d, P, pn.abits, pn.rbits) - ab));
      }
    }
  };
  const float qscale = kLog2e * rsqrtf((float)d);
  __syncthreads();  // barriers + counters initialised

  if (warp < ADA_NL) {
    // ---------------- logit warps ----------------
    ptx::griddep_wait();
    ptx::griddep_launch_dependents();
    ptx::mbar_wait(lut_bar, 0);
    int j = -1, ubase = 0, unt = 0;
    const TileEntry* tl = tl0;
    uint32_t qoff = p.smem_q;
    for (;;) {
      int k = 0;
      if (lane == 0) k = atomicAdd(&ctr[0], 1);
      k = __shfl_sync(0xffffffffu, k, 0);
      bool end = false;
      while (j < 0 || k >= ubase + unt) {  // move to the unit holding tile k
        ++j;
        if (lane == 0)
          while (*reinterpret_cast<volatile int*>(&ctr[1]) <= j) __nanosleep(64);
        __syncwarp();
        __threadfence_block();
        const volatile int4* vin = &info[j];
        const int4 in = make_int4(vin->x, vin->y, vin->z, vin->w);
        if (in.y < 0) {
          end = true;
          break;
        }
        ubase = in.x;
        unt = in.y;
        tl = (j & 1) ? tl1 : tl0;
        qoff = (j & 1) ? p.smem_q2 : p.smem_q;
      }
      if (end) break;
      const int kl = k - ubase;
      if (lane == 0) prefetch_tile(tl, kl + SPHKV_PF_DIST, unt);
      const TileEntry te = tl[kl];
      const int sub = te.sub_off >> 24;
      const sphkv_page_t pg = st.pages[te.page];
      const int ti = tier_index(st, pg.tier);
      float lg[TK][2 * GP];
      ada_logit_dispatch<GP, -1>(pg.abits, st.codes, d, P, pg, sub, lane, smem, qoff,
                                 p.lut_off[ti], lg);
      uint32_t valid = 0;
#pragma unroll
      for (int kk = 0; kk < TK; ++kk) {
        const int it = sub * TI + 32 * kk + lane;
        if (32 * kk + lane < TI && it < pg.count) valid |= 1u << kk;
      }
      const uint32_t gk = (uint32_t)k;
      const int ps = gk % ADA_NS;
      ptx::mbar_wait(&p_empty[ps], ((gk / ADA_NS) & 1) ^ 1);
      write_pslot<2 * GP>(pslots + ps * p.pslot_bytes, p.prow_bytes, p.prows, TI, lane, p.G, lg,
                          valid, false);
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&p_full[ps]);
    }
  } else {
    // ---------------- PV warp: consumer, unit builder, V producer ----------------
    const uint64_t vpol = ptx::policy_evict_first();
    int nbuilt = 0, tiles_built = 0;  // units built, tiles of the built units
    int last_unit = -1;               // unit id of the last unit built (static stepping)
    bool ended = false;
    // build local unit `jj` (ordinal) = unit id `u` (< 0: end) into buffer jj & 1
    auto build = [&](int u, bool load_q) {
      const int jj = nbuilt;
      if (u < 0 || u >= p.n_units || jj >= PIPE_MAXU - 1) {
        if (lane == 0) info[jj] = make_int4(tiles_built, -1, -1, 0);
        ended = true;
      } else {
        TileEntry* tl = (jj & 1) ? tl1 : tl0;
        int* nts = reinterpret_cast<int*>(tl + PIPE_TILES);
        int nt = build_tiles_std(st, p.units[u], TI, tl, nts, lane, p.fz.ctl_err, PIPE_TILES);
        nt = nt < PIPE_TILES ? nt : PIPE_TILES;
        if (load_q) {
          float2* qs = reinterpret_cast<float2*>(smem + ((jj & 1) ? p.smem_q2 : p.smem_q));
          const float* qg = p.q + (size_t)p.units[u].group * p.G * d;
          for (int i = lane; i < d * GP; i += 32) {
            const int jr = i / GP, g2 = i % GP;
            const float a = (2 * g2 < p.G) ? qg[(size_t)(2 * g2) * d + jr] * qscale : 0.f;
            const float b = (2 * g2 + 1 < p.G) ? qg[(size_t)(2 * g2 + 1) * d + jr] * qscale : 0.f;
            qs[jr * (q_row_bytes(GP) / 8) + g2] = make_float2(a, b);
          }
        }
        __syncwarp();
        if (lane < SPHKV_PF_DIST) prefetch_tile(tl, lane, nt);
        if (lane == 0) info[jj] = make_int4(tiles_built, nt, u, 0);
        tiles_built += nt;
        last_unit = u;
      }
      __syncwarp();
      __threadfence_block();
      if (lane == 0) *reinterpret_cast<volatile int*>(&ctr[1]) = jj + 1;
      ++nbuilt;
    };
    auto next_unit = [&]() -> int {
      if (ended) return -1;
      int u = 0;
      if (p.fz.dynamic) {
        if (lane == 0) u = atomicAdd(&p.fz.ctl[p.fz.n_groups], 1) + (int)gridDim.x;
        u = __shfl_sync(0xffffffffu, u, 0);
      } else {
        u = last_unit + (int)gridDim.x;
      }
      return u;
    };
    // V copy of sequence number s (its unit is built: s < tiles_built); the
    // unit cursor (vj, vb, ve) only moves forward (lane 0's registers)
    int vj = 0, vb = 0, ve = 0;
    auto issue_v = [&](uint32_t s) {
      while ((int)s >= ve) {
        const int4 in = info[++vj];
        vb = in.x;
        ve = in.x + (in.y > 0 ? in.y : 0);
      }
      const TileEntry* tl = (vj & 1) ? tl1 : tl0;
      const TileEntry te = tl[s - vb];
      const int sub = te.sub_off >> 24;
      const int vs = s % ADA_NV;
      ptx::mbar_wait(&v_empty[vs], ((s / ADA_NV) & 1) ^ 1);
      const uint16_t* src = st.values + ((size_t)te.page * P + (size_t)sub * TI) * dvp;
      ptx::fence_proxy_async();
      ptx::mbar_arrive_expect_tx(&v_full[vs], vbytes);
      ptx::bulk_g2s_hint(vslots + (size_t)vs * vbytes, src, vbytes, &v_full[vs], vpol);
    };
    uint32_t v_next = 0;
    // prologue: unit 0 (static: blockIdx.x) tile list + V copies before the
    // wait; its q rows, the second unit and the claims after it
    {
      const int u0 = (int)blockIdx.x;
      if (u0 < p.n_units) {
        TileEntry* tl = tl0;
        int* nts = reinterpret_cast<int*>(tl + PIPE_TILES);
        int nt = build_tiles_std(st, p.units[u0], TI, tl, nts, lane, p.fz.ctl_err, PIPE_TILES);
        nt = nt < PIPE_TILES ? nt : PIPE_TILES;
        __syncwarp();
        if (lane < SPHKV_PF_DIST) prefetch_tile(tl, lane, nt);
        if (lane == 0) {
          info[0] = make_int4(0, nt, u0, 0);
          for (; v_next < (uint32_t)nt && v_next < (uint32_t)ADA_NV; ++v_next) {
            const TileEntry te = tl[v_next];
            const int vs = v_next % ADA_NV;
            const uint16_t* src = st.values + ((size_t)te.page * P + (size_t)(te.sub_off >> 24) * TI) * dvp;
            ptx::mbar_arrive_expect_tx(&v_full[vs], vbytes);
            ptx::bulk_g2s_hint(vslots + (size_t)vs * vbytes, src, vbytes, &v_full[vs], vpol);
          }
        }
        tiles_built = nt;
        last_unit = u0;
        ve = nt;
      }
      ptx::griddep_wait();
#ifdef SPHKV_DBG_TIMING
      if (lane == 0 && blockIdx.x < 1024) g_cta_t[2 * blockIdx.x] = gtimer();
#endif
      if (u0 < p.n_units) {
        float2* qs = reinterpret_cast<float2*>(smem + p.smem_q);
        const float* qg = p.q + (size_t)p.units[u0].group * p.G * d;
        for (int i = lane; i < d * GP; i += 32) {
          const int jr = i / GP, g2 = i % GP;
          const float a = (2 * g2 < p.G) ? qg[(size_t)(2 * g2) * d + jr] * qscale : 0.f;
          const float b = (2 * g2 + 1 < p.G) ? qg[(size_t)(2 * g2 + 1) * d + jr] * qscale : 0.f;
          qs[jr * (q_row_bytes(GP) / 8) + g2] = make_float2(a, b);
        }
        __syncwarp();
        __threadfence_block();
        if (lane == 0) *reinterpret_cast<volatile int*>(&ctr[1]) = 1;
        nbuilt = 1;
        build(next_unit(), true);
      } else {
        build(-1, false);
      }
    }
    ptx::griddep_launch_dependents();
    PVState<ADA_MTW> s;
    const bool fast_pv = (dvp == 128 && TI == ADA_TI && MT == ADA_MTW);
    const bool fast64 = (dvp == 64 && TI == ADA_TI);
    for (int j = 0;; ++j) {
      const int4 in = info[j];
      if (in.y < 0) break;
      pv_init(s);
      for (int k = 0; k < in.y; ++k) {
        const uint32_t gk = (uint32_t)(in.x + k);
        const int vs = gk % ADA_NV, ps = gk % ADA_NS;
        ptx::mbar_wait(&v_full[vs], (gk / ADA_NV) & 1);
        ptx::mbar_wait(&p_full[ps], (gk / ADA_NS) & 1);
        if (fast_pv)
          pv_tile_128<ADA_MTW>(s, pslots + ps * p.pslot_bytes, vslots + (size_t)vs * vbytes,
                               p.prow_bytes, p.prows, 0, p.G, lane, false);
        else if (fast64)
          pv_tile_128<ADA_MTW, ADA_TI / 16, 64, 4>(s, pslots + ps * p.pslot_bytes,
                                                   vslots + (size_t)vs * vbytes, p.prow_bytes,
                                                   p.prows, 0, p.G, lane, false);
        else
          pv_tile<ADA_MTW>(s, pslots + ps * p.pslot_bytes, vslots + (size_t)vs * vbytes,
                           p.prow_bytes, p.prows, TI, dvp, 0, MT, p.G, lane, false);
        __syncwarp();
        if (lane == 0) {
          ptx::mbar_arrive(&p_empty[ps]);
          ptx::mbar_arrive(&v_empty[vs]);
          for (; v_next < gk + 1 + ADA_NV && v_next < (uint32_t)tiles_built; ++v_next) issue_v(v_next);
        }
        __syncwarp();
      }
      const sphkv_unit_t unit = p.units[in.z];
      float* part = p.partials + (size_t)unit.out_slot * ((size_t)p.G * (st.d_v + 2));
      pv_write<ADA_MTW>(s, part, p.G, st.d_v, 0, MT, true, lane, nullptr);
      // merge count; the last split of a group defers the (block-wide) merge
      // to the CTA's end
      if (p.fz.slot_group != nullptr) {
        __threadfence();
        __syncwarp();
        const int gi = p.fz.slot_group[unit.out_slot];
        if (lane == 0 && gi >= 0) {
          const int ns = p.fz.slot_begin[gi + 1] - p.fz.slot_begin[gi];
          if (atomicAdd(&p.fz.ctl[gi], 1) == ns - 1) mlist[ctr[2]++] = gi;
        }
      }
      // the buffers of unit j are free: build unit j + 2
      if (!ended) build(next_unit(), true);
      if (lane == 0)
        for (; v_next < (uint32_t)(in.x + in.y) + ADA_NV && v_next < (uint32_t)tiles_built; ++v_next)
          issue_v(v_next);
      __syncwarp();
    }
    if (p.fz.dynamic && lane == 0) {
      __threadfence();
      if (atomicAdd(&p.fz.ctl[p.fz.n_groups + 1], 1) == (int)gridDim.x - 1) {
        p.fz.ctl[p.fz.n_groups] = 0;
        p.fz.ctl[p.fz.n_groups + 1] = 0;
      }
    }
  }
  __syncthreads();
  {
    float* s_ml = reinterpret_cast<float*>(bars + 2 * ADA_NS + 2 * ADA_NV + 2);
    const int nm = ctr[2];
    for (int i = 0; i < nm; ++i)
      merge_group_block(p.fz.slot_begin, p.fz.ctl, p.fz.out, p.partials, mlist[i], p.G, st.d_v, s_ml);
  }
#ifdef SPHKV_DBG_TIMING
  if (threadIdx.x == 0 && blockIdx.x < 1024) g_cta_t[2 * blockIdx.x + 1] = gtimer();
#endif
}

// ---------------------------------------------------------------------------
// Dense bf16 paged decode (baseline), same unit / partial contract
// ---------------------------------------------------------------------------
constexpr int DN_NL = 4;
constexpr int DN_TI = 64;
#ifndef SPHKV_DN_NK
#define SPHKV_DN_NK 8
#endif
#ifndef SPHKV_DN_NV
#define SPHKV_DN_NV 4
#endif
constexpr int DN_NK = SPHKV_DN_NK;  // K ring slots (64-item tiles)
constexpr int DN_NV = SPHKV_DN_NV;  // V ring slots
constexpr int DN_NS = 8;
// Two launch shapes (dense_threads): d_v = 128 runs two PV warps (each half
// of the d_v m-tiles) and separate K and V producer warps -- a single
// producer blocked on a full V ring starved the logit warps of K (c5:
// 0.77 -> 0.84 of the copy peak); narrower values keep one PV warp and one
// producer, which measured faster there (c4, d_v = 64).
__host__ __device__ constexpr int dense_threads(int npv, bool sep) {
  return (DN_NL + npv + (sep ? 2 : 1)) * 32;
}

struct DenseParams {
  sphkv_dense_store_t st;
  const float* q;
  int G;
  const sphkv_unit_t* units;
  int n_units;
  float* partials;
  int dp, dvp;            // padded key / value widths
  int tok_lo;             // first attended token (sliding window); 0 = all
  uint32_t smem_k, smem_v, smem_p, smem_bar;
  int pslot_bytes, prow_bytes;
  FusedCtl fz;
};

// DVF: 128 / 64 = the unrolled P.V path for that padded d_v, 0 = generic
template <int NPV, bool SEP, int DVF>
__global__ void __launch_bounds__(dense_threads(NPV, SEP), 1) k_dense_decode(const DenseParams p) {
  constexpr int MTW = 8 / NPV;
  extern __shared__ __align__(128) uint8_t smem[];
  const sphkv_dense_store_t& st = p.st;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* kslots = smem + p.smem_k;
  uint8_t* vslots = smem + p.smem_v;
  uint8_t* pslots = smem + p.smem_p;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.smem_bar);
  uint64_t* k_full = bars;
  uint64_t* k_empty = bars + DN_NK;
  uint64_t* v_full = bars + 2 * DN_NK;
  uint64_t* v_empty = v_full + DN_NV;
  uint64_t* p_full = v_empty + DN_NV;
  uint64_t* p_empty = p_full + DN_NS;
  const int P = st.page_size, dp = p.dp, dvp = p.dvp, MT = dvp / 16, KT = dp / 16;
  const uint32_t kbytes = (uint32_t)DN_TI * dp * 2, vbytes = (uint32_t)DN_TI * dvp * 2;
  const int tiles_per_page = P / DN_TI;

  if (threadIdx.x == 0) {
    for (int i = 0; i < DN_NK; ++i) { ptx::mbar_init(&k_full[i], 1); ptx::mbar_init(&k_empty[i], 1); }
    for (int i = 0; i < DN_NV; ++i) { ptx::mbar_init(&v_full[i], 1); ptx::mbar_init(&v_empty[i], NPV); }
    for (int i = 0; i < DN_NS; ++i) { ptx::mbar_init(&p_full[i], 1); ptx::mbar_init(&p_empty[i], NPV); }
    ptx::fence_mbar_init();
  }
  ptx::griddep_wait();  // same PDL contract as the ADA kernel
  __syncthreads();
  ptx::griddep_launch_dependents();
  const float qscale = kLog2e * rsqrtf((float)st.d);
  __shared__ int s_flag, s_next;
  __shared__ float s_ml[16];
  uint32_t gbase = 0;
  for (int u = fused_first_unit(p.fz, &s_next); u < p.n_units;) {
    const sphkv_unit_t unit = p.units[u];
    const int t_begin = max(unit.ptr_begin * tiles_per_page, p.tok_lo / DN_TI);
    int t_end = unit.ptr_end * tiles_per_page;
    const int t_max = (st.tokens + DN_TI - 1) / DN_TI;
    if (t_end > t_max) t_end = t_max;
    const int nt = t_end > t_begin ? t_end - t_begin : 0;
    const size_t gpage0 = (size_t)unit.group * st.n_pages_per_group;

    if (warp < DN_NL) {
      // q^T B-fragments in registers (bf16), g = lane / 4
      uint32_t qb[8][2];
      {
        const int g = lane >> 2;
        const float* qg = p.q + ((size_t)unit.group * p.G + g) * st.d;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            int j = kk * 16 + h * 8 + 2 * (lane & 3);
            float a = (g < p.G && j < st.d) ? qg[j] * qscale : 0.f;
            float b = (g < p.G && j + 1 < st.d) ? qg[j + 1] * qscale : 0.f;
            __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
            qb[kk][h] = *reinterpret_cast<uint32_t*>(&v);
          }
        }
      }
      const int nchunks = dp / 8, smask = (nchunks < 8 ? nchunks : 8) - 1;
      for (int k = warp; k < nt; k += DN_NL) {
        const uint32_t gk = gbase + k;
        const int ks = gk % DN_NK, ps = gk % DN_NS;
        ptx::mbar_wait(&k_full[ks], (gk / DN_NK) & 1);
        const uint32_t kb = ptx::smem_u32(kslots + (size_t)ks * kbytes);
        float c[DN_TI / 16][4];
#pragma unroll
        for (int mi = 0; mi < DN_TI / 16; ++mi) {
#pragma unroll
          for (int r = 0; r < 4; ++r) c[mi][r] = 0.f;
          const int item = mi * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            if (kk < KT) {
              int chunk = 2 * kk + (lane >> 4);
              int sw = chunk ^ (item & smask);
              uint32_t a0, a1, a2, a3;
              ptx::ldsm_x4(kb + (item * dp + sw * 8) * 2, a0, a1, a2, a3);
              ptx::mma_bf16(c[mi], a0, a1, a2, a3, qb[kk][0], qb[kk][1]);
            }
          }
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&k_empty[ks]);
        // softmax over the tile per head column
        const int tok0 = (t_begin + k) * DN_TI;
        uint8_t* slot = pslots + ps * p.pslot_bytes;
        ptx::mbar_wait(&p_empty[ps], ((gk / DN_NS) & 1) ^ 1);
        float* hdr = reinterpret_cast<float*>(slot + 8 * p.prow_bytes);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int g = 2 * (lane & 3) + h;
          float m = -INFINITY;
#pragma unroll
          for (int mi = 0; mi < DN_TI / 16; ++mi) {
            int i0 = mi * 16 + (lane >> 2);
            if (tok0 + i0 < st.tokens && tok0 + i0 >= p.tok_lo) m = fmaxf(m, c[mi][h]);
            if (tok0 + i0 + 8 < st.tokens && tok0 + i0 + 8 >= p.tok_lo) m = fmaxf(m, c[mi][2 + h]);
          }
          m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 4));
          m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 8));
          m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 16));
          float s = 0.f;
#pragma unroll
          for (int mi = 0; mi < DN_TI / 16; ++mi) {
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
              int i0 = mi * 16 + (lane >> 2) + rr * 8;
              float e = (tok0 + i0 < st.tokens && tok0 + i0 >= p.tok_lo)
                            ? exp2f(c[mi][2 * rr + h] - m) : 0.f;
              __half hv = __float2half_rn(e);
              s += __half2float(hv);
              if (g < p.G) *reinterpret_cast<__half*>(slot + g * p.prow_bytes + i0 * 2) = hv;
            }
          }
          s += __shfl_xor_sync(0xffffffffu, s, 4);
          s += __shfl_xor_sync(0xffffffffu, s, 8);
          s += __shfl_xor_sync(0xffffffffu, s, 16);
          if ((lane >> 2) == 0) {
            hdr[g] = m;
            hdr[8 + g] = s;
          }
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&p_full[ps]);
      }
    } else if (warp < DN_NL + NPV) {
      // NPV warps split the d_v m-tiles; each consumes every tile
      const int pw = warp - DN_NL;
      const int mt0 = NPV == 1 ? 0 : pw * MTW;  // compile-time 0 with one PV warp
      const int mtn = max(0, min(MTW, MT - mt0));
      PVState<MTW> s;
      pv_init(s);
      for (int k = 0; k < nt; ++k) {
        const uint32_t gk = gbase + k;
        const int vs = gk % DN_NV, ps = gk % DN_NS;
        ptx::mbar_wait(&v_full[vs], (gk / DN_NV) & 1);
        ptx::mbar_wait(&p_full[ps], (gk / DN_NS) & 1);
        if constexpr (DVF == 128)
          pv_tile_128<MTW, DN_TI / 16>(s, pslots + ps * p.pslot_bytes,
                                          vslots + (size_t)vs * vbytes, p.prow_bytes, 8, mt0,
                                          p.G, lane);
        else if constexpr (DVF == 64 && NPV == 1)
          pv_tile_128<MTW, DN_TI / 16, 64, 4>(s, pslots + ps * p.pslot_bytes,
                                              vslots + (size_t)vs * vbytes, p.prow_bytes, 8, 0,
                                              p.G, lane);
        else
          pv_tile<MTW>(s, pslots + ps * p.pslot_bytes, vslots + (size_t)vs * vbytes,
                          p.prow_bytes, 8, DN_TI, dvp, mt0, mtn, p.G, lane);
        __syncwarp();
        if (lane == 0) {
          ptx::mbar_arrive(&p_empty[ps]);
          ptx::mbar_arrive(&v_empty[vs]);
        }
      }
      float* part = p.partials + (size_t)unit.out_slot * ((size_t)p.G * (st.d_v + 2));
      pv_write<MTW>(s, part, p.G, st.d_v, mt0, mtn, pw == 0, lane);
    } else if (!SEP) {
      if (lane == 0) {
        for (int k = 0; k < nt; ++k) {
          const uint32_t gk = gbase + k;
          const int ks = gk % DN_NK, vs = gk % DN_NV;
          const size_t item0 = gpage0 * P + (size_t)(t_begin + k) * DN_TI;
          ptx::mbar_wait(&k_empty[ks], ((gk / DN_NK) & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(&k_full[ks], kbytes);
          ptx::bulk_g2s(kslots + (size_t)ks * kbytes, st.keys + item0 * dp, kbytes, &k_full[ks]);
          ptx::mbar_wait(&v_empty[vs], ((gk / DN_NV) & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(&v_full[vs], vbytes);
          ptx::bulk_g2s(vslots + (size_t)vs * vbytes, st.values + item0 * dvp, vbytes, &v_full[vs]);
        }
      }
    } else if (lane == 0 && warp == DN_NL + NPV) {  // K producer
      for (int k = 0; k < nt; ++k) {
        const uint32_t gk = gbase + k;
        const int ks = gk % DN_NK;
        const size_t item0 = gpage0 * P + (size_t)(t_begin + k) * DN_TI;
        ptx::mbar_wait(&k_empty[ks], ((gk / DN_NK) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&k_full[ks], kbytes);
        ptx::bulk_g2s(kslots + (size_t)ks * kbytes, st.keys + item0 * dp, kbytes, &k_full[ks]);
      }
    } else if (lane == 0) {  // V producer
      for (int k = 0; k < nt; ++k) {
        const uint32_t gk = gbase + k;
        const int vs = gk % DN_NV;
        const size_t item0 = gpage0 * P + (size_t)(t_begin + k) * DN_TI;
        ptx::mbar_wait(&v_empty[vs], ((gk / DN_NV) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&v_full[vs], vbytes);
        ptx::bulk_g2s(vslots + (size_t)vs * vbytes, st.values + item0 * dvp, vbytes, &v_full[vs]);
      }
    }
    gbase += nt;
    __syncthreads();
    fused_unit_done(p.fz, p.partials, unit.out_slot, p.G, st.d_v, p.n_units, &s_flag, s_ml,
                    &s_next);
    u = p.fz.dynamic ? s_next : u + gridDim.x;
  }
  fused_kernel_exit(p.fz);
}

// ---------------------------------------------------------------------------
// LSE merge
// ---------------------------------------------------------------------------
// Group grp's splits: slots [sb[grp], sb[grp+1]) when sb is given, else the
// rank-major layout of an all-gather, slot = grp + s * split_stride for
// s < n_splits.  state_out = 0: normalized output rows [n_groups*G][d_v];
// state_out = 1: one partial slot per group (m = log2-sum-exp, l = 1,
// acc = normalized output; an all-empty group stays m = -inf, l = 0, acc = 0),
// which is again a valid split state for the next merge level.
__global__ void k_lse_merge(const float* __restrict__ partials, const int32_t* __restrict__ sb,
                            int n_splits, int64_t split_stride, int n_groups, int G, int d_v,
                            float* __restrict__ out, int state_out) {
  const int gid = blockIdx.x;  // group * G + g
  if (gid >= n_groups * G) return;
  const int grp = gid / G, g = gid % G;
  int64_t b, step;
  int cnt;
  if (sb != nullptr) {
    b = sb[grp];
    cnt = sb[grp + 1] - sb[grp];
    step = 1;
  } else {
    b = grp;
    cnt = n_splits;
    step = split_stride;
  }
  const int64_t stride = (int64_t)G * (d_v + 2);
  float M = -INFINITY;
  for (int s = 0; s < cnt; ++s) M = fmaxf(M, partials[(b + s * step) * stride + g]);
  float L = 0.f;
  for (int s = 0; s < cnt; ++s) {
    const float* ps = partials + (b + s * step) * stride;
    float m = ps[g];
    if (m != -INFINITY) L += ps[G + g] * exp2f(m - M);
  }
  float* o = state_out ? out + (int64_t)grp * stride + 2 * G + (int64_t)g * d_v
                       : out + (int64_t)gid * d_v;
  for (int j = threadIdx.x; j < d_v; j += blockDim.x) {
    float a = 0.f;
    for (int s = 0; s < cnt; ++s) {
      const float* ps = partials + (b + s * step) * stride;
      float m = ps[g];
      if (m != -INFINITY) a += ps[2 * G + (int64_t)g * d_v + j] * exp2f(m - M);
    }
    o[j] = (L > 0.f) ? a / L : 0.f;
  }
  if (state_out && threadIdx.x == 0) {
    float* st = out + (int64_t)grp * stride;
    st[g] = (L > 0.f) ? M + log2f(L) : -INFINITY;
    st[G + g] = (L > 0.f) ? 1.f : 0.f;
  }
}

}  // namespace sphkv

using namespace sphkv;

// ---------------------------------------------------------------------------
// host entry points
// ---------------------------------------------------------------------------
static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

extern "C" int64_t sphkv_partial_floats(int G, int d_v) { return (int64_t)G * (d_v + 2); }

// Shared memory of a GP <= 2 launch besides the LUT and the h-byte tables
// (q rows, tile list, P slots, V ring, barriers), rounded up.
static size_t ada_other_smem(int d, int d_v, int P) {
  const int TI = P < ADA_TI ? P : ADA_TI;
  const size_t dvp = (size_t)(d_v + 15) / 16 * 16;
  const size_t prow = (size_t)TI * 2 + PROW_PAD;
  return (size_t)d * q_row_bytes(2) + MAX_UNIT_TILES * sizeof(TileEntry) + 16 +
         ADA_NS * ((4 * prow + 96 + 15) / 16 * 16) + ADA_NV * TI * dvp * 2 + 1024 + 4 * 128;
}

// Does this launch decode the 2-bit tier through the h-byte tables?  The
// caller opts in per store (lut_flags bit 0, with the matching prebuilt LUT);
// launches outside the mode's limits (G > 4, other d, narrow pages) use the
// quad-row table (in-kernel LUT fill if the prebuilt one is the h-byte layout).
static bool ada_use_hb(const sphkv_store_t* st, int GP) {
#ifdef SPHKV_NO_HB  // experiment builds: the 2-bit tier through the quad-row table
  return false;
#endif
  if (!(st->lut_flags & 1)) return false;
  if (GP > 2 || !hb_supported(st->d) || st->page_size % ADA_TI != 0) return false;
  for (int t = 1; t < st->n_tiers; ++t)
    if (st->tiers[t].angle_bits == 2) return true;
  return false;
}

// LUT placement for a launch mode: the h-byte mode drops the 2-bit table and
// gives the LUT what the h-byte tables leave of the opt-in shared memory.
static int lut_layout(const sphkv_store_t* st, int off[SPHKV_MAX_TIERS], int hb) {
  int budget = 0;
  if (hb) {
    const long left = 232448L - (long)hb_bytes(st->d) - (long)ada_other_smem(st->d, st->d_v,
                                                                             st->page_size);
    budget = (int)(left < LUT_BUDGET_BYTES ? (left / 16) * 16 : LUT_BUDGET_BYTES);
    if (budget < 16) budget = 16;
  }
  return lut_layout_tiers(st->tiers, st->n_tiers, off, st->lut_items, hb, budget);
}

namespace sphkv {
__global__ void k_build_lut(sphkv_store_t st) {
  lut_fill(reinterpret_cast<uint8_t*>(st.lut), st.tiers, st.n_tiers, st.lut_off,
           blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}
}  // namespace sphkv

extern "C" int sphkv_ada_tile_items(void) { return ADA_TI; }
extern "C" int sphkv_unit_tile_cap(void) { return MAX_UNIT_TILES; }

extern "C" int64_t sphkv_lut_floats(const sphkv_store_t* st) {
  int off[SPHKV_MAX_TIERS];
  return lut_layout(st, off, st->lut_flags & 1) / 4 + 4;
}

extern "C" int sphkv_store_build_lut(sphkv_store_t* st, cudaStream_t stream) {
  if (!st || !st->lut) return fail(SPHKV_E_VALUE, "store lut buffer missing");
  int used = lut_layout(st, st->lut_off, st->lut_flags & 1);
  if (used == 0) return SPHKV_OK;
  k_build_lut<<<64, 256, 0, stream>>>(*st);
  SPHKV_LAUNCH_CHECK();
  return SPHKV_OK;
}

// Launch with programmatic stream serialization (PDL): the kernel's
// prologue may start while the previous grid on the stream drains; it waits
// (griddepcontrol.wait) before touching any input.
template <typename Kern, typename Params>
static int launch_pdl(Kern kern, const Params& p, int grid, int threads, size_t smem,
                      cudaStream_t stream, bool pdl = true) {
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  SPHKV_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, p));
  SPHKV_LAUNCH_CHECK();
  return SPHKV_OK;
}

template <int GP, int DK>
static int launch_ada_dk(AdaParams& p, size_t smem, int grid, cudaStream_t stream, bool pdl) {
  auto kern = k_ada_decode<GP, DK>;
  cudaFuncAttributes fa;
  SPHKV_CUDA_TRY(cudaFuncGetAttributes(&fa, kern));
  int dev = 0, optin = 0;
  SPHKV_CUDA_TRY(cudaGetDevice(&dev));
  SPHKV_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  if (smem + fa.sharedSizeBytes > (size_t)optin)
    return fail(SPHKV_E_UNSUPPORTED, "ADA decode needs %zu B shared memory (+%zu static) > %d",
                smem, (size_t)fa.sharedSizeBytes, optin);
  SPHKV_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  return launch_pdl(kern, p, grid, ADA_THREADS, smem, stream, pdl);
}

template <int GP>
static int launch_ada_std(AdaParams& p, size_t smem, int grid, cudaStream_t stream, bool pdl) {
  auto kern = k_ada_decode_std<GP>;
  cudaFuncAttributes fa;
  SPHKV_CUDA_TRY(cudaFuncGetAttributes(&fa, kern));
  int dev = 0, optin = 0;
  SPHKV_CUDA_TRY(cudaGetDevice(&dev));
  SPHKV_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  if (smem + fa.sharedSizeBytes > (size_t)optin)
    return fail(SPHKV_E_UNSUPPORTED, "ADA decode needs %zu B shared memory (+%zu static) > %d",
                smem, (size_t)fa.sharedSizeBytes, optin);
  SPHKV_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  return launch_pdl(kern, p, grid, ADA_THREADS, smem, stream, pdl);
}

template <int GP>
static int launch_ada_pipe(AdaParams& p, size_t smem, int grid, cudaStream_t stream, bool pdl) {
  auto kern = k_ada_decode_pipe<GP>;
  SPHKV_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  return launch_pdl(kern, p, grid, ADA_THREADS, smem, stream, pdl);
}

template <int GP>
static int launch_ada(AdaParams& p, size_t smem, int grid, cudaStream_t stream, bool pdl) {
  if (p.pipe) return launch_ada_pipe<GP>(p, smem, grid, stream, pdl);
  // the fused path (outputs, gate margins, absolute rows, live units) runs the
  // round-1 kernel body (see k_ada_decode_std); state output, debug logits
  // and the h-byte tables take the general kernel
  if (p.fz.flag_units && p.fz.ctl_err != nullptr && !p.hb && p.logits_dbg == nullptr &&
      !p.fz.state_out)
    return launch_ada_std<GP>(p, smem, grid, stream, pdl);
  switch (p.st.d) {
    case 128: return launch_ada_dk<GP, 128>(p, smem, grid, stream, pdl);
    case 64: return launch_ada_dk<GP, 64>(p, smem, grid, stream, pdl);
    default: return launch_ada_dk<GP, 0>(p, smem, grid, stream, pdl);
  }
}

static int ada_decode_impl(const sphkv_store_t* st, const float* q, int G,
                           const sphkv_unit_t* units, int n_units, float* partials,
                           float* logits_dbg, const int64_t* dbg_offsets, int grid,
                           const FusedCtl& fz, cudaStream_t stream, bool live = false) {
  if (!st || !q || !units || !partials) return fail(SPHKV_E_VALUE, "null argument");
  if (G < 1 || G > 8) return fail(SPHKV_E_UNSUPPORTED, "GQA group size %d outside [1, 8]", G);
  if (st->d < 3 || st->d > 256) return fail(SPHKV_E_UNSUPPORTED, "d=%d outside [3, 256]", st->d);
  if (st->d_v < 1 || st->d_v > 128) return fail(SPHKV_E_UNSUPPORTED, "d_v=%d outside [1, 128]", st->d_v);
  if (st->page_size % 32 != 0 || st->page_size < 32 || st->page_size > 1024 ||
      (st->page_size > 128 && st->page_size % 128 != 0))
    return fail(SPHKV_E_UNSUPPORTED, "page_size=%d unsupported", st->page_size);
  if (logits_dbg && !dbg_offsets) return fail(SPHKV_E_VALUE, "dbg offsets missing");
  for (int t = 1; t < st->n_tiers; ++t)
    if (st->tiers[t].angle_bits > 16 || st->tiers[t].radius_bits > 16)
      return fail(SPHKV_E_UNSUPPORTED, "tier %d: code widths above 16 bits", st->tiers[t].id);
  if (n_units == 0) return SPHKV_OK;

  AdaParams p;
  memset(&p, 0, sizeof(p));
  p.st = *st;
  p.q = q;
  p.G = G;
  p.units = units;
  p.n_units = n_units;
  p.partials = partials;
  p.logits_dbg = logits_dbg;
  p.dbg_off = dbg_offsets;
  p.fz = fz;
  p.TI = st->page_size < ADA_TI ? st->page_size : ADA_TI;
  p.dvp = (st->d_v + 15) / 16 * 16;
  const int GP = (G + 1) / 2;
  p.hb = ada_use_hb(st, GP) ? 1 : 0;
  int used = lut_layout(st, p.lut_off, p.hb);
  p.lut_bytes = used;
  p.lut_global = nullptr;
  if (st->lut != nullptr && (st->lut_flags & 1) == p.hb) {
    bool same = true;
    for (int t = 0; t < SPHKV_MAX_TIERS; ++t) same = same && (st->lut_off[t] == p.lut_off[t]);
    if (same) p.lut_global = reinterpret_cast<const uint8_t*>(st->lut);
  }
  size_t off = align_up((size_t)used, 128);
  if (p.hb) {
    if (off == 0) off = 128;  // smem_hb == 0 means "no tables" to the tile dispatch
    p.smem_hb = (uint32_t)off;
    off = align_up(off + hb_bytes(st->d), 128);
  }
  p.smem_q = (uint32_t)off;
  off = align_up(off + (size_t)st->d * q_row_bytes(GP), 128);
  p.smem_tiles = (uint32_t)off;
  off = align_up(off + MAX_UNIT_TILES * sizeof(TileEntry) + 16, 128);
  // pipelined unit transitions (experiment, SPHKV_PIPE=1): plain fused
  // outputs only (no margins / state / live / debug logits / h-byte tables)
  {
    const char* e = getenv("SPHKV_PIPE");
    p.pipe = (e != nullptr && e[0] == '1' && ADA_NPV == 1 && fz.flag_units && fz.ctl_err != nullptr && !p.hb &&
              logits_dbg == nullptr && !fz.state_out && fz.margins == nullptr &&
              fz.slot_group != nullptr && !fz.abs_rows && !live) ? 1 : 0;
  }
  if (p.pipe) {  // two PIPE_TILES lists (+ count word each) inside the tile-list region
    static_assert(2 * (PIPE_TILES * sizeof(TileEntry) + 16) <= MAX_UNIT_TILES * sizeof(TileEntry) + 16 + 128,
                  "pipe tile lists fit the standard tile-list region");
    p.smem_tiles2 = p.smem_tiles + (uint32_t)align_up(PIPE_TILES * sizeof(TileEntry) + 16, 16);
    p.smem_info = (uint32_t)off;
    off = align_up(off + PIPE_MAXU * 16 + 16 + PIPE_MAXU * 4, 128);
    p.smem_q2 = (uint32_t)off;
    off = align_up(off + (size_t)st->d * q_row_bytes(GP), 128);
  }
  p.prow_bytes = p.TI * 2 + PROW_PAD;
  p.prows = G <= 4 ? 4 : 8;
  p.pslot_bytes = (int)align_up(p.prows * p.prow_bytes + 96, 16);  // hdr: m, sum, top-2
  p.smem_p = (uint32_t)off;
  off += (size_t)ADA_NS * p.pslot_bytes;
  off = align_up(off, 1024);
  p.smem_v = (uint32_t)off;
  off += (size_t)ADA_NV * p.TI * p.dvp * 2;
  p.smem_bar = (uint32_t)off;
  off += (2 * ADA_NS + 2 * ADA_NV + 1) * 8 + 8 + 64;  // barriers, s_flag/s_next, s_ml[16]
  size_t smem = off;
  if (smem > 232448) return fail(SPHKV_E_UNSUPPORTED, "ADA smem %zu exceeds 227 KB", smem);
  if (grid <= 0) grid = SM_COUNT;
  if (grid > n_units) grid = n_units;
#ifdef SPHKV_ONLY_GP  // fast experimental builds: one GQA width only
  if (GP != SPHKV_ONLY_GP) return fail(SPHKV_E_UNSUPPORTED, "built for GP=%d only", SPHKV_ONLY_GP);
  return launch_ada<SPHKV_ONLY_GP>(p, smem, grid, stream, !live);
#else
  switch (GP) {
    case 1: return launch_ada<1>(p, smem, grid, stream, !live);
    case 2: return launch_ada<2>(p, smem, grid, stream, !live);
    case 3: return launch_ada<3>(p, smem, grid, stream, !live);
    default: return launch_ada<4>(p, smem, grid, stream, !live);
  }
#endif
}

static int dense_decode_impl(const sphkv_dense_store_t* st, const float* q, int G,
                             const sphkv_unit_t* units, int n_units, float* partials, int grid,
                             const FusedCtl& fz, cudaStream_t stream, int tok_lo = 0) {
  if (!st || !q || !units || !partials) return fail(SPHKV_E_VALUE, "null argument");
  if (G < 1 || G > 8) return fail(SPHKV_E_UNSUPPORTED, "GQA group size %d outside [1, 8]", G);
  if (st->d > 128 || st->d_v > 128) return fail(SPHKV_E_UNSUPPORTED, "d/d_v above 128");
  if (st->page_size % DN_TI != 0) return fail(SPHKV_E_UNSUPPORTED, "page_size %% 64 != 0");
  if (n_units == 0) return SPHKV_OK;
  DenseParams p;
  memset(&p, 0, sizeof(p));
  p.st = *st;
  p.q = q;
  p.G = G;
  p.units = units;
  p.n_units = n_units;
  p.partials = partials;
  p.fz = fz;
  p.dp = (st->d + 15) / 16 * 16;
  p.dvp = (st->d_v + 15) / 16 * 16;
  if (tok_lo < 0 || tok_lo > st->tokens) return fail(SPHKV_E_VALUE, "token_begin %d", tok_lo);
  p.tok_lo = tok_lo;
  p.prow_bytes = DN_TI * 2 + PROW_PAD;
  p.pslot_bytes = (int)align_up(8 * p.prow_bytes + 64, 128);
  size_t off = 0;
  p.smem_k = 0;
  off += (size_t)DN_NK * DN_TI * p.dp * 2;
  off = align_up(off, 1024);
  p.smem_v = (uint32_t)off;
  off += (size_t)DN_NV * DN_TI * p.dvp * 2;
  off = align_up(off, 128);
  p.smem_p = (uint32_t)off;
  off += (size_t)DN_NS * p.pslot_bytes;
  off = align_up(off, 8);
  p.smem_bar = (uint32_t)off;
  off += (2 * DN_NK + 2 * DN_NV + 2 * DN_NS) * 8;
  size_t smem = off;
  if (smem > 227 * 1024) return fail(SPHKV_E_UNSUPPORTED, "dense smem %zu exceeds 227 KB", smem);
  if (grid <= 0) grid = SM_COUNT;
  if (grid > n_units) grid = n_units;
  if (p.dvp == 128) {
    SPHKV_CUDA_TRY(cudaFuncSetAttribute(k_dense_decode<2, true, 128>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    return launch_pdl(k_dense_decode<2, true, 128>, p, grid, dense_threads(2, true), smem, stream);
  }
#ifndef SPHKV_DN_NO64
  if (p.dvp == 64) {
    SPHKV_CUDA_TRY(cudaFuncSetAttribute(k_dense_decode<1, false, 64>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    return launch_pdl(k_dense_decode<1, false, 64>, p, grid, dense_threads(1, false), smem, stream);
  }
#endif
  SPHKV_CUDA_TRY(cudaFuncSetAttribute(k_dense_decode<1, false, 0>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  return launch_pdl(k_dense_decode<1, false, 0>, p, grid, dense_threads(1, false), smem, stream);
}

static int make_fused(FusedCtl& f, const int32_t* slot_group, const int32_t* slot_begin,
                      int n_groups, int32_t* ctl, float* out, int dynamic) {
  // ctl: [n_groups] split counters, queue head, CTAs done, error word
  memset(&f, 0, sizeof(f));
  if (slot_group != nullptr && (!slot_begin || !ctl || !out || n_groups < 1))
    return fail(SPHKV_E_VALUE, "fused merge needs slot_begin, ctl and out");
  if (dynamic && !ctl) return fail(SPHKV_E_VALUE, "dynamic unit queue needs ctl");
  f.slot_group = slot_group;
  f.slot_begin = slot_begin;
  f.ctl = ctl;
  f.out = out;
  f.n_groups = n_groups;
  f.dynamic = dynamic;
  f.ctl_err = (slot_group != nullptr && ctl != nullptr) ? ctl + n_groups + 2 : nullptr;
  return SPHKV_OK;
}

extern "C" int sphkv_ada_decode(const sphkv_store_t* st, const float* q, int G,
                                const sphkv_unit_t* units, int n_units, float* partials,
                                float* logits_dbg, const int64_t* dbg_offsets, int grid,
                                cudaStream_t stream) {
  FusedCtl f;
  make_fused(f, nullptr, nullptr, 0, nullptr, nullptr, 0);
  return ada_decode_impl(st, q, G, units, n_units, partials, logits_dbg, dbg_offsets, grid, f,
                         stream);
}

extern "C" int sphkv_ada_decode_fused(const sphkv_store_t* st, const float* q, int G,
                                      const sphkv_unit_t* units, int n_units, float* partials,
                                      const int32_t* slot_group, const int32_t* slot_begin,
                                      int n_groups, int32_t* ctl, float* out, int dynamic,
                                      int grid, cudaStream_t stream) {
  FusedCtl f;
  int rc = make_fused(f, slot_group, slot_begin, n_groups, ctl, out, dynamic);
  if (rc) return rc;
  f.flag_units = 1;
  return ada_decode_impl(st, q, G, units, n_units, partials, nullptr, nullptr, grid, f, stream);
}

extern "C" int sphkv_ada_decode_margins(const sphkv_store_t* st, const float* q, int G,
                                        const sphkv_unit_t* units, int n_units, float* partials,
                                        const int32_t* slot_group, const int32_t* slot_begin,
                                        int n_groups, int32_t* ctl, float* out, int dynamic,
                                        float* top2, float* margins, int grid,
                                        cudaStream_t stream) {
  if (!slot_group || !top2 || !margins)
    return fail(SPHKV_E_VALUE, "margins need the fused merge (slot_group), top2 and margins");
  FusedCtl f;
  int rc = make_fused(f, slot_group, slot_begin, n_groups, ctl, out, dynamic);
  if (rc) return rc;
  f.top2 = top2;
  f.margins = margins;
  return ada_decode_impl(st, q, G, units, n_units, partials, nullptr, nullptr, grid, f, stream);
}

extern "C" int sphkv_ada_decode_live(const sphkv_store_t* st, const float* q, int G,
                                     const sphkv_unit_t* units, int n_units, float* partials,
                                     const int32_t* slot_group, const int32_t* slot_begin,
                                     int n_groups, int32_t* ctl, float* out, float* top2,
                                     float* margins, int flags, int grid, cudaStream_t stream) {
  FusedCtl f;
  int rc = make_fused(f, slot_group, slot_begin, n_groups, ctl, out, 0);
  if (rc) return rc;
  if (!slot_group) return fail(SPHKV_E_VALUE, "the live decode needs the fused merge");
  if ((top2 == nullptr) != (margins == nullptr)) return fail(SPHKV_E_VALUE, "top2 with margins");
  f.top2 = top2;
  f.margins = margins;
  f.abs_rows = (flags & SPHKV_LIVE_ABS_ROWS) ? 1 : 0;
  f.flag_units = 1;
  return ada_decode_impl(st, q, G, units, n_units, partials, nullptr, nullptr, grid, f, stream,
                         (flags & SPHKV_LIVE_AFTER_MUTATION) != 0);
}

extern "C" int sphkv_ada_decode_state(const sphkv_store_t* st, const float* q, int G,
                                      const sphkv_unit_t* units, int n_units, float* partials,
                                      const int32_t* slot_group, const int32_t* slot_begin,
                                      int n_groups, int32_t* ctl, float* state_out, int grid,
                                      cudaStream_t stream) {
  FusedCtl f;
  int rc = make_fused(f, slot_group, slot_begin, n_groups, ctl, state_out, 0);
  if (rc) return rc;
  if (!slot_group) return fail(SPHKV_E_VALUE, "the state output needs the fused merge");
  f.state_out = 1;
  return ada_decode_impl(st, q, G, units, n_units, partials, nullptr, nullptr, grid, f, stream);
}

extern "C" int sphkv_dense_decode(const sphkv_dense_store_t* st, const float* q, int G,
                                  const sphkv_unit_t* units, int n_units, float* partials,
                                  int grid, cudaStream_t stream) {
  FusedCtl f;
  make_fused(f, nullptr, nullptr, 0, nullptr, nullptr, 0);
  return dense_decode_impl(st, q, G, units, n_units, partials, grid, f, stream);
}

extern "C" int sphkv_dense_decode_fused(const sphkv_dense_store_t* st, const float* q, int G,
                                        const sphkv_unit_t* units, int n_units, float* partials,
                                        const int32_t* slot_group, const int32_t* slot_begin,
                                        int n_groups, int32_t* ctl, float* out, int dynamic,
                                        int grid, cudaStream_t stream) {
  FusedCtl f;
  int rc = make_fused(f, slot_group, slot_begin, n_groups, ctl, out, dynamic);
  if (rc) return rc;
  return dense_decode_impl(st, q, G, units, n_units, partials, grid, f, stream);
}

extern "C" int sphkv_dense_decode_window(const sphkv_dense_store_t* st, const float* q, int G,
                                         const sphkv_unit_t* units, int n_units, float* partials,
                                         const int32_t* slot_group, const int32_t* slot_begin,
                                         int n_groups, int32_t* ctl, float* out, int dynamic,
                                         int token_begin, int grid, cudaStream_t stream) {
  FusedCtl f;
  int rc = make_fused(f, slot_group, slot_begin, n_groups, ctl, out, dynamic);
  if (rc) return rc;
  return dense_decode_impl(st, q, G, units, n_units, partials, grid, f, stream, token_begin);
}

// Debug builds (-DSPHKV_DBG_TIMING) only: per-CTA (start, end) globaltimer of
// the last ADA launch, 2 * n values; not declared in the public header.
extern "C" int sphkv_debug_cta_times(unsigned long long* out_host, int n) {
#ifdef SPHKV_DBG_TIMING
  SPHKV_CUDA_TRY(cudaMemcpyFromSymbol(out_host, g_cta_t, sizeof(unsigned long long) * 2 * n));
  return SPHKV_OK;
#else
  (void)out_host;
  (void)n;
  return fail(SPHKV_E_UNSUPPORTED, "built without SPHKV_DBG_TIMING");
#endif
}

extern "C" int sphkv_lse_merge_ex(const float* partials, const int32_t* slot_begin,
                                  int n_splits, int64_t split_stride, int n_groups, int G,
                                  int d_v, float* out, int state_out, cudaStream_t stream) {
  if (!partials || !out) return fail(SPHKV_E_VALUE, "null argument");
  if (!slot_begin && (n_splits < 0 || split_stride < n_groups))
    return fail(SPHKV_E_VALUE, "bad split layout (n_splits=%d, stride=%lld)", n_splits,
                (long long)split_stride);
  if (G < 1 || d_v < 1) return fail(SPHKV_E_VALUE, "bad G/d_v");
  if (n_groups == 0) return SPHKV_OK;
  int threads = d_v >= 128 ? 128 : ((d_v + 31) / 32) * 32;
  k_lse_merge<<<n_groups * G, threads, 0, stream>>>(partials, slot_begin, n_splits, split_stride,
                                                    n_groups, G, d_v, out, state_out);
  SPHKV_LAUNCH_CHECK();
  return SPHKV_OK;
}

extern "C" int sphkv_lse_merge(const float* partials, const int32_t* slot_begin, int n_groups,
                               int G, int d_v, float* out, cudaStream_t stream) {
  if (!slot_begin) return fail(SPHKV_E_VALUE, "null argument");
  return sphkv_lse_merge_ex(partials, slot_begin, 0, 0, n_groups, G, d_v, out, 0, stream);
}
