/*
 * sphkv_b200.h -- C ABI of the B200-native Spherical-KV decode hot path.
 *
 * One shared library, libsphkv_b200.so, built for sm_100a only.  Every entry
 * point is `extern "C"`, takes plain pointers / sizes / a cudaStream_t, and
 * returns an int status (0 == SPHKV_OK).  All data buffers are caller-owned
 * DEVICE pointers unless the parameter name ends in `_host`.  The library
 * keeps no global mutable state; `sphkv_last_error()` is thread-local.
 *
 * The reference (arXiv 2605.18856, read-only `sphkv` Python package, paths
 * below relative to pkg/src/sphkv/) has no FFI: its boundary is the Python
 * API exported from __init__.py:4-18.  Each entry point cites the reference
 * function it replaces; INTEGRATION.md shows the ctypes binding a maintainer
 * would add on the reference side.
 *
 * Device page format:
 *   code pool  : per page a 16-byte aligned block.  Angle part, "word-
 *                interleaved item-major": item i's d-1 codes are one LSB-first
 *                bit string (code j at bits [j*b, j*b+b)) padded to W words
 *                (ceil((d-1)*b/32) rounded up to a multiple of 4); 16-byte
 *                quad w4 of item i is stored at quad ((i/32)*(W/4) + w4)*32 +
 *                i%32 (granules of 32 items: a warp loads one quad of 32 items
 *                as one coalesced 512-byte load and each lane holds its item's
 *                codes in registers).
 *                Then one radius row of page_size*radius_bits bits (LSB-
 *                first), padded to 16 bytes.  sphkv_export_streams() converts
 *                to the reference's coordinate-major SoA streams
 *                (store.py:205-211) bit for bit.
 *   value pool : fp16 [page][page_size][d_v]; inside each row the 16-byte
 *                chunk c of item i is stored at chunk (c ^ (i & 7)) so that
 *                1-D bulk copies land ldmatrix-conflict-free in shared memory.
 */
#ifndef SPHKV_B200_H
#define SPHKV_B200_H

#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPHKV_ABI_VERSION 1

enum {
  SPHKV_OK = 0,
  SPHKV_E_VALUE = 1,        /* -> ValueError   (bad argument / range)          */
  SPHKV_E_KEY = 2,          /* -> KeyError     (unknown head / missing state)  */
  SPHKV_E_INFEASIBLE = 3,   /* -> InfeasibleProtectionError (controller.py:46) */
  SPHKV_E_UNSUPPORTED = 4,  /* -> ValueError   (outside the kernel contract)   */
  SPHKV_E_CUDA = 5,         /* -> RuntimeError (CUDA error)                    */
  SPHKV_E_CAPACITY = 6      /* -> RuntimeError (store pool exhausted)          */
};

enum { SPHKV_F32 = 0, SPHKV_F64 = 1, SPHKV_BF16 = 2, SPHKV_F16 = 3 };

#define SPHKV_MAX_TIERS 16

/* One precision tier (codec.py:73-107 TierSpec + TierTable eps constants). */
typedef struct {
  int32_t id;
  int32_t angle_bits;
  int32_t radius_bits;
  int32_t meta_bits;
  double eps_theta;
  double eps_r;
} sphkv_tier_t;

/* Device page descriptor, 32 bytes (the reference Page, store.py:136-211). */
typedef struct {
  uint64_t code_off;     /* byte offset of the page's code block             */
  double radius_scale;   /* page radius scale (fp64, store.py:465 / :264)   */
  float rscale;          /* (float)(radius_scale / (2^radius_bits - 1))      */
  int32_t count;         /* items stored                                     */
  int32_t group;         /* (seq*layers + layer)*heads + head                */
  uint8_t tier;          /* tier id                                          */
  uint8_t abits;
  uint8_t rbits;
  uint8_t mbits;
} sphkv_page_t;

/* Paged store: pools and tables (PagedStore, store.py:214-427). */
typedef struct {
  int32_t batch, layers, heads, d, d_v, page_size;
  int32_t n_tiers;            /* entries in `tiers`, drop tier first          */
  int32_t max_pages;          /* capacity of the page-indexed pools          */
  int32_t ptr_cap;            /* pointer-list capacity per group             */
  int32_t lut_flags;          /* bit 0: the prebuilt LUT omits the 2-bit tier,
                                 which decodes from per-query h-byte tables
                                 (launches with G <= 4 query heads, d = 64/128) */
  uint64_t code_cap;          /* bytes in `codes`                             */
  sphkv_tier_t tiers[SPHKV_MAX_TIERS];
  sphkv_page_t* pages;        /* [max_pages]                                  */
  int32_t* ptr;               /* [groups * ptr_cap] page ids, pointer order   */
  int32_t* ptr_len;           /* [groups]                                     */
  int32_t* group_last;        /* [groups * SPHKV_MAX_TIERS] last page / -1    */
  uint8_t* codes;             /* code pool                                    */
  uint16_t* values;           /* fp16 value pool [max_pages][P][d_v]          */
  uint8_t* protect;           /* [max_pages][P]                               */
  int64_t* token_ids;         /* [max_pages][P]                               */
  uint64_t* counters;         /* [0]=n_pages [1]=code bytes used (device)     */
  float* lut;                 /* prebuilt (cos, sin) tables, filled by
                                 sphkv_store_build_lut; NULL -> computed in-kernel */
  int32_t lut_off[SPHKV_MAX_TIERS];  /* (byte offset << 2) | mode per tier, -1 = none */
  int64_t lut_items[SPHKV_MAX_TIERS];  /* items stored per tier index: LUT placement hint
                                          (all zero = unknown, every tier gets a table) */
} sphkv_store_t;

/* Dense bf16-K / fp16-V paged store used by the dense baseline kernel
 * (DenseStore, store.py:485-569). K pages are [P][d] bf16, swizzled like V. */
typedef struct {
  int32_t batch, layers, heads, d, d_v, page_size;
  int32_t n_pages_per_group;  /* ceil(T / P)                                  */
  int32_t tokens;             /* T (items per group)                          */
  uint16_t* keys;             /* bf16 [groups][n_pages][P][d]                 */
  uint16_t* values;           /* fp16 [groups][n_pages][P][d_v]               */
} sphkv_dense_store_t;

/* One decode work unit: a contiguous range of one group's pointer list. */
typedef struct {
  int32_t group;              /* (seq*layers + layer)*heads + head            */
  int32_t ptr_begin;          /* first pointer-list position                  */
  int32_t ptr_end;            /* one past the last; < 0: the list's current end
                                 (sphkv_ada_decode_live only)                  */
  int32_t out_slot;           /* index into the partial buffer                */
} sphkv_unit_t;

/* Controller features (ControllerFeatures, controller.py:77-96). */
typedef struct {
  const double* u_hat;        /* [layers*heads] (per sequence if batched: [B*L*H]) */
  const double* s_hat;        /* same shape as u_hat                          */
  const double* omega_tok;    /* [tokens] omega of each prefill token         */
  double r_q;
  double alpha_theta;
  double alpha_r;
  double omega_recent;        /* omega of decode-appended states (:96)         */
} sphkv_features_t;

int sphkv_abi_version(void);
const char* sphkv_last_error(void);
int sphkv_device_ok(void);

/* ---- encode (codec.py:222-257, decode.py:457-459) ------------------------ */

/* radii[n] = || keys[n, :] || in fp64 with numpy's pairwise summation order. */
int sphkv_encode_radii(const void* keys, int dtype, int64_t n, int d,
                       double* radii, cudaStream_t stream);

/* to_spherical / angles_from_unit, batched: radii[n] and angles[n, d-1]. */
int sphkv_encode(const void* keys, int dtype, int64_t n, int d,
                 double* radii, double* angles, cudaStream_t stream);

/* angles_from_unit (codec.py:239-257) on rows that are already unit length. */
int sphkv_angles_from_unit(const double* u, int64_t n, int d, double* angles,
                           cudaStream_t stream);

/* quantize_angles (codec.py:326-340): codes[n, d-1] (uint32) at `bits`. */
int sphkv_quantize_angles(const double* angles, int64_t n, int dm1, int bits,
                          uint32_t* codes, cudaStream_t stream);

/* ---- RDR controller (controller.py:201-386) ----------------------------- */

/* score_states: best_tier int16, score/nu/d_drop fp64 over [n = L*H*T]
 * states.  `seg_omega` is omega per token (length T), u_hat/s_hat per
 * (l, h) [L*H].  Bit-exact with numpy's fp64 operation order. */
int sphkv_rdr_score(const double* radii, const double* u_hat, const double* s_hat,
                    const double* seg_omega, double r_q, double alpha_theta,
                    double alpha_r, const sphkv_tier_t* tiers_host, int n_tiers,
                    double lam, const uint8_t* protect, int layers, int heads,
                    int tokens, int d, int16_t* best_tier, double* score,
                    double* nu, double* d_drop, cudaStream_t stream);

/* Scratch bytes for allocate_greedy / downtier over n states. */
int64_t sphkv_rdr_workspace_bytes(int64_t n);

/* allocate_greedy: z int8 / tier int16 outputs.  Exact parallel form: stable
 * radix sort on (-nu, flat index) then <= (#distinct rates) filtered scans.
 * Returns SPHKV_E_INFEASIBLE when protected demand exceeds the budget. */
int sphkv_rdr_allocate_greedy(const int16_t* best_tier, const double* nu,
                              const uint8_t* protect, int64_t n,
                              const sphkv_tier_t* tiers_host, int n_tiers, int d,
                              int64_t budget_bits, void* workspace, int8_t* z,
                              int16_t* tier, cudaStream_t stream);

/* downtier_before_drop from the full best-tier start (controller.py:349-398). */
int sphkv_rdr_downtier(const int16_t* best_tier, const double* nu,
                       const uint8_t* protect, int64_t n,
                       const sphkv_tier_t* tiers_host, int n_tiers, int d,
                       int64_t budget_bits, void* workspace, int8_t* z,
                       int16_t* tier, cudaStream_t stream);

/* ---- paged store (store.py:214-482) ------------------------------------- */

/* Fill st->lut (caller-allocated, sphkv_lut_floats() floats) and st->lut_off
 * with fp32-rounded fp64 (cos, sin) of every polar grid point of each tier
 * whose angle width fits the shared-memory LUT budget. */
int64_t sphkv_lut_floats(const sphkv_store_t* st);
int sphkv_store_build_lut(sphkv_store_t* st, cudaStream_t stream);

/* Reset counters / pointer lists of a store (pools are zeroed by caller). */
int sphkv_store_reset(const sphkv_store_t* st, cudaStream_t stream);

/* pack_pages_arrays fused with the encoder: dense keys [B*L*H*T, d] (fp32 /
 * bf16 / fp64), fp16 values, assignment (z int8, tier int16, protect u8)
 * and fp64 radii -> pages in pointer order (l, h) -> tier -> chunk.
 * `angles` may be NULL (encode from keys) or fp64 [.., d-1] (drop-in path
 * with caller-supplied angles, as pack_pages_arrays takes them). */
int sphkv_pack_pages(const sphkv_store_t* st, const void* keys, int key_dtype,
                     const double* angles, const double* radii,
                     const uint16_t* values, const int8_t* z, const int16_t* tier,
                     const uint8_t* protect, int tokens, void* workspace,
                     int64_t workspace_bytes, cudaStream_t stream);
/* Same, for the contiguous groups [group0, group0 + n_groups) only: every
 * input array is relative to group0 ([n_groups * tokens] states).  Packs one
 * sequence (or one shard) at a time into a shared store, so the raw K/V of
 * only that part needs to be resident; pages append after the existing ones
 * and pointer lists of other groups are untouched. */
int sphkv_pack_pages_groups(const sphkv_store_t* st, int group0, int n_groups, const void* keys,
                            int key_dtype, const double* angles, const double* radii,
                            const uint16_t* values, const int8_t* z, const int16_t* tier,
                            const uint8_t* protect, int tokens, void* workspace,
                            int64_t workspace_bytes, cudaStream_t stream);
int64_t sphkv_pack_workspace_bytes(int batch, int layers, int heads, int tokens);

/* PagedStore.append_item for one new state per group (decode.py:454-498):
 * keys [groups, d] (fp64 radius/angles computed on device unless `angles`
 * given), values fp16 [groups, d_v], tier_ids int16 [groups] (0 = drop),
 * protect u8 [groups], token id per group.  Pages open in group order. */
int sphkv_append(const sphkv_store_t* st, const void* keys, int key_dtype,
                 const double* radii, const double* angles, const uint16_t* values,
                 const int16_t* tier_ids, const uint8_t* protect,
                 const int64_t* token_ids, const uint8_t* active, void* workspace,
                 cudaStream_t stream);
int64_t sphkv_append_workspace_bytes(int groups);

/* score_and_best_tier for appended states (controller.py:181-198). */
int sphkv_score_append(const double* radii, int groups_per_seq, int heads,
                       const double* u_hat, const double* s_hat, double r_q,
                       double omega, double alpha_theta, double alpha_r,
                       const sphkv_tier_t* tiers_host, int n_tiers, double lam,
                       int d, int64_t n, int16_t* tier_out, double* score_out,
                       double* nu_out, cudaStream_t stream);

/* Dense baseline store fill (DenseStore.bulk_load, store.py:524-531): keys
 * [groups*T, d] (dtype), values fp16 [groups*T, d_v] -> swizzled pages. */
int sphkv_dense_fill(const sphkv_dense_store_t* st, const void* keys, int key_dtype,
                     const uint16_t* values, cudaStream_t stream);

/* Same for the contiguous groups [group0, group0 + n_groups) (inputs relative
 * to group0): fills one sequence / shard of a batched dense store. */
int sphkv_dense_fill_groups(const sphkv_dense_store_t* st, int group0, int n_groups,
                            const void* keys, int key_dtype, const uint16_t* values,
                            cudaStream_t stream);

/* fp64 -> fp16 with one round-to-nearest-even (numpy astype(np.float16),
 * the SPHKV1 value type, store.py:383); torch's double->half conversion
 * rounds through fp32 and differs for some inputs. */
int sphkv_f64_to_f16(const double* in, int64_t n, uint16_t* out, cudaStream_t stream);

/* Reference-format streams of every page: angle stream (stride = count),
 * radius stream, fp16 values un-swizzled [count][d_v], protect bytes.
 * offsets_host give each page's byte offset in `out`. */
int sphkv_export_streams(const sphkv_store_t* st, int n_pages,
                         const int64_t* offsets, uint8_t* out, cudaStream_t stream);

/* Inverse of sphkv_export_streams (SPHKV1 import, store.py:391-427): with the
 * page descriptors st->pages[0..n_pages) already set (code_off, count,
 * group, tier and widths, radius_scale), rebuild each page's device code
 * block, value rows and protect flags from the same per-page stream layout
 * (angle stream, radius stream, fp16 values, protect bytes at offsets[pid]);
 * token ids become -1. */
int sphkv_import_streams(const sphkv_store_t* st, int n_pages, const int64_t* offsets,
                         const uint8_t* in, cudaStream_t stream);

/* ---- controller features (controller.py:99-142) --------------------------- */

/* Dense prefill pass over sampled rows for every query group: keys
 * [groups / q_per_key, tokens, d] (key_dtype; q_per_key consecutive query
 * groups share one key group -- the G query heads of a KV head), q_rows fp64
 * [groups, R, d] (the queries at the sampled rows), rows [R] ascending token
 * indices.  Per group: u_raw = mean over rows
 * of the causal softmax weight on tokens j <= row - window; inv_margin = mean
 * over rows >= 1 of 1 / (top-1 - top-2 logit + 1e-6).  fp64 throughout.
 * workspace: sphkv_controller_workspace_bytes(groups, R) bytes. */
int64_t sphkv_controller_workspace_bytes(int64_t groups, int R);
int sphkv_controller_stats(const void* keys, int key_dtype, const double* q_rows,
                           const int32_t* rows, int R, int64_t groups, int tokens, int d,
                           int window, int q_per_key, double* u_raw, double* inv_margin,
                           void* workspace, cudaStream_t stream);

/* ---- decode (decode.py:291-355) ------------------------------------------ */

/* Tile geometry the decode kernels were built with, for the host planner:
 * items per tile (min(P, this) for narrow pages) and the tile cap of one
 * work unit: the planner cuts units to it; the general kernel runs a longer
 * unit (a direct caller's) as several segments; the standard fused kernel
 * flags it in ctl[n_groups + 2] = SPHKV_E_CAPACITY (its outputs are then
 * unusable -- re-plan or use sphkv_ada_decode). */
int sphkv_ada_tile_items(void);
int sphkv_unit_tile_cap(void);

/* ADA paged decode: q fp32 [B, L, H*G, d]; per unit writes the partial
 * softmax state (m[G], l[G], acc[G][d_v]) in base-2 logit units to
 * partials[out_slot].  logits_dbg (optional, fp32) receives logits (natural
 * units) at [unit item index] for parity checks; pass NULL in production. */
int sphkv_ada_decode(const sphkv_store_t* st, const float* q, int G,
                     const sphkv_unit_t* units, int n_units, float* partials,
                     float* logits_dbg, const int64_t* dbg_offsets, int grid,
                     cudaStream_t stream);

/* ADA decode with the split merge fused in: the CTA that finishes the last
 * split of a plan group merges that group's partial slots into `out` fp32
 * [n_groups*G, d_v] (same result as sphkv_lse_merge).  slot_group int32
 * [n_slots] gives each partial slot's plan group (-1 = scratch slot);
 * slot_begin as for sphkv_lse_merge; ctl int32 [n_groups + 3] must be zero
 * before the first call and is left zero (CUDA-graph replay safe) except the
 * error word ctl[n_groups + 2] (set to SPHKV_E_CAPACITY when a unit exceeds
 * sphkv_unit_tile_cap() tiles; sticky until the caller clears it).
 * dynamic != 0: CTAs claim units from a global queue in list order (plan the
 * list longest-first) instead of the static u += grid assignment. */
int sphkv_ada_decode_fused(const sphkv_store_t* st, const float* q, int G,
                           const sphkv_unit_t* units, int n_units, float* partials,
                           const int32_t* slot_group, const int32_t* slot_begin, int n_groups,
                           int32_t* ctl, float* out, int dynamic, int grid,
                           cudaStream_t stream);

/* sphkv_ada_decode_fused plus the decode-time gate's input: margins fp32
 * [n_groups * G] = top-1 minus top-2 logit of each (group, query head) over
 * all of the group's items in natural logit units (+inf with fewer than two
 * items) -- gate.margin (gate.py:50-56) of the head's logits
 * (decode.py:433-436).  top2: fp32 scratch [n_slots + 1][G]. */
int sphkv_ada_decode_margins(const sphkv_store_t* st, const float* q, int G,
                             const sphkv_unit_t* units, int n_units, float* partials,
                             const int32_t* slot_group, const int32_t* slot_begin, int n_groups,
                             int32_t* ctl, float* out, int dynamic, float* top2, float* margins,
                             int grid, cudaStream_t stream);

/* Dense bf16 paged decode with the same unit/partial contract. */
int sphkv_dense_decode(const sphkv_dense_store_t* st, const float* q, int G,
                       const sphkv_unit_t* units, int n_units, float* partials,
                       int grid, cudaStream_t stream);

/* Dense decode with the fused split merge / dynamic queue (as above). */
int sphkv_dense_decode_fused(const sphkv_dense_store_t* st, const float* q, int G,
                             const sphkv_unit_t* units, int n_units, float* partials,
                             const int32_t* slot_group, const int32_t* slot_begin,
                             int n_groups, int32_t* ctl, float* out, int dynamic, int grid,
                             cudaStream_t stream);

/* Fused ADA decode whose in-kernel merge writes each planned group's STATE
 * (one partial slot [G*(d_v+2)] per group: m = log2-sum-exp, l = 1, acc =
 * normalized output; all-empty: -inf, 0, 0) instead of output rows -- a
 * rank's page-range share in one launch, ready for the all-gather and
 * sphkv_lse_merge_ex over ranks. */
int sphkv_ada_decode_state(const sphkv_store_t* st, const float* q, int G,
                           const sphkv_unit_t* units, int n_units, float* partials,
                           const int32_t* slot_group, const int32_t* slot_begin, int n_groups,
                           int32_t* ctl, float* state_out, int grid, cudaStream_t stream);

/* Decode-time append decision for one new key per group (decode.py:454-498):
 * the key's radius (fp64, numpy pairwise order), its best tier
 * (score_and_best_tier, controller.py:181-198, omega = the recent-segment
 * weight), and with use_gate the hysteretic gate (gate.py:59-74): danger =
 * max over the G query heads of alpha * logit_drift_bound(|q|, r_max,
 * eps_r * r_max, eps_theta, d) / (margin + 1e-9) clamped to 10 (0 for an
 * infinite margin), probe tier = best tier or the max tier for a drop, r_max =
 * max page radius scale of the group; a protected head appends at the max
 * tier with the protect flag.  keys [groups, d] (key_dtype), q fp32 [groups,
 * G, d], margins fp32 [groups*G] (natural units, from the decode), u_hat /
 * s_hat fp64 [groups], mode int8 [groups] gate state (0 compressible,
 * 1 held, 2 protected; updated in place).  Outputs tier_out int16 [groups],
 * protect_out uint8 [groups], danger_out fp32 [groups] (may be NULL). */
int sphkv_decode_gate(const sphkv_store_t* st, const void* keys, int key_dtype, const float* q,
                      int G, const float* margins, const double* u_hat, const double* s_hat,
                      double r_q, double omega, double alpha_theta, double alpha_r, double lam,
                      int use_gate, double tau_drop, double tau_prot, double gate_alpha,
                      int8_t* mode, int16_t* tier_out, uint8_t* protect_out, float* danger_out,
                      cudaStream_t stream);

/* Decode over a store that decode steps grow: the fused ADA decode with the
 * gate margins (top2/margins may both be NULL); units with ptr_end < 0 run to
 * the group's current pointer-list end, so one plan (and one captured CUDA
 * graph) serves every step.  flags: SPHKV_LIVE_AFTER_MUTATION -- the
 * previous work on the stream may have changed the store (an append): no
 * programmatic-dependent launch, the prologue may not read the page table
 * early; SPHKV_LIVE_ABS_ROWS -- out [groups*G, d_v] and margins [groups*G]
 * rows are indexed by absolute group id (one buffer for all layer launches).
 * As with sphkv_ada_decode_fused, a unit whose pages exceed
 * sphkv_unit_tile_cap() tiles is not decoded: ctl[n_groups + 2] is set to
 * SPHKV_E_CAPACITY (the caller re-plans; planner units of a growing store stay
 * far below the cap). */
enum { SPHKV_LIVE_AFTER_MUTATION = 1, SPHKV_LIVE_ABS_ROWS = 2 };
int sphkv_ada_decode_live(const sphkv_store_t* st, const float* q, int G,
                          const sphkv_unit_t* units, int n_units, float* partials,
                          const int32_t* slot_group, const int32_t* slot_begin, int n_groups,
                          int32_t* ctl, float* out, float* top2, float* margins, int flags,
                          int grid, cudaStream_t stream);

/* Fused dense decode restricted to tokens >= token_begin of every planned
 * group (a sliding-window layer: the window's last W tokens only). */
int sphkv_dense_decode_window(const sphkv_dense_store_t* st, const float* q, int G,
                              const sphkv_unit_t* units, int n_units, float* partials,
                              const int32_t* slot_group, const int32_t* slot_begin, int n_groups,
                              int32_t* ctl, float* out, int dynamic, int token_begin, int grid,
                              cudaStream_t stream);

/* Reconstruct-then-dot negative control (decode.py:195-217):
 * decode the codes of pages[i] (pointer order) into dense key rows
 * k~ = r~ * unit(angles), written at rows [item_off[i], item_off[i] + count)
 * of `out` ([n, d], out_dtype SPHKV_F32 or SPHKV_F16) -- the staging write the
 * ADA kernel avoids. */
int sphkv_recon_keys(const sphkv_store_t* st, const int32_t* pages, const int64_t* item_off,
                     int n_pages, void* out, int out_dtype, cudaStream_t stream);

/* The dot's re-read of the staged rows: out[i*G + g] = q_g . stage_i / sqrt(d)
 * for rows i < n of `stage` ([n, d], SPHKV_F32 or SPHKV_F16), q fp32 [G, d],
 * G <= 8.  Rows must be whole 16-byte chunks (d*esize % 16 == 0, d <= 256). */
int sphkv_recon_dot(const void* stage, int stage_dtype, int64_t n, int d, const float* q,
                    int G, float* out, cudaStream_t stream);

/* dense_logits(q, keys) = keys @ q / sqrt(d) in fp64 (decode.py:63-69):
 * q [d], keys [n, d] row-major, out [n]. */
int sphkv_dense_logits(const double* q, const double* keys, int64_t n, int d, double* out,
                       cudaStream_t stream);

/* Logits of every token of one dense-store group for G <= 8 query heads
 * (the dense branch of _head_attend, decode.py:302-307, store.py:533-546):
 * out fp32 [tokens][G] = q_g . k_t / sqrt(d) over the bf16 pages. */
int sphkv_dense_store_logits(const sphkv_dense_store_t* st, const float* q, int G, int group,
                             float* out, cudaStream_t stream);

/* Split-context LSE merge: out fp32 [n_groups*G, d_v]; group g's partials
 * are slots [slot_begin[g], slot_begin[g+1]). Empty splits carry m = -inf. */
int sphkv_lse_merge(const float* partials, const int32_t* slot_begin,
                    int n_groups, int G, int d_v, float* out, cudaStream_t stream);

/* General form.  slot_begin == NULL selects the rank-major layout an
 * all-gather produces: group g's splits are slots g + s*split_stride, s <
 * n_splits.  state_out != 0 writes one partial slot per group instead of
 * normalized rows (m = log2-sum-exp, l = 1, acc = normalized output; all-empty
 * groups keep m = -inf, l = 0, acc = 0) -- a valid split state, so per-rank
 * results can be all-gathered and merged again by this same call (the
 * multi-GPU page-range split of SURVEY 8(e)). */
int sphkv_lse_merge_ex(const float* partials, const int32_t* slot_begin, int n_splits,
                       int64_t split_stride, int n_groups, int G, int d_v, float* out,
                       int state_out, cudaStream_t stream);

/* Bytes per partial slot for G query heads and d_v. */
int64_t sphkv_partial_floats(int G, int d_v);

#ifdef __cplusplus
}
#endif
#endif /* SPHKV_B200_H */
