// Reconstruct-then-dot negative control.
//
// Reference behaviour replaced (pkg/src/sphkv/):
//   decode.py:195-217  recon_logits: each streamed page is decoded to a dense
//                      key block, staged through a real buffer write and
//                      re-read by the dot product (the "densification tax",
//                      metered as dense_k_write + dense_k_read, d*2 B/item each)
//   decode.py:272-288  _page_dense_block / codec.reconstruct_from_trig
//
// k_recon_keys decodes the listed pages' angle/radius codes (device WI layout)
// into dense key rows k~ = r~ * unit(angles) -- the staging write the ADA
// kernel exists to avoid.  The dot product then re-reads the rows.
#include "common.cuh"

namespace sphkv {

// one warp per page chunk of 32 items, lane = item; rows written as fp32 or fp16
template <typename OutT>
__global__ void k_recon_keys(sphkv_store_t st, const int32_t* __restrict__ pages,
                             const int64_t* __restrict__ item_off, int n_pages,
                             OutT* __restrict__ out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int chunks = (st.page_size + 31) / 32;
  if (warp >= n_pages * chunks) return;
  const int pi = warp / chunks, slot = (warp % chunks) * 32 + lane;
  const sphkv_page_t pg = st.pages[pages[pi]];
  if (slot >= pg.count) return;
  const int d = st.d, b = pg.abits, W = item_words(d, b);
  const uint32_t* words = reinterpret_cast<const uint32_t*>(st.codes + pg.code_off);
  auto code = [&](int bit, int n) -> uint32_t {
    const int w0 = bit >> 5, sh = bit & 31;
    const uint32_t lo = words[wi_word(slot, w0, W)];
    const uint32_t hi = (sh + n > 32) ? words[wi_word(slot, w0 + 1, W)] : 0u;
    return __funnelshift_r(lo, hi, sh) & ((1u << n) - 1u);
  };
  // decoded radius r~ = code / levels * scale (decode.py:137-139)
  const uint64_t rbit = angle_part_bytes(d, st.page_size, b) * 8 + (uint64_t)slot * pg.rbits;
  const uint32_t* rw = words + (rbit >> 5);
  const int rsh = (int)(rbit & 31);
  const uint32_t rhi = (rsh + pg.rbits > 32) ? rw[1] : 0u;
  const uint32_t rc = __funnelshift_r(rw[0], rhi, rsh) & ((1u << pg.rbits) - 1u);
  const float r = (float)((double)rc / (double)((1u << pg.rbits) - 1u) * pg.radius_scale);
  OutT* row = out + (item_off[pi] + slot) * (int64_t)d;
  const float pstep = 1.0f / (float)((1u << b) - 1u);  // angle / pi
  float prod = r;
  for (int j = 0; j < d - 2; ++j) {
    float sn, cs;
    sincospif((float)code(j * b, b) * pstep, &sn, &cs);
    row[j] = (OutT)(prod * cs);
    prod *= sn;
  }
  float sn, cs;  // circular last angle: step 2 pi / 2^b
  sincospif((float)code((d - 2) * b, b) * (1.0f / (float)(1u << (b - 1))), &sn, &cs);
  row[d - 2] = (OutT)(prod * cs);
  row[d - 1] = (OutT)(prod * sn);
}

}  // namespace sphkv

using namespace sphkv;

extern "C" int sphkv_recon_keys(const sphkv_store_t* st, const int32_t* pages,
                                const int64_t* item_off, int n_pages, void* out, int out_dtype,
                                cudaStream_t stream) {
  if (!st || !pages || !item_off || !out) return fail(SPHKV_E_VALUE, "null argument");
  if (st->d < 3) return fail(SPHKV_E_UNSUPPORTED, "d=%d", st->d);
  for (int t = 1; t < st->n_tiers; ++t)
    if (st->tiers[t].angle_bits > 16 || st->tiers[t].radius_bits > 16)
      return fail(SPHKV_E_UNSUPPORTED, "tier %d: code widths above 16 bits", st->tiers[t].id);
  if (n_pages == 0) return SPHKV_OK;
  const int chunks = (st->page_size + 31) / 32;
  const int64_t threads = (int64_t)n_pages * chunks * 32;
  const int block = 256;
  const int grid = (int)div_up(threads, block);
  if (out_dtype == SPHKV_F32)
    k_recon_keys<float><<<grid, block, 0, stream>>>(*st, pages, item_off, n_pages,
                                                    static_cast<float*>(out));
  else if (out_dtype == SPHKV_F16)
    k_recon_keys<__half><<<grid, block, 0, stream>>>(*st, pages, item_off, n_pages,
                                                     static_cast<__half*>(out));
  else
    return fail(SPHKV_E_UNSUPPORTED, "recon output dtype %d (f32 / f16 only)", out_dtype);
  SPHKV_LAUNCH_CHECK();
  return SPHKV_OK;
}
