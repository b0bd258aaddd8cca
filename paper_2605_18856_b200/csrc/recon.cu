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
// kernel exists to avoid.  k_recon_dot then re-reads the rows for the logits
// of all G query heads.  Both are plain HBM streams (coalesced 16-byte
// accesses through shared memory), so their DRAM counters measure the tax
// itself rather than a slow kernel.
#include "common.cuh"

#include <algorithm>

namespace sphkv {

constexpr int RC_WARPS = 4;
// shared-memory row stride in 32-bit words for d elements of `esz` bytes: odd
__host__ __device__ inline int recon_row_words(int d, int esz) { return (d * esz / 4) | 1; }

// One warp per 32-item chunk of a page, lane = item.  A lane runs the
// feature recurrence of its item into a shared-memory row (fp32 math, output
// type OutT); the warp then writes the 32 rows out as contiguous words
// (consecutive lanes -> consecutive addresses, 128 bytes per warp store).
template <typename OutT>
__global__ void __launch_bounds__(RC_WARPS * 32) k_recon_keys(sphkv_store_t st,
                                                              const int32_t* __restrict__ pages,
                                                              const int64_t* __restrict__ item_off,
                                                              int n_pages, OutT* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t rc_smem[];
  const int d = st.d;
  // padded row: an odd number of 32-bit words, so the 32 lanes' row writes
  // (one row per lane) fall in distinct banks
  const int rsw = recon_row_words(d, (int)sizeof(OutT)), rs = rsw * 4 / (int)sizeof(OutT);
  OutT* rows = reinterpret_cast<OutT*>(rc_smem) + (size_t)(threadIdx.x >> 5) * 32 * rs;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int chunks = (st.page_size + 31) / 32;
  if (warp >= n_pages * chunks) return;
  const int pi = warp / chunks, slot0 = (warp % chunks) * 32, slot = slot0 + lane;
  const sphkv_page_t pg = st.pages[pages[pi]];
  const int n_here = min(32, pg.count - slot0);
  if (n_here <= 0) return;
  if (slot < pg.count) {
    const int b = pg.abits, W = item_words(d, b);
    const uint32_t* words = reinterpret_cast<const uint32_t*>(st.codes + pg.code_off);
    auto code = [&](int bit, int n) -> uint32_t {
      const int w0 = bit >> 5, sh = bit & 31;
      const uint32_t lo = __ldg(words + wi_word(slot, w0, W));
      const uint32_t hi = (sh + n > 32) ? __ldg(words + wi_word(slot, w0 + 1, W)) : 0u;
      return __funnelshift_r(lo, hi, sh) & ((1u << n) - 1u);
    };
    // decoded radius r~ = code / levels * scale (decode.py:137-139)
    const uint64_t rbit = angle_part_bytes(d, st.page_size, b) * 8 + (uint64_t)slot * pg.rbits;
    const uint32_t* rw = words + (rbit >> 5);
    const int rsh = (int)(rbit & 31);
    const uint32_t rhi = (rsh + pg.rbits > 32) ? rw[1] : 0u;
    const uint32_t rc = __funnelshift_r(rw[0], rhi, rsh) & ((1u << pg.rbits) - 1u);
    const float r = (float)((double)rc / (double)((1u << pg.rbits) - 1u) * pg.radius_scale);
    OutT* row = rows + (size_t)lane * rs;
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
  __syncwarp();
  // coalesced write-out: the chunk's rows are contiguous in `out`
  OutT* dst = out + (item_off[pi] + slot0) * (int64_t)d;
  const int wpr = d * (int)sizeof(OutT) / 4;  // whole words per row (d even for fp16)
  const uint32_t* src = reinterpret_cast<const uint32_t*>(rows);
  uint32_t* dw = reinterpret_cast<uint32_t*>(dst);
  for (int c = lane; c < n_here * wpr; c += 32) dw[c] = src[(c / wpr) * rsw + c % wpr];
}

// Re-read of the staged rows: out[i * G + g] = q_g . k_i / sqrt(d) for the
// rows of one group (rows [row0, row0 + n)).  A block stages 128 rows in
// shared memory with coalesced 16-byte loads, then thread pairs form one
// row's dots for all G heads (q in shared memory).
template <typename InT>
__global__ void __launch_bounds__(256) k_recon_dot(const InT* __restrict__ stage, int64_t n, int d,
                                                   const float* __restrict__ q, int G,
                                                   float* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t rd_smem[];
  const int rsw = recon_row_words(d, (int)sizeof(InT));
  uint32_t* tile = reinterpret_cast<uint32_t*>(rd_smem);
  float* qs = reinterpret_cast<float*>(rd_smem + (size_t)128 * rsw * 4);
  for (int i = threadIdx.x; i < G * d; i += blockDim.x) qs[i] = q[i];
  const float inv = rsqrtf((float)d);
  const int per_row = d * (int)sizeof(InT) / 16;  // 16-byte chunks per row
  for (int64_t r0 = (int64_t)blockIdx.x * 128; r0 < n; r0 += (int64_t)gridDim.x * 128) {
    const int nr = (n - r0 < 128) ? (int)(n - r0) : 128;
    __syncthreads();
    const uint4* src = reinterpret_cast<const uint4*>(stage + r0 * d);
    for (int c = threadIdx.x; c < nr * per_row; c += blockDim.x) {
      const uint4 v = __ldcs(src + c);  // streamed once: evict-first
      uint32_t* t = tile + (c / per_row) * rsw + (c % per_row) * 4;
      t[0] = v.x;
      t[1] = v.y;
      t[2] = v.z;
      t[3] = v.w;
    }
    __syncthreads();
    const int rr = threadIdx.x >> 1, half = threadIdx.x & 1;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (rr < nr) {
      const InT* row = reinterpret_cast<const InT*>(tile + (size_t)rr * rsw);
      for (int j = half; j < d; j += 2) {
        const float k = (float)row[j];
#pragma unroll
        for (int g = 0; g < 8; ++g)
          if (g < G) acc[g] += k * qs[g * d + j];
      }
    }
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      const float v = acc[g] + __shfl_xor_sync(0xffffffffu, acc[g], 1);
      if (g < G && half == 0 && rr < nr) out[(r0 + rr) * G + g] = v * inv;
    }
  }
}

}  // namespace sphkv

using namespace sphkv;

extern "C" int sphkv_recon_keys(const sphkv_store_t* st, const int32_t* pages,
                                const int64_t* item_off, int n_pages, void* out, int out_dtype,
                                cudaStream_t stream) {
  if (!st || !pages || !item_off || !out) return fail(SPHKV_E_VALUE, "null argument");
  if (st->d < 3 || st->d > 256) return fail(SPHKV_E_UNSUPPORTED, "d=%d outside [3, 256]", st->d);
  for (int t = 1; t < st->n_tiers; ++t)
    if (st->tiers[t].angle_bits > 16 || st->tiers[t].radius_bits > 16)
      return fail(SPHKV_E_UNSUPPORTED, "tier %d: code widths above 16 bits", st->tiers[t].id);
  if (n_pages == 0) return SPHKV_OK;
  const int chunks = (st->page_size + 31) / 32;
  const int64_t warps = (int64_t)n_pages * chunks;
  const int grid = (int)div_up(warps, RC_WARPS);
  if (out_dtype == SPHKV_F32) {
    const size_t smem = (size_t)RC_WARPS * 32 * recon_row_words(st->d, 4) * 4;
    SPHKV_CUDA_TRY(cudaFuncSetAttribute(k_recon_keys<float>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_recon_keys<float><<<grid, RC_WARPS * 32, smem, stream>>>(*st, pages, item_off, n_pages,
                                                               static_cast<float*>(out));
  } else if (out_dtype == SPHKV_F16) {
    if (st->d % 2) return fail(SPHKV_E_UNSUPPORTED, "fp16 staging needs an even d (d=%d)", st->d);
    const size_t smem = (size_t)RC_WARPS * 32 * recon_row_words(st->d, 2) * 4;
    SPHKV_CUDA_TRY(cudaFuncSetAttribute(k_recon_keys<__half>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_recon_keys<__half><<<grid, RC_WARPS * 32, smem, stream>>>(*st, pages, item_off, n_pages,
                                                                static_cast<__half*>(out));
  } else {
    return fail(SPHKV_E_UNSUPPORTED, "recon output dtype %d (f32 / f16 only)", out_dtype);
  }
  SPHKV_LAUNCH_CHECK();
  return SPHKV_OK;
}

extern "C" int sphkv_recon_dot(const void* stage, int stage_dtype, int64_t n, int d,
                               const float* q, int G, float* out, cudaStream_t stream) {
  if (n < 0 || d < 1) return fail(SPHKV_E_VALUE, "bad shape");
  if (n == 0) return SPHKV_OK;
  if (!stage || !q || !out) return fail(SPHKV_E_VALUE, "null argument");
  if (G < 1 || G > 8) return fail(SPHKV_E_UNSUPPORTED, "GQA group size %d outside [1, 8]", G);
  const int esz = stage_dtype == SPHKV_F32 ? 4 : 2;
  if (stage_dtype != SPHKV_F32 && stage_dtype != SPHKV_F16)
    return fail(SPHKV_E_UNSUPPORTED, "stage dtype %d (f32 / f16 only)", stage_dtype);
  if ((d * esz) % 16 != 0 || d > 256)
    return fail(SPHKV_E_UNSUPPORTED, "d=%d: rows must be whole 16-byte chunks, d <= 256", d);
  const size_t smem = (size_t)128 * recon_row_words(d, esz) * 4 + (size_t)G * d * 4;
  const int grid = (int)std::min<int64_t>(div_up(n, 128), 4 * SM_COUNT);
  if (stage_dtype == SPHKV_F32) {
    SPHKV_CUDA_TRY(cudaFuncSetAttribute(k_recon_dot<float>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_recon_dot<float><<<grid, 256, smem, stream>>>(static_cast<const float*>(stage), n, d, q, G,
                                                    out);
  } else {
    SPHKV_CUDA_TRY(cudaFuncSetAttribute(k_recon_dot<__half>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_recon_dot<__half><<<grid, 256, smem, stream>>>(static_cast<const __half*>(stage), n, d, q,
                                                     G, out);
  }
  SPHKV_LAUNCH_CHECK();
  return SPHKV_OK;
}
