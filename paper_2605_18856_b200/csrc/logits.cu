// Dense logit kernels for the reference-shaped API (not the decode hot path).
//
// Reference behaviour replaced (pkg/src/sphkv/):
//   decode.py:63-69    dense_logits(q, keys) = keys @ q / sqrt(d), fp64
//   decode.py:302-307  _head_attend("dense"): the dense store's logits of one
//                      (layer, head) in token order (store.py:533-546)
#include "common.cuh"

namespace sphkv {

// one warp per key row, fp64 products, warp-tree sum, then / sqrt(d) as numpy
// does (a division by math.sqrt(d), decode.py:69)
__global__ void k_dense_logits_f64(const double* __restrict__ q, const double* __restrict__ keys,
                                   int64_t n, int d, double* __restrict__ out) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const double* k = keys + row * d;
  double acc = 0.0;
  for (int j = lane; j < d; j += 32) acc = fma(k[j], q[j], acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) out[row] = acc / sqrt((double)d);
}

// Logits of every token of one dense-store group for G query heads:
// out[t * G + g] = q_g . k_t / sqrt(d) (fp32 math over the bf16 pages).
// One warp per token row; the row's swizzled 16-byte chunks are read as
// 32-bit pairs.
__global__ void k_dense_store_logits(sphkv_dense_store_t st, const float* __restrict__ q, int G,
                                     int group, float* __restrict__ out) {
  extern __shared__ float qs[];  // [G][dp]
  const int dp = (st.d + 15) / 16 * 16;
  for (int i = threadIdx.x; i < G * dp; i += blockDim.x) {
    const int g = i / dp, e = i % dp;
    qs[i] = e < st.d ? q[g * st.d + e] : 0.f;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (t >= st.tokens) return;
  const int P = st.page_size;
  const int64_t item0 = ((int64_t)group * st.n_pages_per_group * P + (t / P) * P);
  const int i = (int)(t % P);
  const uint16_t* row = st.keys + item0 * dp;
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int e = 2 * lane; e < st.d; e += 64) {
    const uint32_t w = *reinterpret_cast<const uint32_t*>(row + vswz(i, e, dp));
    const float k0 = __uint_as_float(w << 16), k1 = __uint_as_float(w & 0xffff0000u);
    for (int g = 0; g < G && g < 8; ++g) acc[g] += k0 * qs[g * dp + e] + k1 * qs[g * dp + e + 1];
  }
  const float inv = rsqrtf((float)st.d);
  for (int g = 0; g < G && g < 8; ++g) {
    float v = acc[g];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) out[t * G + g] = v * inv;
  }
}

}  // namespace sphkv

using namespace sphkv;

extern "C" int sphkv_dense_logits(const double* q, const double* keys, int64_t n, int d,
                                  double* out, cudaStream_t stream) {
  if (n < 0 || d < 1) return fail(SPHKV_E_VALUE, "bad shape n=%lld d=%d", (long long)n, d);
  if (n == 0) return SPHKV_OK;
  if (!q || !keys || !out) return fail(SPHKV_E_VALUE, "null argument");
  const int64_t threads = n * 32;
  k_dense_logits_f64<<<(unsigned)div_up(threads, 256), 256, 0, stream>>>(q, keys, n, d, out);
  SPHKV_LAUNCH_CHECK();
  return SPHKV_OK;
}

extern "C" int sphkv_dense_store_logits(const sphkv_dense_store_t* st, const float* q, int G,
                                        int group, float* out, cudaStream_t stream) {
  if (!st || !q || !out) return fail(SPHKV_E_VALUE, "null argument");
  if (G < 1 || G > 8) return fail(SPHKV_E_UNSUPPORTED, "GQA group size %d outside [1, 8]", G);
  if (st->d < 2 || st->d % 2 != 0 || st->d > 256)
    return fail(SPHKV_E_UNSUPPORTED, "d=%d (even, <= 256)", st->d);
  const int64_t groups = (int64_t)st->batch * st->layers * st->heads;
  if (group < 0 || group >= groups) return fail(SPHKV_E_KEY, "group %d outside [0, %lld)", group,
                                                (long long)groups);
  if (st->tokens == 0) return SPHKV_OK;
  const int dp = (st->d + 15) / 16 * 16;
  const int64_t threads = (int64_t)st->tokens * 32;
  k_dense_store_logits<<<(unsigned)div_up(threads, 256), 256, G * dp * sizeof(float), stream>>>(
      *st, q, G, group, out);
  SPHKV_LAUNCH_CHECK();
  return SPHKV_OK;
}
