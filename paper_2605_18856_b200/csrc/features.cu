// Controller features from a sampled dense prefill pass.
//
// Reference behaviour replaced (pkg/src/sphkv/controller.py:99-142,
// compute_features): per (layer, head), for <= 512 sampled prefill rows r,
//   logits_j = q_r . k_j / sqrt(d) for j <= r (causal), softmax over j,
//   reuse   u_r = sum of the weights of "old" tokens j <= r - window,
//   margin  m_r = top-1 minus top-2 logit (rows r >= 1),
// u_raw = mean_r u_r, inv_margin = mean_{r >= 1} 1 / (m_r + 1e-6).  The host
// normalizes across heads (u_hat = u_raw / max, s_hat = 1 - inv / max).
//
// One block per (group, 16 sampled rows): the 16 fp64 query rows stay in
// shared memory, keys stream through a 64-token fp64 tile (one padded row
// per token: conflict-free column reads), every thread keeps an online
// softmax state (max, sum, old-token sum, top-2) for one row over a strided
// token subset; the 16 threads of a row merge their states with shuffles.
// Everything is fp64 (the reference's numpy dtype); summation order differs
// from numpy's (BLAS dot, pairwise sums) at the 1e-16 relative level.
#include "common.cuh"

namespace sphkv {

constexpr int CF_ROWS = 16;    // sampled rows per block
constexpr int CF_TOK = 64;     // tokens per key tile
constexpr int CF_THREADS = 256;

struct RowState {
  double m, s, so, t1, t2;  // running max, sum exp(l - m), old-token sum, top-2 logits
};

__device__ __forceinline__ void rs_add(RowState& a, double l, bool old) {
  if (l > a.m) {
    const double c = exp(a.m - l);  // (a.m = -inf: c = 0)
    a.s = a.s * c + 1.0;
    a.so = a.so * c + (old ? 1.0 : 0.0);
    a.m = l;
  } else {
    const double e = exp(l - a.m);
    a.s += e;
    if (old) a.so += e;
  }
  if (l > a.t1) {
    a.t2 = a.t1;
    a.t1 = l;
  } else if (l > a.t2) {
    a.t2 = l;
  }
}

__device__ __forceinline__ void rs_merge(RowState& a, const RowState& b) {
  const double M = fmax(a.m, b.m);
  const double ca = (a.m == -INFINITY) ? 0.0 : exp(a.m - M);
  const double cb = (b.m == -INFINITY) ? 0.0 : exp(b.m - M);
  a.s = a.s * ca + b.s * cb;
  a.so = a.so * ca + b.so * cb;
  a.m = M;
  const double hi = fmax(a.t1, b.t1);
  const double lo = fmax(fmin(a.t1, b.t1), fmax(a.t2, b.t2));
  a.t1 = hi;
  a.t2 = lo;
}

template <typename T>
__global__ void __launch_bounds__(CF_THREADS) k_ctrl_rows(const T* __restrict__ keys,
                                                          const double* __restrict__ q,
                                                          const int32_t* __restrict__ rows, int R,
                                                          int T_, int d, int window, int qpk,
                                                          double* __restrict__ row_out) {
  extern __shared__ double cf_smem[];
  const int blocks_per_group = (R + CF_ROWS - 1) / CF_ROWS;
  const int64_t g = blockIdx.x / blocks_per_group;
  const int r0 = (blockIdx.x % blocks_per_group) * CF_ROWS;
  const int dp = d + 1;  // padded fp64 row (bank-conflict free column reads)
  double* qs = cf_smem;                 // [CF_ROWS][dp]
  double* ks = cf_smem + CF_ROWS * dp;  // [CF_TOK][dp]
  const int nr = min(CF_ROWS, R - r0);
  for (int i = threadIdx.x; i < CF_ROWS * d; i += blockDim.x) {
    const int rr = i / d, c = i % d;
    qs[rr * dp + c] = rr < nr ? q[((g * R) + r0 + rr) * (int64_t)d + c] : 0.0;
  }
  const int ri = threadIdx.x / 16, sub = threadIdx.x % 16;  // row, token lane
  const int row = ri < nr ? rows[r0 + ri] : -1;
  int max_row = 0;
  for (int i = 0; i < nr; ++i) max_row = max(max_row, rows[r0 + i]);
  RowState st{-INFINITY, 0.0, 0.0, -INFINITY, -INFINITY};
  const double inv_sqrt_d = 1.0 / sqrt((double)d);
  const T* kg = keys + (g / qpk) * (int64_t)T_ * d;  // qpk query groups share a key group
  for (int t0 = 0; t0 <= max_row; t0 += CF_TOK) {  // causal: tokens beyond every row skipped
    __syncthreads();
    for (int i = threadIdx.x; i < CF_TOK * d; i += blockDim.x) {
      const int tk = i / d, c = i % d;
      ks[tk * dp + c] = (t0 + tk < T_) ? load_as_double(kg + (int64_t)(t0 + tk) * d + c) : 0.0;
    }
    __syncthreads();
    if (row < 0) continue;
#pragma unroll
    for (int k = 0; k < CF_TOK / 16; ++k) {
      const int tk = sub + 16 * k, j = t0 + tk;
      if (j > row || j >= T_) continue;
      const double* kr = ks + tk * dp;
      const double* qr = qs + ri * dp;
      double acc = 0.0;
      for (int c = 0; c < d; ++c) acc = fma(qr[c], kr[c], acc);
      rs_add(st, acc * inv_sqrt_d, j <= row - window);
    }
  }
  // merge the 16 token lanes of each row (lanes of one row are contiguous)
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) {
    RowState b;
    b.m = __shfl_xor_sync(0xffffffffu, st.m, o);
    b.s = __shfl_xor_sync(0xffffffffu, st.s, o);
    b.so = __shfl_xor_sync(0xffffffffu, st.so, o);
    b.t1 = __shfl_xor_sync(0xffffffffu, st.t1, o);
    b.t2 = __shfl_xor_sync(0xffffffffu, st.t2, o);
    rs_merge(st, b);
  }
  if (sub == 0 && row >= 0) {
    double* o = row_out + ((g * R) + r0 + ri) * 2;
    o[0] = st.so / st.s;                                           // old-token weight
    o[1] = row >= 1 ? 1.0 / ((st.t1 - st.t2) + 1e-6) : 0.0;        // inverse margin
  }
}

// per group: means over the sampled rows (sequential sums, row order)
__global__ void k_ctrl_reduce(const double* __restrict__ row_out, const int32_t* __restrict__ rows,
                              int R, int64_t groups, double* __restrict__ u_raw,
                              double* __restrict__ inv_margin) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= groups) return;
  double su = 0.0, sm = 0.0;
  int nm = 0;
  for (int i = 0; i < R; ++i) {
    su += row_out[(g * R + i) * 2];
    if (rows[i] >= 1) {
      sm += row_out[(g * R + i) * 2 + 1];
      ++nm;
    }
  }
  u_raw[g] = su / (double)R;
  inv_margin[g] = nm ? sm / (double)nm : 0.0;
}

}  // namespace sphkv

using namespace sphkv;

extern "C" int64_t sphkv_controller_workspace_bytes(int64_t groups, int R) {
  return groups * (int64_t)R * 2 * (int64_t)sizeof(double) + 256;
}

extern "C" int sphkv_controller_stats(const void* keys, int key_dtype, const double* q_rows,
                                      const int32_t* rows, int R, int64_t groups, int tokens,
                                      int d, int window, int q_per_key, double* u_raw,
                                      double* inv_margin, void* workspace, cudaStream_t stream) {
  if (groups < 0 || R < 0 || tokens < 0 || d < 1) return fail(SPHKV_E_VALUE, "bad shape");
  if (groups == 0 || R == 0) return SPHKV_OK;
  if (!keys || !q_rows || !rows || !u_raw || !inv_margin || !workspace)
    return fail(SPHKV_E_VALUE, "null argument");
  if (d > 256) return fail(SPHKV_E_UNSUPPORTED, "d=%d > 256", d);
  if (q_per_key < 1 || groups % q_per_key) return fail(SPHKV_E_VALUE, "q_per_key %d", q_per_key);
  const int bpg = (R + CF_ROWS - 1) / CF_ROWS;
  if (groups * bpg > 0x7fffffffLL) return fail(SPHKV_E_UNSUPPORTED, "too many groups");
  const size_t smem = (size_t)(CF_ROWS + CF_TOK) * (d + 1) * sizeof(double);
  double* row_out = static_cast<double*>(workspace);
  const unsigned grid = (unsigned)(groups * bpg);
#define SPHKV_CF(T)                                                                        \
  do {                                                                                     \
    SPHKV_CUDA_TRY(cudaFuncSetAttribute(k_ctrl_rows<T>,                                    \
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                                        (int)smem));                                       \
    k_ctrl_rows<T><<<grid, CF_THREADS, smem, stream>>>((const T*)keys, q_rows, rows, R,    \
                                                       tokens, d, window, q_per_key,       \
                                                       row_out);                           \
  } while (0)
  switch (key_dtype) {
    case SPHKV_F32: SPHKV_CF(float); break;
    case SPHKV_F64: SPHKV_CF(double); break;
    case SPHKV_BF16: SPHKV_CF(__nv_bfloat16); break;
    case SPHKV_F16: SPHKV_CF(__half); break;
    default: return fail(SPHKV_E_VALUE, "unknown key dtype %d", key_dtype);
  }
#undef SPHKV_CF
  SPHKV_LAUNCH_CHECK();
  k_ctrl_reduce<<<(unsigned)((groups + 127) / 128), 128, 0, stream>>>(row_out, rows, R, groups,
                                                                      u_raw, inv_margin);
  SPHKV_LAUNCH_CHECK();
  return SPHKV_OK;
}
