// RDR controller: vectorized scoring, greedy allocation and down-tiering.
// Compiled with --fmad=false (bit-exact fp64, numpy operation order).
//
// Reference behaviour replaced (pkg/src/sphkv/controller.py):
//   :213-245  score_states  (w_theta, w_r, strict-> argmax, nu)
//   :301-346  allocate_greedy  lexsort(-nu, l, h, tok) + sequential fit
//   :349-398  downtier_before_drop from the full best-tier start
//
// Exact parallel forms:
//   greedy  : stable radix sort of the free states on (-nu); then rounds of
//             "inclusive scan of eligible costs -> first overflow -> cap".  A
//             rejection at cost c rejects every later item of cost >= c since
//             the remaining budget only shrinks, so rounds <= #distinct rates.
//   downtier: the while-loop drops a prefix of the ascending-nu order and
//             partially demotes one boundary state: one scan + a scalar step.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include "common.cuh"

namespace sphkv {

__global__ void k_rdr_score(const double* __restrict__ radii, const double* __restrict__ u_hat,
                            const double* __restrict__ s_hat, const double* __restrict__ seg_omega,
                            double r_q, double at, double ar, const TierSet tiers_arr,
                            int NT, double lam, const uint8_t* __restrict__ protect, int LH, int T,
                            int d, int16_t* best_tier, double* score, double* nu, double* d_drop_out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)LH * T) return;
  const int lh = (int)(i / T), tok = (int)(i % T);
  const double sqrt_d = __dsqrt_rn((double)d);
  const double om = seg_omega[tok];
  // w_theta = alpha_theta * u_hat[:,:,None] * om * (r_q * radii / sqrt_d)
  const double w_theta = __dmul_rn(__dmul_rn(__dmul_rn(at, u_hat[lh]), om),
                                   __ddiv_rn(__dmul_rn(r_q, radii[i]), sqrt_d));
  // w_r = alpha_r * (1.0 - s_hat[:,:,None]) * om * (r_q / sqrt_d)
  const double w_r = __dmul_rn(__dmul_rn(__dmul_rn(ar, __dadd_rn(1.0, -s_hat[lh])), om),
                               __ddiv_rn(r_q, sqrt_d));
  const double dd = __dadd_rn(w_theta, w_r);
  int best = 0;
  double bs = protect[i] ? -INFINITY : -dd;
  for (int t = 1; t < NT; ++t) {
    const sphkv_tier_t tt = tiers_arr.t[t];
    const int rate = (d - 1) * tt.angle_bits + tt.radius_bits + tt.meta_bits;
    double s = __dadd_rn(-__dadd_rn(__dmul_rn(w_theta, tt.eps_theta), __dmul_rn(w_r, tt.eps_r)),
                         -__dmul_rn(lam, (double)rate));
    if (s > bs) {
      bs = s;
      best = t;
    }
  }
  double db, rb;
  if (best == 0) {
    db = __dadd_rn(__dmul_rn(w_theta, 1.0), __dmul_rn(w_r, 1.0));
    rb = 0.0;
  } else {
    const sphkv_tier_t tt = tiers_arr.t[best];
    db = __dadd_rn(__dmul_rn(w_theta, tt.eps_theta), __dmul_rn(w_r, tt.eps_r));
    rb = (double)((d - 1) * tt.angle_bits + tt.radius_bits + tt.meta_bits);
  }
  best_tier[i] = (int16_t)tiers_arr.t[best].id;
  if (score) score[i] = bs;
  if (nu) nu[i] = __ddiv_rn(__dadd_rn(dd, -db), __dadd_rn(rb, 1e-12));
  if (d_drop_out) d_drop_out[i] = dd;
}

// order-preserving uint64 of a double, -0.0 canonicalized to +0.0; protected
// states get the max key so they sort past every free state
__device__ __forceinline__ uint64_t okey(double x) {
  if (x == 0.0) x = 0.0;
  uint64_t b = (uint64_t)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void k_keys(const double* __restrict__ nu, const uint8_t* __restrict__ protect,
                       int64_t n, int negate, uint64_t* keys, int64_t* idx) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = negate ? -nu[i] : nu[i];
  keys[i] = protect[i] ? ~0ull : okey(v);
  idx[i] = i;
}

struct TierRates {
  int id[SPHKV_MAX_TIERS];
  int rate[SPHKV_MAX_TIERS];
  int below[SPHKV_MAX_TIERS];  // tier id one step down (controller.py:360)
  int n;
};

__device__ __forceinline__ int rate_of(const TierRates& tr, int id) {
  for (int t = 0; t < tr.n; ++t)
    if (tr.id[t] == id) return tr.rate[t];
  return 0;
}

__global__ void k_init_assign(const int16_t* __restrict__ start, const uint8_t* __restrict__ protect,
                              int64_t n, int max_id, int keep_start, int8_t* z, int16_t* tier) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int t = protect[i] ? max_id : (keep_start ? start[i] : 0);
  tier[i] = (int16_t)t;
  z[i] = t != 0 ? 1 : 0;
}

// per sorted position: cost of the state's best tier (0 = never retained)
__global__ void k_costs(const int64_t* __restrict__ sidx, const int16_t* __restrict__ best,
                        const uint8_t* __restrict__ protect, int64_t n, TierRates tr,
                        int32_t* cost) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t s = sidx[i];
  cost[i] = protect[s] ? 0 : rate_of(tr, best[s]);
}

// Device-resident state of the greedy rounds (no host round trips): the
// scan position p, the remaining budget R, the cost cap and the first
// rejected sorted position of the current round.
struct GreedyState {
  long long p, R;
  int cap, finished;
  unsigned long long first;
};

__global__ void k_greedy_init(GreedyState* gs, const unsigned long long* n_prot, long long budget,
                              long long max_rate, int* status) {
  const long long R = budget - (long long)*n_prot * max_rate;
  gs->p = 0;
  gs->R = R;
  gs->cap = 0x7fffffff;
  gs->finished = R < 0;
  gs->first = ~0ull;
  *status = R < 0 ? 1 : 0;  // 1: infeasible protection (controller.py:316-322)
}

__global__ void k_masked(const int32_t* __restrict__ cost, const uint8_t* __restrict__ done,
                         int64_t n, const GreedyState* __restrict__ gs, int64_t* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t c = cost[i];
  out[i] = (!gs->finished && i >= gs->p && !done[i] && c > 0 && c < gs->cap) ? (int64_t)c : 0;
}

// masked[i] = 0 below p, so scan[i] is the cost taken since p
__global__ void k_first_over_gs(const int64_t* __restrict__ scan, const int64_t* __restrict__ masked,
                                int64_t n, GreedyState* gs) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n || gs->finished || i < gs->p) return;
  if (masked[i] > 0 && scan[i] > gs->R) atomicMin(&gs->first, (unsigned long long)i);
}

__global__ void k_accept_gs(const int64_t* __restrict__ sidx, const int16_t* __restrict__ best,
                            const int64_t* __restrict__ masked, int64_t n,
                            const GreedyState* __restrict__ gs, uint8_t* done, int8_t* z,
                            int16_t* tier) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n || gs->finished || i < gs->p || (unsigned long long)i >= gs->first) return;
  if (masked[i] > 0) {
    int64_t s = sidx[i];
    z[s] = 1;
    tier[s] = best[s];
    done[i] = 1;
  }
}

// end of a round: the first rejected item shrinks the budget and the cap
__global__ void k_greedy_update(const int64_t* __restrict__ scan, const int32_t* __restrict__ cost,
                                int64_t n, GreedyState* gs) {
  if (gs->finished) return;
  const unsigned long long first = gs->first;
  if (first == ~0ull) {
    gs->finished = 1;
    return;
  }
  const int64_t hi = (int64_t)first;
  gs->R -= hi > 0 ? scan[hi - 1] : 0;
  gs->cap = min(gs->cap, cost[hi]);
  gs->p = hi + 1;
  gs->first = ~0ull;
  if (gs->p >= n) gs->finished = 1;
}

__global__ void k_first_over(const int64_t* __restrict__ scan, const int64_t* __restrict__ masked,
                             int64_t n, int64_t p, int64_t R, unsigned long long* first) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < p || i >= n) return;
  if (masked[i] > 0 && scan[i] > R) atomicMin(first, (unsigned long long)i);
}

__global__ void k_accept(const int64_t* __restrict__ sidx, const int16_t* __restrict__ best,
                         const int64_t* __restrict__ masked, int64_t lo, int64_t hi, uint8_t* done,
                         int8_t* z, int16_t* tier) {
  int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= hi) return;
  if (masked[i] > 0) {
    int64_t s = sidx[i];
    z[s] = 1;
    tier[s] = best[s];
    done[i] = 1;
  }
}

__global__ void k_rates_sorted(const int64_t* __restrict__ sidx, const int16_t* __restrict__ tier,
                               const uint8_t* __restrict__ protect, int64_t n, TierRates tr,
                               int64_t* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t s = sidx[i];
  out[i] = protect[s] ? 0 : (int64_t)rate_of(tr, tier[s]);
}

__global__ void k_total_rate(const int16_t* __restrict__ tier, int64_t n, TierRates tr,
                             unsigned long long* total) {
  __shared__ unsigned long long red[32];
  unsigned long long s = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    s += (unsigned long long)rate_of(tr, tier[i]);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    atomicAdd(total, s);
  }
}

__global__ void k_count_protect(const uint8_t* __restrict__ protect, int64_t n,
                                unsigned long long* cnt) {
  unsigned long long s = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    s += protect[i] ? 1 : 0;
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(cnt, s);
}

__global__ void k_drop_prefix(const int64_t* __restrict__ sidx, int64_t k, int8_t* z,
                              int16_t* tier, const uint8_t* __restrict__ protect) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= k) return;
  int64_t s = sidx[i];
  if (protect[s]) return;
  z[s] = 0;
  tier[s] = 0;
}

}  // namespace sphkv

using namespace sphkv;

static TierRates make_rates(const sphkv_tier_t* tiers, int NT, int d) {
  TierRates tr;
  memset(&tr, 0, sizeof(tr));
  tr.n = NT;
  for (int t = 0; t < NT; ++t) {
    tr.id[t] = tiers[t].id;
    tr.rate[t] = t == 0 ? 0 : (d - 1) * tiers[t].angle_bits + tiers[t].radius_bits + tiers[t].meta_bits;
    tr.below[t] = t == 0 ? 0 : tiers[t - 1].id;
  }
  return tr;
}

extern "C" int sphkv_rdr_score(const double* radii, const double* u_hat, const double* s_hat,
                               const double* seg_omega, double r_q, double alpha_theta,
                               double alpha_r, const sphkv_tier_t* tiers_host, int n_tiers,
                               double lam, const uint8_t* protect, int layers, int heads,
                               int tokens, int d, int16_t* best_tier, double* score, double* nu,
                               double* d_drop, cudaStream_t stream) {
  if (n_tiers < 1 || n_tiers > SPHKV_MAX_TIERS) return fail(SPHKV_E_VALUE, "bad tier count");
  if (d < 2) return fail(SPHKV_E_VALUE, "head dimension must be >= 2");
  int64_t n = (int64_t)layers * heads * tokens;
  if (n == 0) return SPHKV_OK;
  k_rdr_score<<<(int)div_up(n, 256), 256, 0, stream>>>(radii, u_hat, s_hat, seg_omega, r_q,
                                                       alpha_theta, alpha_r,
                                                       make_tierset(tiers_host, n_tiers), n_tiers,
                                                       lam, protect, layers * heads, tokens, d,
                                                       best_tier, score, nu, d_drop);
  SPHKV_LAUNCH_CHECK();
  return SPHKV_OK;
}

namespace {
struct RdrWs {
  uint64_t *k0, *k1;
  int64_t *i0, *i1;
  int32_t* cost;
  int64_t *masked, *scan;
  uint8_t* done;
  unsigned long long* scal;  // [0]=first [1]=count/total
  void* cub;
  size_t cub_bytes;
};

size_t cub_need(int64_t n) {
  size_t a = 0, b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, (uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (int64_t*)nullptr, (int64_t*)nullptr, (int)n);
  cub::DeviceScan::InclusiveSum(nullptr, b, (int64_t*)nullptr, (int64_t*)nullptr, (int)n);
  return (a > b ? a : b) + 256;
}

RdrWs carve(void* base, int64_t n) {
  uint8_t* p = (uint8_t*)base;
  auto take = [&](size_t bytes) {
    uint8_t* r = p;
    p += (bytes + 255) / 256 * 256;
    return r;
  };
  RdrWs w;
  w.k0 = (uint64_t*)take(n * 8);
  w.k1 = (uint64_t*)take(n * 8);
  w.i0 = (int64_t*)take(n * 8);
  w.i1 = (int64_t*)take(n * 8);
  w.cost = (int32_t*)take(n * 4);
  w.masked = (int64_t*)take(n * 8);
  w.scan = (int64_t*)take(n * 8);
  w.done = (uint8_t*)take(n);
  w.scal = (unsigned long long*)take(64);
  w.cub_bytes = cub_need(n);
  w.cub = take(w.cub_bytes);
  return w;
}

// stable sort of all states by key; returns sorted index array
int sort_states(RdrWs& w, const double* nu, const uint8_t* protect, int64_t n, int negate,
                int64_t** sidx, cudaStream_t stream) {
  k_keys<<<(int)div_up(n, 256), 256, 0, stream>>>(nu, protect, n, negate, w.k0, w.i0);
  SPHKV_LAUNCH_CHECK();
  size_t tb = w.cub_bytes;
  SPHKV_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.cub, tb, w.k0, w.k1, w.i0, w.i1, (int)n, 0, 64,
                                                 stream));
  *sidx = w.i1;
  return SPHKV_OK;
}
}  // namespace

extern "C" int64_t sphkv_rdr_workspace_bytes(int64_t n) {
  int64_t per = 8 * 4 + 4 + 8 * 2 + 1;
  return n * per + 16 * 256 + 64 + (int64_t)cub_need(n) + 4096;
}

extern "C" int sphkv_rdr_allocate_greedy(const int16_t* best_tier, const double* nu,
                                         const uint8_t* protect, int64_t n,
                                         const sphkv_tier_t* tiers_host, int n_tiers, int d,
                                         int64_t budget_bits, void* workspace, int8_t* z,
                                         int16_t* tier, cudaStream_t stream) {
  if (budget_bits < 0) return fail(SPHKV_E_VALUE, "budget must be nonnegative");
  if (n_tiers < 2) return fail(SPHKV_E_VALUE, "tier table has no non-drop tiers");
  if (n > 0x7fffffffLL) return fail(SPHKV_E_UNSUPPORTED, "more than 2^31 states");
  if (n == 0) return SPHKV_OK;
  TierRates tr = make_rates(tiers_host, n_tiers, d);
  const int max_id = tiers_host[n_tiers - 1].id;
  const int64_t max_rate = tr.rate[n_tiers - 1];
  RdrWs w = carve(workspace, n);
  const int nb = (int)div_up(n, 256);
  // protected demand (controller.py:316-322) and the round state, on the device
  GreedyState* gs = reinterpret_cast<GreedyState*>(w.scal + 2);
  int* status = reinterpret_cast<int*>(w.scal + 7);
  SPHKV_CUDA_TRY(cudaMemsetAsync(w.scal, 0, 64, stream));
  k_count_protect<<<4 * SM_COUNT, 256, 0, stream>>>(protect, n, w.scal + 1);
  SPHKV_LAUNCH_CHECK();
  k_greedy_init<<<1, 1, 0, stream>>>(gs, w.scal + 1, (long long)budget_bits, (long long)max_rate,
                                     status);
  SPHKV_LAUNCH_CHECK();
  k_init_assign<<<nb, 256, 0, stream>>>(best_tier, protect, n, max_id, 0, z, tier);
  SPHKV_LAUNCH_CHECK();
  int64_t* sidx = nullptr;
  if (int e = sort_states(w, nu, protect, n, 1, &sidx, stream)) return e;
  k_costs<<<nb, 256, 0, stream>>>(sidx, best_tier, protect, n, tr, w.cost);
  SPHKV_LAUNCH_CHECK();
  SPHKV_CUDA_TRY(cudaMemsetAsync(w.done, 0, n, stream));
  // Every round rejects one item whose cost is below the cap, so the cap
  // strictly decreases: at most (distinct non-drop rates) + 1 rounds.  They
  // are all enqueued; finished rounds are no-ops on the device.
  for (int round = 0; round < n_tiers + 1; ++round) {
    k_masked<<<nb, 256, 0, stream>>>(w.cost, w.done, n, gs, w.masked);
    SPHKV_LAUNCH_CHECK();
    size_t tb = w.cub_bytes;
    SPHKV_CUDA_TRY(cub::DeviceScan::InclusiveSum(w.cub, tb, w.masked, w.scan, (int)n, stream));
    k_first_over_gs<<<nb, 256, 0, stream>>>(w.scan, w.masked, n, gs);
    SPHKV_LAUNCH_CHECK();
    k_accept_gs<<<nb, 256, 0, stream>>>(sidx, best_tier, w.masked, n, gs, w.done, z, tier);
    SPHKV_LAUNCH_CHECK();
    k_greedy_update<<<1, 1, 0, stream>>>(w.scan, w.cost, n, gs);
    SPHKV_LAUNCH_CHECK();
  }
  // one host read at the end: the infeasibility status and convergence
  int host[2] = {0, 0};
  SPHKV_CUDA_TRY(cudaMemcpyAsync(&host[0], status, 4, cudaMemcpyDeviceToHost, stream));
  SPHKV_CUDA_TRY(cudaMemcpyAsync(&host[1], &gs->finished, 4, cudaMemcpyDeviceToHost, stream));
  SPHKV_CUDA_TRY(cudaStreamSynchronize(stream));
  if (host[0] == 1)
    return fail(SPHKV_E_INFEASIBLE, "protected demand exceeds budget %lld bits",
                (long long)budget_bits);
  if (!host[1]) return fail(SPHKV_E_CUDA, "greedy allocation did not converge");
  return SPHKV_OK;
}

extern "C" int sphkv_rdr_downtier(const int16_t* best_tier, const double* nu,
                                  const uint8_t* protect, int64_t n,
                                  const sphkv_tier_t* tiers_host, int n_tiers, int d,
                                  int64_t budget_bits, void* workspace, int8_t* z, int16_t* tier,
                                  cudaStream_t stream) {
  if (budget_bits < 0) return fail(SPHKV_E_VALUE, "budget must be nonnegative");
  if (n_tiers < 2) return fail(SPHKV_E_VALUE, "tier table has no non-drop tiers");
  if (n > 0x7fffffffLL) return fail(SPHKV_E_UNSUPPORTED, "more than 2^31 states");
  if (n == 0) return SPHKV_OK;
  TierRates tr = make_rates(tiers_host, n_tiers, d);
  const int max_id = tiers_host[n_tiers - 1].id;
  RdrWs w = carve(workspace, n);
  const int nb = (int)div_up(n, 256);
  k_init_assign<<<nb, 256, 0, stream>>>(best_tier, protect, n, max_id, 1, z, tier);
  SPHKV_LAUNCH_CHECK();
  SPHKV_CUDA_TRY(cudaMemsetAsync(w.scal, 0, 64, stream));
  k_total_rate<<<4 * SM_COUNT, 256, 0, stream>>>(tier, n, tr, w.scal + 1);
  SPHKV_LAUNCH_CHECK();
  unsigned long long total = 0;
  SPHKV_CUDA_TRY(cudaMemcpyAsync(&total, w.scal + 1, 8, cudaMemcpyDeviceToHost, stream));
  SPHKV_CUDA_TRY(cudaStreamSynchronize(stream));
  if ((int64_t)total <= budget_bits) return SPHKV_OK;
  int64_t* sidx = nullptr;
  if (int e = sort_states(w, nu, protect, n, 0, &sidx, stream)) return e;
  k_rates_sorted<<<nb, 256, 0, stream>>>(sidx, tier, protect, n, tr, w.masked);
  SPHKV_LAUNCH_CHECK();
  size_t tb = w.cub_bytes;
  SPHKV_CUDA_TRY(cub::DeviceScan::InclusiveSum(w.cub, tb, w.masked, w.scan, (int)n, stream));
  // first k with total - scan[k] <= budget  (monotone: binary search on host
  // over device values would need syncs; do it with one more kernel pass)
  SPHKV_CUDA_TRY(cudaMemsetAsync(w.scal, 0xff, 8, stream));
  k_first_over<<<nb, 256, 0, stream>>>(w.scan, w.scan, n, 0,
                                       (int64_t)total - budget_bits - 1, w.scal);
  SPHKV_LAUNCH_CHECK();
  unsigned long long k = 0;
  SPHKV_CUDA_TRY(cudaMemcpyAsync(&k, w.scal, 8, cudaMemcpyDeviceToHost, stream));
  SPHKV_CUDA_TRY(cudaStreamSynchronize(stream));
  if (k == ~0ull)
    return fail(SPHKV_E_INFEASIBLE, "protected demand exceeds budget %lld", (long long)budget_bits);
  // state k is the boundary: states [0, k) drop entirely
  if (k > 0) {
    k_drop_prefix<<<(int)div_up((int64_t)k, 256), 256, 0, stream>>>(sidx, (int64_t)k, z, tier,
                                                                     protect);
    SPHKV_LAUNCH_CHECK();
  }
  int64_t before = 0, s = 0;
  int16_t cur = 0;
  if (k > 0) SPHKV_CUDA_TRY(cudaMemcpyAsync(&before, w.scan + k - 1, 8, cudaMemcpyDeviceToHost, stream));
  SPHKV_CUDA_TRY(cudaMemcpyAsync(&s, sidx + k, 8, cudaMemcpyDeviceToHost, stream));
  SPHKV_CUDA_TRY(cudaStreamSynchronize(stream));
  SPHKV_CUDA_TRY(cudaMemcpyAsync(&cur, tier + s, 2, cudaMemcpyDeviceToHost, stream));
  SPHKV_CUDA_TRY(cudaStreamSynchronize(stream));
  int64_t tot = (int64_t)total - before;
  int t_idx = 0;
  for (int t = 0; t < n_tiers; ++t)
    if (tr.id[t] == cur) t_idx = t;
  while (tot > budget_bits && t_idx > 0) {
    tot -= tr.rate[t_idx] - tr.rate[t_idx - 1];
    t_idx -= 1;
  }
  int16_t nt = (int16_t)tr.id[t_idx];
  int8_t nz = nt != 0 ? 1 : 0;
  SPHKV_CUDA_TRY(cudaMemcpyAsync(tier + s, &nt, 2, cudaMemcpyHostToDevice, stream));
  SPHKV_CUDA_TRY(cudaMemcpyAsync(z + s, &nz, 1, cudaMemcpyHostToDevice, stream));
  SPHKV_CUDA_TRY(cudaStreamSynchronize(stream));
  return SPHKV_OK;
}
