// ADA key encoder, tier-homogeneous page packer, decode-time append, stream
// export and the dense baseline store fill.  Compiled with --fmad=false: every
// fp64 expression follows numpy's operation order so codes are bit-exact.
//
// Reference behaviour replaced (pkg/src/sphkv/):
//   codec.py:222-257   to_spherical / angles_from_unit
//   codec.py:318-377   quantize_angles, quantize_radius, encode_key
//   store.py:430-482   pack_pages_arrays (grouping, chunking, page scale, SoA)
//   store.py:249-274   PagedStore.append_item (page open rule, headroom)
//   store.py:205-211   Page.angle_stream / radius_stream (export)
//   controller.py:181-198  score_and_best_tier (append scoring)
#include "common.cuh"

namespace sphkv {

// ---------------------------------------------------------------------------
// encoder
// ---------------------------------------------------------------------------
template <typename T>
struct KeyRow {
  const T* p;
  __device__ double operator()(int i) const { return load_as_double(p + i); }
};

template <typename T>
__device__ double key_radius(const T* row, int d) {
  auto sq = [row](int i) {
    double v = load_as_double(row + i);
    return __dmul_rn(v, v);
  };
  return __dsqrt_rn(np_pairwise_sum(sq, 0, d));
}

// Calls emit(j, angle) for the circular angle j = d-2 first, then the polar
// angles j = d-3 .. 0 (descending), exactly as angles_from_unit computes them
// on u = k / (r + 1e-12).  Zero radius emits all-zero angles (codec.py:234).
template <typename T, typename Emit>
__device__ void encode_desc(const T* row, int d, double r, Emit emit, bool unit_input = false) {
  if (r == 0.0 && !unit_input) {
    for (int j = d - 2; j >= 0; --j) emit(j, 0.0);
    return;
  }
  // unit_input: angles_from_unit(u) on rows already normalized (codec.py:239)
  const double den = unit_input ? 1.0 : __dadd_rn(r, kNormEps);
  auto u = [&](int i) { return __ddiv_rn(load_as_double(row + i), den); };
  double ul = u(d - 1), up = u(d - 2);
  double last = atan2(ul, up);
  if (last < 0.0) last = __dadd_rn(last, kTwoPi);
  emit(d - 2, last);
  if (d > 2) {
    double acc = __dmul_rn(ul, ul);           // cumsum[0] of the reversed squares
    acc = __dadd_rn(acc, __dmul_rn(up, up));  // tail^2 at index d-2
    for (int j = d - 3; j >= 0; --j) {
      double uj = u(j);
      double a = atan2(__dsqrt_rn(acc), uj);
      a = fmin(fmax(a, 0.0), kPi);
      emit(j, a);
      acc = __dadd_rn(acc, __dmul_rn(uj, uj));
    }
  }
}

template <typename T>
__global__ void k_encode_radii(const T* __restrict__ keys, int64_t n, int d, double* radii) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  radii[i] = key_radius(keys + i * d, d);
}

template <typename T>
__global__ void k_encode(const T* __restrict__ keys, int64_t n, int d, double* radii,
                         double* angles, int unit_input) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const T* row = keys + i * d;
  double r = unit_input ? 1.0 : key_radius(row, d);
  if (radii) radii[i] = r;
  double* out = angles + i * (d - 1);
  encode_desc(row, d, r, [&](int j, double a) { out[j] = a; }, unit_input != 0);
}

__global__ void k_quantize(const double* __restrict__ angles, int64_t n, int dm1, int bits,
                           uint32_t* codes) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n * dm1) return;
  int j = (int)(e % dm1);
  double a = angles[e];
  codes[e] = (j == dm1 - 1) ? quant_circ(a, circular_step(bits), bits)
                            : quant_polar(a, polar_step(bits), bits);
}

// ---------------------------------------------------------------------------
// store helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ int tier_idx(const sphkv_store_t& st, int id) {
  for (int i = 0; i < st.n_tiers; ++i)
    if (st.tiers[i].id == id) return i;
  return -1;
}

__global__ void k_store_reset(sphkv_store_t st) {
  const int groups = st.batch * st.layers * st.heads;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < groups * SPHKV_MAX_TIERS;
       i += gridDim.x * blockDim.x) {
    st.group_last[i] = -1;
    if (i < groups) st.ptr_len[i] = 0;
    if (i < 4) st.counters[i] = 0;
  }
}

// per group, per tier-index retained counts
// (block = group g0 + blockIdx.x; input arrays are relative to group g0)
__global__ void k_pack_count(sphkv_store_t st, int T, int g0, const int8_t* __restrict__ z,
                             const int16_t* __restrict__ tier, int* counts, int* err) {
  __shared__ int c[SPHKV_MAX_TIERS];
  if (threadIdx.x < SPHKV_MAX_TIERS) c[threadIdx.x] = 0;
  __syncthreads();
  const int64_t g = g0 + blockIdx.x;
  for (int i = threadIdx.x; i < T; i += blockDim.x) {
    int64_t s = (int64_t)blockIdx.x * T + i;
    if (z[s] == 1) {
      int ti = tier_idx(st, tier[s]);
      if (ti <= 0) { atomicExch(err, 1); continue; }  // retained state at drop tier
      atomicAdd(&c[ti], 1);
    } else if (z[s] != 0) {
      atomicExch(err, 2);
    }
  }
  __syncthreads();
  if (threadIdx.x < st.n_tiers) counts[g * SPHKV_MAX_TIERS + threadIdx.x] = c[threadIdx.x];
}

// single block: page bases and code offsets for (group, tier) entries in
// pointer order (group -> tier ascending), store.py:453-466
__global__ void k_pack_plan(sphkv_store_t st, const int* __restrict__ counts, int* page_base,
                            uint64_t* code_base, int* err) {
  const int groups = st.batch * st.layers * st.heads;
  const int NT = st.n_tiers;
  const int E = groups * NT;
  __shared__ int s_np[1024];
  __shared__ unsigned long long s_nb[1024];
  const int per = (E + blockDim.x - 1) / blockDim.x;
  const int e0 = threadIdx.x * per, e1 = min(E, e0 + per);
  int np = 0;
  unsigned long long nb = 0;
  for (int e = e0; e < e1; ++e) {
    int t = e % NT;
    if (t == 0) continue;
    int c = counts[(e / NT) * SPHKV_MAX_TIERS + t];
    int k = (c + st.page_size - 1) / st.page_size;
    np += k;
    nb += (unsigned long long)k *
          code_block_bytes(st.d, st.page_size, st.tiers[t].angle_bits, st.tiers[t].radius_bits);
  }
  s_np[threadIdx.x] = np;
  s_nb[threadIdx.x] = nb;
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = 0;
    unsigned long long b = 0;
    for (int i = 0; i < (int)blockDim.x; ++i) {
      int x = s_np[i];
      unsigned long long y = s_nb[i];
      s_np[i] = a;
      s_nb[i] = b;
      a += x;
      b += y;
    }
    unsigned long long p0 = st.counters[0], c0 = st.counters[1];
    if (p0 + a > (unsigned long long)st.max_pages || c0 + b > st.code_cap) atomicExch(err, 3);
    st.counters[0] = p0 + a;
    st.counters[1] = c0 + b;
    s_np[1023] = (int)p0;  // stash (blockDim <= 1023 entries used above)
    s_nb[1023] = c0;
  }
  __syncthreads();
  int pb = s_np[1023] + s_np[threadIdx.x];
  unsigned long long cb = s_nb[1023] + s_nb[threadIdx.x];
  for (int e = e0; e < e1; ++e) {
    int t = e % NT;
    page_base[e] = pb;
    code_base[e] = cb;
    if (t == 0) continue;
    int c = counts[(e / NT) * SPHKV_MAX_TIERS + t];
    int k = (c + st.page_size - 1) / st.page_size;
    pb += k;
    cb += (unsigned long long)k *
          code_block_bytes(st.d, st.page_size, st.tiers[t].angle_bits, st.tiers[t].radius_bits);
  }
}

// one block per (group, tier) entry: page descriptors, pointer lists
__global__ void k_pack_pages_init(sphkv_store_t st, const int* __restrict__ counts,
                                  const int* __restrict__ page_base,
                                  const uint64_t* __restrict__ code_base, int* err) {
  const int NT = st.n_tiers;
  const int e = blockIdx.x;
  const int g = e / NT, t = e % NT;
  if (t == 0) return;
  const int c = counts[g * SPHKV_MAX_TIERS + t];
  const int k = (c + st.page_size - 1) / st.page_size;
  if (k == 0) return;
  const sphkv_tier_t tt = st.tiers[t];
  const uint64_t blk = code_block_bytes(st.d, st.page_size, tt.angle_bits, tt.radius_bits);
  const int first_of_group = page_base[g * NT];
  const int base_len = st.ptr_len[g];
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    int pid = page_base[e] + i;
    if (pid >= st.max_pages) { atomicExch(err, 3); continue; }
    sphkv_page_t pg;
    pg.code_off = code_base[e] + (uint64_t)i * blk;
    pg.radius_scale = 0.0;
    pg.rscale = 0.f;
    pg.count = min(st.page_size, c - i * st.page_size);
    pg.group = g;
    pg.tier = (uint8_t)tt.id;
    pg.abits = (uint8_t)tt.angle_bits;
    pg.rbits = (uint8_t)tt.radius_bits;
    pg.mbits = (uint8_t)tt.meta_bits;
    st.pages[pid] = pg;
    int pos = base_len + (pid - first_of_group);
    if (pos < st.ptr_cap) st.ptr[(int64_t)g * st.ptr_cap + pos] = pid;
    else atomicExch(err, 4);
    if (i == k - 1) st.group_last[g * SPHKV_MAX_TIERS + t] = pid;
  }
}

__global__ void k_pack_ptrlen(sphkv_store_t st, const int* __restrict__ page_base, int* err) {
  const int groups = st.batch * st.layers * st.heads;
  const int NT = st.n_tiers;
  int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= groups) return;
  int first = page_base[g * NT];
  int next = (g + 1 < groups) ? page_base[(g + 1) * NT] : (int)st.counters[0];
  int len = st.ptr_len[g] + (next - first);
  if (len > st.ptr_cap) atomicExch(err, 4);
  st.ptr_len[g] = min(len, st.ptr_cap);
}

// per group: rank of each retained token inside its (group, tier) in token
// order -> page_items[page * P + slot] = state index
__global__ void __launch_bounds__(1024) k_pack_rank(sphkv_store_t st, int T, int g0,
                                                    const int8_t* __restrict__ z,
                                                    const int16_t* __restrict__ tier,
                                                    const int* __restrict__ page_base,
                                                    int first, int* page_items) {
  __shared__ int wc[32][SPHKV_MAX_TIERS];
  __shared__ int running[SPHKV_MAX_TIERS];
  const int NT = st.n_tiers;
  const int64_t gr = blockIdx.x, g = g0 + gr;  // relative / absolute group
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < SPHKV_MAX_TIERS) running[threadIdx.x] = 0;
  __syncthreads();
  for (int base = 0; base < T; base += blockDim.x) {
    const int i = base + threadIdx.x;
    int ti = -1;
    if (i < T && z[gr * T + i] == 1) ti = tier_idx(st, tier[gr * T + i]);
    int my_rank_in_warp = 0;
    for (int t = 1; t < NT; ++t) {
      unsigned m = __ballot_sync(0xffffffffu, ti == t);
      if (lane == 0) wc[warp][t] = __popc(m);
      if (ti == t) my_rank_in_warp = __popc(m & ((1u << lane) - 1u));
    }
    __syncthreads();
    if (ti > 0) {
      int r = running[ti] + my_rank_in_warp;
      for (int w = 0; w < warp; ++w) r += wc[w][ti];
      int pid = page_base[g * NT + ti] + r / st.page_size;
      page_items[(int64_t)(pid - first) * st.page_size + r % st.page_size] = (int)(gr * T + i);
    }
    __syncthreads();
    if (threadIdx.x < NT && threadIdx.x > 0) {
      int s = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += wc[w][threadIdx.x];
      running[threadIdx.x] += s;
    }
    __syncthreads();
  }
}

// page scale = max(max radius in chunk, 1e-9)  (store.py:465)
__global__ void k_pack_scale(sphkv_store_t st, int first_page, int n_pages,
                             const int* __restrict__ page_items, const double* __restrict__ radii) {
  int pid = first_page + blockIdx.x;
  if (pid >= first_page + n_pages) return;
  sphkv_page_t& pg = st.pages[pid];
  double m = -1.0;
  for (int s = threadIdx.x; s < pg.count; s += blockDim.x)
    m = fmax(m, radii[page_items[(int64_t)(pid - first_page) * st.page_size + s]]);
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    double scale = fmax(m, 1e-9);
    pg.radius_scale = scale;
    pg.rscale = (float)__ddiv_rn(scale, (double)((1u << pg.rbits) - 1u));
  }
}

// Assemble one bit row of 32 consecutive slots (b bits each) in a warp and
// store it: `dst` points at the first 32-bit word of the 32-slot chunk.
__device__ __forceinline__ void warp_store_bits(uint32_t* wbuf, uint32_t* dst, uint32_t code,
                                                int b, int lane) {
  if (lane < b) wbuf[lane] = 0u;
  __syncwarp();
  const int bit = lane * b;
  atomicOr(&wbuf[bit >> 5], code << (bit & 31));
  if ((bit & 31) + b > 32) atomicOr(&wbuf[(bit >> 5) + 1], code >> (32 - (bit & 31)));
  __syncwarp();
  if (lane < b) dst[lane] = wbuf[lane];
  __syncwarp();
}

// warp per (page, 32-slot chunk): encode + quantize + SoA bit rows, radius
// row, swizzled fp16 values, protect, token ids.
template <typename T>
__global__ void k_pack_write(sphkv_store_t st, int first_page, int n_pages, int T_,
                             const T* __restrict__ keys, const double* __restrict__ angles,
                             const double* __restrict__ radii, const uint16_t* __restrict__ values,
                             const uint8_t* __restrict__ protect,
                             const int* __restrict__ page_items) {
  __shared__ uint32_t wbuf_all[8][17];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* wbuf = wbuf_all[warp];
  const int chunks = st.page_size / 32;
  const int64_t job = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (job >= (int64_t)n_pages * chunks) return;
  const int pid = first_page + (int)(job / chunks);
  const int chunk = (int)(job % chunks);
  const sphkv_page_t pg = st.pages[pid];
  const int d = st.d, P = st.page_size, b = pg.abits, rb = pg.rbits;
  const int slot = chunk * 32 + lane;
  const bool valid = slot < pg.count;
  const int idx = valid ? page_items[(int64_t)(pid - first_page) * P + slot] : 0;
  const double r = valid ? radii[idx] : 0.0;
  uint32_t* block = reinterpret_cast<uint32_t*>(st.codes + pg.code_off);
  const int W = item_words(d, b);
  const double ps = polar_step(b), cs = circular_step(b);
  // Codes arrive in descending row order (circular d-2, then polar d-3..0),
  // so the lane assembles its item string word by word from the top and
  // stores each finished word once (coalesced across the warp's 32 items).
  uint32_t acc = 0;
  int cur = W - 1;
  auto put_word = [&](int w, uint32_t v) {
    while (cur > w) {
      block[wi_word(slot, cur, W)] = acc;
      acc = 0;
      --cur;
    }
    acc |= v;
  };
  auto emit = [&](int j, double a) {
    uint32_t c = 0;
    if (valid) c = (j == d - 2) ? quant_circ(a, cs, b) : quant_polar(a, ps, b);
    const int bit = j * b, w = bit >> 5, sh = bit & 31;
    if (sh + b > 32) put_word(w + 1, c >> (32 - sh));
    put_word(w, c << sh);
  };
  if (angles != nullptr) {
    const double* ar = angles + (int64_t)idx * (d - 1);
    for (int j = d - 2; j >= 0; --j) emit(j, valid ? ar[j] : 0.0);
  } else if (__all_sync(0xffffffffu, valid)) {
    encode_desc(keys + (int64_t)idx * d, d, r, emit);
  } else {
    // ragged last chunk: every lane walks the same row sequence
    double rr = valid ? r : 0.0;
    encode_desc(keys + (int64_t)idx * d, d, rr, emit);
  }
  put_word(-1, 0u);  // flush word 0 (and any untouched padding words above)
  // radius row (SoA, LSB-first) after the angle part
  {
    const double levels = (double)((1u << rb) - 1u);
    uint32_t c = 0;
    if (valid) {
      double x = __ddiv_rn(r, pg.radius_scale);
      x = fmin(fmax(x, 0.0), 1.0);
      c = (uint32_t)rint(__dmul_rn(x, levels));
    }
    uint32_t* rrow = block + angle_part_bytes(d, P, b) / 4;
    warp_store_bits(wbuf, rrow + chunk * rb, c, rb, lane);
  }
  // values (swizzled, zero padded), protect, token id
  const int dv = st.d_v, dvp = (dv + 15) / 16 * 16;
  uint16_t* vrow = st.values + (int64_t)pid * P * dvp;
  for (int e = 0; e < dvp; ++e) {
    uint16_t v = (valid && e < dv) ? values[(int64_t)idx * dv + e] : (uint16_t)0;
    vrow[vswz(slot, e, dvp)] = v;
  }
  st.protect[(int64_t)pid * P + slot] = valid ? protect[idx] : 0;
  st.token_ids[(int64_t)pid * P + slot] = valid ? (int64_t)(idx % T_) : -1;
}

// ---------------------------------------------------------------------------
// append (store.py:249-274)
// ---------------------------------------------------------------------------
struct AppendWs {
  int* flag;       // [n] opens a page
  int* slot;       // [n] page id used
  double* radius;  // [n]
  double* angles;  // [n, d-1]
  int* err;
};

__global__ void k_append_decide(sphkv_store_t st, int n, const double* __restrict__ radii_in,
                                const int16_t* __restrict__ tier_ids,
                                const uint8_t* __restrict__ active, AppendWs ws) {
  int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  ws.flag[g] = 0;
  ws.slot[g] = -1;
  if ((active && !active[g]) || tier_ids[g] == 0) return;
  int ti = tier_idx(st, tier_ids[g]);
  if (ti <= 0) { atomicExch(ws.err, 5); return; }
  double r = radii_in ? radii_in[g] : ws.radius[g];
  ws.radius[g] = r;
  int last = st.group_last[g * SPHKV_MAX_TIERS + ti];
  bool need = last < 0;
  if (!need) {
    const sphkv_page_t pg = st.pages[last];
    need = pg.count >= st.page_size || r > pg.radius_scale;
  }
  ws.flag[g] = need ? 1 : 0;
  ws.slot[g] = need ? -1 : last;
}

// single block: new page ids and code blocks in group order
__global__ void k_append_alloc(sphkv_store_t st, int n, const int16_t* __restrict__ tier_ids,
                               AppendWs ws) {
  __shared__ int s_np[1024];
  __shared__ unsigned long long s_nb[1024];
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int g0 = threadIdx.x * per, g1 = min(n, g0 + per);
  int np = 0;
  unsigned long long nb = 0;
  for (int g = g0; g < g1; ++g) {
    if (!ws.flag[g]) continue;
    int ti = tier_idx(st, tier_ids[g]);
    np += 1;
    nb += code_block_bytes(st.d, st.page_size, st.tiers[ti].angle_bits, st.tiers[ti].radius_bits);
  }
  s_np[threadIdx.x] = np;
  s_nb[threadIdx.x] = nb;
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = 0;
    unsigned long long b = 0;
    for (int i = 0; i < (int)blockDim.x; ++i) {
      int x = s_np[i];
      unsigned long long y = s_nb[i];
      s_np[i] = a;
      s_nb[i] = b;
      a += x;
      b += y;
    }
    unsigned long long p0 = st.counters[0], c0 = st.counters[1];
    if (p0 + a > (unsigned long long)st.max_pages || c0 + b > st.code_cap) {
      atomicExch(ws.err, 3);
      a = 0;
      b = 0;
    }
    st.counters[0] = p0 + a;
    st.counters[1] = c0 + b;
    s_np[1023] = (int)p0;
    s_nb[1023] = c0;
  }
  __syncthreads();
  if (*ws.err == 3) return;
  int pid = s_np[1023] + s_np[threadIdx.x];
  unsigned long long cb = s_nb[1023] + s_nb[threadIdx.x];
  for (int g = g0; g < g1; ++g) {
    if (!ws.flag[g]) continue;
    int ti = tier_idx(st, tier_ids[g]);
    const sphkv_tier_t tt = st.tiers[ti];
    const double r = ws.radius[g];
    double scale = fmax(__dmul_rn(r, 1.25), 1e-9);
    if (st.group_last[g * SPHKV_MAX_TIERS + ti] < 0 && r == 0.0) scale = 1e-9;
    sphkv_page_t pg;
    pg.code_off = cb;
    pg.radius_scale = scale;
    pg.rscale = (float)__ddiv_rn(scale, (double)((1u << tt.radius_bits) - 1u));
    pg.count = 0;
    pg.group = g;
    pg.tier = (uint8_t)tt.id;
    pg.abits = (uint8_t)tt.angle_bits;
    pg.rbits = (uint8_t)tt.radius_bits;
    pg.mbits = (uint8_t)tt.meta_bits;
    st.pages[pid] = pg;
    int len = st.ptr_len[g];
    if (len >= st.ptr_cap) atomicExch(ws.err, 4);
    else {
      st.ptr[(int64_t)g * st.ptr_cap + len] = pid;
      st.ptr_len[g] = len + 1;
    }
    st.group_last[g * SPHKV_MAX_TIERS + ti] = pid;
    ws.slot[g] = pid;
    pid += 1;
    cb += code_block_bytes(st.d, st.page_size, tt.angle_bits, tt.radius_bits);
  }
}

// warp per appended state
__global__ void k_append_write(sphkv_store_t st, int n, const int16_t* __restrict__ tier_ids,
                               const uint16_t* __restrict__ values,
                               const uint8_t* __restrict__ protect,
                               const int64_t* __restrict__ token_ids, AppendWs ws) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= n) return;
  const int g = warp;
  const int pid = ws.slot[g];
  if (pid < 0 || *ws.err) return;
  sphkv_page_t& pgr = st.pages[pid];
  const sphkv_page_t pg = pgr;
  const int d = st.d, P = st.page_size, b = pg.abits, rb = pg.rbits;
  uint8_t* blk = st.codes + pg.code_off;
  if (pg.count == 0) {  // fresh page: clear its code block
    uint64_t bytes = code_block_bytes(d, P, b, rb);
    for (uint64_t i = lane * 16; i < bytes; i += 32 * 16)
      *reinterpret_cast<uint4*>(blk + i) = make_uint4(0, 0, 0, 0);
    __syncwarp();
  }
  const int pos = pg.count;
  uint32_t* words = reinterpret_cast<uint32_t*>(blk);
  const double* ang = ws.angles + (int64_t)g * (d - 1);
  const double ps = polar_step(b), cs = circular_step(b);
  const int W = item_words(d, b);
  // lanes write different codes of the same item string: OR atomically
  for (int j = lane; j < d - 1; j += 32) {
    uint32_t c = (j == d - 2) ? quant_circ(ang[j], cs, b) : quant_polar(ang[j], ps, b);
    const int bit = j * b, w = bit >> 5, sh = bit & 31;
    atomicOr(words + wi_word(pos, w, W), c << sh);
    if (sh + b > 32) atomicOr(words + wi_word(pos, w + 1, W), c >> (32 - sh));
  }
  if (lane == 0) {
    // quantize_radius: Python round() == round-half-even (codec.py:353-355)
    double x = fmin(fmax(__ddiv_rn(ws.radius[g], pg.radius_scale), 0.0), 1.0);
    uint32_t rc = (uint32_t)rint(__dmul_rn(x, (double)((1u << rb) - 1u)));
    const uint64_t bit = angle_part_bytes(d, P, b) * 8 + (uint64_t)pos * rb;
    const int sh = (int)(bit & 31);
    atomicOr(words + (bit >> 5), rc << sh);
    if (sh + rb > 32) atomicOr(words + (bit >> 5) + 1, rc >> (32 - sh));
  }
  const int dv = st.d_v, dvp = (dv + 15) / 16 * 16;
  uint16_t* vrow = st.values + (int64_t)pid * P * dvp;
  for (int e = lane; e < dvp; e += 32)
    vrow[vswz(pos, e, dvp)] = e < dv ? values[(int64_t)g * dv + e] : (uint16_t)0;
  __syncwarp();
  if (lane == 0) {
    st.protect[(int64_t)pid * P + pos] = protect ? protect[g] : 0;
    st.token_ids[(int64_t)pid * P + pos] = token_ids ? token_ids[g] : -1;
    __threadfence();
    pgr.count = pos + 1;
  }
}

// score_and_best_tier per appended state (controller.py:163-198)
__global__ void k_score_append(const double* __restrict__ radii, int groups_per_seq, int heads,
                               const double* __restrict__ u_hat, const double* __restrict__ s_hat,
                               double r_q, double om, double at, double ar, const TierSet ts,
                               int NT, double lam, int d, int64_t n, int16_t* tier_out,
                               double* score_out, double* nu_out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int lh = (int)(i % groups_per_seq);
  const double sqrt_d = __dsqrt_rn((double)d);
  const double w_theta =
      __dmul_rn(__dmul_rn(__dmul_rn(at, u_hat[lh]), om), __ddiv_rn(__dmul_rn(r_q, radii[i]), sqrt_d));
  const double w_r = __dmul_rn(__dmul_rn(__dmul_rn(ar, __dadd_rn(1.0, -s_hat[lh])), om),
                               __ddiv_rn(r_q, sqrt_d));
  int best = -1;
  double best_s = -INFINITY;
  for (int t = 0; t < NT; ++t) {
    double et = t == 0 ? 1.0 : ts.t[t].eps_theta, er = t == 0 ? 1.0 : ts.t[t].eps_r;
    double dist = __dadd_rn(__dmul_rn(w_theta, et), __dmul_rn(w_r, er));
    int rate = t == 0 ? 0 : (d - 1) * ts.t[t].angle_bits + ts.t[t].radius_bits + ts.t[t].meta_bits;
    double s = __dadd_rn(-dist, -__dmul_rn(lam, (double)rate));
    if (s > best_s) {
      best_s = s;
      best = t;
    }
  }
  double d_drop = __dadd_rn(w_theta, w_r);
  double et = best == 0 ? 1.0 : ts.t[best].eps_theta, er = best == 0 ? 1.0 : ts.t[best].eps_r;
  double d_best = __dadd_rn(__dmul_rn(w_theta, et), __dmul_rn(w_r, er));
  int rate = best == 0 ? 0
                       : (d - 1) * ts.t[best].angle_bits + ts.t[best].radius_bits +
                             ts.t[best].meta_bits;
  tier_out[i] = (int16_t)ts.t[best].id;
  if (score_out) score_out[i] = best_s;
  if (nu_out) nu_out[i] = __ddiv_rn(__dadd_rn(d_drop, -d_best), __dadd_rn((double)rate, 1e-12));
}

// Decode-time append decision (decode.py:454-498): one warp per group.
template <typename T>
__global__ void k_decode_gate(sphkv_store_t st, const T* __restrict__ keys,
                              const float* __restrict__ q, int G,
                              const float* __restrict__ margins, const double* __restrict__ u_hat,
                              const double* __restrict__ s_hat, double r_q, double om, double at,
                              double ar, double lam, int use_gate, double tau_drop,
                              double tau_prot, double galpha, int8_t* mode, int16_t* tier_out,
                              uint8_t* prot_out, float* danger_out) {
  const int groups = st.batch * st.layers * st.heads;
  const int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (g >= groups) return;
  const int d = st.d, NT = st.n_tiers;
  const double sqrt_d = __dsqrt_rn((double)d);
  // best tier of the new key (score_and_best_tier, controller.py:181-198)
  const double radius = key_radius(keys + (int64_t)g * d, d);
  const double w_theta =
      __dmul_rn(__dmul_rn(__dmul_rn(at, u_hat[g]), om), __ddiv_rn(__dmul_rn(r_q, radius), sqrt_d));
  const double w_r =
      __dmul_rn(__dmul_rn(__dmul_rn(ar, __dadd_rn(1.0, -s_hat[g])), om), __ddiv_rn(r_q, sqrt_d));
  int best = -1;
  double best_s = -INFINITY;
  for (int t = 0; t < NT; ++t) {
    const double et = t == 0 ? 1.0 : st.tiers[t].eps_theta, er = t == 0 ? 1.0 : st.tiers[t].eps_r;
    const double dist = __dadd_rn(__dmul_rn(w_theta, et), __dmul_rn(w_r, er));
    const int rate = t == 0 ? 0 : (d - 1) * st.tiers[t].angle_bits + st.tiers[t].radius_bits +
                                     st.tiers[t].meta_bits;
    const double sc = __dadd_rn(-dist, -__dmul_rn(lam, (double)rate));
    if (sc > best_s) {
      best_s = sc;
      best = t;
    }
  }
  int tid = st.tiers[best].id;
  uint8_t prot = 0;
  float danger_f = 0.f;
  if (use_gate) {
    // probe tier, calibrated RMS constants (eps_r scale-relative), r_max
    const int probe = best != 0 ? best : NT - 1;
    const double eps_t = st.tiers[probe].eps_theta, eps_r_rel = st.tiers[probe].eps_r;
    double r_max = 0.0;
    const int n = st.ptr_len[g];
    for (int i = lane; i < n; i += 32)
      r_max = fmax(r_max, st.pages[st.ptr[(int64_t)g * st.ptr_cap + i]].radius_scale);
    for (int o = 16; o > 0; o >>= 1) r_max = fmax(r_max, __shfl_xor_sync(0xffffffffu, r_max, o));
    const double eps_r = __dmul_rn(eps_r_rel, r_max);
    const double inner = __dadd_rn(__dadd_rn(__dmul_rn(r_max, eps_t), eps_r), __dmul_rn(eps_r, eps_t));
    double danger = 0.0;
    if (lane < G) {
      const float* qi = q + ((int64_t)g * G + lane) * d;
      auto sq = [qi](int i) {
        const double v = (double)qi[i];
        return __dmul_rn(v, v);
      };
      const double qn = __dsqrt_rn(np_pairwise_sum(sq, 0, d));
      const double bound = __dmul_rn(galpha, __dmul_rn(__ddiv_rn(qn, sqrt_d), inner));
      const double m = (double)margins[(int64_t)g * G + lane];
      danger = isinf(m) ? 0.0 : fmin(__ddiv_rn(bound, __dadd_rn(m, 1e-9)), 10.0);
    }
    for (int o = 16; o > 0; o >>= 1) danger = fmax(danger, __shfl_xor_sync(0xffffffffu, danger, o));
    int md = mode[g];
    if (danger >= tau_prot) md = 2;
    else if (danger <= tau_drop) md = 0;
    if (md == 2) {
      tid = st.tiers[NT - 1].id;
      prot = 1;
    }
    if (lane == 0) mode[g] = (int8_t)md;
    danger_f = (float)danger;
  }
  if (lane == 0) {
    tier_out[g] = (int16_t)tid;
    prot_out[g] = prot;
    if (danger_out) danger_out[g] = danger_f;
  }
}

// ---------------------------------------------------------------------------
// export: reference-format streams per page (stride = count)
// ---------------------------------------------------------------------------
__global__ void k_export(sphkv_store_t st, const int64_t* __restrict__ offsets, uint8_t* out) {
  const int pid = blockIdx.x;
  const sphkv_page_t pg = st.pages[pid];
  const int d = st.d, P = st.page_size, b = pg.abits, rb = pg.rbits, n = pg.count;
  const uint32_t* words = reinterpret_cast<const uint32_t*>(st.codes + pg.code_off);
  uint8_t* o = out + offsets[pid];
  const int64_t abytes = ((int64_t)n * (d - 1) * b + 7) / 8;
  const int64_t rbytes = ((int64_t)n * rb + 7) / 8;
  auto bit_at = [&](uint64_t bit) { return (words[bit >> 5] >> (bit & 31)) & 1u; };
  const int W = item_words(d, b);
  for (int64_t k = threadIdx.x; k < abytes; k += blockDim.x) {
    uint32_t byte = 0;
    for (int bb = 0; bb < 8; ++bb) {
      int64_t pos = k * 8 + bb;
      if (pos >= (int64_t)n * (d - 1) * b) break;
      int64_t ci = pos / b;  // reference SoA order: code (j, i) at j * count + i
      int bit = (int)(pos % b);
      int64_t j = ci / n, i = ci % n;
      const int sb = (int)j * b + bit;  // bit of item i's string
      byte |= ((words[wi_word((int)i, sb >> 5, W)] >> (sb & 31)) & 1u) << bb;
    }
    o[k] = (uint8_t)byte;
  }
  const uint64_t rbase = angle_part_bytes(d, P, b) * 8;
  for (int64_t k = threadIdx.x; k < rbytes; k += blockDim.x) {
    uint32_t byte = 0;
    for (int bb = 0; bb < 8; ++bb) {
      int64_t pos = k * 8 + bb;
      if (pos >= (int64_t)n * rb) break;
      byte |= bit_at(rbase + (uint64_t)pos) << bb;
    }
    o[abytes + k] = (uint8_t)byte;
  }
  const int dv = st.d_v, dvp = (dv + 15) / 16 * 16;
  uint16_t* vo = reinterpret_cast<uint16_t*>(o + abytes + rbytes);  // caller keeps 2-B alignment
  const uint16_t* vrow = st.values + (int64_t)pid * P * dvp;
  for (int e = threadIdx.x; e < n * dv; e += blockDim.x) {
    int i = e / dv, c = e % dv;
    uint16_t v = vrow[vswz(i, c, dvp)];
    uint8_t* dst = reinterpret_cast<uint8_t*>(vo) + 2 * (int64_t)e;
    dst[0] = (uint8_t)(v & 0xff);
    dst[1] = (uint8_t)(v >> 8);
  }
  uint8_t* po = o + abytes + rbytes + 2 * (int64_t)n * dv;
  for (int i = threadIdx.x; i < n; i += blockDim.x) po[i] = st.protect[(int64_t)pid * P + i];
}

// import: the inverse of k_export (SPHKV1 from_file, store.py:391-427).  The
// page descriptors are already in st.pages; `in` holds per page the reference
// angle stream (stride = count), radius stream, fp16 values [count][d_v] and
// one protect byte per item at offsets[pid].  One block per page writes the
// word-interleaved code block, the radius row, the swizzled value rows,
// protect flags and token ids (-1, as the reference's from_file leaves them).
__global__ void k_import(sphkv_store_t st, const int64_t* __restrict__ offsets,
                         const uint8_t* __restrict__ in) {
  const int pid = blockIdx.x;
  const sphkv_page_t pg = st.pages[pid];
  const int d = st.d, P = st.page_size, b = pg.abits, rb = pg.rbits, n = pg.count;
  const uint8_t* src = in + offsets[pid];
  uint32_t* words = reinterpret_cast<uint32_t*>(st.codes + pg.code_off);
  const int W = item_words(d, b);
  const int64_t nbits = (int64_t)(d - 1) * b;  // valid bits of one item string
  const int64_t abytes = ((int64_t)n * (d - 1) * b + 7) / 8;
  const int64_t rbytes = ((int64_t)n * rb + 7) / 8;
  auto in_bit = [&](int64_t pos) -> uint32_t { return (src[pos >> 3] >> (pos & 7)) & 1u; };
  const int64_t awords = (int64_t)angle_part_bytes(d, P, b) / 4;
  for (int64_t k = threadIdx.x; k < awords; k += blockDim.x) {
    // WI word k -> (item i, string word w)
    const int64_t quad = k >> 2;
    const int lane = (int)(quad & 31), w = (int)(((quad >> 5) % (W >> 2)) * 4 + (k & 3));
    const int i = (int)((quad >> 5) / (W >> 2)) * 32 + lane;
    uint32_t v = 0;
    if (i < n)
      for (int bit = 0; bit < 32; ++bit) {
        const int64_t sb = (int64_t)w * 32 + bit;
        if (sb >= nbits) break;
        const int64_t j = sb / b, cb = sb % b;  // code j of item i, bit cb
        v |= in_bit((j * n + i) * b + cb) << bit;
      }
    words[k] = v;
  }
  // radius row: the reference radius stream, bit for bit, zero-padded to P*rb
  uint32_t* rw = words + awords;
  const int64_t rwords = ((int64_t)P * rb + 31) / 32;
  for (int64_t k = threadIdx.x; k < rwords; k += blockDim.x) {
    uint32_t v = 0;
    for (int by = 0; by < 4; ++by) {
      const int64_t byte = k * 4 + by;
      if (byte < rbytes) v |= (uint32_t)src[abytes + byte] << (8 * by);
    }
    rw[k] = v;
  }
  const int dv = st.d_v, dvp = (dv + 15) / 16 * 16;
  const uint8_t* vin = src + abytes + rbytes;
  uint16_t* vrow = st.values + (int64_t)pid * P * dvp;
  for (int e = threadIdx.x; e < P * dvp; e += blockDim.x) {
    const int i = e / dvp, c = e % dvp;
    uint16_t v = 0;
    if (i < n && c < dv) {
      const uint8_t* x = vin + 2 * ((int64_t)i * dv + c);
      v = (uint16_t)(x[0] | (x[1] << 8));
    }
    vrow[vswz(i, c, dvp)] = v;
  }
  const uint8_t* pin = vin + 2 * (int64_t)n * dv;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    st.protect[(int64_t)pid * P + i] = i < n ? pin[i] : 0;
    st.token_ids[(int64_t)pid * P + i] = -1;
  }
}

// dense baseline store: bf16 K and fp16 V pages, swizzled rows
template <typename T>
__global__ void k_dense_fill(sphkv_dense_store_t st, int64_t g0, int64_t groups,
                             const T* __restrict__ keys, const uint16_t* __restrict__ values) {
  const int dp = (st.d + 15) / 16 * 16, dvp = (st.d_v + 15) / 16 * 16;
  const int64_t per_group = (int64_t)st.n_pages_per_group * st.page_size;
  const int64_t n = groups * per_group;
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < n;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = it / per_group, pos = it % per_group;
    const int i = (int)(pos % st.page_size);
    const bool valid = pos < st.tokens;
    const int64_t src = g * st.tokens + pos;  // relative to group g0
    const int64_t dst = it + g0 * per_group;
    uint16_t* krow = st.keys + (dst - i) * dp;
    for (int e = 0; e < dp; ++e) {
      float v = (valid && e < st.d) ? (float)load_as_double(keys + src * st.d + e) : 0.f;
      __nv_bfloat16 h = __float2bfloat16_rn(v);
      krow[vswz(i, e, dp)] = *reinterpret_cast<uint16_t*>(&h);
    }
    uint16_t* vrow = st.values + (dst - i) * dvp;
    for (int e = 0; e < dvp; ++e)
      vrow[vswz(i, e, dvp)] = (valid && e < st.d_v) ? values[src * st.d_v + e] : (uint16_t)0;
  }
}

}  // namespace sphkv

using namespace sphkv;

// ---------------------------------------------------------------------------
// host entry points
// ---------------------------------------------------------------------------
static int check_dtype(int dtype) {
  if (dtype != SPHKV_F32 && dtype != SPHKV_F64 && dtype != SPHKV_BF16 && dtype != SPHKV_F16)
    return fail(SPHKV_E_VALUE, "unknown key dtype %d", dtype);
  return SPHKV_OK;
}

#define SPHKV_DTYPE_DISPATCH(dtype, KERN, ...)                                       \
  switch (dtype) {                                                                 \
    case SPHKV_F32: KERN<float><<<__VA_ARGS__>>>; break;                            \
    case SPHKV_F64: KERN<double><<<__VA_ARGS__>>>; break;                           \
    case SPHKV_BF16: KERN<__nv_bfloat16><<<__VA_ARGS__>>>; break;                   \
    default: KERN<__half><<<__VA_ARGS__>>>; break;                                  \
  }

extern "C" int sphkv_encode_radii(const void* keys, int dtype, int64_t n, int d, double* radii,
                                  cudaStream_t stream) {
  if (check_dtype(dtype)) return SPHKV_E_VALUE;
  if (d < 2) return fail(SPHKV_E_VALUE, "need d >= 2, got %d", d);
  if (n == 0) return SPHKV_OK;
  int blocks = (int)div_up(n, 128);
  switch (dtype) {
    case SPHKV_F32: k_encode_radii<float><<<blocks, 128, 0, stream>>>((const float*)keys, n, d, radii); break;
    case SPHKV_F64: k_encode_radii<double><<<blocks, 128, 0, stream>>>((const double*)keys, n, d, radii); break;
    case SPHKV_BF16: k_encode_radii<__nv_bfloat16><<<blocks, 128, 0, stream>>>((const __nv_bfloat16*)keys, n, d, radii); break;
    default: k_encode_radii<__half><<<blocks, 128, 0, stream>>>((const __half*)keys, n, d, radii); break;
  }
  SPHKV_LAUNCH_CHECK();
  return SPHKV_OK;
}

extern "C" int sphkv_encode(const void* keys, int dtype, int64_t n, int d, double* radii,
                            double* angles, cudaStream_t stream) {
  if (check_dtype(dtype)) return SPHKV_E_VALUE;
  if (d < 2) return fail(SPHKV_E_VALUE, "need d >= 2, got %d", d);
  if (n == 0) return SPHKV_OK;
  int blocks = (int)div_up(n, 128);
  switch (dtype) {
    case SPHKV_F32: k_encode<float><<<blocks, 128, 0, stream>>>((const float*)keys, n, d, radii, angles, 0); break;
    case SPHKV_F64: k_encode<double><<<blocks, 128, 0, stream>>>((const double*)keys, n, d, radii, angles, 0); break;
    case SPHKV_BF16: k_encode<__nv_bfloat16><<<blocks, 128, 0, stream>>>((const __nv_bfloat16*)keys, n, d, radii, angles, 0); break;
    default: k_encode<__half><<<blocks, 128, 0, stream>>>((const __half*)keys, n, d, radii, angles, 0); break;
  }
  SPHKV_LAUNCH_CHECK();
  return SPHKV_OK;
}

extern "C" int sphkv_angles_from_unit(const double* u, int64_t n, int d, double* angles,
                                      cudaStream_t stream) {
  if (d < 2) return fail(SPHKV_E_VALUE, "need d >= 2, got %d", d);
  if (n == 0) return SPHKV_OK;
  k_encode<double><<<(int)div_up(n, 128), 128, 0, stream>>>(u, n, d, nullptr, angles, 1);
  SPHKV_LAUNCH_CHECK();
  return SPHKV_OK;
}

extern "C" int sphkv_quantize_angles(const double* angles, int64_t n, int dm1, int bits,
                                     uint32_t* codes, cudaStream_t stream) {
  if (bits < 1 || bits > 31) return fail(SPHKV_E_UNSUPPORTED, "angle bits %d outside [1, 31]", bits);
  if (dm1 < 1) return fail(SPHKV_E_VALUE, "need at least one angle");
  int64_t total = n * dm1;
  if (total == 0) return SPHKV_OK;
  k_quantize<<<(int)div_up(total, 256), 256, 0, stream>>>(angles, n, dm1, bits, codes);
  SPHKV_LAUNCH_CHECK();
  return SPHKV_OK;
}

static int validate_store(const sphkv_store_t* st) {
  if (!st) return fail(SPHKV_E_VALUE, "null store");
  if (st->page_size < 32 || st->page_size % 32 != 0)
    return fail(SPHKV_E_UNSUPPORTED, "device page_size must be a positive multiple of 32 (got %d)",
                st->page_size);
  if (st->d < 2 || st->d > 256) return fail(SPHKV_E_UNSUPPORTED, "d=%d outside [2, 256]", st->d);
  if (st->n_tiers < 2 || st->n_tiers > SPHKV_MAX_TIERS)
    return fail(SPHKV_E_VALUE, "tier table needs 2..%d entries", SPHKV_MAX_TIERS);
  if (st->tiers[0].id != 0) return fail(SPHKV_E_VALUE, "tier table must start with the drop tier");
  for (int t = 1; t < st->n_tiers; ++t) {
    const sphkv_tier_t& x = st->tiers[t];
    if (x.angle_bits < 1 || x.angle_bits > 16 || x.radius_bits < 1 || x.radius_bits > 16)
      return fail(SPHKV_E_UNSUPPORTED, "tier %d: device codes support 1..16 bits", x.id);
    if (x.id <= st->tiers[t - 1].id) return fail(SPHKV_E_VALUE, "tier ids must ascend");
  }
  return SPHKV_OK;
}

extern "C" int sphkv_store_reset(const sphkv_store_t* st, cudaStream_t stream) {
  if (int e = validate_store(st)) return e;
  k_store_reset<<<64, 256, 0, stream>>>(*st);
  SPHKV_LAUNCH_CHECK();
  return SPHKV_OK;
}

extern "C" int64_t sphkv_pack_workspace_bytes(int batch, int layers, int heads, int tokens) {
  int64_t groups = (int64_t)batch * layers * heads;
  int64_t e = groups * SPHKV_MAX_TIERS;
  // counts, page_base (int), code_base (u64), err, page_items (int per state + slack)
  return 256 + e * 4 * 2 + e * 8 + 64 + (groups * tokens + groups * SPHKV_MAX_TIERS * 1024) * 4;
}

extern "C" int sphkv_pack_pages_groups(const sphkv_store_t* st, int group0, int n_groups,
                                       const void* keys, int key_dtype, const double* angles,
                                       const double* radii, const uint16_t* values,
                                       const int8_t* z, const int16_t* tier,
                                       const uint8_t* protect, int tokens, void* workspace,
                                       int64_t workspace_bytes, cudaStream_t stream) {
  if (int e = validate_store(st)) return e;
  if (!radii || !values || !z || !tier || !protect || !workspace)
    return fail(SPHKV_E_VALUE, "null argument");
  if (!angles && (!keys || check_dtype(key_dtype))) return fail(SPHKV_E_VALUE, "need keys or angles");
  const int groups = st->batch * st->layers * st->heads;
  if (group0 < 0 || n_groups < 0 || group0 + n_groups > groups)
    return fail(SPHKV_E_KEY, "groups [%d, %d) outside the store's %d", group0, group0 + n_groups,
                groups);
  if (n_groups == 0) return SPHKV_OK;
  const int NT = st->n_tiers;
  const int P = st->page_size;
  if (groups * NT > 1023 * 64) return fail(SPHKV_E_UNSUPPORTED, "too many (group, tier) entries");
  int64_t need = sphkv_pack_workspace_bytes(st->batch, st->layers, st->heads, tokens);
  need -= (int64_t)(groups - n_groups) * tokens * 4;  // page_items of the packed groups only
  if (workspace_bytes < need) return fail(SPHKV_E_VALUE, "pack workspace too small (%lld < %lld)",
                                          (long long)workspace_bytes, (long long)need);
  uint8_t* ws = (uint8_t*)workspace;
  const int64_t E = (int64_t)groups * SPHKV_MAX_TIERS;
  int* err = (int*)ws;
  int* counts = (int*)(ws + 256);
  int* page_base = counts + E;
  uint64_t* code_base = (uint64_t*)(ws + 256 + E * 8);
  int* page_items = (int*)(ws + 256 + E * 8 + E * 8 + 64);
  SPHKV_CUDA_TRY(cudaMemsetAsync(err, 0, 256, stream));
  SPHKV_CUDA_TRY(cudaMemsetAsync(counts, 0, E * 4, stream));

  // read the current page count (fresh stores: 0) for the page range we write
  uint64_t host_counters[2];
  SPHKV_CUDA_TRY(cudaMemcpyAsync(host_counters, st->counters, 16, cudaMemcpyDeviceToHost, stream));
  k_pack_count<<<n_groups, 256, 0, stream>>>(*st, tokens, group0, z, tier, counts, err);
  SPHKV_LAUNCH_CHECK();
  k_pack_plan<<<1, 1023, 0, stream>>>(*st, counts, page_base, code_base, err);
  SPHKV_LAUNCH_CHECK();
  k_pack_pages_init<<<groups * NT, 128, 0, stream>>>(*st, counts, page_base, code_base, err);
  SPHKV_LAUNCH_CHECK();
  k_pack_ptrlen<<<(groups + 255) / 256, 256, 0, stream>>>(*st, page_base, err);
  SPHKV_LAUNCH_CHECK();
  uint64_t after[2];
  int herr = 0;
  SPHKV_CUDA_TRY(cudaMemcpyAsync(after, st->counters, 16, cudaMemcpyDeviceToHost, stream));
  SPHKV_CUDA_TRY(cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, stream));
  SPHKV_CUDA_TRY(cudaStreamSynchronize(stream));
  if (herr == 1 || herr == 2) return fail(SPHKV_E_VALUE, "retained state assigned to the drop tier / bad z");
  if (herr == 3) return fail(SPHKV_E_CAPACITY, "store pool exhausted (pages or code bytes)");
  if (herr == 4) return fail(SPHKV_E_CAPACITY, "pointer list capacity exceeded");
  const int first = (int)host_counters[0];
  const int n_new = (int)(after[0] - host_counters[0]);
  if (n_new == 0) return SPHKV_OK;
  k_pack_rank<<<n_groups, 1024, 0, stream>>>(*st, tokens, group0, z, tier, page_base, first,
                                             page_items);
  SPHKV_LAUNCH_CHECK();
  k_pack_scale<<<n_new, 128, 0, stream>>>(*st, first, n_new, page_items, radii);
  SPHKV_LAUNCH_CHECK();
  const int64_t jobs = (int64_t)n_new * (P / 32);
  const int blocks = (int)div_up(jobs, 8);
  if (angles) {
    k_pack_write<float><<<blocks, 256, 0, stream>>>(*st, first, n_new, tokens, nullptr, angles,
                                                     radii, values, protect, page_items);
  } else {
    switch (key_dtype) {
      case SPHKV_F32: k_pack_write<float><<<blocks, 256, 0, stream>>>(*st, first, n_new, tokens, (const float*)keys, nullptr, radii, values, protect, page_items); break;
      case SPHKV_F64: k_pack_write<double><<<blocks, 256, 0, stream>>>(*st, first, n_new, tokens, (const double*)keys, nullptr, radii, values, protect, page_items); break;
      case SPHKV_BF16: k_pack_write<__nv_bfloat16><<<blocks, 256, 0, stream>>>(*st, first, n_new, tokens, (const __nv_bfloat16*)keys, nullptr, radii, values, protect, page_items); break;
      default: k_pack_write<__half><<<blocks, 256, 0, stream>>>(*st, first, n_new, tokens, (const __half*)keys, nullptr, radii, values, protect, page_items); break;
    }
  }
  SPHKV_LAUNCH_CHECK();
  return SPHKV_OK;
}

extern "C" int sphkv_pack_pages(const sphkv_store_t* st, const void* keys, int key_dtype,
                                const double* angles, const double* radii, const uint16_t* values,
                                const int8_t* z, const int16_t* tier, const uint8_t* protect,
                                int tokens, void* workspace, int64_t workspace_bytes,
                                cudaStream_t stream) {
  if (!st) return fail(SPHKV_E_VALUE, "null argument");
  return sphkv_pack_pages_groups(st, 0, st->batch * st->layers * st->heads, keys, key_dtype,
                                 angles, radii, values, z, tier, protect, tokens, workspace,
                                 workspace_bytes, stream);
}

extern "C" int64_t sphkv_append_workspace_bytes(int groups) {
  return 256 + (int64_t)groups * (4 + 4 + 8) + (int64_t)groups * 255 * 8 + 64;
}

extern "C" int sphkv_append(const sphkv_store_t* st, const void* keys, int key_dtype,
                            const double* radii, const double* angles, const uint16_t* values,
                            const int16_t* tier_ids, const uint8_t* protect,
                            const int64_t* token_ids, const uint8_t* active, void* workspace,
                            cudaStream_t stream) {
  if (int e = validate_store(st)) return e;
  if (!values || !tier_ids || !workspace) return fail(SPHKV_E_VALUE, "null argument");
  const int n = st->batch * st->layers * st->heads;
  const int d = st->d;
  uint8_t* ws8 = (uint8_t*)workspace;
  AppendWs ws;
  ws.err = (int*)ws8;
  ws.flag = (int*)(ws8 + 256);
  ws.slot = ws.flag + n;
  ws.radius = (double*)(ws8 + 256 + (((int64_t)n * 8 + 63) / 64) * 64);
  ws.angles = ws.radius + n;
  SPHKV_CUDA_TRY(cudaMemsetAsync(ws.err, 0, 4, stream));
  if (angles) {
    SPHKV_CUDA_TRY(cudaMemcpyAsync(ws.angles, angles, (size_t)n * (d - 1) * 8,
                                   cudaMemcpyDeviceToDevice, stream));
    if (radii) SPHKV_CUDA_TRY(cudaMemcpyAsync(ws.radius, radii, (size_t)n * 8, cudaMemcpyDeviceToDevice, stream));
    else return fail(SPHKV_E_VALUE, "angles given without radii");
  } else {
    if (!keys || check_dtype(key_dtype)) return fail(SPHKV_E_VALUE, "need keys or angles");
    if (int e = sphkv_encode(keys, key_dtype, n, d, ws.radius, ws.angles, stream)) return e;
    if (radii) SPHKV_CUDA_TRY(cudaMemcpyAsync(ws.radius, radii, (size_t)n * 8, cudaMemcpyDeviceToDevice, stream));
  }
  k_append_decide<<<(n + 127) / 128, 128, 0, stream>>>(*st, n, nullptr, tier_ids, active, ws);
  SPHKV_LAUNCH_CHECK();
  k_append_alloc<<<1, 1023, 0, stream>>>(*st, n, tier_ids, ws);
  SPHKV_LAUNCH_CHECK();
  k_append_write<<<(n * 32 + 127) / 128, 128, 0, stream>>>(*st, n, tier_ids, values, protect,
                                                            token_ids, ws);
  SPHKV_LAUNCH_CHECK();
  return SPHKV_OK;
}

extern "C" int sphkv_score_append(const double* radii, int groups_per_seq, int heads,
                                  const double* u_hat, const double* s_hat, double r_q,
                                  double omega, double alpha_theta, double alpha_r,
                                  const sphkv_tier_t* tiers_host, int n_tiers, double lam, int d,
                                  int64_t n, int16_t* tier_out, double* score_out, double* nu_out,
                                  cudaStream_t stream) {
  (void)heads;
  if (n_tiers < 2 || n_tiers > SPHKV_MAX_TIERS) return fail(SPHKV_E_VALUE, "bad tier count");
  if (n == 0) return SPHKV_OK;
  k_score_append<<<(int)div_up(n, 128), 128, 0, stream>>>(radii, groups_per_seq, heads, u_hat,
                                                          s_hat, r_q, omega, alpha_theta, alpha_r,
                                                          make_tierset(tiers_host, n_tiers),
                                                          n_tiers, lam, d, n, tier_out, score_out,
                                                          nu_out);
  SPHKV_LAUNCH_CHECK();
  return SPHKV_OK;
}

extern "C" int sphkv_decode_gate(const sphkv_store_t* st, const void* keys, int key_dtype,
                                 const float* q, int G, const float* margins,
                                 const double* u_hat, const double* s_hat, double r_q,
                                 double omega, double alpha_theta, double alpha_r, double lam,
                                 int use_gate, double tau_drop, double tau_prot,
                                 double gate_alpha, int8_t* mode, int16_t* tier_out,
                                 uint8_t* protect_out, float* danger_out, cudaStream_t stream) {
  if (int e = validate_store(st)) return e;
  if (!keys || !u_hat || !s_hat || !tier_out || !protect_out) return fail(SPHKV_E_VALUE, "null argument");
  if (use_gate && (!q || !margins || !mode)) return fail(SPHKV_E_VALUE, "the gate needs q, margins, mode");
  if (G < 1 || G > 32) return fail(SPHKV_E_UNSUPPORTED, "G=%d", G);
  if (use_gate && !(tau_drop < tau_prot)) return fail(SPHKV_E_VALUE, "tau_drop < tau_prot");
  if (check_dtype(key_dtype)) return SPHKV_E_VALUE;
  const int groups = st->batch * st->layers * st->heads;
  const int blocks = (groups * 32 + 127) / 128;
#define SPHKV_GATE_ARGS                                                                       \
  *st, (const T*)keys, q, G, margins, u_hat, s_hat, r_q, omega, alpha_theta, alpha_r, lam,     \
      use_gate, tau_drop, tau_prot, gate_alpha, mode, tier_out, protect_out, danger_out
  switch (key_dtype) {
    case SPHKV_F32: { using T = float; k_decode_gate<T><<<blocks, 128, 0, stream>>>(SPHKV_GATE_ARGS); break; }
    case SPHKV_F64: { using T = double; k_decode_gate<T><<<blocks, 128, 0, stream>>>(SPHKV_GATE_ARGS); break; }
    case SPHKV_BF16: { using T = __nv_bfloat16; k_decode_gate<T><<<blocks, 128, 0, stream>>>(SPHKV_GATE_ARGS); break; }
    default: { using T = __half; k_decode_gate<T><<<blocks, 128, 0, stream>>>(SPHKV_GATE_ARGS); break; }
  }
#undef SPHKV_GATE_ARGS
  SPHKV_LAUNCH_CHECK();
  return SPHKV_OK;
}

extern "C" int sphkv_export_streams(const sphkv_store_t* st, int n_pages, const int64_t* offsets,
                                    uint8_t* out, cudaStream_t stream) {
  if (int e = validate_store(st)) return e;
  if (n_pages == 0) return SPHKV_OK;
  k_export<<<n_pages, 256, 0, stream>>>(*st, offsets, out);
  SPHKV_LAUNCH_CHECK();
  return SPHKV_OK;
}

extern "C" int sphkv_import_streams(const sphkv_store_t* st, int n_pages, const int64_t* offsets,
                                    const uint8_t* in, cudaStream_t stream) {
  if (int e = validate_store(st)) return e;
  if (n_pages < 0 || n_pages > st->max_pages) return fail(SPHKV_E_CAPACITY, "n_pages %d", n_pages);
  if (n_pages == 0) return SPHKV_OK;
  if (!offsets || !in) return fail(SPHKV_E_VALUE, "null argument");
  k_import<<<n_pages, 256, 0, stream>>>(*st, offsets, in);
  SPHKV_LAUNCH_CHECK();
  return SPHKV_OK;
}

extern "C" int sphkv_dense_fill_groups(const sphkv_dense_store_t* st, int group0, int n_groups,
                                       const void* keys, int key_dtype, const uint16_t* values,
                                       cudaStream_t stream) {
  if (!st || !keys || !values) return fail(SPHKV_E_VALUE, "null argument");
  if (check_dtype(key_dtype)) return SPHKV_E_VALUE;
  const int groups = st->batch * st->layers * st->heads;
  if (group0 < 0 || n_groups < 0 || group0 + n_groups > groups)
    return fail(SPHKV_E_KEY, "groups [%d, %d) outside the store's %d", group0, group0 + n_groups,
                groups);
  if (n_groups == 0) return SPHKV_OK;
  const int64_t g0 = group0, ng = n_groups;
  switch (key_dtype) {
    case SPHKV_F32: k_dense_fill<float><<<4 * SM_COUNT, 256, 0, stream>>>(*st, g0, ng, (const float*)keys, values); break;
    case SPHKV_F64: k_dense_fill<double><<<4 * SM_COUNT, 256, 0, stream>>>(*st, g0, ng, (const double*)keys, values); break;
    case SPHKV_BF16: k_dense_fill<__nv_bfloat16><<<4 * SM_COUNT, 256, 0, stream>>>(*st, g0, ng, (const __nv_bfloat16*)keys, values); break;
    default: k_dense_fill<__half><<<4 * SM_COUNT, 256, 0, stream>>>(*st, g0, ng, (const __half*)keys, values); break;
  }
  SPHKV_LAUNCH_CHECK();
  return SPHKV_OK;
}

extern "C" int sphkv_dense_fill(const sphkv_dense_store_t* st, const void* keys, int key_dtype,
                                const uint16_t* values, cudaStream_t stream) {
  if (!st) return fail(SPHKV_E_VALUE, "null argument");
  return sphkv_dense_fill_groups(st, 0, st->batch * st->layers * st->heads, keys, key_dtype,
                                 values, stream);
}

namespace sphkv {
__global__ void k_f64_to_f16(const double* __restrict__ in, int64_t n, __half* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __double2half(in[i]);  // single rounding, RN-even
}
}  // namespace sphkv

extern "C" int sphkv_f64_to_f16(const double* in, int64_t n, uint16_t* out, cudaStream_t stream) {
  if (n < 0 || (n > 0 && (!in || !out))) return fail(SPHKV_E_VALUE, "null argument");
  if (n == 0) return SPHKV_OK;
  const int64_t blocks = (n + 255) / 256;
  k_f64_to_f16<<<(int)(blocks < 8 * SM_COUNT ? blocks : 8 * SM_COUNT), 256, 0, stream>>>(
      in, n, reinterpret_cast<__half*>(out));
  SPHKV_LAUNCH_CHECK();
  return SPHKV_OK;
}
