// dpq_ivf.cuh — inverted-file search (IVFIndex, ivf.py:107-277) and the
// sharded-flat split API.  Included at the end of dpq_flat.cu
// (same translation unit: the kernels are header-defined).
//
// IVF derived batch (nb queries, ma probes each):
//   probe (f64 centre distances, top-ma with lower-id ties)
//   -> slots (query, probe) of non-empty lists, grouped by cell into query
//      tiles of QT slots: every list is streamed once per tile of queries
//      probing it ("query-by-list batching")
//   -> K1 twice: small tables per slot; qmin/qmax from the first non-empty
//      probed list of each query (ivf.py:205-217); quantize every slot with
//      its query's bounds
//   -> guard per query from per-list sampled histograms
//   -> the flat scan kernel over (tile, list row range) units, emitting into
//      per-query lists (one candidate pool per query, ivf.py:222-236)
//   -> K3 per query -> refine each candidate in its own cell's residual
//      frame (ivf.py:253-268), ids = sorted_ids_.
#pragma once

namespace dpq {

// ---------------------------------------------------------------------------
// probe: d2[c] = sum_t (c_t - y_t)^2 in f64, ascending, ties to lower cell.
// ---------------------------------------------------------------------------
template <int BUF, int NT>
__global__ void __launch_bounds__(NT) k_probe(const float* __restrict__ y, int d,
                                              const float* __restrict__ centers, int K, int ma,
                                              int64_t* __restrict__ cells) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem);
  int64_t* ids = reinterpret_cast<int64_t*>(keys + BUF);
  float* ys = reinterpret_cast<float*>(ids + BUF);
  __shared__ int fill;
  __shared__ uint64_t thr_k;
  __shared__ int64_t thr_i;
  const int q = blockIdx.x;
  for (int i = threadIdx.x; i < d; i += NT) ys[i] = y[(int64_t)q * d + i];
  if (threadIdx.x == 0) { fill = 0; thr_k = ~0ull; thr_i = INT64_MAX; }
  __syncthreads();
  for (int base = 0; base < K; base += NT) {
    const int c = base + threadIdx.x;
    bool keep = false;
    uint64_t key = 0;
    if (c < K) {
      const float* cr = centers + (int64_t)c * d;
      double acc = 0.0;
      for (int t = 0; t < d; ++t) {
        const double df = __dsub_rn((double)cr[t], (double)ys[t]);
        acc = __dadd_rn(acc, __dmul_rn(df, df));
      }
      key = (uint64_t)__double_as_longlong(acc);
      keep = pair_less(key, c, thr_k, thr_i);
    }
    if (keep) {
      const int p = atomicAdd(&fill, 1);
      keys[p] = key;
      ids[p] = c;
    }
    __syncthreads();
    const int f = fill;
    __syncthreads();
    if (f > BUF - NT) {
      for (int i = f + threadIdx.x; i < BUF; i += NT) { keys[i] = ~0ull; ids[i] = INT64_MAX; }
      __syncthreads();
      sort_pairs<NT>(keys, ids, BUF);
      if (threadIdx.x == 0) {
        const int nf = min(f, ma);
        fill = nf;
        if (nf == ma) { thr_k = keys[nf - 1]; thr_i = ids[nf - 1]; }
      }
      __syncthreads();
    }
  }
  const int f = fill;
  for (int i = f + threadIdx.x; i < BUF; i += NT) { keys[i] = ~0ull; ids[i] = INT64_MAX; }
  __syncthreads();
  sort_pairs<NT>(keys, ids, BUF);
  for (int i = threadIdx.x; i < ma; i += NT) cells[(int64_t)q * ma + i] = ids[i];
}

// Query-tiled probe (K <= 8192): k_probe_dist computes d2 for a tile of 16
// queries x 256 centres per CTA with the centres staged through shared memory
// (each centre row read once per 16 queries instead of once per query), same
// f64 arithmetic as k_probe; k_probe_select keeps each query's ma smallest
// (d2, cell) pairs — ties to the lower cell — and writes them sorted.
constexpr int kProbeQT = 16, kProbeCT = 256, kProbeDC = 32;
__global__ void __launch_bounds__(kProbeCT) k_probe_dist(const float* __restrict__ y, int d, int nq,
                                                          const float* __restrict__ centers, int K,
                                                          double* __restrict__ d2) {
  __shared__ float cs[kProbeCT][kProbeDC + 1];
  __shared__ float ys[kProbeQT][kProbeDC];
  const int c0 = blockIdx.x * kProbeCT, q0 = blockIdx.y * kProbeQT, tid = threadIdx.x;
  double acc[kProbeQT];
#pragma unroll
  for (int q = 0; q < kProbeQT; ++q) acc[q] = 0.0;
  for (int t0 = 0; t0 < d; t0 += kProbeDC) {
    const int dc = min(kProbeDC, d - t0);
    __syncthreads();
    for (int i = tid; i < kProbeCT * kProbeDC; i += kProbeCT) {
      const int r = i / kProbeDC, t = i % kProbeDC;
      cs[r][t] = (c0 + r < K && t < dc) ? centers[(int64_t)(c0 + r) * d + t0 + t] : 0.f;
    }
    for (int i = tid; i < kProbeQT * kProbeDC; i += kProbeCT) {
      const int q = i / kProbeDC, t = i % kProbeDC;
      ys[q][t] = (q0 + q < nq && t < dc) ? y[(int64_t)(q0 + q) * d + t0 + t] : 0.f;
    }
    __syncthreads();
    for (int t = 0; t < dc; ++t) {
      const double c = (double)cs[tid][t];
#pragma unroll
      for (int q = 0; q < kProbeQT; ++q) {
        const double df = __dsub_rn(c, (double)ys[q][t]);
        acc[q] = __dadd_rn(acc[q], __dmul_rn(df, df));
      }
    }
  }
  if (c0 + tid < K)
#pragma unroll
    for (int q = 0; q < kProbeQT; ++q)
      if (q0 + q < nq) d2[(int64_t)(q0 + q) * K + c0 + tid] = acc[q];
}

template <int NT, int EPT>
__global__ void __launch_bounds__(NT, 1) k_probe_select(const double* __restrict__ d2, int K, int ma,
                                                        int64_t* __restrict__ cells) {
  // the ma smallest (d2, cell) pairs of the query's K: exact radix select
  // (select_r, the refine's), then a bitonic sort of the ma kept pairs
  extern __shared__ __align__(16) uint8_t probe_smem[];
  uint64_t* keys = reinterpret_cast<uint64_t*>(probe_smem);
  int64_t* ids = reinterpret_cast<int64_t*>(keys + NT * EPT);
  __shared__ SelShared S;
  __shared__ uint64_t thr_k;
  __shared__ int64_t thr_i;
  const int q = blockIdx.x;
  for (int i = threadIdx.x; i < K; i += NT) {
    keys[i] = (uint64_t)__double_as_longlong(d2[(int64_t)q * K + i]);  // d2 >= 0: bits order as values
    ids[i] = i;
  }
  __syncthreads();
  if (K > ma) select_r<NT, EPT>(keys, ids, K, ma, S, thr_k, thr_i);
  const int f = min(K, ma);
  int P = 2;
  while (P < f) P <<= 1;
  for (int i = f + threadIdx.x; i < P; i += NT) { keys[i] = ~0ull; ids[i] = INT64_MAX; }
  __syncthreads();
  sort_pairs<NT>(keys, ids, P);
  for (int i = threadIdx.x; i < ma; i += NT) cells[(int64_t)q * ma + i] = ids[i];
}

// Tensor-core probe (ivf.py:107-120 on the 5th-generation tensor cores).
// The squared distances of a query to all K centres come from the 3xTF32
// table GEMM of dpq_tctab.cu (centres = an m = 1 codebook, kbar = 1, so the
// entries are in centre order) with rigorous bounds: |approx_c - d2_c| <=
// E_c = gamma (||y - mu|| + ||c - mu||)^2 <= eps (the query's bound with
// the largest centre norm).  Per query (one 256-thread CTA, K <= 8192):
// A = the ma-th smallest approx (4-pass radix select on order-preserving
// 32-bit keys), tau = A + eps >= the ma-th smallest upper bound, candidates
// = {c : approx_c - E_c <= tau} (a superset of the exact ma nearest); their
// d2 is recomputed with k_probe_dist's f64 arithmetic and the ma smallest
// (d2, cell) pairs are written in order — the f64 probe's cells, from ~ma
// exact distances instead of K.  More than kPtcCand candidates (not seen):
// every centre is recomputed exactly.
constexpr int kPtcThreads = 256, kPtcEpt = 32, kPtcCand = 1024;
__device__ __forceinline__ uint32_t f32_order_key(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__global__ void __launch_bounds__(kPtcThreads) k_probe_select_tc(const float* __restrict__ approx,
                                                                 const double* __restrict__ eps,
                                                                 const double* __restrict__ ny,
                                                                 const float* __restrict__ cnorm, double gamma,
                                                                 const float* __restrict__ y, int d,
                                                                 const float* __restrict__ centers, int K, int ma,
                                                                 int64_t* __restrict__ cells,
                                                                 unsigned long long* __restrict__ n_exact) {
  __shared__ uint32_t hist[256];
  __shared__ uint32_t s_pfx, s_need;
  __shared__ int ncand;
  __shared__ uint64_t ckey[kPtcCand];
  __shared__ int64_t cid[kPtcCand];
  __shared__ float ys[128];
  const int q = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* aq = approx + (int64_t)q * K;
  uint32_t key[kPtcEpt];
#pragma unroll
  for (int e = 0; e < kPtcEpt; ++e) {
    const int c = tid + e * kPtcThreads;
    key[e] = c < K ? f32_order_key(aq[c]) : 0xFFFFFFFFu;
  }
  for (int i = tid; i < d; i += kPtcThreads) ys[i] = y[(int64_t)q * d + i];
  if (tid == 0) { s_pfx = 0u; s_need = (uint32_t)ma; ncand = 0; }
  // the ma-th smallest key: 4 digit passes (prefix known above the digit)
  for (int pass = 0; pass < 4; ++pass) {
    const int sft = 24 - 8 * pass;
    for (int i = tid; i < 256; i += kPtcThreads) hist[i] = 0u;
    __syncthreads();
    const uint32_t pfx = s_pfx, hmask = pass == 0 ? 0u : (0xFFFFFFFFu << (sft + 8));
#pragma unroll
    for (int e = 0; e < kPtcEpt; ++e)
      if ((key[e] & hmask) == pfx && tid + e * kPtcThreads < K) atomicAdd(&hist[(key[e] >> sft) & 0xFFu], 1u);
    __syncthreads();
    if (warp == 0) {
      const uint32_t need = s_need;
      uint32_t ls = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) ls += hist[lane * 8 + i];
      uint32_t incl = ls;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const int L = __ffs(__ballot_sync(0xffffffffu, incl >= need)) - 1;
      if (lane == L) {
        uint32_t below = incl - ls;
        int dg = lane * 8;
        for (int i = 0; i < 8; ++i) {
          const uint32_t hb = hist[lane * 8 + i];
          if (below + hb >= need) { dg = lane * 8 + i; break; }
          below += hb;
        }
        s_need = need - below;
        s_pfx = pfx | ((uint32_t)dg << sft);
      }
    }
    __syncthreads();
  }
  const uint32_t kth = s_pfx;
  const float A = __uint_as_float((kth & 0x80000000u) ? (kth & 0x7FFFFFFFu) : ~kth);
  const double tau = (double)A + eps[q] * (1.0 + 1e-9);
  const double nyq = ny[q];
  const double loose = tau + eps[q] * (1.0 + 1e-9);  // approx_c <= tau + E_c <= tau + eps
#pragma unroll
  for (int e = 0; e < kPtcEpt; ++e) {
    const int c = tid + e * kPtcThreads;
    if (c < K) {
      const double a = (double)aq[c];
      if (a <= loose) {
        const double sn = nyq + (double)cnorm[c];
        if (a - gamma * sn * sn * (1.0 + 1e-9) <= tau) {
          const int p = atomicAdd(&ncand, 1);
          if (p < kPtcCand) cid[p] = c;
        }
      }
    }
  }
  __syncthreads();
  const int nc = ncand;
  auto exact = [&](int c) {  // k_probe_dist's arithmetic (sequential f64)
    const float* cr = centers + (int64_t)c * d;
    double acc = 0.0;
    for (int t = 0; t < d; ++t) {
      const double df = __dsub_rn((double)cr[t], (double)ys[t]);
      acc = __dadd_rn(acc, __dmul_rn(df, df));
    }
    return acc;
  };
  if (nc <= kPtcCand) {
    for (int i = tid; i < nc; i += kPtcThreads) ckey[i] = (uint64_t)__double_as_longlong(exact((int)cid[i]));
    int P = 2;
    while (P < nc) P <<= 1;
    for (int i = nc + tid; i < P; i += kPtcThreads) { ckey[i] = ~0ull; cid[i] = INT64_MAX; }
    __syncthreads();
    sort_pairs<kPtcThreads>(ckey, cid, P);
    for (int i = tid; i < ma; i += kPtcThreads) cells[(int64_t)q * ma + i] = cid[i];
  } else {
    // (degenerate bounds) exact top-ma of all K: running buffer of kPtcCand / 2
    const int half = kPtcCand / 2;
    int fill = 0;
    for (int base = 0; base < K; base += half) {
      const int n = min(half, K - base);
      for (int i = tid; i < n; i += kPtcThreads) {
        ckey[fill + i] = (uint64_t)__double_as_longlong(exact(base + i));
        cid[fill + i] = base + i;
      }
      for (int i = fill + n + tid; i < kPtcCand; i += kPtcThreads) { ckey[i] = ~0ull; cid[i] = INT64_MAX; }
      __syncthreads();
      sort_pairs<kPtcThreads>(ckey, cid, kPtcCand);
      fill = min(ma, fill + n);
    }
    for (int i = tid; i < ma; i += kPtcThreads) cells[(int64_t)q * ma + i] = cid[i];
  }
  if (tid == 0 && n_exact) atomicAdd(n_exact, (unsigned long long)(nc <= kPtcCand ? nc : K));
}

// residuals y - centre in f32 (ivf.py:120), natural (query, probe) order
__global__ void k_residuals(const float* __restrict__ y, const float* __restrict__ centers,
                            const int64_t* __restrict__ cells, int nq, int ma, int d,
                            float* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)nq * ma * d;
  if (i >= total) return;
  const int t = (int)(i % d);
  const int64_t s = i / d;
  const int q = (int)(s / ma);
  out[i] = __fsub_rn(y[(int64_t)q * d + t], centers[cells[s] * d + t]);
}

// per tile-slot copy of its (query, probe) residual; zeros for padding
// bounds of every slot = (qmin, qmax) of its query's first non-empty list
__global__ void k_slot_bounds(const double* __restrict__ qmin, const double* __restrict__ qmax,
                              const int* __restrict__ bound_ts, const int* __restrict__ slot_query,
                              int nts, double* __restrict__ bounds) {
  const int ts = blockIdx.x * blockDim.x + threadIdx.x;
  if (ts >= nts) return;
  const int q = slot_query[ts];
  const int b = q < 0 ? -1 : bound_ts[q];
  bounds[2 * ts] = b < 0 ? 0.0 : qmin[b];
  bounds[2 * ts + 1] = b < 0 ? 0.0 : qmax[b];
}

// per-query histograms from the live slots' histograms (padding slots skipped)
__global__ void k_expand_gword(const uint16_t* __restrict__ gq, const int* __restrict__ slot_query, int nts,
                               uint16_t* __restrict__ gts) {
  const int ts = blockIdx.x * blockDim.x + threadIdx.x;
  if (ts >= nts) return;
  const int q = slot_query[ts];
  gts[ts] = q < 0 ? (uint16_t)0x7F7F : gq[q];
}

// Conventional IVF scan (ivf.py:162-193): every row of every probed list is
// a candidate; exact entries computed per row in its cell's frame.
struct IvfConvArgs {
  const int64_t* cells; const int64_t* offsets; int ma;
  const void* codes; int code_bytes; int m, k, dsub;
  const float* cb; const float* ynat; const int64_t* sorted_ids;
  int r; double* out_d; int64_t* out_i;
  int y_in_smem = 1;  // residual block staged in shared memory (else read from global)
};

template <int BUF, int NT>
__global__ void __launch_bounds__(NT) k_ivf_conventional(IvfConvArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem);
  int64_t* ids = reinterpret_cast<int64_t*>(keys + BUF);
  float* ys_s = reinterpret_cast<float*>(ids + BUF);
  __shared__ int fill;
  __shared__ uint64_t thr_k;
  __shared__ int64_t thr_i;
  const int q = blockIdx.x;
  const int d = a.m * a.dsub;
  const float* ys = a.y_in_smem ? ys_s : a.ynat + (int64_t)q * a.ma * d;
  if (a.y_in_smem)
    for (int i = threadIdx.x; i < a.ma * d; i += NT) ys_s[i] = a.ynat[(int64_t)q * a.ma * d + i];
  if (threadIdx.x == 0) { fill = 0; thr_k = ~0ull; thr_i = INT64_MAX; }
  __syncthreads();
  for (int p = 0; p < a.ma; ++p) {
    const int64_t cell = a.cells[(int64_t)q * a.ma + p];
    const int64_t lo = a.offsets[cell], hi = a.offsets[cell + 1];
    for (int64_t base = lo; base < hi; base += NT) {
      const int64_t row = base + threadIdx.x;
      bool keep = false;
      uint64_t key = 0;
      int64_t id = 0;
      if (row < hi) {
        double dist = 0.0;
        for (int j = 0; j < a.m; ++j) {
          const uint32_t c = code_at(a.codes, a.code_bytes, row * a.m + j);
          const float t = pw_sqdist(a.cb + ((int64_t)j * a.k + c) * a.dsub, ys + p * d + j * a.dsub, a.dsub);
          dist = __dadd_rn(dist, (double)t);
        }
        key = (uint64_t)__double_as_longlong(dist);
        id = a.sorted_ids[row];
        keep = pair_less(key, id, thr_k, thr_i);
      }
      if (keep) {
        const int pp = atomicAdd(&fill, 1);
        keys[pp] = key;
        ids[pp] = id;
      }
      __syncthreads();
      const int f = fill;
      __syncthreads();
      if (f > BUF - NT) {
        for (int i = f + threadIdx.x; i < BUF; i += NT) { keys[i] = ~0ull; ids[i] = INT64_MAX; }
        __syncthreads();
        sort_pairs<NT>(keys, ids, BUF);
        if (threadIdx.x == 0) {
          const int nf = min(f, a.r);
          fill = nf;
          if (nf == a.r) { thr_k = keys[nf - 1]; thr_i = ids[nf - 1]; }
        }
        __syncthreads();
      }
    }
  }
  const int f = fill;
  for (int i = f + threadIdx.x; i < BUF; i += NT) { keys[i] = ~0ull; ids[i] = INT64_MAX; }
  __syncthreads();
  sort_pairs<NT>(keys, ids, BUF);
  const int got = min(f, a.r);
  for (int i = threadIdx.x; i < a.r; i += NT) {
    const int64_t o = (int64_t)q * a.r + i;
    a.out_d[o] = i < got ? __longlong_as_double((long long)keys[i]) : INFINITY;
    a.out_i[o] = i < got ? ids[i] : -1;
  }
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
// Page-locked host allocator: the plan's per-slot arrays (~1M entries per
// 4096-query batch) are DMA'd to the device every batch.
template <class T>
struct PinnedAllocator {
  using value_type = T;
  PinnedAllocator() = default;
  template <class U>
  PinnedAllocator(const PinnedAllocator<U>&) {}
  T* allocate(size_t n) {
    void* p = nullptr;
    if (cudaMallocHost(&p, n * sizeof(T)) != cudaSuccess) {
      cudaGetLastError();
      throw std::bad_alloc();
    }
    return static_cast<T*>(p);
  }
  void deallocate(T* p, size_t) { cudaFreeHost(p); }
  template <class U>
  bool operator==(const PinnedAllocator<U>&) const { return true; }
  template <class U>
  bool operator!=(const PinnedAllocator<U>&) const { return false; }
};
template <class T>
using pinned_vector = std::vector<T, PinnedAllocator<T>>;


struct IvfPlan {
  int nq = 0, ma = 0, nts = 0, ntiles = 0;
  int nph = 0;                         // shard: bound-source slots after the tile slots (list empty here)
  pinned_vector<int> phantom;          // their slot indices
  std::vector<int64_t> nr_global;      // shard: rows of the probed GLOBAL lists per query
  pinned_vector<int64_t> cells;        // (nq, ma)
  pinned_vector<int> slot_query, slot_probe;
  std::vector<int> tile_cell;
  pinned_vector<int> bound_ts;
  std::vector<int> cnt, first, tile0, ts_first, cnt_t, base_t;  // scratch of ivf_plan (capacity kept)
  std::vector<int64_t> nr, sq;
  pinned_vector<int> live, bsrc;       // live (non-padding) slots; bound-source slots
  pinned_vector<int64_t> pre_off, pre_len, tile_row0, tile_nsamp, ns_tmp;
  pinned_vector<int> unit_tile;
  pinned_vector<int64_t> unit_r0, unit_r1;
  pinned_vector<double> lambda;        // per query, <0 = exact histogram
  int64_t stride = 1, max_nsamp = 0;
  bool dev = false;                    // built on the device (ivf_plan_dev): the vectors above are unused
  int nlive = 0, nbsrc = 0, n_units = 0;  // (device plan: n_units is an upper bound, the count is B.pl_nunits)
};

struct IvfBuffers {
  IvfPlan plan;  // host plan of the last batch (reused: no per-batch allocation)
  int cap_q = 0, cap_ts = 0, cap_units = 0, cap_tiles = 0, cap_ma = 0;
  int64_t* cells = nullptr;
  float* ynat = nullptr;
  float* yts = nullptr;
  int* bound_ts = nullptr;
  int* live = nullptr;                 // [cap_ts]
  int* bsrc = nullptr;                 // [cap_q]
  double* lambda = nullptr;
  uint32_t* hist_q = nullptr;
  uint16_t* gword_q = nullptr;
  uint16_t* guard_q = nullptr;
  int* unit_tile = nullptr;
  int64_t* unit_r0 = nullptr;
  int64_t* unit_r1 = nullptr;
  int64_t* tile_row0 = nullptr;
  int64_t* tile_nsamp = nullptr;
  int* phantom = nullptr;              // [cap_q] shard bound-source slots
  double* d2 = nullptr;                // probe distances (nq, K)
  int64_t cap_d2 = 0;
  // tensor-core probe: centres as an m = 1 codebook (dpq_tctab.cu)
  void* ptc = nullptr;
  int ptc_state = 0;                   // 0 untried, 1 ready, -1 unavailable
  float* papprox = nullptr;            // (nq, K) approximate squared distances
  double* peps = nullptr;              // (nq) entry bound of the query (unused: per-entry bounds below)
  double* pny = nullptr;               // (nq) ||y - mu||
  int64_t cap_pa = 0;
  int cap_pq = 0;
  cudaEvent_t ev_cells = nullptr;      // probe cells copied to the host
  // device plan (ivf_plan_dev)
  int cap_pp = 0, cap_pk = 0, cap_ptiles = 0;
  size_t cap_ptmp = 0;
  int *pl_key = nullptr, *pl_val = nullptr, *pl_key2 = nullptr, *pl_val2 = nullptr;
  int *pl_cnt = nullptr, *pl_cstart = nullptr, *pl_tpc = nullptr, *pl_tile0 = nullptr;
  int *pl_first = nullptr, *pl_flag = nullptr, *pl_pos = nullptr;
  int64_t* pl_nr = nullptr;
  int64_t* pl_tile_len = nullptr;
  int *pl_tile_units = nullptr, *pl_ustart = nullptr, *pl_nunits = nullptr;
  void* pl_tmp = nullptr;
  unsigned long long* pl_sc = nullptr;     // device scalars
  unsigned long long* pl_sc_h = nullptr;   // pinned copy
  int64_t max_len = -1;                    // longest inverted list (host, once)
};

static IvfBuffers& ivf_bufs(Index* h) { return *reinterpret_cast<IvfBuffers*>(h->ivf_state); }

static int ivf_ensure(Index* h, int nq, int ma, int nts, int ntiles, int nunits) {
  IvfBuffers& b = ivf_bufs(h);
  const int d = h->d;
  if (nq > b.cap_q || ma > b.cap_ma) {
    b.cap_q = std::max(nq, b.cap_q);
    b.cap_ma = std::max(ma, b.cap_ma);
    DPQ_TRY(dmalloc(&b.cells, (size_t)b.cap_q * b.cap_ma));
    DPQ_TRY(dmalloc(&b.ynat, (size_t)b.cap_q * b.cap_ma * d));
    DPQ_TRY(dmalloc(&b.bound_ts, (size_t)b.cap_q));
    DPQ_TRY(dmalloc(&b.bsrc, (size_t)b.cap_q));
    DPQ_TRY(dmalloc(&b.lambda, (size_t)b.cap_q));
    DPQ_TRY(dmalloc(&b.hist_q, (size_t)b.cap_q * 256));
    DPQ_TRY(dmalloc(&b.gword_q, (size_t)b.cap_q));
    DPQ_TRY(dmalloc(&b.guard_q, (size_t)b.cap_q));
    DPQ_TRY(dmalloc(&b.phantom, (size_t)b.cap_q));
  }
  if (nts > b.cap_ts) {
    b.cap_ts = nts;
    DPQ_TRY(dmalloc(&b.live, (size_t)b.cap_ts));
  }
  if (ntiles > b.cap_tiles) {
    b.cap_tiles = ntiles;
    DPQ_TRY(dmalloc(&b.tile_row0, (size_t)ntiles));
    DPQ_TRY(dmalloc(&b.tile_nsamp, (size_t)ntiles));
  }
  if (nunits > b.cap_units) {
    b.cap_units = nunits;
    DPQ_TRY(dmalloc(&b.unit_tile, (size_t)nunits));
    DPQ_TRY(dmalloc(&b.unit_r0, (size_t)nunits));
    DPQ_TRY(dmalloc(&b.unit_r1, (size_t)nunits));
  }
  return DPQ_OK;
}

static void ivf_free(Index* h) {
  if (!h->ivf_state) return;
  IvfBuffers& b = ivf_bufs(h);
  void* p[] = {b.cells, b.ynat, b.yts, b.bound_ts, b.live, b.bsrc, b.lambda, b.hist_q, b.gword_q, b.guard_q,
               b.unit_tile, b.unit_r0, b.unit_r1, b.tile_row0, b.tile_nsamp, b.d2, b.phantom,
               b.papprox, b.peps, b.pny};
  for (void* x : p)
    if (x) cudaFree(x);
  tct_free(b.ptc);
  if (b.ev_cells) cudaEventDestroy(b.ev_cells);
  void* pl[] = {b.pl_key, b.pl_val, b.pl_key2, b.pl_val2, b.pl_cnt, b.pl_cstart, b.pl_tpc, b.pl_tile0, b.pl_first,
                b.pl_flag, b.pl_pos, b.pl_nr, b.pl_tile_len, b.pl_tile_units, b.pl_ustart, b.pl_nunits, b.pl_tmp,
                b.pl_sc};
  for (void* x : pl)
    if (x) cudaFree(x);
  if (b.pl_sc_h) cudaFreeHost(b.pl_sc_h);
  delete reinterpret_cast<IvfBuffers*>(h->ivf_state);
  h->ivf_state = nullptr;
  if (h->g_prefix) cudaFree(h->g_prefix);
  h->g_prefix = nullptr;
}

// Probe on device: cells (nb, ma) into bufs.cells.
static int ivf_probe_dev(Index* h, int nb, int ma) {
  IvfBuffers& b = ivf_bufs(h);
  // tensor-core probe (h->probe_tc: 0 off, 1 auto = K >= 1024, 2 forced)
  const int probe_tc = h->probe_tc;
  const int K = h->n_cells;
  if (nb > 0 && K <= 8192 && h->d <= 128 && ma < K && ma <= kPtcCand / 2 && tct_supported(1, K, 1, h->d) &&
      (probe_tc == 2 || (probe_tc == 1 && K >= 1024))) {
    if (b.ptc_state == 0)
      b.ptc_state = tct_prepare(h->device, h->centers, 1, K, 1, h->d, h->stream, &b.ptc) == DPQ_OK ? 1 : -1;
    if (b.ptc_state == 1) {
      if ((int64_t)nb * K > b.cap_pa) {
        if (b.papprox) cudaFree(b.papprox);
        b.papprox = nullptr;
        b.cap_pa = (int64_t)nb * K;
        DPQ_TRY(dmalloc(&b.papprox, (size_t)b.cap_pa));
      }
      if (nb > b.cap_pq) {
        if (b.peps) cudaFree(b.peps);
        if (b.pny) cudaFree(b.pny);
        b.peps = b.pny = nullptr;
        b.cap_pq = nb;
        DPQ_TRY(dmalloc(&b.peps, (size_t)nb));
        DPQ_TRY(dmalloc(&b.pny, (size_t)nb));
      }
      DPQ_TRY(tct_build(b.ptc, h->ws.y, h->d, nb, b.papprox, b.peps, b.pny, 1.0, h->stream));
      DPQ_LAUNCHED(h);
      k_probe_select_tc<<<nb, kPtcThreads, 0, h->stream>>>(b.papprox, b.peps, b.pny, tct_cnorm(b.ptc),
                                                           tct_gamma(b.ptc, 1.0), h->ws.y, h->d, h->centers, K, ma,
                                                           b.cells, h->d_nrows + 4);
      DPQ_LAUNCHED(h);
      return DPQ_OK;
    }
    cudaGetLastError();  // tct_prepare failed: the f64 path below
  }
  if (h->n_cells <= 8192 && nb > 0) {  // query-tiled distances + block radix sort per query
    if ((int64_t)nb * h->n_cells > b.cap_d2) {
      if (b.d2) cudaFree(b.d2);
      b.d2 = nullptr;
      b.cap_d2 = (int64_t)nb * h->n_cells;
      DPQ_TRY(dmalloc(&b.d2, (size_t)b.cap_d2));
    }
    const dim3 grid((unsigned)((h->n_cells + kProbeCT - 1) / kProbeCT), (unsigned)((nb + kProbeQT - 1) / kProbeQT));
    k_probe_dist<<<grid, kProbeCT, 0, h->stream>>>(h->ws.y, h->d, nb, h->centers, h->n_cells, b.d2);
    DPQ_LAUNCHED(h);
    const size_t smem = (size_t)1024 * 8 * 16;  // 8192 (key, id) pairs
    DPQ_TRY(set_smem(h, k_probe_select<1024, 8>, smem));
    k_probe_select<1024, 8><<<nb, 1024, smem, h->stream>>>(b.d2, h->n_cells, ma, b.cells);
    DPQ_LAUNCHED(h);
    return DPQ_OK;
  }
  const int need = ma + 256;
  const size_t ys = (size_t)h->d * 4;
  auto go = [&](auto kern, int BUF) -> int {
    const size_t smem = (size_t)BUF * 16 + ys;
    DPQ_TRY(set_smem(h, kern, smem));
    kern<<<nb, 256, smem, h->stream>>>(h->ws.y, h->d, h->centers, h->n_cells, ma, b.cells);
    return DPQ_OK;
  };
  if (need <= 1024) DPQ_TRY(go(k_probe<1024, 256>, 1024));
  else if (need <= 2048) DPQ_TRY(go(k_probe<2048, 256>, 2048));
  else if (need <= 4096) DPQ_TRY(go(k_probe<4096, 256>, 4096));
  else if (need <= 8192) DPQ_TRY(go(k_probe<8192, 256>, 8192));
  else { set_error("ma too large for the device probe (<= 7936)"); return DPQ_ERR_ARG; }
  DPQ_LAUNCHED(h);
  return DPQ_OK;
}

// Build the slot / tile / unit plan on the host from the probe result.
static void ivf_plan(Index* h, IvfPlan& P, int nb, int ma, int r2) {
  const int qt = qt_of(h);
  static const bool ptrace = getenv("DPQ_HOST_TRACE") != nullptr;
  double tm[8];
  int nm = 0;
  auto mark = [&]() { if (ptrace && nm < 8) tm[nm++] = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  mark();
  const int64_t* off = h->h_offsets.data();
  const int K = h->n_cells;
  P.nq = nb;
  P.ma = ma;
  // Non-empty probes grouped by cell, (query, probe) order kept inside a
  // cell: a counting sort over the K cells, parallel over contiguous query
  // ranges with per-thread cell counts (thread t's probes of cell c follow
  // those of threads < t, so the order is the sequential one).
  static const int ncpu = std::max(1, omp_get_num_procs());
  const int T = std::max(1, std::min(std::min(16, ncpu), nb / 256));
  P.cnt_t.assign((size_t)T * K, 0);
  std::vector<int>& first = P.first;
  first.assign(nb, -1);
  P.nr.assign(nb, 0);
  P.sq.assign(nb, 0);
  const int64_t* cells = P.cells.data();
  const bool shard = h->ivf_shard;
  const int64_t* goff = shard ? h->g_offsets.data() : off;  // bound source and sampling follow the global lists
  if (shard) P.nr_global.assign(nb, 0);
#pragma omp parallel num_threads(T)
  {
    const int t = omp_get_thread_num();
    int* ct = P.cnt_t.data() + (size_t)t * K;
    for (int q = nb * t / T; q < nb * (t + 1) / T; ++q)
      for (int p = 0; p < ma; ++p) {
        const int64_t c = cells[(size_t)q * ma + p];
        if (shard) {
          const int64_t glen = goff[c + 1] - goff[c];
          if (glen > 0 && first[q] < 0) first[q] = p;
          P.nr_global[q] += glen;
        }
        const int64_t len = off[c + 1] - off[c];
        if (len <= 0) continue;
        if (!shard && first[q] < 0) first[q] = p;
        ++ct[c];
        P.nr[q] += len;
      }
  }
  mark();
  // tiles per cell, the first tile of each cell, per-thread slot bases
  std::vector<int>& cnt = P.cnt;
  std::vector<int>& tile0 = P.tile0;
  cnt.assign(K, 0);
  tile0.assign(K + 1, 0);
  P.base_t.assign((size_t)T * K, 0);
  for (int c = 0; c < K; ++c) {
    int acc = 0;
    for (int t = 0; t < T; ++t) {
      P.base_t[(size_t)t * K + c] = acc;
      acc += P.cnt_t[(size_t)t * K + c];
    }
    cnt[c] = acc;
    tile0[c + 1] = tile0[c] + (acc + qt - 1) / qt;
  }
  int64_t tot_rows = 0;
  for (int q = 0; q < nb; ++q) tot_rows += P.nr[q];
  P.ntiles = tile0[K];
  P.nts = P.ntiles * qt;
  P.tile_cell.resize(P.ntiles);
  for (int c = 0; c < K; ++c)
    for (int t = tile0[c]; t < tile0[c + 1]; ++t) P.tile_cell[t] = c;
  // guard sampling: one stride for the batch, exact when lists are short
  // (shard: from the global lists, so every shard samples alike)
  if (shard) {
    tot_rows = 0;
    for (int q = 0; q < nb; ++q) tot_rows += P.nr_global[q];
  }
  const int64_t avg = nb > 0 ? tot_rows / std::max(1, nb) : 0;
  P.stride = (avg <= h->exact_limit) ? 1 : std::max<int64_t>(1, avg / std::max<int64_t>(1, h->sample));
  const int64_t stride = P.stride;
  P.slot_query.resize(P.nts + nb);  // (+ room for shard bound-source slots)
  P.slot_probe.resize(P.nts + nb);
  std::vector<int>& ts_first = P.ts_first;  // slot of each query's first non-empty probe
  ts_first.assign(nb, -1);
  int* sqv = P.slot_query.data();
  int* spv = P.slot_probe.data();
  const int nts = P.nts;
#pragma omp parallel num_threads(T)
  {
#pragma omp for schedule(static)
    for (int i = 0; i < nts; ++i) { sqv[i] = -1; spv[i] = 0; }
    const int t = omp_get_thread_num();
    int* bt = P.base_t.data() + (size_t)t * K;
    for (int q = nb * t / T; q < nb * (t + 1) / T; ++q)
      for (int p = 0; p < ma; ++p) {
        const int64_t c = cells[(size_t)q * ma + p];
        const int64_t len = off[c + 1] - off[c];
        if (len <= 0) continue;
        const int ts = tile0[c] * qt + bt[c]++;  // slots of a cell's tiles fill front to back
        sqv[ts] = q;
        spv[ts] = p;
        if (p == first[q]) ts_first[q] = ts;
        if (stride > 1) P.sq[q] += (len + stride - 1) / stride;
      }
  }
  mark();
  int nne = 0;
  for (int c = 0; c < K; ++c) nne += cnt[c];
  P.live.resize(nne);
  int k = 0;
  for (int c = 0; c < K; ++c)  // live slots in slot order
    for (int i = 0; i < cnt[c]; ++i) P.live[k++] = tile0[c] * qt + i;
  mark();
  // qmax prefix: first min(r2, len) rows of each query's first non-empty
  // list, one entry per bound-source slot (list order of P.bsrc).  A shard
  // takes them from the replicated global prefixes; when that list is empty
  // on this shard the bound source is an extra slot after the tile slots.
  P.bound_ts.assign(nb, -1);
  P.bsrc.clear();
  P.pre_off.clear();
  P.pre_len.clear();
  P.phantom.clear();
  P.nph = 0;
  for (int q = 0; q < nb; ++q) {
    if (first[q] < 0) continue;
    const int64_t c = P.cells[(size_t)q * ma + first[q]];
    int ts = ts_first[q];
    if (ts < 0) {  // (shard only)
      ts = P.nts + P.nph++;
      P.slot_query[ts] = q;
      P.slot_probe[ts] = first[q];
      P.phantom.push_back(ts);
    }
    P.bound_ts[q] = ts;
    P.bsrc.push_back(ts);
    if (shard) {
      P.pre_off.push_back(h->g_pre_off[c]);
      P.pre_len.push_back(std::min<int64_t>(r2, goff[c + 1] - goff[c]));
    } else {
      P.pre_off.push_back(off[c]);
      P.pre_len.push_back(std::min<int64_t>(r2, off[c + 1] - off[c]));
    }
  }
  mark();
  P.slot_query.resize(P.nts + P.nph);
  P.slot_probe.resize(P.nts + P.nph);
  P.tile_row0.assign(P.ntiles, 0);
  P.tile_nsamp.assign(P.ntiles, 0);
  P.max_nsamp = 0;
  for (int t = 0; t < P.ntiles; ++t) {
    const int64_t c = P.tile_cell[t];
    const int64_t len = off[c + 1] - off[c];
    P.tile_row0[t] = off[c];
    P.tile_nsamp[t] = (len + P.stride - 1) / P.stride;
    P.max_nsamp = std::max(P.max_nsamp, P.tile_nsamp[t]);
  }
  P.lambda.assign(nb, -1.0);
  if (P.stride > 1)
    for (int q = 0; q < nb; ++q)
      P.lambda[q] = P.nr[q] > 0 ? (double)r2 * (double)P.sq[q] / (double)P.nr[q] : -1.0;
  mark();
  // scan units: each tile's list split into row ranges, ~8 units per SM
  const int sms = num_sms(h);
  const int64_t target = std::max<int64_t>(1, (8LL * sms));
  int64_t tot_tile_rows = 0;
  for (int t = 0; t < P.ntiles; ++t) tot_tile_rows += off[P.tile_cell[t] + 1] - off[P.tile_cell[t]];
  int64_t per = std::max<int64_t>(4096, (tot_tile_rows + target - 1) / target);
  P.unit_tile.clear(); P.unit_r0.clear(); P.unit_r1.clear();
  for (int t = 0; t < P.ntiles; ++t) {
    const int64_t lo = off[P.tile_cell[t]], hi = off[P.tile_cell[t] + 1];
    for (int64_t r0 = lo; r0 < hi; r0 += per) {
      P.unit_tile.push_back(t);
      P.unit_r0.push_back(r0);
      P.unit_r1.push_back(std::min(hi, r0 + per));
    }
  }
  mark();
  if (ptrace) {
    fprintf(stderr, "[dpq ivf plan]");
    for (int i = 1; i < nm; ++i) fprintf(stderr, " %.0f", tm[i] - tm[i - 1]);
    fprintf(stderr, " us\n");
  }
}

template <class T, class A>
static int h2d(T* dst, const std::vector<T, A>& v, cudaStream_t s) {
  if (v.empty()) return DPQ_OK;
  DPQ_CUDA(cudaMemcpyAsync(dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  return DPQ_OK;
}

// ---------------------------------------------------------------------------
// Device-built plan (unsharded IVF): the host plan's counting sort of the
// non-empty probes by cell, as kernels over the probe result already in HBM.
// A stable radix sort of (cell, probe index) pairs keeps (query, probe) order
// inside a cell, so slots, tiles, bound sources and units are exactly the
// host plan's.  One 64-byte D2H of counts (replacing the host's cells copy)
// sizes the buffers; everything else stays on the device.
// ---------------------------------------------------------------------------
enum { SC_TOT_ROWS = 0, SC_TOT_TILE_ROWS, SC_NNE, SC_NTILES, SC_NBSRC, SC_N };

__global__ void k_plan_probe(const int64_t* __restrict__ cells, const int64_t* __restrict__ off, int nb, int ma,
                             int K, int* __restrict__ key, int* __restrict__ val, int* __restrict__ cnt,
                             int* __restrict__ first, int64_t* __restrict__ nr, int* __restrict__ flag,
                             unsigned long long* __restrict__ sc) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nb) return;
  int f = -1;
  int64_t s = 0;
  for (int p = 0; p < ma; ++p) {
    const int i = q * ma + p;
    const int64_t c = cells[i];
    const int64_t len = off[c + 1] - off[c];
    if (len > 0) {
      if (f < 0) f = p;
      s += len;
      key[i] = (int)c;
      atomicAdd(&cnt[c], 1);
    } else {
      key[i] = K;  // sorts last
    }
    val[i] = i;
  }
  first[q] = f;
  nr[q] = s;
  flag[q] = f >= 0;
  atomicAdd(&sc[SC_TOT_ROWS], (unsigned long long)s);
}

// tiles per cell and the rows all tiles of the cell will scan
__global__ void k_plan_tpc(const int* __restrict__ cnt, const int64_t* __restrict__ off, int K, int qt,
                           int* __restrict__ tpc, unsigned long long* __restrict__ sc) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > K) return;
  const int t = c < K ? (cnt[c] + qt - 1) / qt : 0;
  tpc[c] = t;
  if (t) atomicAdd(&sc[SC_TOT_TILE_ROWS], (unsigned long long)t * (unsigned long long)(off[c + 1] - off[c]));
}

__global__ void k_plan_counts(const int* __restrict__ cstart, const int* __restrict__ tile0,
                              const int* __restrict__ pos, int K, int nb, unsigned long long* __restrict__ sc) {
  sc[SC_NNE] = (unsigned long long)cstart[K];
  sc[SC_NTILES] = (unsigned long long)tile0[K];
  sc[SC_NBSRC] = (unsigned long long)pos[nb];
}

// slot of every non-empty probe (sorted position i -> rank inside its cell)
__global__ void k_plan_place(const int* __restrict__ key, const int* __restrict__ val, int n, int K, int ma, int qt,
                             const int* __restrict__ cstart, const int* __restrict__ tile0,
                             const int* __restrict__ first, int* __restrict__ slot_query,
                             int* __restrict__ slot_probe, int* __restrict__ live, int* __restrict__ bound_ts) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = key[i];
  if (c >= K) return;
  const int pi = val[i], q = pi / ma, p = pi % ma;
  const int ts = tile0[c] * qt + (i - cstart[c]);
  slot_query[ts] = q;
  slot_probe[ts] = p;
  live[i] = ts;
  if (p == first[q]) bound_ts[q] = ts;
}

// per cell: padding slots of its last tile, tile rows / samples / unit counts
__global__ void k_plan_cells(const int* __restrict__ cnt, const int* __restrict__ tile0,
                             const int64_t* __restrict__ off, int K, int qt, int64_t stride, int64_t per,
                             int* __restrict__ slot_query, int* __restrict__ slot_probe,
                             int64_t* __restrict__ tile_row0, int64_t* __restrict__ tile_nsamp,
                             int64_t* __restrict__ tile_len, int* __restrict__ tile_units) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= K) return;
  const int t0 = tile0[c], t1 = tile0[c + 1];
  if (t0 == t1) return;
  const int64_t len = off[c + 1] - off[c];
  for (int ts = t0 * qt + cnt[c]; ts < t1 * qt; ++ts) {
    slot_query[ts] = -1;
    slot_probe[ts] = 0;
  }
  for (int t = t0; t < t1; ++t) {
    tile_row0[t] = off[c];
    tile_nsamp[t] = (len + stride - 1) / stride;
    tile_len[t] = len;
    tile_units[t] = (int)((len + per - 1) / per);
  }
}

__global__ void k_plan_units(const int* __restrict__ ustart, const int* __restrict__ tile_units,
                             const int64_t* __restrict__ tile_row0, const int64_t* __restrict__ tile_len,
                             int ntiles, int64_t per, int* __restrict__ unit_tile, int64_t* __restrict__ unit_r0,
                             int64_t* __restrict__ unit_r1, int* __restrict__ n_units) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  const int u0 = ustart[t], nu = tile_units[t];
  const int64_t lo = tile_row0[t], hi = lo + tile_len[t];
  for (int j = 0; j < nu; ++j) {
    unit_tile[u0 + j] = t;
    unit_r0[u0 + j] = lo + (int64_t)j * per;
    unit_r1[u0 + j] = min(hi, lo + (int64_t)(j + 1) * per);
  }
  if (t == ntiles - 1) *n_units = u0 + nu;
}

// bound sources in query order (ivf.py:205-217) and the per-query sampling rate
__global__ void k_plan_queries(const int64_t* __restrict__ cells, const int64_t* __restrict__ off, int nb, int ma,
                               int r2, int64_t stride, const int* __restrict__ first, const int* __restrict__ pos,
                               const int64_t* __restrict__ nr, const int* __restrict__ bound_ts,
                               int* __restrict__ bsrc, int64_t* __restrict__ pre_off, int64_t* __restrict__ pre_len,
                               double* __restrict__ lambda) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nb) return;
  const int f = first[q];
  if (f >= 0) {
    const int k = pos[q];
    const int64_t c = cells[(int64_t)q * ma + f];
    bsrc[k] = bound_ts[q];
    pre_off[k] = off[c];
    pre_len[k] = min((int64_t)r2, off[c + 1] - off[c]);
  }
  double lam = -1.0;
  if (stride > 1 && nr[q] > 0) {
    int64_t sq = 0;
    for (int p = 0; p < ma; ++p) {
      const int64_t c = cells[(int64_t)q * ma + p];
      const int64_t len = off[c + 1] - off[c];
      if (len > 0) sq += (len + stride - 1) / stride;
    }
    lam = (double)r2 * (double)sq / (double)nr[q];
  }
  lambda[q] = lam;
}

__global__ void k_plan_nsamp(const int64_t* __restrict__ tile_len, int ntiles, int64_t stride,
                             int64_t* __restrict__ tile_nsamp) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < ntiles) tile_nsamp[t] = (tile_len[t] + stride - 1) / stride;
}

static int ivf_plan_dev(Index* h, IvfPlan& P, int nb, int ma, int r, int r2) {
  IvfBuffers& B = ivf_bufs(h);
  cudaStream_t st = h->stream;
  const int K = h->n_cells, qt = qt_of(h), n = nb * ma;
  if (B.max_len < 0) {
    B.max_len = 0;
    for (int c = 0; c < K; ++c) B.max_len = std::max(B.max_len, h->h_offsets[c + 1] - h->h_offsets[c]);
  }
  // buffers (probe-, cell- and query-indexed)
  if (n > B.cap_pp || nb + 1 > B.cap_pk) {
    // (dmalloc releases the previous buffer itself: freeing it here as well
    // would free it twice, and the second free could hit a buffer just handed out again)
    B.cap_pp = std::max(n, B.cap_pp);
    B.cap_pk = std::max(nb + 1, B.cap_pk);
    DPQ_TRY(dmalloc(&B.pl_key, (size_t)B.cap_pp));
    DPQ_TRY(dmalloc(&B.pl_val, (size_t)B.cap_pp));
    DPQ_TRY(dmalloc(&B.pl_key2, (size_t)B.cap_pp));
    DPQ_TRY(dmalloc(&B.pl_val2, (size_t)B.cap_pp));
    DPQ_TRY(dmalloc(&B.pl_first, (size_t)B.cap_pk));
    DPQ_TRY(dmalloc(&B.pl_flag, (size_t)B.cap_pk));
    DPQ_TRY(dmalloc(&B.pl_pos, (size_t)B.cap_pk));
    DPQ_TRY(dmalloc(&B.pl_nr, (size_t)B.cap_pk));
  }
  if (!B.pl_cnt) {
    DPQ_TRY(dmalloc(&B.pl_cnt, (size_t)K + 1));
    DPQ_TRY(dmalloc(&B.pl_cstart, (size_t)K + 1));
    DPQ_TRY(dmalloc(&B.pl_tpc, (size_t)K + 1));
    DPQ_TRY(dmalloc(&B.pl_tile0, (size_t)K + 1));
    DPQ_TRY(dmalloc(&B.pl_sc, (size_t)SC_N));
    DPQ_TRY(dmalloc(&B.pl_nunits, (size_t)1));
    DPQ_CUDA(cudaHostAlloc((void**)&B.pl_sc_h, SC_N * sizeof(unsigned long long), cudaHostAllocDefault));
  }
  int end_bit = 1;
  while ((1 << end_bit) <= K) ++end_bit;
  size_t t_sort = 0, t_scan1 = 0, t_scan2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t_sort, B.pl_key, B.pl_key2, B.pl_val, B.pl_val2, n, 0, end_bit, st);
  cub::DeviceScan::ExclusiveSum(nullptr, t_scan1, B.pl_cnt, B.pl_cstart, K + 1, st);
  cub::DeviceScan::ExclusiveSum(nullptr, t_scan2, B.pl_flag, B.pl_pos, nb + 1, st);
  const size_t need_tmp = std::max(t_sort, std::max(t_scan1, t_scan2)) + 256;
  if (need_tmp > B.cap_ptmp) {
    if (B.pl_tmp) cudaFree(B.pl_tmp);
    B.pl_tmp = nullptr;
    DPQ_CUDA(cudaMalloc(&B.pl_tmp, need_tmp));
    B.cap_ptmp = need_tmp;
  }
  // phase 1: counts
  DPQ_CUDA(cudaMemsetAsync(B.pl_cnt, 0, (size_t)(K + 1) * 4, st));
  DPQ_CUDA(cudaMemsetAsync(B.pl_flag + nb, 0, 4, st));
  DPQ_CUDA(cudaMemsetAsync(B.pl_sc, 0, SC_N * 8, st));
  k_plan_probe<<<(nb + 127) / 128, 128, 0, st>>>(B.cells, h->offsets, nb, ma, K, B.pl_key, B.pl_val, B.pl_cnt,
                                                 B.pl_first, B.pl_nr, B.pl_flag, B.pl_sc);
  DPQ_LAUNCHED(h);
  size_t tb = B.cap_ptmp;
  DPQ_CUDA(cub::DeviceRadixSort::SortPairs(B.pl_tmp, tb, B.pl_key, B.pl_key2, B.pl_val, B.pl_val2, n, 0, end_bit,
                                           st));
  k_plan_tpc<<<(K + 256) / 256, 256, 0, st>>>(B.pl_cnt, h->offsets, K, qt, B.pl_tpc, B.pl_sc);
  DPQ_LAUNCHED(h);
  tb = B.cap_ptmp;
  DPQ_CUDA(cub::DeviceScan::ExclusiveSum(B.pl_tmp, tb, B.pl_cnt, B.pl_cstart, K + 1, st));
  tb = B.cap_ptmp;
  DPQ_CUDA(cub::DeviceScan::ExclusiveSum(B.pl_tmp, tb, B.pl_tpc, B.pl_tile0, K + 1, st));
  tb = B.cap_ptmp;
  DPQ_CUDA(cub::DeviceScan::ExclusiveSum(B.pl_tmp, tb, B.pl_flag, B.pl_pos, nb + 1, st));
  k_plan_counts<<<1, 1, 0, st>>>(B.pl_cstart, B.pl_tile0, B.pl_pos, K, nb, B.pl_sc);
  DPQ_LAUNCHED(h);
  DPQ_CUDA(cudaMemcpyAsync(B.pl_sc_h, B.pl_sc, SC_N * 8, cudaMemcpyDeviceToHost, st));
  DPQ_CUDA(cudaStreamSynchronize(st));
  const unsigned long long* sc = B.pl_sc_h;
  P.nq = nb;
  P.ma = ma;
  P.dev = true;
  P.nph = 0;
  P.ntiles = (int)sc[SC_NTILES];
  P.nts = P.ntiles * qt;
  P.nlive = (int)sc[SC_NNE];
  P.nbsrc = (int)sc[SC_NBSRC];
  const int64_t tot_rows = (int64_t)sc[SC_TOT_ROWS];
  const int64_t avg = nb > 0 ? tot_rows / std::max(1, nb) : 0;
  P.stride = (avg <= h->exact_limit) ? 1 : std::max<int64_t>(1, avg / std::max<int64_t>(1, h->sample));
  P.max_nsamp = (B.max_len + P.stride - 1) / P.stride;
  const int64_t target = std::max<int64_t>(1, (8LL * num_sms(h)));
  const int64_t per = std::max<int64_t>(4096, ((int64_t)sc[SC_TOT_TILE_ROWS] + target - 1) / target);
  P.n_units = (int)std::min<int64_t>((int64_t)P.ntiles + target + 1,
                                     (int64_t)P.ntiles + ((int64_t)sc[SC_TOT_TILE_ROWS] + per - 1) / per);
  if (h->ws.cap == 0 && h->cap0 == 0) {  // first emit capacity, as the host plan
    int64_t c = std::max<int64_t>(16384, std::min<int64_t>(tot_rows / std::max(nb, 1) / 256, (int64_t)1 << 20));
    int64_t p2 = 1;
    while (p2 < c) p2 <<= 1;
    h->cap0 = p2;
  }
  if (P.nts == 0) return DPQ_OK;
  // phase 2: placement, tiles, units, bound sources (capacities now exact)
  DPQ_TRY(ensure_ws(h, P.nts, r, h->d, nb));
  DPQ_TRY(ivf_ensure(h, nb, ma, P.nts, P.ntiles, std::max(P.n_units, 1)));
  if (P.ntiles + 1 > B.cap_ptiles) {
    if (B.pl_tile_len) cudaFree(B.pl_tile_len);
    if (B.pl_tile_units) cudaFree(B.pl_tile_units);
    if (B.pl_ustart) cudaFree(B.pl_ustart);
    B.pl_tile_len = nullptr; B.pl_tile_units = nullptr; B.pl_ustart = nullptr;
    B.cap_ptiles = P.ntiles + 1;
    DPQ_TRY(dmalloc(&B.pl_tile_len, (size_t)B.cap_ptiles));
    DPQ_TRY(dmalloc(&B.pl_tile_units, (size_t)B.cap_ptiles));
    DPQ_TRY(dmalloc(&B.pl_ustart, (size_t)B.cap_ptiles));
    size_t t3 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, t3, B.pl_tile_units, B.pl_ustart, B.cap_ptiles, st);
    if (t3 + 256 > B.cap_ptmp) {
      cudaFree(B.pl_tmp);
      B.pl_tmp = nullptr;
      DPQ_CUDA(cudaMalloc(&B.pl_tmp, t3 + 256));
      B.cap_ptmp = t3 + 256;
    }
  }
  Workspace& w = h->ws;
  DPQ_CUDA(cudaMemsetAsync(B.bound_ts, 0xFF, (size_t)nb * 4, st));
  k_plan_place<<<(n + 255) / 256, 256, 0, st>>>(B.pl_key2, B.pl_val2, n, K, ma, qt, B.pl_cstart, B.pl_tile0,
                                                B.pl_first, w.slot_query, w.slot_probe, B.live, B.bound_ts);
  DPQ_LAUNCHED(h);
  k_plan_cells<<<(K + 255) / 256, 256, 0, st>>>(B.pl_cnt, B.pl_tile0, h->offsets, K, qt, P.stride, per, w.slot_query,
                                                w.slot_probe, B.tile_row0, B.tile_nsamp, B.pl_tile_len,
                                                B.pl_tile_units);
  DPQ_LAUNCHED(h);
  DPQ_CUDA(cudaMemsetAsync(B.pl_tile_units + P.ntiles, 0, 4, st));
  tb = B.cap_ptmp;
  DPQ_CUDA(cub::DeviceScan::ExclusiveSum(B.pl_tmp, tb, B.pl_tile_units, B.pl_ustart, P.ntiles + 1, st));
  k_plan_units<<<(P.ntiles + 255) / 256, 256, 0, st>>>(B.pl_ustart, B.pl_tile_units, B.tile_row0, B.pl_tile_len,
                                                       P.ntiles, per, B.unit_tile, B.unit_r0, B.unit_r1,
                                                       B.pl_nunits);
  DPQ_LAUNCHED(h);
  k_plan_queries<<<(nb + 127) / 128, 128, 0, st>>>(B.cells, h->offsets, nb, ma, r2, P.stride, B.pl_first, B.pl_pos,
                                                   B.pl_nr, B.bound_ts, B.bsrc, w.slot_pre_off, w.slot_pre_len,
                                                   B.lambda);
  DPQ_LAUNCHED(h);
  return DPQ_OK;
}

static bool use_dev_plan(const Index* h) { return !h->ivf_shard && h->ivf_dev_plan; }

// Probe (or take the caller's cells) and form the residuals in natural
// (query, probe) order: B.cells, P.cells (host), B.ynat.
static int ivf_probe_residuals(Index* h, int nb, int ma, const float* res_rot, const int64_t* cells_in) {
  Workspace& w = h->ws;
  IvfBuffers& B = ivf_bufs(h);
  IvfPlan& P = B.plan;
  const int d = h->d;
  DPQ_TRY(ivf_ensure(h, nb, ma, 0, 0, 0));
  P.cells.resize((size_t)nb * ma);
  if (cells_in) {
    memcpy(P.cells.data(), cells_in, P.cells.size() * 8);
    DPQ_TRY(h2d(B.cells, P.cells, h->stream));
  } else {
    DPQ_TRY(ivf_probe_dev(h, nb, ma));
    if (!use_dev_plan(h)) {  // the host plan reads the cells
      DPQ_CUDA(cudaMemcpyAsync(P.cells.data(), B.cells, P.cells.size() * 8, cudaMemcpyDeviceToHost, h->stream));
      if (!B.ev_cells) DPQ_CUDA(cudaEventCreateWithFlags(&B.ev_cells, cudaEventDisableTiming));
      DPQ_CUDA(cudaEventRecord(B.ev_cells, h->stream));
    }
  }
  ev_rec(h, 1);
  // the residuals are enqueued behind the cell copy, so they run while the
  // host plans (the caller synchronises on ev_cells before ivf_plan)
  if (res_rot) {
    DPQ_CUDA(cudaMemcpyAsync(B.ynat, res_rot, (size_t)nb * ma * d * 4, cudaMemcpyHostToDevice, h->stream));
  } else {
    const int64_t tot = (int64_t)nb * ma * d;
    k_residuals<<<(unsigned)((tot + 255) / 256), 256, 0, h->stream>>>(w.y, h->centers, B.cells, nb, ma, d, B.ynat);
    DPQ_LAUNCHED(h);
  }
  if (!cells_in && !use_dev_plan(h)) DPQ_CUDA(cudaEventSynchronize(B.ev_cells));
  return DPQ_OK;
}

// ---------------------------------------------------------------------------
// Derived-mode pieces shared by ivf_batch and the list-split shard protocol.
// ---------------------------------------------------------------------------
// After probe + residuals (B.cells, B.ynat): plan, uploads, slot residuals,
// K1 pass A (qmin/qmax of each query's bound-source slot, from the first
// min(r2, len) rows of its first non-empty probed list — the replicated
// global prefixes on a shard) and pass B (every live slot quantized with its
// query's bounds).  *empty: no probed list holds rows here.
static int ivf_derived_setup(Index* h, int nb, int r, int ma, int r2, bool* empty) {
  Workspace& w = h->ws;
  IvfBuffers& B = ivf_bufs(h);
  IvfPlan& P = B.plan;
  const int d = h->d;
  if (use_dev_plan(h)) {
    DPQ_TRY(ivf_plan_dev(h, P, nb, ma, r, r2));
    DPQ_TRY(ensure_ws(h, std::max(P.nts, 1), r, d, nb));
    DPQ_CUDA(cudaMemsetAsync(w.emit_cnt, 0, (size_t)nb * 4, h->stream));
    *empty = P.nts == 0;
    if (*empty) return DPQ_OK;
  } else {
  try {
    ivf_plan(h, P, nb, ma, r2);
  } catch (const std::bad_alloc&) {
    set_error("ivf plan: pinned host allocation failed");
    return DPQ_ERR_NOMEM;
  }
  P.dev = false;
  P.nlive = (int)P.live.size();
  P.nbsrc = (int)P.bsrc.size();
  P.n_units = (int)P.unit_tile.size();
  if (h->ws.cap == 0 && h->cap0 == 0) {
    // first emit capacity per query from the probed rows (a query emits ~r2
    // to a few r2 rows; growth covers outliers): avg probed / 256, pow2
    int64_t probed = 0;
    for (int q = 0; q < nb; ++q)
      for (int p = 0; p < ma; ++p) {
        const int64_t c = P.cells[(size_t)q * ma + p];
        probed += h->h_offsets[c + 1] - h->h_offsets[c];
      }
    int64_t c = std::max<int64_t>(16384, std::min<int64_t>(probed / std::max(nb, 1) / 256, (int64_t)1 << 20));
    int64_t p2 = 1;
    while (p2 < c) p2 <<= 1;
    h->cap0 = p2;
  }
  const int nslot0 = P.nts + P.nph;
  DPQ_TRY(ensure_ws(h, std::max(nslot0, 1), r, d, nb));
  DPQ_TRY(ivf_ensure(h, nb, ma, std::max(nslot0, 1), std::max(P.ntiles, 1), std::max(P.n_units, 1)));
  DPQ_TRY(h2d(w.slot_query, P.slot_query, h->stream));
  DPQ_TRY(h2d(w.slot_probe, P.slot_probe, h->stream));
  DPQ_TRY(h2d(w.slot_pre_off, P.pre_off, h->stream));
  DPQ_TRY(h2d(w.slot_pre_len, P.pre_len, h->stream));
  DPQ_TRY(h2d(B.bound_ts, P.bound_ts, h->stream));
  DPQ_TRY(h2d(B.lambda, P.lambda, h->stream));
  DPQ_TRY(h2d(B.tile_row0, P.tile_row0, h->stream));
  DPQ_TRY(h2d(B.tile_nsamp, P.tile_nsamp, h->stream));
  DPQ_TRY(h2d(B.unit_tile, P.unit_tile, h->stream));
  DPQ_TRY(h2d(B.unit_r0, P.unit_r0, h->stream));
  DPQ_TRY(h2d(B.unit_r1, P.unit_r1, h->stream));
  DPQ_CUDA(cudaMemsetAsync(w.emit_cnt, 0, (size_t)nb * 4, h->stream));
  *empty = P.nts == 0;
  if (*empty) return DPQ_OK;
  DPQ_TRY(h2d(B.live, P.live, h->stream));
  DPQ_TRY(h2d(B.bsrc, P.bsrc, h->stream));
  }
  const int nslot = P.nts + P.nph;
  const int nlive = P.nlive, nbsrc = P.nbsrc;
  // (K1 reads each slot's residual row q * ma + p of ynat directly: no gathered copy)
  const void* prefix = h->ivf_shard ? h->g_prefix : h->codes;
  // K1 pass A: qmin/qmax of the bound-source slots only (their tables are
  // recomputed in pass B; padding slots are never computed)
  DPQ_TRY(run_small_tables(h, nslot, prefix, 0, w.slot_pre_off, w.slot_pre_len, nullptr, false, B.ynat, B.bsrc, nbsrc,
                           false, nullptr, w.slot_query, w.slot_probe, ma));
  k_slot_bounds<<<(P.nts + 255) / 256, 256, 0, h->stream>>>(w.qmin, w.qmax, B.bound_ts, w.slot_query, P.nts,
                                                            w.bounds);
  DPQ_LAUNCHED(h);
  // K1 pass B: quantize every slot with its query's bounds -> LUT tiles
  DPQ_TRY(run_small_tables(h, P.nts, prefix, 0, nullptr, nullptr, w.bounds, false, B.ynat, B.live, nlive, true,
                           w.slot_query, w.slot_query, w.slot_probe, ma));
  ev_rec(h, 2);
  return DPQ_OK;
}

// Per-query score histograms (B.hist_q) of every stride-th row of the live
// slots' lists (stride 1: exact).
static int ivf_sample_hist(Index* h, int nb, int64_t stride) {
  Workspace& w = h->ws;
  IvfBuffers& B = ivf_bufs(h);
  IvfPlan& P = B.plan;
  DPQ_CUDA(cudaMemsetAsync(B.hist_q, 0, (size_t)nb * 256 * 4, h->stream));
  if (P.nts == 0) return DPQ_OK;
  int64_t mx = 0;
  if (P.dev) {  // per-tile sample counts on the device (upper bound of the max for the grid)
    if (stride != P.stride) {
      k_plan_nsamp<<<(P.ntiles + 255) / 256, 256, 0, h->stream>>>(B.pl_tile_len, P.ntiles, stride, B.tile_nsamp);
      DPQ_LAUNCHED(h);
    }
    mx = (B.max_len + stride - 1) / stride;
  } else {
    pinned_vector<int64_t>& ns = P.ns_tmp;
    ns.resize(P.ntiles);
    for (int t = 0; t < P.ntiles; ++t) {
      const int64_t len = h->h_offsets[P.tile_cell[t] + 1] - h->h_offsets[P.tile_cell[t]];
      ns[t] = (len + stride - 1) / stride;
      mx = std::max(mx, ns[t]);
    }
    DPQ_TRY(h2d(B.tile_nsamp, ns, h->stream));
  }
  DPQ_TRY(build_lut(h, P.nts, nullptr, nullptr, w.slot_query));  // histograms need unclamped entries
  // sampled counts of every slot straight into its query's histogram (B.hist_q)
  DPQ_TRY(launch_hist(h, P.ntiles, nullptr, stride, mx, h->plane, B.tile_row0, B.tile_nsamp, w.slot_query,
                      B.hist_q));
  return DPQ_OK;
}

// Guards from B.hist_q (sampled: per-query lambda in B.lambda; exact: r2),
// then the clamped LUT tiles.  only: recompute the flagged queries only.
static int ivf_set_guards(Index* h, int nb, int r2, bool exact, const uint8_t* only) {
  Workspace& w = h->ws;
  IvfBuffers& B = ivf_bufs(h);
  IvfPlan& P = B.plan;
  k_guard<<<(nb + kGuardSlotsPerCta - 1) / kGuardSlotsPerCta, 32 * kGuardSlotsPerCta, 0, h->stream>>>(B.hist_q, nb, r2, 0.0, exact ? 1 : 0, only, B.guard_q, B.gword_q,
                                                    exact ? nullptr : B.lambda);
  DPQ_LAUNCHED(h);
  if (P.nts == 0) return DPQ_OK;
  k_expand_gword<<<(P.nts + 255) / 256, 256, 0, h->stream>>>(B.gword_q, w.slot_query, P.nts, w.gword);
  DPQ_LAUNCHED(h);
  DPQ_TRY(build_lut(h, P.nts, w.gword, nullptr, w.slot_query));
  return DPQ_OK;
}

// First-pass scan of the planned units + K3 (hist_out: export the local
// candidate histogram instead of deciding b*, shard protocol).
static int ivf_scan(Index* h, int nb, int r2, int32_t* hist_out) {
  Workspace& w = h->ws;
  IvfBuffers& B = ivf_bufs(h);
  IvfPlan& P = B.plan;
  DPQ_CUDA(cudaMemsetAsync(w.emit_cnt, 0, (size_t)nb * 4, h->stream));
  if (P.nts > 0) {
    EmitArgs ea;
    ea.plane = h->plane; ea.row_begin = 0; ea.row_end = h->n; ea.rows_per_cta = 0;
    ea.lut = w.lut; ea.gword = w.gword; ea.tile_list = nullptr;
    ea.slot_query = w.slot_query; ea.slot_probe = w.slot_probe;
    ea.emit_cnt = w.emit_cnt; ea.emit = w.emit; ea.cap = w.cap; ea.emit32 = (int)h->emit32;
    ea.unit_tile = B.unit_tile; ea.unit_r0 = B.unit_r0; ea.unit_r1 = B.unit_r1;
    ea.n_units = P.n_units; ea.units_per_tile = 1;
    ea.n_units_dev = P.dev ? B.pl_nunits : nullptr;
    DPQ_TRY(launch_emit(h, ea, P.ntiles, 0));
  }
  k_threshold<256><<<nb, 256, 0, h->stream>>>(w.emit, w.emit_cnt, w.cap, B.guard_q, r2, nullptr, w.bstar, w.ncand,
                                              w.flags, hist_out, h->d_nemit, (int)h->emit32);
  DPQ_LAUNCHED(h);
  return DPQ_OK;
}

// Grow the emit lists to the largest flagged (overflowed) count; 100 = split the batch.
static int ivf_grow_emit(Index* h, int nb) {
  Workspace& w = h->ws;
  DPQ_CUDA(cudaMemcpyAsync(w.h_cnt, w.emit_cnt, (size_t)nb * 4, cudaMemcpyDeviceToHost, h->stream));
  DPQ_CUDA(cudaStreamSynchronize(h->stream));
  uint32_t need = 0;
  for (int q = 0; q < nb; ++q)
    if (w.h_flags[q] == 2) need = std::max(need, w.h_cnt[q]);
  if ((size_t)w.qcap_emit * need * 8 > h->emit_budget && nb > 1) return 100;
  DPQ_TRY(grow_emit(h, need));
  return DPQ_OK;
}

// One IVF batch: raw queries in ws.y (nb x d).  res_rot / cells_in are host
// arrays for the OPQ path (residuals rotated by the caller), else NULL.
static int ivf_batch(Index* h, int nb, int r, int ma, int r2, bool derived, const float* res_rot,
                     const int64_t* cells_in) {
  Workspace& w = h->ws;
  IvfBuffers& B = ivf_bufs(h);
  const int d = h->d;
  const int qt = qt_of(h);
  ev_rec(h, 0);
  IvfPlan& P = B.plan;  // persistent: vectors keep their capacity (no re-faulting per batch)
  DPQ_TRY(ivf_probe_residuals(h, nb, ma, res_rot, cells_in));
  if (!derived) {
    IvfConvArgs a;
    a.cells = B.cells; a.offsets = h->offsets; a.ma = ma;
    a.codes = h->codes; a.code_bytes = h->code_bytes; a.m = h->m; a.k = h->k; a.dsub = h->dsub;
    a.cb = h->cb; a.ynat = B.ynat; a.sorted_ids = h->sorted_ids;
    a.r = r; a.out_d = w.out_d; a.out_i = w.out_i;
    const size_t ysm = (size_t)ma * d * 4;
    auto go = [&](auto kern, int BUF) -> int {
      // residuals staged in shared memory when they fit, else read from global
      a.y_in_smem = (size_t)BUF * 16 + ysm <= kRefineSmemMax ? 1 : 0;
      const size_t smem = (size_t)BUF * 16 + (a.y_in_smem ? ysm : 0);
      DPQ_TRY(set_smem(h, kern, smem));
      kern<<<nb, 256, smem, h->stream>>>(a);
      return DPQ_OK;
    };
    const int need = r + 256;
    if (need <= 1024) DPQ_TRY(go(k_ivf_conventional<1024, 256>, 1024));
    else if (need <= 2048) DPQ_TRY(go(k_ivf_conventional<2048, 256>, 2048));
    else if (need <= 4096) DPQ_TRY(go(k_ivf_conventional<4096, 256>, 4096));
    else if (need <= 8192) DPQ_TRY(go(k_ivf_conventional<8192, 256>, 8192));
    else { set_error("r exceeds the device top-r limit (7936)"); return DPQ_ERR_ARG; }
    DPQ_LAUNCHED(h);
    ev_rec(h, 6);
    if (h->timing) {
      DPQ_CUDA(cudaEventSynchronize(h->ev[6]));
      h->phase_ms[PH_GUARD] = 0.f;  // index phase reported separately below
      h->phase_ms[PH_TABLES] = 0.f;
      h->phase_ms[PH_SCAN] = ev_ms(h, 1, 6);
      h->phase_ms[PH_REFINE] = 0.f;
      h->phase_ms[PH_THRESH] = 0.f;
      h->phase_ms[PH_FALLBACK] = ev_ms(h, 0, 1);  // probe
      h->phase_ms[PH_TOTAL] = ev_ms(h, 0, 6);
    }
    h->counters[1] += nb;
    return DPQ_OK;
  }
  static const bool trace = getenv("DPQ_HOST_TRACE") != nullptr;
  auto now = []() { return std::chrono::duration<double, std::micro>(
                        std::chrono::steady_clock::now().time_since_epoch()).count(); };
  const double t_plan0 = trace ? now() : 0.0;
  bool empty = false;
  DPQ_TRY(ivf_derived_setup(h, nb, r, ma, r2, &empty));
  const double t_plan1 = trace ? now() : 0.0;
  if (empty) {  // every probed list is empty: empty results (ivf.py:230-233)
    DPQ_CUDA(cudaMemsetAsync(w.bstar, 0xFF, (size_t)nb * 4, h->stream));
  } else {
    DPQ_TRY(ivf_sample_hist(h, nb, P.stride));
    DPQ_TRY(ivf_set_guards(h, nb, r2, P.stride == 1, nullptr));
    ev_rec(h, 3);
    for (int attempt = 0; attempt < 8; ++attempt) {
      DPQ_TRY(ivf_scan(h, nb, r2, nullptr));
      DPQ_CUDA(cudaMemcpyAsync(w.h_flags, w.flags, nb, cudaMemcpyDeviceToHost, h->stream));
      DPQ_CUDA(cudaStreamSynchronize(h->stream));
      bool any_exact = false, any_over = false;
      for (int q = 0; q < nb; ++q) {
        any_exact |= w.h_flags[q] == 1;
        any_over |= w.h_flags[q] == 2;
      }
      if (!any_exact && !any_over) break;
      if (attempt == 7) { set_error("ivf first pass did not converge"); return DPQ_ERR_CUDA; }
      h->counters[4]++;
      if (any_over) {
        const int rc = ivf_grow_emit(h, nb);
        if (rc != DPQ_OK) return rc;
      }
      if (any_exact) {
        for (int q = 0; q < nb; ++q) w.h_flags[q] = w.h_flags[q] == 1;
        DPQ_CUDA(cudaMemcpyAsync(w.only, w.h_flags, nb, cudaMemcpyHostToDevice, h->stream));
        DPQ_TRY(ivf_sample_hist(h, nb, 1));
        DPQ_TRY(ivf_set_guards(h, nb, r2, true, w.only));
      }
    }
  }
  ev_rec(h, 4);
  if (trace && P.nts > 0) {  // guard and tile-mode histograms of this batch
    std::vector<uint16_t> gq(nb);
    std::vector<int> tf(P.ntiles);
    cudaMemcpyAsync(gq.data(), B.guard_q, (size_t)nb * 2, cudaMemcpyDeviceToHost, h->stream);
    cudaMemcpyAsync(tf.data(), w.tile_fast, (size_t)P.ntiles * 4, cudaMemcpyDeviceToHost, h->stream);
    cudaStreamSynchronize(h->stream);
    int gc[5] = {0, 0, 0, 0, 0}, tc[8] = {0};
    for (int q = 0; q < nb; ++q) gc[gq[q] <= 30 ? 0 : gq[q] <= 62 ? 1 : gq[q] <= 126 ? 2 : gq[q] <= 254 ? 3 : 4]++;
    for (int t = 0; t < P.ntiles; ++t) tc[std::min(7, std::max(0, tf[t]))]++;
    fprintf(stderr, "[dpq ivf] guards <=30 %d, <=62 %d, <=126 %d, <=254 %d, other %d | tiles generic %d wide5 %d "
            "wide6 %d 7bit %d\n", gc[0], gc[1], gc[2], gc[3], gc[4], tc[0], tc[5], tc[6], tc[7]);
  }
  if (trace)
    fprintf(stderr, "[dpq ivf] plan %.1f us | uploads+first pass (host) %.1f us | live %zu of %d slots, %d tiles\n",
            t_plan1 - t_plan0, now() - t_plan1, (size_t)P.nlive, P.nts, P.ntiles);
  RefineArgs ra = make_refine_args(h, r);
  ra.y = B.ynat;
  ra.ystride = ma * d;
  ra.row_ids = h->sorted_ids;
  ra.id_base = 0;
  DPQ_TRY(launch_refine<MODE_EMIT>(h, ra, nb));
  ev_rec(h, 6);
  h->counters[1] += nb;
  if (h->timing) {
    DPQ_CUDA(cudaEventSynchronize(h->ev[6]));
    h->phase_ms[PH_FALLBACK] = ev_ms(h, 0, 1);  // probe ("index_us")
    h->phase_ms[PH_TABLES] = P.nts ? ev_ms(h, 1, 2) : 0.f;
    h->phase_ms[PH_GUARD] = P.nts ? ev_ms(h, 2, 3) : 0.f;
    h->phase_ms[PH_SCAN] = P.nts ? ev_ms(h, 3, 4) : 0.f;
    h->phase_ms[PH_THRESH] = 0.f;
    h->phase_ms[PH_REFINE] = ev_ms(h, 4, 6);
    h->phase_ms[PH_TOTAL] = ev_ms(h, 0, 6);
  }
  return DPQ_OK;
}

// host-buffer driver for ivf (queries + optional rotated residuals/cells)
static int ivf_driver(Index* h, const float* y, int64_t nq, int r, int ma, int r2, bool derived,
                      const float* res_rot, const int64_t* cells, double* dists, int64_t* ids, double* phase_us) {
  static const int env_batch = getenv("DPQ_IVF_BATCH") ? atoi(getenv("DPQ_IVF_BATCH")) : 0;
  // IVF tiles are per cell: larger batches fill them (tile occupancy ~ nq * ma / cells), so the IVF
  // batch is at least 2^18 / ma probes' worth of queries (4096 at ma = 64), capped at 4096 queries
  int bsz = env_batch > 0 ? env_batch
                          : std::max(1, std::max(std::min(h->batch, (1 << 16) / std::max(ma, 1)),
                                                 std::min(4096, (1 << 18) / std::max(ma, 1))));
  struct HostOutReset {
    Index* h;
    ~HostOutReset() { h->host_out = false; }
  } host_out_reset{h};
  int64_t q0 = 0;
  while (q0 < nq) {
    const int nb = (int)std::min<int64_t>(bsz, nq - q0);
    DPQ_TRY(ensure_ws(h, nb, r, h->d, nb));
    Workspace& w = h->ws;
    DPQ_CUDA(cudaMemcpyAsync(w.y, y + q0 * h->d, (size_t)nb * h->d * 4, cudaMemcpyHostToDevice, h->stream));
    const bool want_t = phase_us != nullptr;
    const bool old_t = h->timing;
    if (want_t) h->timing = true;
    // derived: the refine writes its rows straight into the pinned staging buffers (see host_driver)
    h->host_out = derived && r > 0;
    int rc = ivf_batch(h, nb, r, ma, r2, derived, res_rot ? res_rot + q0 * ma * h->d : nullptr,
                       cells ? cells + q0 * ma : nullptr);
    h->timing = old_t;
    if (rc == 100) { bsz = std::max(1, nb / 2); continue; }
    if (rc != DPQ_OK) return rc;
    if (!h->host_out) {
      DPQ_CUDA(cudaMemcpyAsync(w.h_d, w.out_d, (size_t)nb * r * 8, cudaMemcpyDeviceToHost, h->stream));
      DPQ_CUDA(cudaMemcpyAsync(w.h_i, w.out_i, (size_t)nb * r * 8, cudaMemcpyDeviceToHost, h->stream));
    }
    DPQ_CUDA(sync_copy_out(h->stream, dists + q0 * r, w.h_d, (size_t)nb * r * 8, ids + q0 * r, w.h_i,
                           (size_t)nb * r * 8));
    if (want_t) {
      const double per = 1000.0 / nb;
      for (int i = 0; i < nb; ++i) {
        double* t = phase_us + (q0 + i) * 4;
        t[0] = h->phase_ms[PH_FALLBACK] * per;  // probe
        t[1] = h->phase_ms[PH_TABLES] * per;
        t[2] = (h->phase_ms[PH_GUARD] + h->phase_ms[PH_SCAN]) * per;
        t[3] = h->phase_ms[PH_REFINE] * per;
      }
    }
    q0 += nb;
  }
  return DPQ_OK;
}

}  // namespace dpq

extern "C" {

int dpq_ivf_create(int device, int m, int k, int kbar, int dsub, const float* codebooks,
                   const float* derived_codebooks, int n_cells, const float* centers, const int64_t* offsets,
                   const void* sorted_codes, int code_bytes, const int64_t* sorted_ids, int64_t n,
                   dpq_index_t** out) {
  if (!out || !codebooks || !derived_codebooks || !centers || !offsets || n_cells < 1 || n < 0 ||
      (n > 0 && (!sorted_codes || !sorted_ids))) {
    set_error("null pointer or bad size");
    return DPQ_ERR_ARG;
  }
  if (offsets[0] != 0 || offsets[n_cells] != n) { set_error("offsets must span [0, n]"); return DPQ_ERR_ARG; }
  Index* h = new Index();
  h->kind = KIND_IVF;
  int rc = index_common_init(h, device, m, k, kbar, dsub, codebooks, derived_codebooks, code_bytes);
  if (rc != DPQ_OK) { index_free(h); return rc; }
  h->ivf_state = new IvfBuffers();
  if (const char* e = getenv("DPQ_PROBE_TC")) h->probe_tc = atoi(e);
  if (const char* e = getenv("DPQ_IVF_DEVPLAN")) h->ivf_dev_plan = atoi(e) != 0;
  // per-cell tiles: 64 queries per tile for m <= 4 (DPQ_IVF_QT=128: the flat geometry)
  if (h->mpad == 4) h->qt = getenv("DPQ_IVF_QT") && atoi(getenv("DPQ_IVF_QT")) == 128 ? 128 : 64;
  h->n = n;
  h->n_cells = n_cells;
  h->h_offsets.assign(offsets, offsets + n_cells + 1);
  const size_t cbytes = (size_t)n * m * code_bytes;
  if ((rc = dmalloc((uint8_t**)&h->codes, cbytes + 16)) != DPQ_OK ||
      (rc = dmalloc(&h->centers, (size_t)n_cells * h->d)) != DPQ_OK ||
      (rc = dmalloc(&h->offsets, (size_t)n_cells + 1)) != DPQ_OK ||
      (rc = dmalloc(&h->sorted_ids, (size_t)std::max<int64_t>(n, 1))) != DPQ_OK) {
    index_free(h);
    return rc;
  }
  bool ok = cudaMemcpy(h->centers, centers, (size_t)n_cells * h->d * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
            cudaMemcpy(h->offsets, offsets, (size_t)(n_cells + 1) * 8, cudaMemcpyHostToDevice) == cudaSuccess;
  if (n > 0)
    ok = ok && cudaMemcpy(h->codes, sorted_codes, cbytes, cudaMemcpyDefault) == cudaSuccess &&
         cudaMemcpy(h->sorted_ids, sorted_ids, (size_t)n * 8, cudaMemcpyDefault) == cudaSuccess;
  if (!ok) { set_error("ivf upload failed"); index_free(h); return DPQ_ERR_CUDA; }
  h->prefix = h->codes;
  h->n_prefix = n;
  if ((rc = make_plane(h)) != DPQ_OK) { index_free(h); return rc; }
  if (cudaStreamSynchronize(h->stream) != cudaSuccess) { set_error("index build failed"); index_free(h); return DPQ_ERR_CUDA; }
  *out = reinterpret_cast<dpq_index_t*>(h);
  return DPQ_OK;
}

int dpq_ivf_probe(dpq_index_t* index, const float* y, int64_t nq, int ma, int64_t* cells) {
  Index* h = reinterpret_cast<Index*>(index);
  if (!h || h->kind != KIND_IVF) { set_error("not an ivf index"); return DPQ_ERR_STATE; }
  if (ma < 1 || ma > h->n_cells) {
    set_error("ma must be in [1, " + std::to_string(h->n_cells) + "], got " + std::to_string(ma));
    return DPQ_ERR_ARG;
  }
  cudaSetDevice(h->device);
  for (int64_t q0 = 0; q0 < nq; q0 += h->batch) {
    const int nb = (int)std::min<int64_t>(h->batch, nq - q0);
    DPQ_TRY(ensure_ws(h, nb, 1, h->d, nb));
    DPQ_TRY(ivf_ensure(h, nb, ma, 0, 0, 0));
    DPQ_CUDA(cudaMemcpyAsync(h->ws.y, y + q0 * h->d, (size_t)nb * h->d * 4, cudaMemcpyHostToDevice, h->stream));
    DPQ_TRY(ivf_probe_dev(h, nb, ma));
    DPQ_CUDA(cudaMemcpyAsync(cells + q0 * ma, ivf_bufs(h).cells, (size_t)nb * ma * 8, cudaMemcpyDeviceToHost,
                             h->stream));
    DPQ_CUDA(cudaStreamSynchronize(h->stream));
  }
  return DPQ_OK;
}

int dpq_ivf_search_derived(dpq_index_t* index, const float* y, int64_t nq, int r, int ma, int r2, int capped,
                           const float* res_rot, const int64_t* cells, double* dists, int64_t* ids,
                           double* phase_us) {
  (void)capped;
  Index* h = reinterpret_cast<Index*>(index);
  if (!h || h->kind != KIND_IVF) { set_error("not an ivf index"); return DPQ_ERR_STATE; }
  if (nq < 0 || r < 1 || r2 < 1 || r > r2) { set_error("need 1 <= r <= r2"); return DPQ_ERR_ARG; }
  if (ma < 1 || ma > h->n_cells) { set_error("ma out of range"); return DPQ_ERR_ARG; }
  cudaSetDevice(h->device);
  dbg_pending("ivf_search_derived entry");
  const int rc_ = ivf_driver(h, y, nq, r, ma, r2, true, res_rot, cells, dists, ids, phase_us);
  dbg_pending("ivf_search_derived exit");
  return rc_;
}

int dpq_ivf_search_conventional(dpq_index_t* index, const float* y, int64_t nq, int r, int ma,
                                const float* res_rot, const int64_t* cells, double* dists, int64_t* ids,
                                double* phase_us) {
  Index* h = reinterpret_cast<Index*>(index);
  if (!h || h->kind != KIND_IVF) { set_error("not an ivf index"); return DPQ_ERR_STATE; }
  if (nq < 0 || r < 1) { set_error("need r >= 1"); return DPQ_ERR_ARG; }
  if (ma < 1 || ma > h->n_cells) { set_error("ma out of range"); return DPQ_ERR_ARG; }
  cudaSetDevice(h->device);
  dbg_pending("ivf_search_conventional entry");
  const int rc_ = ivf_driver(h, y, nq, r, ma, 1, false, res_rot, cells, dists, ids, phase_us);
  dbg_pending("ivf_search_conventional exit");
  return rc_;
}

// ------------------------------------------------- ivf list-split shards --
int dpq_ivf_set_shard(dpq_index_t* index, const int64_t* global_offsets, const void* prefix_codes,
                      const int64_t* prefix_offsets, int64_t prefix_rows) {
  Index* h = reinterpret_cast<Index*>(index);
  if (!h || h->kind != KIND_IVF) { set_error("not an ivf index"); return DPQ_ERR_STATE; }
  if (!global_offsets || !prefix_offsets || prefix_rows < 1) { set_error("bad shard arguments"); return DPQ_ERR_ARG; }
  const int K = h->n_cells;
  if (global_offsets[0] != 0 || prefix_offsets[0] != 0) { set_error("offsets must start at 0"); return DPQ_ERR_ARG; }
  for (int c = 0; c < K; ++c) {
    const int64_t glen = global_offsets[c + 1] - global_offsets[c], llen = h->h_offsets[c + 1] - h->h_offsets[c];
    const int64_t plen = prefix_offsets[c + 1] - prefix_offsets[c];
    if (glen < llen || plen != std::min(glen, prefix_rows)) {
      set_error("shard lists inconsistent with the global lists / prefixes at cell " + std::to_string(c));
      return DPQ_ERR_ARG;
    }
  }
  cudaSetDevice(h->device);
  const int64_t rows = prefix_offsets[K];
  const size_t bytes = (size_t)std::max<int64_t>(rows, 1) * h->m * h->code_bytes;
  if (h->g_prefix) { cudaFree(h->g_prefix); h->g_prefix = nullptr; }
  DPQ_TRY(dmalloc((uint8_t**)&h->g_prefix, bytes));
  if (rows > 0 && !prefix_codes) { set_error("null prefix codes"); return DPQ_ERR_ARG; }
  if (rows > 0) DPQ_CUDA(cudaMemcpy(h->g_prefix, prefix_codes, (size_t)rows * h->m * h->code_bytes,
                                    cudaMemcpyHostToDevice));
  h->g_offsets.assign(global_offsets, global_offsets + K + 1);
  h->g_pre_off.assign(prefix_offsets, prefix_offsets + K + 1);
  h->g_pre_rows = prefix_rows;
  h->ivf_shard = true;
  return DPQ_OK;
}

int dpq_ivf_shard_begin(dpq_index_t* index, const float* y, int64_t nq, int ma, int r2, int exact,
                        const float* res_rot, const int64_t* cells, int32_t* sample_hist, int64_t* n_sampled,
                        int64_t* n_rows) {
  Index* h = reinterpret_cast<Index*>(index);
  if (!h || h->kind != KIND_IVF || !h->ivf_shard) { set_error("not an ivf shard (dpq_ivf_set_shard)"); return DPQ_ERR_STATE; }
  if (nq < 1 || nq > (1 << 20) || r2 < 1 || !y || !sample_hist || !n_sampled || !n_rows || (res_rot && !cells)) {
    set_error("bad ivf_shard_begin arguments"); return DPQ_ERR_ARG;
  }
  if (ma < 1 || ma > h->n_cells) { set_error("ma out of range"); return DPQ_ERR_ARG; }
  if (r2 > h->g_pre_rows) {
    set_error("r2 = " + std::to_string(r2) + " exceeds the replicated list prefixes (" + std::to_string(h->g_pre_rows) +
              " rows)");
    return DPQ_ERR_ARG;
  }
  cudaSetDevice(h->device);
  const int nb = (int)nq;
  DPQ_TRY(ensure_ws(h, nb, 1, h->d, nb));
  DPQ_CUDA(cudaMemcpyAsync(h->ws.y, y, (size_t)nb * h->d * 4, cudaMemcpyHostToDevice, h->stream));
  DPQ_TRY(ivf_probe_residuals(h, nb, ma, res_rot, cells));
  bool empty = false;
  DPQ_TRY(ivf_derived_setup(h, nb, 1, ma, r2, &empty));
  IvfBuffers& B = ivf_bufs(h);
  IvfPlan& P = B.plan;
  const int64_t stride = exact ? 1 : P.stride;
  DPQ_TRY(ivf_sample_hist(h, nb, stride));
  DPQ_CUDA(cudaMemcpyAsync(sample_hist, B.hist_q, (size_t)nb * 256 * 4, cudaMemcpyDeviceToHost, h->stream));
  DPQ_CUDA(cudaStreamSynchronize(h->stream));
  for (int q = 0; q < nb; ++q) {
    n_sampled[q] = stride > 1 ? P.sq[q] : P.nr[q];
    n_rows[q] = P.nr_global[q];
  }
  h->shard_nq = nb;
  h->shard_ma = ma;
  h->shard_stride = stride;
  return DPQ_OK;
}

int dpq_ivf_shard_scan(dpq_index_t* index, const int32_t* sample_hist_sum, const int64_t* sampled_sum,
                       const int64_t* rows_sum, int r2, int32_t* cand_hist) {
  Index* h = reinterpret_cast<Index*>(index);
  if (!h || h->kind != KIND_IVF || !h->ivf_shard || h->shard_nq < 1) { set_error("ivf_shard_begin first"); return DPQ_ERR_STATE; }
  if (!sample_hist_sum || !sampled_sum || !rows_sum || !cand_hist) { set_error("null argument"); return DPQ_ERR_ARG; }
  cudaSetDevice(h->device);
  const int nb = h->shard_nq;
  Workspace& w = h->ws;
  IvfBuffers& B = ivf_bufs(h);
  DPQ_CUDA(cudaMemcpyAsync(B.hist_q, sample_hist_sum, (size_t)nb * 256 * 4, cudaMemcpyHostToDevice, h->stream));
  const bool exact = h->shard_stride == 1;
  std::vector<double> lam(nb, -1.0);  // (exact histograms: lambda < 0)
  if (!exact)
    for (int q = 0; q < nb; ++q)
      lam[q] = rows_sum[q] > 0 ? (double)r2 * (double)sampled_sum[q] / (double)rows_sum[q] : -1.0;
  DPQ_CUDA(cudaMemcpyAsync(B.lambda, lam.data(), (size_t)nb * 8, cudaMemcpyHostToDevice, h->stream));
  DPQ_TRY(ivf_set_guards(h, nb, r2, exact, nullptr));
  for (int attempt = 0; attempt < 4; ++attempt) {
    DPQ_TRY(ivf_scan(h, nb, r2, w.hist_i));
    DPQ_CUDA(cudaMemcpyAsync(w.h_flags, w.flags, nb, cudaMemcpyDeviceToHost, h->stream));
    DPQ_CUDA(cudaStreamSynchronize(h->stream));
    bool over = false;
    for (int q = 0; q < nb; ++q) over |= w.h_flags[q] == 2;
    if (!over) {
      DPQ_CUDA(cudaMemcpy(cand_hist, w.hist_i, (size_t)nb * 256 * 4, cudaMemcpyDeviceToHost));
      return DPQ_OK;
    }
    const int rc = ivf_grow_emit(h, nb);
    if (rc == 100) { set_error("ivf shard scan: emit budget exceeded, use a smaller batch"); return DPQ_ERR_NOMEM; }
    if (rc != DPQ_OK) return rc;
  }
  set_error("ivf shard scan: emit buffer did not converge");
  return DPQ_ERR_NOMEM;
}

int dpq_ivf_shard_finish(dpq_index_t* index, const int32_t* cand_hist_sum, int r, int r2, double* dists,
                         int64_t* ids, uint8_t* need_exact) {
  Index* h = reinterpret_cast<Index*>(index);
  if (!h || h->kind != KIND_IVF || !h->ivf_shard || h->shard_nq < 1) { set_error("ivf_shard_begin first"); return DPQ_ERR_STATE; }
  if (r < 1 || r > r2 || !cand_hist_sum || !dists || !ids || !need_exact) { set_error("bad arguments"); return DPQ_ERR_ARG; }
  cudaSetDevice(h->device);
  const int nb = h->shard_nq, ma = h->shard_ma;
  DPQ_TRY(ensure_ws(h, std::max(ivf_bufs(h).plan.nts + ivf_bufs(h).plan.nph, 1), r, h->d, nb));
  Workspace& w = h->ws;
  IvfBuffers& B = ivf_bufs(h);
  DPQ_CUDA(cudaMemcpyAsync(w.hist_i, cand_hist_sum, (size_t)nb * 256 * 4, cudaMemcpyHostToDevice, h->stream));
  k_bstar_from_hist<<<(nb + 127) / 128, 128, 0, h->stream>>>(w.hist_i, B.guard_q, nb, r2, w.bstar, w.ncand, w.flags);
  DPQ_LAUNCHED(h);
  RefineArgs ra = make_refine_args(h, r);
  ra.y = B.ynat;
  ra.ystride = ma * h->d;
  ra.row_ids = h->sorted_ids;  // global ids
  ra.id_base = 0;
  DPQ_TRY(launch_refine<MODE_EMIT>(h, ra, nb));
  DPQ_CUDA(cudaMemcpyAsync(w.h_d, w.out_d, (size_t)nb * r * 8, cudaMemcpyDeviceToHost, h->stream));
  DPQ_CUDA(cudaMemcpyAsync(w.h_i, w.out_i, (size_t)nb * r * 8, cudaMemcpyDeviceToHost, h->stream));
  DPQ_CUDA(cudaMemcpyAsync(need_exact, w.flags, nb, cudaMemcpyDeviceToHost, h->stream));
  DPQ_CUDA(cudaStreamSynchronize(h->stream));
  memcpy(dists, w.h_d, (size_t)nb * r * 8);
  memcpy(ids, w.h_i, (size_t)nb * r * 8);
  for (int q = 0; q < nb; ++q) need_exact[q] = need_exact[q] != 0;
  h->counters[1] += nb;
  return DPQ_OK;
}

int dpq_shard_begin(dpq_index_t* index, const float* yr, int64_t nq, int r2, int64_t n_global, int exact,
                    int32_t* sample_hist, int64_t* n_sampled) {
  Index* h = reinterpret_cast<Index*>(index);
  if (!h || h->kind != KIND_FLAT) { set_error("not a flat index"); return DPQ_ERR_STATE; }
  if (nq < 1 || nq > (1 << 20) || r2 < 1 || !yr || !sample_hist || !n_sampled) {
    set_error("bad shard_begin arguments"); return DPQ_ERR_ARG;
  }
  const int64_t npre = std::min<int64_t>(r2, n_global);
  if (h->n_prefix < npre) {
    set_error("shard prefix holds " + std::to_string(h->n_prefix) + " rows, need min(r2, N) = " +
              std::to_string(npre));
    return DPQ_ERR_ARG;
  }
  cudaSetDevice(h->device);
  const int nb = (int)nq;
  DPQ_TRY(ensure_ws(h, nb, 1, h->d, -1));
  Workspace& w = h->ws;
  const int qt = qt_of(h);
  const int tiles = tiles_of(nb, h);
  DPQ_CUDA(cudaMemcpyAsync(w.y, yr, (size_t)nb * h->d * 4, cudaMemcpyHostToDevice, h->stream));
  DPQ_TRY(run_small_tables(h, nb, h->prefix, npre, nullptr, nullptr, nullptr, false, nullptr));
  DPQ_CUDA(cudaMemsetAsync(w.gword, 0x7F, (size_t)tiles * qt * 2, h->stream));
  DPQ_CUDA(cudaMemsetAsync(w.hist, 0, (size_t)tiles * qt * 256 * 4, h->stream));
  const bool ex = exact || n_global <= h->exact_limit;
  const int64_t ns = h->n == 0 ? 0 : (ex ? h->n : std::min<int64_t>(h->n, h->sample));
  const int64_t stride = ns ? h->n / ns : 1;
  if (ns > 0) DPQ_TRY(launch_hist(h, tiles, nullptr, stride, ns, h->plane));
  DPQ_CUDA(cudaMemcpyAsync(sample_hist, w.hist, (size_t)nb * 256 * 4, cudaMemcpyDeviceToHost, h->stream));
  DPQ_CUDA(cudaStreamSynchronize(h->stream));
  *n_sampled = ns;
  h->shard_nq = nb;
  return DPQ_OK;
}

int dpq_shard_scan(dpq_index_t* index, const int32_t* sample_hist_sum, int64_t n_global, int64_t sample_global,
                   int r2, int exact, int32_t* cand_hist) {
  Index* h = reinterpret_cast<Index*>(index);
  if (!h || h->kind != KIND_FLAT || h->shard_nq < 1) { set_error("shard_begin first"); return DPQ_ERR_STATE; }
  cudaSetDevice(h->device);
  const int nb = h->shard_nq;
  Workspace& w = h->ws;
  const int tiles = tiles_of(nb, h);
  DPQ_CUDA(cudaMemcpyAsync(w.hist, sample_hist_sum, (size_t)nb * 256 * 4, cudaMemcpyHostToDevice, h->stream));
  const bool ex = exact || n_global <= h->exact_limit;
  const double lambda = (double)r2 * (double)sample_global / (double)std::max<int64_t>(n_global, 1);
  k_guard<<<(nb + kGuardSlotsPerCta - 1) / kGuardSlotsPerCta, 32 * kGuardSlotsPerCta, 0, h->stream>>>(w.hist, nb, r2, lambda, ex ? 1 : 0, nullptr, w.guard_b, w.gword,
                                                    nullptr);
  DPQ_LAUNCHED(h);
  // same scan preparation as the single-GPU first pass (slot clustering,
  // clamped tiles, run-filtered chunk lists over this shard's sorted rows)
  ScanPlan sp;
  DPQ_TRY(plan_flat_scan(h, nb, sp));
  DPQ_TRY(prepare_flat_scan(h, nb, sp));
  sp.scan_hist = sp.direct && scan_hist_on(h);  // (ws.hist is free once k_guard has read it)
  for (int attempt = 0; attempt < 4; ++attempt) {
    DPQ_CUDA(cudaMemsetAsync(w.emit_cnt, 0, (size_t)nb * 4, h->stream));
    if (sp.scan_hist) DPQ_CUDA(cudaMemsetAsync(w.hist, 0, (size_t)nb * 256 * 4, h->stream));
    if (h->n > 0) {
      EmitArgs ea;
      ea.plane = h->plane; ea.row_begin = 0; ea.row_end = h->n; ea.rows_per_cta = 0;
      ea.lut = w.lut; ea.tile_list = nullptr; ea.slot_probe = nullptr;
      plan_emit_args(h, sp, ea);
      ea.unit_tile = nullptr; ea.unit_r0 = nullptr; ea.unit_r1 = nullptr;
      ea.emit_cnt = w.emit_cnt; ea.emit = w.emit; ea.cap = w.cap; ea.emit32 = (int)h->emit32;
      DPQ_TRY(launch_emit(h, ea, tiles, h->n));
      DPQ_TRY(launch_direct(h, sp));
      if (!sp.list) h->counters[2] += (int64_t)nb * h->n;
    }
    k_threshold<256><<<nb, 256, 0, h->stream>>>(w.emit, w.emit_cnt, w.cap, w.guard_b, r2, nullptr, w.bstar,
                                                w.ncand, w.flags, w.hist_i, h->d_nemit, (int)h->emit32,
                                                sp.scan_hist ? w.hist : nullptr, w.gword);
    DPQ_LAUNCHED(h);
    DPQ_CUDA(cudaMemcpyAsync(w.h_flags, w.flags, nb, cudaMemcpyDeviceToHost, h->stream));
    DPQ_CUDA(cudaMemcpyAsync(w.h_cnt, w.emit_cnt, (size_t)nb * 4, cudaMemcpyDeviceToHost, h->stream));
    DPQ_CUDA(cudaStreamSynchronize(h->stream));
    uint32_t need = 0;
    for (int q = 0; q < nb; ++q)
      if (w.h_flags[q] == 2) need = std::max(need, w.h_cnt[q]);
    if (!need) {
      DPQ_CUDA(cudaMemcpy(cand_hist, w.hist_i, (size_t)nb * 256 * 4, cudaMemcpyDeviceToHost));
      return DPQ_OK;
    }
    DPQ_TRY(grow_emit(h, need));
  }
  set_error("shard scan: emit buffer did not converge");
  return DPQ_ERR_NOMEM;
}

int dpq_shard_finish(dpq_index_t* index, const int32_t* cand_hist_sum, int r, int r2, double* dists, int64_t* ids,
                     uint8_t* need_exact) {
  Index* h = reinterpret_cast<Index*>(index);
  if (!h || h->kind != KIND_FLAT || h->shard_nq < 1) { set_error("shard_begin first"); return DPQ_ERR_STATE; }
  if (r < 1 || r > r2) { set_error("need 1 <= r <= r2"); return DPQ_ERR_ARG; }
  cudaSetDevice(h->device);
  const int nb = h->shard_nq;
  DPQ_TRY(ensure_ws(h, nb, r, h->d, -1));
  Workspace& w = h->ws;
  DPQ_CUDA(cudaMemcpyAsync(w.hist_i, cand_hist_sum, (size_t)nb * 256 * 4, cudaMemcpyHostToDevice, h->stream));
  k_bstar_from_hist<<<(nb + 127) / 128, 128, 0, h->stream>>>(w.hist_i, w.guard_b, nb, r2, w.bstar, w.ncand,
                                                              w.flags);
  DPQ_LAUNCHED(h);
  RefineArgs ra = make_refine_args(h, r);
  if (group_tables_fit(h, nb)) {
    DPQ_TRY(run_group_tables(h, nb, h->d));
    ra.tables = w.tables;
    DPQ_TRY(h->emit32 ? launch_refine<MODE_EMIT_TABLE32>(h, ra, nb) : launch_refine<MODE_EMIT_TABLE>(h, ra, nb));
  } else {
    DPQ_TRY(launch_refine<MODE_EMIT>(h, ra, nb));
  }
  DPQ_CUDA(cudaMemcpyAsync(w.h_d, w.out_d, (size_t)nb * r * 8, cudaMemcpyDeviceToHost, h->stream));
  DPQ_CUDA(cudaMemcpyAsync(w.h_i, w.out_i, (size_t)nb * r * 8, cudaMemcpyDeviceToHost, h->stream));
  DPQ_CUDA(cudaMemcpyAsync(need_exact, w.flags, nb, cudaMemcpyDeviceToHost, h->stream));
  DPQ_CUDA(cudaStreamSynchronize(h->stream));
  memcpy(dists, w.h_d, (size_t)nb * r * 8);
  memcpy(ids, w.h_i, (size_t)nb * r * 8);
  for (int q = 0; q < nb; ++q) need_exact[q] = need_exact[q] == 1;
  h->counters[1] += nb;
  return DPQ_OK;
}


// ---------------------------------------------------------------------------
// Device-resident shard protocol: the same three phases on device buffers,
// enqueued on the index stream with no host synchronisation, so the caller
// runs the histogram all-reduces (NCCL) in place on the same stream.  Guard
// too tight / emit overflow are flagged per query (flags: 1 / 2) instead of
// being handled synchronously; the caller all-reduces the flags (max) and
// redoes a flagged batch through the host-staged protocol above.
// ---------------------------------------------------------------------------
int dpq_shard_begin_dev(dpq_index_t* index, const float* yr, int64_t nq, int r2, int64_t n_global, int exact,
                        int32_t* sample_hist, int64_t* n_sampled) {
  Index* h = reinterpret_cast<Index*>(index);
  if (!h || h->kind != KIND_FLAT) { set_error("not a flat index"); return DPQ_ERR_STATE; }
  if (nq < 1 || nq > (1 << 20) || r2 < 1 || !yr || !sample_hist || !n_sampled) {
    set_error("bad shard_begin_dev arguments"); return DPQ_ERR_ARG;
  }
  const int64_t npre = std::min<int64_t>(r2, n_global);
  if (h->n_prefix < npre) {
    set_error("shard prefix holds " + std::to_string(h->n_prefix) + " rows, need min(r2, N) = " +
              std::to_string(npre));
    return DPQ_ERR_ARG;
  }
  cudaSetDevice(h->device);
  const int nb = (int)nq;
  DPQ_TRY(ensure_ws(h, nb, 1, h->d, -1));
  Workspace& w = h->ws;
  const int qt = qt_of(h);
  const int tiles = tiles_of(nb, h);
  DPQ_CUDA(cudaMemcpyAsync(w.y, yr, (size_t)nb * h->d * 4, cudaMemcpyDeviceToDevice, h->stream));
  DPQ_TRY(run_small_tables(h, nb, h->prefix, npre, nullptr, nullptr, nullptr, false, nullptr));
  DPQ_CUDA(cudaMemsetAsync(w.gword, 0x7F, (size_t)tiles * qt * 2, h->stream));
  DPQ_CUDA(cudaMemsetAsync(w.hist, 0, (size_t)tiles * qt * 256 * 4, h->stream));
  const bool ex = exact || n_global <= h->exact_limit;
  const int64_t ns = h->n == 0 ? 0 : (ex ? h->n : std::min<int64_t>(h->n, h->sample));
  const int64_t stride = ns ? h->n / ns : 1;
  if (ns > 0) DPQ_TRY(launch_hist(h, tiles, nullptr, stride, ns, h->plane));
  DPQ_CUDA(cudaMemcpyAsync(sample_hist, w.hist, (size_t)nb * 256 * 4, cudaMemcpyDeviceToDevice, h->stream));
  *n_sampled = ns;
  h->shard_nq = nb;
  return DPQ_OK;
}

int dpq_shard_scan_dev(dpq_index_t* index, const int32_t* sample_hist_sum, int64_t n_global, int64_t sample_global,
                       int r2, int exact, int32_t* cand_hist) {
  Index* h = reinterpret_cast<Index*>(index);
  if (!h || h->kind != KIND_FLAT || h->shard_nq < 1) { set_error("shard_begin first"); return DPQ_ERR_STATE; }
  if (!sample_hist_sum || !cand_hist) { set_error("null histogram"); return DPQ_ERR_ARG; }
  cudaSetDevice(h->device);
  const int nb = h->shard_nq;
  Workspace& w = h->ws;
  const int tiles = tiles_of(nb, h);
  DPQ_CUDA(cudaMemcpyAsync(w.hist, sample_hist_sum, (size_t)nb * 256 * 4, cudaMemcpyDeviceToDevice, h->stream));
  const bool ex = exact || n_global <= h->exact_limit;
  const double lambda = (double)r2 * (double)sample_global / (double)std::max<int64_t>(n_global, 1);
  k_guard<<<(nb + kGuardSlotsPerCta - 1) / kGuardSlotsPerCta, 32 * kGuardSlotsPerCta, 0, h->stream>>>(w.hist, nb, r2, lambda, ex ? 1 : 0, nullptr, w.guard_b, w.gword,
                                                    nullptr);
  DPQ_LAUNCHED(h);
  ScanPlan sp;
  DPQ_TRY(plan_flat_scan(h, nb, sp));
  DPQ_TRY(prepare_flat_scan(h, nb, sp));
  sp.scan_hist = sp.direct && scan_hist_on(h);  // (ws.hist is free once k_guard has read it)
  DPQ_CUDA(cudaMemsetAsync(w.emit_cnt, 0, (size_t)nb * 4, h->stream));
  if (sp.scan_hist) DPQ_CUDA(cudaMemsetAsync(w.hist, 0, (size_t)nb * 256 * 4, h->stream));
  if (h->n > 0) {
    EmitArgs ea;
    ea.plane = h->plane; ea.row_begin = 0; ea.row_end = h->n; ea.rows_per_cta = 0;
    ea.lut = w.lut; ea.tile_list = nullptr; ea.slot_probe = nullptr;
    plan_emit_args(h, sp, ea);
    ea.unit_tile = nullptr; ea.unit_r0 = nullptr; ea.unit_r1 = nullptr;
    ea.emit_cnt = w.emit_cnt; ea.emit = w.emit; ea.cap = w.cap; ea.emit32 = (int)h->emit32;
    DPQ_TRY(launch_emit(h, ea, tiles, h->n));
    DPQ_TRY(launch_direct(h, sp));
    if (!sp.list) h->counters[2] += (int64_t)nb * h->n;
  }
  k_threshold<256><<<nb, 256, 0, h->stream>>>(w.emit, w.emit_cnt, w.cap, w.guard_b, r2, nullptr, w.bstar, w.ncand,
                                              w.flags, cand_hist, h->d_nemit, (int)h->emit32,
                                              sp.scan_hist ? w.hist : nullptr, w.gword);
  DPQ_LAUNCHED(h);
  return DPQ_OK;
}

int dpq_shard_finish_dev(dpq_index_t* index, const int32_t* cand_hist_sum, int r, int r2, double* dists,
                         int64_t* ids, uint8_t* flags) {
  Index* h = reinterpret_cast<Index*>(index);
  if (!h || h->kind != KIND_FLAT || h->shard_nq < 1) { set_error("shard_begin first"); return DPQ_ERR_STATE; }
  if (r < 1 || r > r2) { set_error("need 1 <= r <= r2"); return DPQ_ERR_ARG; }
  if (!cand_hist_sum || !dists || !ids || !flags) { set_error("null argument"); return DPQ_ERR_ARG; }
  cudaSetDevice(h->device);
  const int nb = h->shard_nq;
  DPQ_TRY(ensure_ws(h, nb, r, h->d, -1));
  Workspace& w = h->ws;
  k_bstar_from_hist<<<(nb + 127) / 128, 128, 0, h->stream>>>(cand_hist_sum, w.guard_b, nb, r2, w.bstar, w.ncand,
                                                              w.flags);
  DPQ_LAUNCHED(h);
  RefineArgs ra = make_refine_args(h, r);
  ra.out_d = dists;
  ra.out_i = ids;
  if (group_tables_fit(h, nb)) {
    DPQ_TRY(run_group_tables(h, nb, h->d));
    ra.tables = w.tables;
    DPQ_TRY(h->emit32 ? launch_refine<MODE_EMIT_TABLE32>(h, ra, nb) : launch_refine<MODE_EMIT_TABLE>(h, ra, nb));
  } else {
    DPQ_TRY(launch_refine<MODE_EMIT>(h, ra, nb));
  }
  DPQ_CUDA(cudaMemcpyAsync(flags, w.flags, nb, cudaMemcpyDeviceToDevice, h->stream));
  h->counters[1] += nb;
  return DPQ_OK;
}

int dpq_merge_topr_dev(dpq_index_t* index, const double* part_dists, const int64_t* part_ids, int n_parts,
                       int64_t nq, int r, double* dists, int64_t* ids) {
  Index* h = reinterpret_cast<Index*>(index);
  if (!h) { set_error("null index"); return DPQ_ERR_ARG; }
  if (n_parts < 1 || nq < 0 || nq > INT32_MAX || r < 1 || (nq > 0 && (!part_dists || !part_ids || !dists || !ids))) {
    set_error("bad merge arguments"); return DPQ_ERR_ARG;
  }
  if (nq == 0) return DPQ_OK;
  cudaSetDevice(h->device);
  k_merge_topr<<<(unsigned)nq, 256, 0, h->stream>>>(part_dists, part_ids, n_parts, (int)nq, r, dists, ids);
  DPQ_LAUNCHED(h);
  return DPQ_OK;
}

int dpq_sync(dpq_index_t* index) {
  Index* h = reinterpret_cast<Index*>(index);
  if (!h) { set_error("null index"); return DPQ_ERR_ARG; }
  cudaSetDevice(h->device);
  DPQ_CUDA(cudaStreamSynchronize(h->stream));
  return DPQ_OK;
}

}  // extern "C"
