// dpq_kernels.cuh — sm_100a kernels of the derived two-pass search.
//
//   K1 k_small_tables   compute_tables(yr, derived) + quantize_tables
//                       (search.py:28-48, twopass.py:41-85)
//   K2 k_scan_hist      score histogram over a row sample (or all rows):
//                       picks a provisional per-query bound ("guard") so the
//                       main scan can drop everything that cannot be a
//                       candidate without a per-code histogram update
//      k_scan_emit      adc_low_batch (twopass.py:99-106) over every code,
//                       query-tiled, emitting (row, score) for score <= guard
//   K3 k_threshold      CappedBuckets bound + refine bucket walk
//                       (twopass.py:171-201, 276-308) in closed form:
//                       b* = min{b : #(s <= b) >= r2}, else 254
//   K5 k_group_tables   LazyTables (twopass.py:220-251) at derived-group
//                       granularity; k_full_tables for the conventional path
//   K6 k_refine_topk    _refine_batch + adc_batch + top-r
//                       (twopass.py:269-273, search.py:64-88): exact f64
//                       distance of every candidate, exact (dist,id) top-r
//
// Data layout in HBM (per index):
//   plane  (n_pad, MPAD) u8   low bbar bits of every sub-code, subspaces
//                             padded to MPAD in {4, 8} with zero bytes; the
//                             first pass reads only this (4 or 8 B/code).
//   codes  (n, m) u8/u16      original codes, gathered per candidate.
//   lut    per query tile of QT = 128 (MPAD 4) / 64 (MPAD 8) queries: u8
//          entries, 4 queries per 32-bit word, see lut_index.
#pragma once
#include <type_traits>

#include "dpq_device.cuh"

namespace dpq {

// ---- emit record: row | probe << 40 | score << 56 -------------------------
constexpr int kRowBits = 40;
constexpr uint64_t kRowMask = (uint64_t(1) << kRowBits) - 1;
__device__ __forceinline__ uint64_t pack_emit(int64_t row, uint32_t probe,
                                              uint32_t score) {
  return (uint64_t)row | ((uint64_t)(probe & 0xFFFF) << kRowBits) |
         ((uint64_t)score << 56);
}
__device__ __forceinline__ int64_t emit_row(uint64_t v) { return (int64_t)(v & kRowMask); }
__device__ __forceinline__ uint32_t emit_probe(uint64_t v) { return (uint32_t)((v >> kRowBits) & 0xFFFF); }
__device__ __forceinline__ uint32_t emit_score(uint64_t v) { return (uint32_t)(v >> 56); }
// Compact 4-byte record (flat shards of < 2^24 rows, probe 0): row | score << 24.
constexpr int kRow32Bits = 24;
__device__ __forceinline__ uint32_t pack_emit32(int64_t row, uint32_t score) {
  return (uint32_t)row | (score << kRow32Bits);
}
__device__ __forceinline__ uint64_t widen_emit32(uint32_t v) {
  return pack_emit(v & ((1u << kRow32Bits) - 1u), 0u, v >> kRow32Bits);
}

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t lds32(const uint8_t* p) {
  return *reinterpret_cast<const uint32_t*>(p);
}

// ---- TMA bulk copies (cp.async.bulk, completion on an mbarrier) -----------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Bounded wait: a copy that never completes traps (a CUDA error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  for (uint32_t spin = 0;; ++spin) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    if (spin > (1u << 26)) __trap();
  }
}

// Tile geometry: MPAD subspaces (4 or 8) x QT queries.  Flat m <= 4 uses
// QT = 128; IVF m <= 4 uses QT = 64 (per-cell tiles are ~25-45% occupied at
// QT = 128, so halving the tile halves the padding work); m = 8 uses 64.
constexpr int default_qt(int mpad) { return mpad == 4 ? 128 : 64; }
template <int MPAD, int QTX = default_qt(MPAD)>
struct ScanGeom {
  static constexpr int QT = QTX;                   // queries per tile
  static constexpr int LPC = QT / 4;               // lanes per code (4 queries/lane)
  static constexpr int CPW = 32 / LPC;             // codes per warp step
  static constexpr int ROWB = QT;                  // bytes of one subspace row (u8)
  static constexpr int SPR = 256 / ROWB;           // subspaces per 256-B row
  static constexpr int CPL = (16 / MPAD) / CPW;    // codes per lane in one 16-B plane word group
  static constexpr int LUT_BYTES = MPAD * 256 * ROWB;  // 128 KB
  static constexpr int CHUNK_ROWS = 512 / MPAD;    // rows per 512-B warp load
};

// LUT layout of one query tile (bytes, one u8 entry per query):
//   [MPAD/SPR tables of 64 KB][256 rows of 256 B][SPR subspaces][QT queries]
// Subspace j, table row i, query qq ->
//   ((j / SPR) * 256 + i) * (SPR * QT) + (j % SPR) * QT + qq
// Lane lic owns queries 4*lic .. 4*lic+3 (one 32-bit word per table row).
// With the tile at a 64-KB aligned shared address, the byte address of that
// word for row i of subspace j is
//   base | i << 8 | (j % SPR) * ROWB | lic * 4   (+ (j / SPR) * 64 KB)
// i.e. ONE byte-permute of the code word into the lane's base word.
// The four u8 entries of a word are split into two u16x2 accumulators
// (bytes 0,2 and 1,3); sums of MPAD entries never carry across halves.
__host__ __device__ __forceinline__ int64_t lut_index(int j, int i, int qq, int spr, int qt) {
  return ((int64_t)(j / spr) * 256 + i) * (spr * qt) + (int64_t)(j % spr) * qt + qq;
}

// ============================================================================
// K1: small tables, qmin/qmax, 8-bit quantization, scan-layout LUT.
// ============================================================================
struct TablesArgs {
  const float* y;          // [nslot][d] queries (flat) or residuals (ivf)
  const int* y_sq = nullptr;  // optional: slot s reads row y_sq[s] * y_ma + y_sp[s] of y (ivf: the
  const int* y_sp = nullptr;  //   natural (query, probe) residual rows, no gathered copy)
  int y_ma = 0;
  const float* dcb;        // [m][kbar][dsub] derived codebooks
  int m, kbar, dsub, mask;
  const void* prefix;      // first rows of the scanned list (qmax)
  int code_bytes;
  int64_t npre;            // min(r2, rows) rows used for qmax
  const int64_t* prefix_off;  // optional per-slot prefix row offset (ivf)
  const int64_t* prefix_len;  // optional per-slot prefix length (ivf)
  const double* bounds_in; // optional [nslot][2] externally chosen bounds
  int nslot;
  float* small_out;        // optional [nslot][m][kbar]
  uint8_t* q8_out;         // optional [nslot][m][kbar]
  double* qmin_out;        // [nslot]
  double* qmax_out;        // [nslot]
  uint8_t* lut;            // [tiles][mpad][256][qt] (see lut_index)
  int mpad, qt;
  uint16_t* cluster = nullptr;  // optional [nslot]: g0* << 8 | g1* (first argmin of the u8 tables)
  unsigned long long negzero2 = kNegZero2;  // runtime (-0, -0) pair for sqdiff2
  const int* slot_list = nullptr;  // optional: CTA b computes slot slot_list[b] (ivf: live slots only);
                                   // prefix_off/prefix_len are then indexed by b
};

__global__ void __launch_bounds__(256) k_small_tables(TablesArgs a) {
  // (the scan-layout LUT is built from q8_out by k_build_lut)
  extern __shared__ __align__(16) float sm_f[];
  __shared__ float red_f[8];
  __shared__ double red_d[8];
  const int s = a.slot_list ? a.slot_list[blockIdx.x] : (int)blockIdx.x, tid = threadIdx.x;
  const int d = a.m * a.dsub, ne = a.m * a.kbar;
  float* ys = sm_f;
  float* st = sm_f + d;
  uint8_t* q8 = reinterpret_cast<uint8_t*>(st + ne);
  const int64_t yrow = a.y_sq ? (int64_t)a.y_sq[s] * a.y_ma + a.y_sp[s] : (int64_t)s;
  for (int i = tid; i < d; i += 256) ys[i] = a.y[yrow * d + i];
  __syncthreads();
  // compute_tables: row_sq_dists per derived centroid (search.py:24-25,46-47)
  float mn = INFINITY;
  const bool v8 = (a.dsub & 7) == 0 && a.dsub <= 128;
  for (int e = tid; e < ne; e += 256) {
    const int j = e / a.kbar;
    float v = v8 ? pw_sqdist_v8(a.dcb + (int64_t)e * a.dsub, ys + j * a.dsub, a.dsub)
                 : pw_sqdist(a.dcb + (int64_t)e * a.dsub, ys + j * a.dsub, a.dsub);
    st[e] = v;
    mn = fminf(mn, v);
  }
  mn = warp_min_f(mn);
  if ((tid & 31) == 0) red_f[tid >> 5] = mn;
  __syncthreads();
  // qmax: max over prefix codes of the f64 masked table sum, j ascending
  // (twopass.py:41-47, 83-84)
  const int pi = a.slot_list ? (int)blockIdx.x : s;  // prefix arrays follow slot_list when given
  int64_t pre_off = a.prefix_off ? a.prefix_off[pi] : 0;
  int64_t npre = a.prefix_len ? a.prefix_len[pi] : a.npre;
  double mx = -INFINITY;
  for (int64_t p = tid; p < npre; p += 256) {
    double acc = 0.0;
    for (int j = 0; j < a.m; ++j) {
      uint32_t c = code_at(a.prefix, a.code_bytes, (pre_off + p) * a.m + j);
      acc = __dadd_rn(acc, (double)st[j * a.kbar + (c & a.mask)]);
    }
    mx = fmax(mx, acc);
  }
  mx = warp_max_d(mx);
  if ((tid & 31) == 0) red_d[tid >> 5] = mx;
  __syncthreads();
  double qmin = (double)red_f[0], qmax = red_d[0];
  for (int w = 1; w < 8; ++w) {
    qmin = fmin(qmin, (double)red_f[w]);
    qmax = fmax(qmax, red_d[w]);
  }
  if (a.bounds_in) {
    qmin = a.bounds_in[2 * s];
    qmax = a.bounds_in[2 * s + 1];
  }
  // quantize_with_bounds (twopass.py:50-60)
  const bool degenerate = !(qmax > qmin);
  const double scale = degenerate ? 0.0 : __ddiv_rn(255.0, __dsub_rn(qmax, qmin));
  const float qmaxf = __double2float_rn(qmax);
  for (int e = tid; e < ne; e += 256) {
    uint8_t q = degenerate ? (uint8_t)0 : quantize_entry(st[e], qmin, scale, qmaxf);
    q8[e] = q;
    if (a.small_out) a.small_out[(int64_t)s * ne + e] = st[e];
    if (a.q8_out) a.q8_out[(int64_t)s * ne + e] = q;
  }
  if (tid == 0) {
    a.qmin_out[s] = qmin;
    a.qmax_out[s] = degenerate ? qmin : qmax;
  }
  if (a.cluster && a.m >= 2) {  // nearest derived group in subspaces 0 and 1 (slot clustering key)
    __syncthreads();
    const int w = tid >> 5, lane = tid & 31;
    __shared__ uint32_t best[2];
    if (w < 2) {
      uint32_t b = 0xFFFFFFFFu;
      for (int g = lane; g < a.kbar; g += 32) b = min(b, ((uint32_t)q8[w * a.kbar + g] << 16) | (uint32_t)g);
      b = __reduce_min_sync(0xffffffffu, b);
      if (lane == 0) best[w] = b & 0xFFu;
    }
    __syncthreads();
    if (tid == 0) a.cluster[s] = (uint16_t)((best[0] << 8) | best[1]);
  }
  __syncthreads();
}

// K1, many-slot form (IVF batches: ~10^5 slots): SPC slots per CTA so each
// derived-codebook row is fetched once per SPC slots instead of once per slot
// (the per-slot kernel re-reads the whole m x kbar x dsub codebook per slot).
// Entry arithmetic is pw_sqdist_v8's, reductions and quantization are
// k_small_tables' — bitwise the same tables, bounds and u8 entries.
// Requires 8 | dsub <= 128 (16-B rows); one warp per slot after the tables.
template <int SPC>
#ifndef DPQ_K1MS_MINB
#define DPQ_K1MS_MINB 2
#endif
__global__ void __launch_bounds__(256, DPQ_K1MS_MINB) k_small_tables_ms(TablesArgs a, int n_slots) {
  extern __shared__ __align__(16) float sm_ms[];
  const int d = a.m * a.dsub, ne = a.m * a.kbar, tid = threadIdx.x;
  float* ys = sm_ms;            // [SPC][d]
  float* st = sm_ms + SPC * d;  // [SPC][ne]
  __shared__ int sl[SPC];
  __shared__ int64_t yr[SPC];
  if (tid < SPC) {
    const int b = blockIdx.x * SPC + tid;
    const int s = b < n_slots ? (a.slot_list ? a.slot_list[b] : b) : -1;
    sl[tid] = s;
    yr[tid] = s < 0 ? 0 : (a.y_sq ? (int64_t)a.y_sq[s] * a.y_ma + a.y_sp[s] : (int64_t)s);
  }
  __syncthreads();
  for (int i = tid; i < SPC * d; i += 256) {
    const int k = i / d, t = i % d;
    ys[i] = sl[k] >= 0 ? a.y[yr[k] * d + t] : 0.f;
  }
  __syncthreads();
  const f32x2_t z2 = a.negzero2;
  for (int e = tid; e < ne; e += 256) {
    const int j = e / a.kbar;
    const ulonglong2* c2 = reinterpret_cast<const ulonglong2*>(a.dcb + (int64_t)e * a.dsub);
    f32x2_t r[SPC][4];
    for (int i = 0; i < a.dsub / 8; ++i) {
      const ulonglong2 ca = c2[2 * i], cb = c2[2 * i + 1];
      const f32x2_t cv[4] = {ca.x, ca.y, cb.x, cb.y};
#pragma unroll
      for (int k = 0; k < SPC; ++k) {
        const ulonglong2* y2 = reinterpret_cast<const ulonglong2*>(ys + k * d + j * a.dsub);
        const ulonglong2 p = y2[2 * i], q = y2[2 * i + 1];
        const f32x2_t yv[4] = {p.x, p.y, q.x, q.y};
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          const f32x2_t v = sqdiff2(cv[l], yv[l], z2);
          r[k][l] = (i == 0) ? v : add2(r[k][l], v);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < SPC; ++k) st[k * ne + e] = pw_combine2(r[k]);
  }
  __syncthreads();
  // Bounds, quantization and cluster keys: WPS = 8 / SPC warps per slot
  // (every warp busy), each over an interleaved share of the entries and the
  // prefix rows; min / max / first-argmin partials combined in shared memory
  // (order-free, so the results are the per-warp form's bit for bit).
  constexpr int WPS = SPC >= 8 ? 1 : 8 / SPC;
  __shared__ float p_min[8];
  __shared__ double p_max[8];
  __shared__ uint32_t p_best[8][2];
  const int w = tid >> 5, lane = tid & 31;
  const int k = w / WPS, sub = w % WPS, step = 32 * WPS, e0 = 32 * sub + lane;
  const int s = k < SPC ? sl[k] : -1;
  const float* t = st + (k < SPC ? k : 0) * ne;
  if (s >= 0) {
    float mn = INFINITY;
    for (int e = e0; e < ne; e += step) mn = fminf(mn, t[e]);
    mn = warp_min_f(mn);
    double mx = -INFINITY;
    if (!a.bounds_in) {
      const int pi = a.slot_list ? blockIdx.x * SPC + k : s;
      const int64_t pre_off = a.prefix_off ? a.prefix_off[pi] : 0;
      const int64_t npre = a.prefix_len ? a.prefix_len[pi] : a.npre;
      if (a.code_bytes == 2 && a.m == 4) {
        // one 8-byte code load per row, four rows in flight per lane
        const uint2* pc = reinterpret_cast<const uint2*>(a.prefix) + pre_off;
        const uint32_t kb = (uint32_t)a.kbar, msk = (uint32_t)a.mask;
        for (int64_t p = e0; p < npre; p += 4 * step) {
          uint2 cv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int64_t pu = p + (int64_t)u * step;
            cv[u] = pu < npre ? __ldg(pc + pu) : make_uint2(0u, 0u);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (p + (int64_t)u * step >= npre) break;
            double acc = 0.0;
            acc = __dadd_rn(acc, (double)t[(cv[u].x & 0xFFFFu) & msk]);
            acc = __dadd_rn(acc, (double)t[kb + ((cv[u].x >> 16) & msk)]);
            acc = __dadd_rn(acc, (double)t[2 * kb + ((cv[u].y & 0xFFFFu) & msk)]);
            acc = __dadd_rn(acc, (double)t[3 * kb + ((cv[u].y >> 16) & msk)]);
            mx = fmax(mx, acc);
          }
        }
      } else {
#pragma unroll 4
        for (int64_t p = e0; p < npre; p += step) {
          double acc = 0.0;
          for (int j = 0; j < a.m; ++j) {
            const uint32_t c = code_at(a.prefix, a.code_bytes, (pre_off + p) * a.m + j);
            acc = __dadd_rn(acc, (double)t[j * a.kbar + (c & a.mask)]);
          }
          mx = fmax(mx, acc);
        }
      }
      mx = warp_max_d(mx);
    }
    if (lane == 0) { p_min[w] = mn; p_max[w] = mx; }
  }
  __syncthreads();
  if (s >= 0) {
    double qmin = (double)p_min[k * WPS], qmax = p_max[k * WPS];
    for (int i = 1; i < WPS; ++i) {
      qmin = fmin(qmin, (double)p_min[k * WPS + i]);
      qmax = fmax(qmax, p_max[k * WPS + i]);
    }
    if (a.bounds_in) {
      qmin = a.bounds_in[2 * s];
      qmax = a.bounds_in[2 * s + 1];
    }
    const bool degenerate = !(qmax > qmin);
    const double scale = degenerate ? 0.0 : __ddiv_rn(255.0, __dsub_rn(qmax, qmin));
    const float qmaxf = __double2float_rn(qmax);
    uint32_t best0 = 0xFFFFFFFFu, best1 = 0xFFFFFFFFu;
    for (int e = e0; e < ne; e += step) {
      const uint8_t q = degenerate ? (uint8_t)0 : quantize_entry(t[e], qmin, scale, qmaxf);
      if (a.small_out) a.small_out[(int64_t)s * ne + e] = t[e];
      if (a.q8_out) a.q8_out[(int64_t)s * ne + e] = q;
      if (e < a.kbar) best0 = min(best0, ((uint32_t)q << 16) | (uint32_t)e);
      else if (e < 2 * a.kbar) best1 = min(best1, ((uint32_t)q << 16) | (uint32_t)(e - a.kbar));
    }
    if (sub == 0 && lane == 0) {
      a.qmin_out[s] = qmin;
      a.qmax_out[s] = degenerate ? qmin : qmax;
    }
    best0 = __reduce_min_sync(0xffffffffu, best0);
    best1 = __reduce_min_sync(0xffffffffu, best1);
    if (lane == 0) { p_best[w][0] = best0; p_best[w][1] = best1; }
  }
  if (a.cluster && a.m >= 2) {
    __syncthreads();
    if (s >= 0 && sub == 0 && lane == 0) {
      uint32_t b0 = p_best[w][0], b1 = p_best[w][1];
      for (int i = 1; i < WPS; ++i) { b0 = min(b0, p_best[w + i][0]); b1 = min(b1, p_best[w + i][1]); }
      a.cluster[s] = (uint16_t)(((b0 & 0xFFu) << 8) | (b1 & 0xFFu));
    }
  }
}

// Scan-layout LUT tiles from the u8 tables q8 [nslot][m][kbar] (see
// lut_index): one thread per (tile, subspace, table row) writes the row's
// LPC lane words (QT/4 queries x 4 bytes, contiguous) with 16-B stores;
// the q8 reads are coalesced across consecutive rows.
//
// With gword given (after the guards are known) a tile whose every query has
// guard B <= 126 is written with entries clamped to 127 and flagged "fast":
// an entry >= 127 > B rules a hit out either way, and every hit has all its
// entries < 127, so hits and their scores are unchanged, while two 7-bit
// words add without carries (k_scan_emit's fast inner loop).
constexpr uint32_t kClampMaxGuard = 126;

// Tile modes (tile_fast[t]), chosen from the largest guard B of the tile:
//   0  generic 8-bit entries
//   7  B <= 126: entries clamped to 127, pair sums in bytes (fast7 loop)
//   6  B <= 62 : entries clamped to 63, four-entry sums <= 252 in bytes
//   5  B <= 30 : entries clamped to 31 and the per-query bias C = 127 - B
//                folded into subspace 0, so a query hits iff bit 7 of its
//                byte sum is clear (C = 128 for slots without a guard)
// Modes 5/6 are scanned by the "wide" loop of k_scan_emit (MPAD = 4): 16
// queries per lane per 128-bit LDS, 4 codes per warp step.
enum { kModeGeneric = 0, kModeWide5 = 5, kModeWide6 = 6, kMode7 = 7 };

__device__ __forceinline__ uint32_t wide_bias(uint32_t gw) {  // C of one slot
  return gw >= 0x8000u ? 127u - (gw - 0x8000u) : 128u;
}

template <int MPAD, int QTX = default_qt(MPAD)>
__global__ void __launch_bounds__(256) k_build_lut(const uint8_t* __restrict__ q8, int nslot, int m, int kbar,
                                                   uint8_t* __restrict__ lut, int ntiles,
                                                   const uint16_t* __restrict__ gword, int* __restrict__ tile_fast,
                                                   int allow_wide, const int* __restrict__ slot_query,
                                                   const int* __restrict__ slot_live,
                                                   const int* __restrict__ live = nullptr) {
  if (live && *live == 0) return;  // every query took the direct scan
  // One CTA per (tile, subspace j): the QT slots' u8 rows of subspace j are
  // staged in shared memory ([slot][group], rows padded to 65 words so the
  // transposed reads below are conflict-free), then written as the tile's
  // 256 table rows of QT bytes with coalesced 32-bit stores.
  using G = ScanGeom<MPAD, QTX>;
  constexpr int RW = 65;  // words per staged row (256 groups + pad)
  __shared__ uint32_t st[G::QT * RW];
  __shared__ uint32_t s_bmax;
  const int t = blockIdx.x, j = blockIdx.y, tid = threadIdx.x;
  if (tid == 0) s_bmax = 0;
  __syncthreads();
  if (gword)
    for (int qq = tid; qq < G::QT; qq += 256) {
      const uint32_t gw = gword[t * G::QT + qq];
      if (gw >= 0x8000u) atomicMax(&s_bmax, gw - 0x8000u);
    }
  const bool live_j = j < m;
  __shared__ uint32_t sbias[G::QT / 4];  // wide-5 bias bytes of slots 4w..4w+3 (subspace 0 only)
  if (gword && j == 0)
    for (int w = tid; w < G::QT / 4; w += 256) {
      uint32_t b4 = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) b4 |= wide_bias(gword[t * G::QT + 4 * w + b]) << (8 * b);
      sbias[w] = b4;
    }
  for (int i = tid; i < G::QT * 64; i += 256) {
    const int sl = i >> 6, w = i & 63;
    const int slot = t * G::QT + sl;
    const int q = slot_query ? slot_query[slot] : slot;
    uint32_t v = 0;
    if (slot_live && slot_live[slot] < 0) {
      v = 0xFFFFFFFFu;  // padding slot (ivf): saturated entries, its q8 row is never computed
    } else if (live_j && q >= 0 && q < nslot && 4 * w < kbar) {
      const uint8_t* row = q8 + ((int64_t)q * m + j) * kbar;
      if ((kbar & 3) == 0) v = *reinterpret_cast<const uint32_t*>(row + 4 * w);
      else
        for (int b = 0; b < 4 && 4 * w + b < kbar; ++b) v |= (uint32_t)row[4 * w + b] << (8 * b);
    }
    st[sl * RW + w] = v;
  }
  __syncthreads();
  int mode = kModeGeneric;
  if (gword) {
    const uint32_t bmax = s_bmax;
    if (MPAD == 4 && G::QT == 128 && allow_wide && bmax <= 30u) mode = kModeWide5;
    else if (MPAD == 4 && G::QT == 128 && allow_wide && bmax <= 62u) mode = kModeWide6;
    else if (bmax <= kClampMaxGuard) mode = kMode7;
  }
  const uint32_t cmax = mode == kModeWide5 ? 31u : (mode == kModeWide6 ? 63u : (mode == kMode7 ? 127u : 255u));
  const bool fold = mode == kModeWide5 && j == 0;
  if (tile_fast && j == 0 && tid == 0) tile_fast[t] = mode;
  uint8_t* tbase = lut + (int64_t)t * G::LUT_BYTES + (int64_t)(j / G::SPR) * 256 * 256 + (j % G::SPR) * G::ROWB;
  constexpr int WPR = G::QT / 4;  // 32-bit words per table row
  constexpr int WG = WPR / 8;     // 8-word groups per table row
  // 4x4 byte transposes: lane (wi, c) of a warp reads staged word (slot
  // 4w + c, groups 4gq..4gq+3) — conflict-free, RW = 65 — the 4 lanes of a
  // quad exchange their words and each keeps byte c of all four, i.e. the
  // table word (group 4gq + c, slots 4w..4w+3); clamped per byte, the wide-5
  // bias added per slot byte (entries <= 31, bias <= 128: no carries).
  const int lane = tid & 31, wi = lane >> 2, c = lane & 3, quad = lane & ~3;
  const uint32_t sel = (uint32_t)c | ((uint32_t)(c + 4) << 4);
  const uint32_t cmax4 = cmax * 0x01010101u;
  for (int blk = tid >> 5; blk < 64 * WG; blk += 8) {
    const int gq = blk / WG, w = (blk % WG) * 8 + wi;
    const uint32_t mine = st[(4 * w + c) * RW + gq];
    const uint32_t i0 = __shfl_sync(0xffffffffu, mine, quad), i1 = __shfl_sync(0xffffffffu, mine, quad + 1);
    const uint32_t i2 = __shfl_sync(0xffffffffu, mine, quad + 2), i3 = __shfl_sync(0xffffffffu, mine, quad + 3);
    const int g = 4 * gq + c;
    uint32_t v = g < kbar ? __byte_perm(__byte_perm(i0, i1, sel), __byte_perm(i2, i3, sel), 0x5410) : 0u;
    if (cmax < 255u) v = __vminu4(v, cmax4);
    if (fold) v += sbias[w];
    reinterpret_cast<uint32_t*>(tbase + (int64_t)g * 256)[w] = v;
  }
}

// Flat batches: query slots ordered so each query tile holds similar
// queries.  With q8 (and nq <= kSortMax) the key is (guard class, g0*, g1*):
// class 0/1/2/3 = B <= 30 / <= 62 / larger / no guard (tile modes 5/6/7),
// g*_j = the derived group nearest to the query in subspace j (first argmin
// of its 8-bit table).  Clustered tiles make the per-tile run filter
// (k_run_potential) skip most rows; otherwise slots are counting-sorted by B.
// slot_query[s] = query in slot s (-1: padding), gword_p[s] = its guard word.
// Only the scan layout changes; emit lists stay per query.
constexpr int kSortMax = 4096;
__global__ void __launch_bounds__(1024) k_sort_slots(const uint16_t* __restrict__ gword,
                                                      const uint16_t* __restrict__ cluster, int nq, int nslot_pad,
                                                      int* __restrict__ slot_query, uint16_t* __restrict__ gword_p,
                                                      const int* __restrict__ live = nullptr) {
  if (live && *live == 0) return;  // every query took the direct scan
  __shared__ uint32_t kv32[kSortMax];
  __shared__ int cnt[258];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto gkey = [&](int q) {
    const uint32_t gw = gword[q];
    return gw >= 0x8000u ? (int)min(gw - 0x8000u, 255u) : 256;
  };
  if (cluster && nq <= kSortMax) {
    // Bitonic sort of P = pow2 >= nq keys, element i = e * 1024 + tid held in
    // register x[e]: partner strides >= 1024 are in-thread swaps, 32..512 go
    // through shared memory, < 32 are warp shuffles (no barrier).
    constexpr int EMAX = kSortMax / 1024;
    int P = 1;
    while (P < nq) P <<= 1;
    const int E = P > 1024 ? P / 1024 : 1;
    uint32_t x[EMAX];  // key = class << 28 | cluster << 12 | q (q < kSortMax = 2^12)
#pragma unroll
    for (int e = 0; e < EMAX; ++e) {
      const int q = e * 1024 + tid;
      x[e] = 0xFFFFFFFFu;
      if (e < E && q < nq) {
        const int B = gkey(q);
        const uint32_t cls = B == 256 ? 3u : (B <= 30 ? 0u : (B <= 62 ? 1u : 2u));
        x[e] = (cls << 28) | ((uint32_t)cluster[q] << 12) | (uint32_t)q;
      }
    }
    // element i keeps the min of (i, i ^ j) iff (i < partner) == ascending
    auto keep = [](uint32_t mine, uint32_t other, bool take_min) {
      return take_min ? (other < mine ? other : mine) : (other > mine ? other : mine);
    };
    for (int size = 2; size <= P; size <<= 1) {
      for (int j = size >> 1; j > 0; j >>= 1) {
        if (j >= 1024) {
          const int ej = j / 1024;
#pragma unroll
          for (int e = 0; e < EMAX; ++e) {
#pragma unroll
            for (int f = e + 1; f < EMAX; ++f) {  // (compile-time indices: x stays in registers)
              if (f >= E || f - e != ej || (e & ej)) continue;
              const int i = e * 1024 + tid;
              const bool asc = (i & size) == 0;
              const uint32_t a0 = x[e], a1 = x[f];
              x[e] = keep(a0, a1, asc);
              x[f] = keep(a1, a0, !asc);
            }
          }
        } else if (j >= 32) {
#pragma unroll
          for (int e = 0; e < EMAX; ++e)
            if (e < E) kv32[e * 1024 + tid] = x[e];
          __syncthreads();
#pragma unroll
          for (int e = 0; e < EMAX; ++e) {
            if (e >= E) continue;
            const int i = e * 1024 + tid;
            if (i >= P) continue;
            const bool asc = (i & size) == 0;
            x[e] = keep(x[e], kv32[i ^ j], ((i & j) == 0) == asc);
          }
          __syncthreads();
        } else {
#pragma unroll
          for (int e = 0; e < EMAX; ++e) {
            if (e >= E) continue;
            const int i = e * 1024 + tid;
            const uint32_t o = __shfl_xor_sync(0xffffffffu, x[e], j);
            const bool asc = (i & size) == 0;
            x[e] = keep(x[e], o, ((i & j) == 0) == asc);
          }
        }
      }
    }
#pragma unroll
    for (int e = 0; e < EMAX; ++e) {
      const int sl = e * 1024 + tid;
      if (e < E && sl < nq) {
        const int q = (int)(x[e] & 0xFFFu);
        slot_query[sl] = q;
        gword_p[sl] = gword[q];
      }
    }
  } else {
    for (int i = tid; i < 258; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    for (int q = tid; q < nq; q += blockDim.x) atomicAdd(&cnt[gkey(q) + 1], 1);
    __syncthreads();
    if (tid == 0)
      for (int i = 1; i < 258; ++i) cnt[i] += cnt[i - 1];  // cnt[k] = first slot of key k
    __syncthreads();
    for (int q = tid; q < nq; q += blockDim.x) {
      const int sl = atomicAdd(&cnt[gkey(q)], 1);
      slot_query[sl] = q;
      gword_p[sl] = gword[q];
    }
  }
  for (int sl = nq + tid; sl < nslot_pad; sl += blockDim.x) {
    slot_query[sl] = -1;
    gword_p[sl] = 0x7F7Fu;
  }
}

// Run filter for indexes whose rows are sorted by key = g0 << 8 | g1 (low
// bytes of subspaces 0 and 1).  Every entry is >= 0, so a row of key
// (g0, g1) can only reach a query's guard B if e0[g0] + e1[g1] <= B.
//   k_run_potential: pot[tile][key] = 1 iff some slot of the tile passes
//     (grid: 256 / kRunG0 x tiles, kRunG0 values of g0 per CTA, 4 of g1 per thread)
//   k_chunk_list: per tile, the scan chunks (512 B of plane) whose key range holds a key
//     with pot = 1 (unordered list + length); the scan visits only those.
// Skipped rows have score > B, so they would never be emitted: exact.
constexpr int kRunG0 = 8;  // values of g0 per k_run_potential CTA
__global__ void __launch_bounds__(256) k_run_potential(const uint8_t* __restrict__ q8, int m, int kbar,
                                                       const int* __restrict__ slot_query,
                                                       const uint16_t* __restrict__ gword, int qt, int nq,
                                                       uint8_t* __restrict__ pot,
                                                       const int* __restrict__ live = nullptr) {
  if (live && *live == 0) return;  // every query took the direct scan
  // CTA = (16 values of g0, tile).  The tile's e1 words are staged once per
  // CTA with eight independent row loads in flight per thread (the load
  // latency, not the arithmetic, bounds this kernel).
  extern __shared__ __align__(16) uint32_t bw[];  // [qt][64] words: 4 x min(e1, 127)
  uint32_t* c4 = bw + qt * 64;                    // [kRunG0][qt] bias words
  __shared__ int sq[256];                         // slot -> query (qt <= 256)
  const int tile = blockIdx.y, tid = threadIdx.x;
  for (int sl = tid; sl < qt; sl += 256) {
    const int q = slot_query ? slot_query[tile * qt + sl] : tile * qt + sl;
    sq[sl] = (q >= 0 && q < nq) ? q : -1;
  }
  __syncthreads();
  auto clamp127 = [](uint32_t v) {  // min(byte, 127) per byte
    const uint32_t hi = v & 0x80808080u;
    return (v & ~(hi | (hi >> 1) | (hi >> 2) | (hi >> 3) | (hi >> 4) | (hi >> 5) | (hi >> 6) | (hi >> 7))) |
           (hi ? (((hi >> 7) * 0x7Fu) & 0x7F7F7F7Fu) : 0u);
  };
  {
    const int g = (tid & 63) * 4;  // this thread's 4 groups; slots tid/64, +4, +8, ...
    constexpr int U = 8;
    for (int sl0 = tid >> 6; sl0 < qt; sl0 += 4 * U) {
      uint32_t v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int sl = sl0 + 4 * u;
        const int q = sl < qt ? sq[sl] : -1;
        v[u] = 0x7F7F7F7Fu;
        if (q >= 0) {
          const uint8_t* row = q8 + ((int64_t)q * m + 1) * kbar;
          if ((kbar & 3) == 0) {
            if (g < kbar) v[u] = __ldg(reinterpret_cast<const uint32_t*>(row + g));
          } else {
            uint32_t w = 0;
            for (int b = 0; b < 4; ++b) w |= (g + b < kbar ? min((uint32_t)row[g + b], 127u) : 127u) << (8 * b);
            v[u] = w;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int sl = sl0 + 4 * u;
        if (sl < qt) bw[sl * 64 + (tid & 63)] = clamp127(v[u]);  // (idempotent on clamped words)
      }
    }
  }
  {
    constexpr int U = (kRunG0 * 256 + 255) / 256;  // (gi, slot) pairs per thread (qt <= 256), loads in flight together
    int ge[U];
    uint32_t gw[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = tid + 256 * u;
      const int gi = i / qt, sl = i % qt, g0 = blockIdx.x * kRunG0 + gi;
      const int q = i < kRunG0 * qt ? sq[sl] : -1;
      gw[u] = q >= 0 ? (uint32_t)gword[tile * qt + sl] : 0u;
      ge[u] = (q >= 0 && g0 < kbar) ? (int)__ldg(q8 + (int64_t)q * m * kbar + g0) : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = tid + 256 * u;
      if (i >= kRunG0 * qt) break;
      const int gi = i / qt, sl = i % qt, g0 = blockIdx.x * kRunG0 + gi;
      uint32_t c = 0x80808080u;  // never
      if (sq[sl] >= 0 && gw[u] >= 0x8000u && g0 < kbar) {
        const int D = (int)(gw[u] - 0x8000u) - ge[u];  // e1 must be <= D
        if (D >= 127) c = 0u;  // any (clamped, <= 127) e1 passes
        else if (D >= 0) c = (uint32_t)(127 - D) * 0x01010101u;
      }
      c4[i] = c;
    }
  }
  __syncthreads();
  const int t = tid & 63;
  for (int gi = tid >> 6; gi < kRunG0; gi += 4) {
    const int g0 = blockIdx.x * kRunG0 + gi;
    uint32_t acc = 0xFFFFFFFFu;
    for (int sl = 0; sl < qt; ++sl) {
      const uint32_t b = bw[sl * 64 + t], c = c4[gi * qt + sl];
      acc &= b | ((b & 0x7F7F7F7Fu) + c);  // bit 7 clear: e1 <= D for this slot
    }
    // byte b of the word = key (g0, 4t + b) has potential
    if (g0 < kbar)
      reinterpret_cast<uint32_t*>(pot + (int64_t)tile * 65536 + g0 * 256)[t] = (~acc & 0x80808080u) >> 7;
  }
}

constexpr int kChunkPerThread = 4;  // k_chunk_list: chunks per thread, their loads in flight together
__global__ void __launch_bounds__(256) k_chunk_list(const uint32_t* __restrict__ chunk_keys, int nchunks, int cr,
                                                    const uint8_t* __restrict__ pot, int* __restrict__ list,
                                                    int* __restrict__ list_len, int64_t n, int nb, int qt,
                                                    unsigned long long* __restrict__ n_rows,
                                                    const int* __restrict__ live = nullptr) {
  if (live && *live == 0) return;  // every query took the direct scan (list lengths stay 0)
  // CTA = (256 * kChunkPerThread chunks, tile); chunk c0 + 256 u + tid for u < kChunkPerThread
  const int tile = blockIdx.y, lane = threadIdx.x & 31;
  const int c0 = blockIdx.x * 256 * kChunkPerThread + threadIdx.x;
  const uint8_t* p = pot + (int64_t)tile * 65536;
  uint32_t kk[kChunkPerThread];
#pragma unroll
  for (int u = 0; u < kChunkPerThread; ++u) {
    const int c = c0 + 256 * u;
    kk[u] = c < nchunks ? __ldg(chunk_keys + c) : 1u;  // (empty key range lo = 1 > hi = 0)
  }
  bool f[kChunkPerThread];
#pragma unroll
  for (int u = 0; u < kChunkPerThread; ++u) {  // first key of each range: loads issued together
    const uint32_t lo = kk[u] & 0xFFFFu;
    f[u] = lo <= (kk[u] >> 16) && p[lo] != 0;
  }
  // rest of the range, 16 keys per load (pot bytes are 0 / 1; bytes outside [lo, hi] masked)
  auto any_in = [](uint4 v, uint32_t base, uint32_t lo, uint32_t hi) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    bool r = false;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int b0 = (int)(base + 4 * k);
      const int s0 = max((int)lo - b0, 0), s1 = min((int)hi - b0, 3);
      if (s0 <= s1) r |= (w[k] & ((0xFFFFFFFFu << (8 * s0)) & (0xFFFFFFFFu >> (8 * (3 - s1))))) != 0u;
    }
    return r;
  };
  const uint4* p4 = reinterpret_cast<const uint4*>(p);
#pragma unroll
  for (int u = 0; u < kChunkPerThread; ++u) {
    const uint32_t lo = (kk[u] & 0xFFFFu) + 1, hi = kk[u] >> 16;
    for (uint32_t v = lo >> 4; v <= (hi >> 4) && lo <= hi && !f[u]; v += 2) {
      const uint4 a = __ldg(p4 + v);
      const bool two = v + 1 <= (hi >> 4);
      const uint4 b = two ? __ldg(p4 + v + 1) : make_uint4(0u, 0u, 0u, 0u);
      f[u] = any_in(a, 16 * v, lo, hi) || (two && any_in(b, 16 * (v + 1), lo, hi));
    }
  }
  // one list reservation per warp for all its chunks
  uint32_t bal[kChunkPerThread];
  int tot = 0;
#pragma unroll
  for (int u = 0; u < kChunkPerThread; ++u) {
    bal[u] = __ballot_sync(0xffffffffu, f[u]);
    tot += __popc(bal[u]);
  }
  int base = 0;
  if (lane == 0 && tot) base = atomicAdd(list_len + tile, tot);
  base = __shfl_sync(0xffffffffu, base, 0);
  unsigned rows = 0;
#pragma unroll
  for (int u = 0; u < kChunkPerThread; ++u) {
    const int c = c0 + 256 * u;
    if (f[u]) {
      list[(int64_t)tile * nchunks + base + __popc(bal[u] & ((1u << lane) - 1u))] = c;
      rows += (unsigned)min((int64_t)cr, n - (int64_t)c * cr);
    }
    base += __popc(bal[u]);
  }
  if (n_rows) {  // query-rows this tile will scan (its real queries x listed rows) and the listed plane rows
    const unsigned wr = __reduce_add_sync(0xffffffffu, rows);
    if (lane == 0 && wr) {
      atomicAdd(n_rows, (unsigned long long)wr * (unsigned long long)min(qt, nb - tile * qt));
      atomicAdd(n_rows + 1, (unsigned long long)wr);
    }
  }
}

// ============================================================================
// Direct first pass (flat indexes whose rows are sorted by key = g0 << 8 | g1).
//
// A row can reach a query's guard B only if e0[g0] + e1[g1] <= B, and on
// clustered data a query has very few such keys (BASELINE configs[1]: a
// median of ONE key, 0.3% of the rows, of which 60% are hits).  So instead of
// testing 128 queries against the union of their rows (k_scan_emit), a query
// whose keys are few is scanned on its own: k_key_select enumerates its keys,
// cuts their row runs (key_start, built with the index) into work items of
// <= kDirSeg rows, and k_scan_direct tests each row with two byte lookups in
// the query's own 8-bit tables; hits are warp-compacted straight into the
// query's emit list (one reservation per 128 rows, no staging, no per-hit
// atomics).  The emitted set is exactly {rows : score <= B}, the same set
// k_scan_emit emits, so K3 / K6 and the results are unchanged.  Queries with
// too many keys or rows (large guards) stay on the tile path: k_key_select
// leaves their guard word in place and replaces a direct query's by "no
// guard" so the tile kernels see it as padding; with no query left they
// return at once (`live`).
// ============================================================================
constexpr int kDirSeg = 1024;         // rows per work item
constexpr uint32_t kDirNullQ = 0x3FFFu;
constexpr int kDirMaxBatch = 0x3FFE;  // queries per batch the item format holds
// item: x = first row, y = e01 | (rows - 1) << 8 | query << 18

__global__ void k_key_starts(const uint32_t* __restrict__ skeys, int64_t n, uint32_t* __restrict__ key_start) {
  // key_start[k] = first row whose key is >= k (k = 0 .. 65536); thread i owns the keys that start at row i
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n) return;
  const uint32_t k = i < n ? skeys[i] : 65536u;
  const uint32_t kp = i > 0 ? skeys[i - 1] + 1u : 0u;
  for (uint32_t key = kp; key <= k; ++key) key_start[key] = (uint32_t)i;
}

// Guard B of one slot from its (sample or exact) score histogram, computed by
// one warp (see k_guard below for the rule): lane l holds bins 8l .. 8l+7.
__device__ __forceinline__ int guard_of_hist(const uint32_t* __restrict__ hist_row, int lane, int r2, double lam,
                                             bool ex) {
  const uint4* h4 = reinterpret_cast<const uint4*>(hist_row) + 2 * lane;
  const uint4 a = __ldg(h4), b = __ldg(h4 + 1);
  const uint32_t v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, lane == 31 ? 0u : b.w};
  const double target = ex ? (double)r2 : lam + 3.0 * sqrt(lam) + 4.0;
  uint64_t tot = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) tot += v[i];
  uint64_t incl = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t x = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += x;
  }
  uint64_t cum = incl - tot;
  int first = 8;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    cum += v[i];
    if (first == 8 && (double)cum >= target) first = i;
  }
  if (lane == 31 && first == 7) first = 8;  // (bin 255)
  const uint32_t bal = __ballot_sync(0xffffffffu, first < 8);
  int B = 254;
  if (bal) {
    const int src = __ffs(bal) - 1;
    B = 8 * src + __shfl_sync(0xffffffffu, first, src);
  }
  return B;
}

struct KeySelArgs {
  const uint8_t* q8;           // [nq][m][kbar]
  int m, kbar;
  uint16_t* guard_b;           // [nq] guard B (read; written when hist is given or a query is handed back, see skip_tiles)
  const uint32_t* hist = nullptr;  // optional [nq][256] score histograms: the guard is computed here (k_guard's rule)
  int r2 = 0, exact = 0;
  double lambda = 0.0;
  int32_t* slack = nullptr;    // optional [nq][m]: k_entry_slack's output, computed here
  int zero_hist = 0;           // (with hist) clear the query's histogram row once the guard is read: the direct
                               // scan then counts its hits by score into it (DirectArgs::hist)
  int skip_tiles = 0;          // the tile kernels are not launched: a query that needs them gets guard 0, which
                               // K3 flags as too tight (the batch is then redone with the tile path)
  uint16_t* gword;             // [nq] guard words: rewritten (direct: 0x7F7F, tile path: 0x8000 + B)
  const uint32_t* key_start;   // [65537]
  uint2* items;
  int* state;                  // [0] items reserved, [1] queries left to the tile path (zeroed before)
  int item_cap, item_qcap, pair_cap;
  unsigned long long* n_rows;  // optional counters: [0] query-rows, [1] plane rows
};

__device__ __forceinline__ int block_scan_256(int v, int* s_warp, int& total) {  // inclusive; blockDim = 256
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();  // (s_warp reuse)
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  int add = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    const int sw = s_warp[w];
    if (w < warp) add += sw;
    tot += sw;
  }
  total = tot;
  return x + add;
}

__global__ void __launch_bounds__(256) k_key_select(KeySelArgs a, int nq) {
  // One CTA per query.  Thread t plays g0 = t while the (g0, g1) pairs are
  // counted, then g1 = t: for every g0 whose e0 leaves room under the guard
  // the CTA tests its 256 keys (g0, t) together, reading the adjacent
  // key_start words with coalesced loads.
  __shared__ int s_cum[256];
  __shared__ int s_warp[8];
  __shared__ int s_act[256];  // g0 values with e0 + min(e1) <= B
  __shared__ uint8_t s_e0[256];
  __shared__ int s_nact, s_base;
  __shared__ int s_rest;  // sum over subspaces j >= 2 of min_g e_j[g]
  __shared__ int s_guard;
  __shared__ int s_min[8];
  const int q = blockIdx.x, t = threadIdx.x;
  if (q >= nq) return;
  if (a.hist) {
    if (t < 32) {
      const int Bh = guard_of_hist(a.hist + (int64_t)q * 256, t, a.r2, a.lambda, a.exact != 0 || a.lambda < 0.0);
      if (t == 0) s_guard = Bh;
    }
    __syncthreads();
    if (a.zero_hist) const_cast<uint32_t*>(a.hist)[(int64_t)q * 256 + t] = 0u;
  }
  const int Bg = a.hist ? s_guard : (int)a.guard_b[q];
  const uint8_t* e = a.q8 + (int64_t)q * a.m * a.kbar;
  const int e0 = t < a.kbar ? (int)e[t] : 255;
  const int e1 = t < a.kbar ? (int)e[a.kbar + t] : 255;
  s_cum[t] = 0;
  s_e0[t] = (uint8_t)e0;
  if (t == 0) { s_nact = 0; s_rest = 0; }
  __syncthreads();
  // a row of key (g0, g1) scores at least e0 + e1 + sum_{j >= 2} min e_j: only keys with
  // e0 + e1 <= B = guard - that sum can hold a hit (the items still carry the full guard)
  for (int j = 0; j < a.m && j < 8; ++j) {
    const unsigned v = __reduce_min_sync(0xffffffffu, t < a.kbar ? (unsigned)e[j * a.kbar + t] : 255u);
    if ((t & 31) == 0) s_cum[j * 8 + (t >> 5)] = (int)v;  // (s_cum reused: cleared below)
  }
  __syncthreads();
  if (t < a.m && t < 8) {
    int mn = 255;
    for (int w = 0; w < 8; ++w) mn = min(mn, s_cum[t * 8 + w]);
    s_min[t] = mn;
    if (t >= 2) atomicAdd(&s_rest, mn);
  }
  __syncthreads();
  if (a.slack && t < a.m && t < 8) {  // slack[q][j] = sum of the other subspaces' smallest entries (k_entry_slack)
    int sum = 0;
    for (int j = 0; j < a.m && j < 8; ++j) sum += s_min[j];
    a.slack[q * a.m + t] = sum - s_min[t];
  }
  const int B = Bg - s_rest;
  s_cum[t] = 0;
  __syncthreads();
  if (t < a.kbar) atomicAdd(&s_cum[e1], 1);
  __syncthreads();
  int tot = 0;
  const int c = block_scan_256(s_cum[t], s_warp, tot);  // c = #g1 with e1 <= t
  __syncthreads();
  s_cum[t] = c;
  __syncthreads();
  const int lim0 = t < a.kbar ? B - e0 : -1;  // (as g0) e1 must be <= lim0
  const int np = lim0 >= 0 ? s_cum[min(lim0, 255)] : 0;
  int pairs = 0;
  block_scan_256(np, s_warp, pairs);
  bool direct = pairs <= a.pair_cap;
  int my_items = 0, items = 0, excl = 0;
  long long my_rows = 0;
  if (direct) {
    if (np > 0) s_act[atomicAdd(&s_nact, 1)] = t;
    __syncthreads();
    const int nact = s_nact;
    // key_start words of 8 values of g0 in flight together (unconditional, coalesced loads)
    for (int i0 = 0; i0 < nact; i0 += 8) {
      uint32_t ks[8], ke[8];
      int lim[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int g0 = s_act[min(i0 + u, nact - 1)];
        lim[u] = i0 + u < nact ? B - (int)s_e0[g0] : -1;
        ks[u] = __ldg(a.key_start + ((g0 << 8) | t));
        ke[u] = __ldg(a.key_start + ((g0 << 8) | t) + 1);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (e1 <= lim[u]) {  // (t >= kbar: e1 = 255 never passes)
          const uint32_t len = ke[u] - ks[u];
          my_items += (int)((len + kDirSeg - 1) / kDirSeg);
          my_rows += len;
        }
    }
    excl = block_scan_256(my_items, s_warp, items) - my_items;
    direct = items <= a.item_qcap;
  }
  if (direct && items > 0) {
    if (t == 0) s_base = atomicAdd(a.state, items);
    __syncthreads();
    const int base = s_base;
    if (base + items > a.item_cap) {  // list full: null items over the reserved part, query stays on the tile path
      direct = false;
      for (int i = base + t; i < min(base + items, a.item_cap); i += 256) a.items[i] = make_uint2(0u, kDirNullQ << 18);
    } else if (my_items > 0) {
      int o = base + excl;
      const int nact = s_nact;
      for (int i0 = 0; i0 < nact; i0 += 8) {
        uint32_t ks[8], ke[8];
        int e0g[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int g0 = s_act[min(i0 + u, nact - 1)];
          e0g[u] = i0 + u < nact ? (int)s_e0[g0] : 1024;
          ks[u] = __ldg(a.key_start + ((g0 << 8) | t));
          ke[u] = __ldg(a.key_start + ((g0 << 8) | t) + 1);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (e1 <= B - e0g[u]) {
            const uint32_t e01 = (uint32_t)(e0g[u] + e1);
            for (uint32_t r0 = ks[u]; r0 < ke[u]; r0 += kDirSeg)
              a.items[o++] =
                  make_uint2(r0, e01 | ((min(ke[u] - r0, (uint32_t)kDirSeg) - 1u) << 8) | ((uint32_t)q << 18));
          }
      }
    }
  }
  if (direct && a.n_rows) {  // rows this query tests (reported with the scan counters)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my_rows += __shfl_xor_sync(0xffffffffu, my_rows, o);
    if ((t & 31) == 0 && my_rows) {
      atomicAdd(a.n_rows, (unsigned long long)my_rows);
      atomicAdd(a.n_rows + 1, (unsigned long long)my_rows);
    }
  }
  if (t == 0) {
    a.gword[q] = direct ? (uint16_t)0x7F7Fu : (uint16_t)(0x8000 + Bg);
    if (a.hist || (a.skip_tiles && !direct)) a.guard_b[q] = (uint16_t)((a.skip_tiles && !direct) ? 0 : Bg);
    if (!direct) atomicAdd(a.state + 1, 1);
  }
}

struct DirectArgs {
  const uint8_t* plane;
  const uint8_t* q8;
  int m, kbar;
  const uint16_t* guard_b;
  const uint2* items;
  const int* state;  // [0] items listed
  int item_cap;
  uint32_t* emit_cnt;
  uint64_t* emit;
  uint32_t cap;
  // optional [nq][256], zeroed: hits counted by score (one atomic per distinct score of 32 rows), so K3
  // takes b* from it without reading the emit lists back
  uint32_t* hist = nullptr;
};

template <int MPAD, bool E32, bool HIST = false>  // HIST: count the hits into a.hist (its own build: 48 vs 40 registers)
__global__ void __launch_bounds__(256, HIST ? 6 : 0) k_scan_direct(DirectArgs a) {  // (HIST: 41 -> 40 registers, 6 CTAs / SM like the plain build)
  constexpr int TB = (MPAD - 2) * 256;  // table bytes per warp: subspaces 2 .. MPAD-1
  __shared__ __align__(16) uint8_t s_tab[8 * TB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* tab = s_tab + warp * TB;
  const uint32_t lt = (1u << lane) - 1u;
  const int n_items = min(*a.state, a.item_cap);
  const int nw = gridDim.x * 8;
  int curq = -1;
  // (items strided over the warps: claiming them from a global counter
  // instead, two ahead, measured slower — 88 -> 98 us — for ~50k claims)
  int i = blockIdx.x * 8 + warp;
  uint2 it = i < n_items ? __ldg(a.items + i) : make_uint2(0u, 0u);
  for (; i < n_items; i += nw) {
    const uint2 cur = it;
    if (i + nw < n_items) it = __ldg(a.items + i + nw);  // next item in flight
    const int q = (int)(cur.y >> 18);
    if (q == (int)kDirNullQ) continue;
    const int len = (int)((cur.y >> 8) & 0x3FFu) + 1;
    const uint32_t e01 = cur.y & 0xFFu;
    // first rows of the item in flight before the tables are (re)loaded
    const int64_t row0 = (int64_t)cur.x;
    auto load_row = [&](int r, uint32_t& w0, uint32_t& w1) {
      if constexpr (MPAD == 4) {
        w0 = __ldg(reinterpret_cast<const uint32_t*>(a.plane) + row0 + r);
        w1 = 0u;
      } else {
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(a.plane) + row0 + r);
        w0 = v.x; w1 = v.y;
      }
    };
    const int Bp = (int)__ldg(a.guard_b + q) - (int)e01;
    if (q != curq) {
      __syncwarp();
      const uint8_t* src = a.q8 + ((int64_t)q * a.m + 2) * a.kbar;
      const int nb = (a.m - 2) * a.kbar;
      if (a.kbar == 256) {
        for (int v = lane; v * 16 < nb; v += 32)
          reinterpret_cast<uint4*>(tab)[v] = __ldg(reinterpret_cast<const uint4*>(src) + v);
      } else {
        for (int b = lane; b < nb; b += 32) tab[(b / a.kbar) * 256 + (b % a.kbar)] = src[b];
      }
      __syncwarp();
      curq = q;
    }
    auto tsum_of = [&](uint32_t w0, uint32_t w1) -> int {
      int tt = 0;
      if (a.m > 2) tt += (int)tab[(w0 >> 16) & 0xFFu];
      if (a.m > 3) tt += (int)tab[256 + (w0 >> 24)];
      if constexpr (MPAD == 8) {
        if (a.m > 4) tt += (int)tab[512 + (w1 & 0xFFu)];
        if (a.m > 5) tt += (int)tab[768 + ((w1 >> 8) & 0xFFu)];
        if (a.m > 6) tt += (int)tab[1024 + ((w1 >> 16) & 0xFFu)];
        if (a.m > 7) tt += (int)tab[1280 + (w1 >> 24)];
      }
      return tt;
    };
    uint32_t* cnt = a.emit_cnt + q;
    uint32_t* e32 = reinterpret_cast<uint32_t*>(a.emit) + (int64_t)q * a.cap;
    uint64_t* e64 = a.emit + (int64_t)q * a.cap;
    // record of row (row0 + r) with score e01 + t:  E32: row | score << 24
    const uint32_t rec0 = (uint32_t)row0 + (uint32_t)lane + (e01 << kRow32Bits);
    for (int r0 = 0; r0 < len; r0 += 128) {
      int ts[4];
      uint32_t bal[4];
      if (r0 + 128 <= len) {  // full group: no bounds tests
        uint32_t w0[4], w1[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) load_row(r0 + 32 * u + lane, w0[u], w1[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          ts[u] = tsum_of(w0[u], w1[u]);
          bal[u] = __ballot_sync(0xffffffffu, ts[u] <= Bp);
        }
      } else {
        uint32_t w0[4], w1[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          w0[u] = 0u; w1[u] = 0u;
          if (r0 + 32 * u + lane < len) load_row(r0 + 32 * u + lane, w0[u], w1[u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          ts[u] = tsum_of(w0[u], w1[u]);
          bal[u] = __ballot_sync(0xffffffffu, r0 + 32 * u + lane < len && ts[u] <= Bp);
        }
      }
      const int tot = __popc(bal[0]) + __popc(bal[1]) + __popc(bal[2]) + __popc(bal[3]);
      if (tot == 0) continue;
      if constexpr (HIST) {
        uint32_t* hq = a.hist + (int64_t)q * 256 + e01;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if ((bal[u] >> lane) & 1u) {
            const unsigned same = __match_any_sync(bal[u], ts[u]);
            if (lane == __ffs(same) - 1) atomicAdd(hq + ts[u], (uint32_t)__popc(same));
          }
        }
      }
      uint32_t pos = 0;
      if (lane == 0) pos = atomicAdd(cnt, (uint32_t)tot);
      pos = __shfl_sync(0xffffffffu, pos, 0);
      if (pos + (uint32_t)tot > a.cap) {  // list overflow (K3 flags the query): store what fits
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t p = pos + (uint32_t)__popc(bal[u] & lt);
          if (((bal[u] >> lane) & 1u) && p < a.cap) {
            if constexpr (E32) e32[p] = rec0 + (uint32_t)(r0 + 32 * u) + ((uint32_t)ts[u] << kRow32Bits);
            else e64[p] = pack_emit(row0 + r0 + 32 * u + lane, 0u, e01 + (uint32_t)ts[u]);
          }
          pos += (uint32_t)__popc(bal[u]);
        }
        continue;
      }
      uint32_t* g32 = e32 + pos;  // (one 64-bit base per group, 32-bit offsets below)
      uint64_t* g64 = e64 + pos;
      uint32_t off = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if ((bal[u] >> lane) & 1u) {
          const uint32_t p = off + (uint32_t)__popc(bal[u] & lt);
          if constexpr (E32) g32[p] = rec0 + (uint32_t)(r0 + 32 * u) + ((uint32_t)ts[u] << kRow32Bits);
          else g64[p] = pack_emit(row0 + r0 + 32 * u + lane, 0u, e01 + (uint32_t)ts[u]);
        }
        off += (uint32_t)__popc(bal[u]);
      }
    }
  }
}

// ============================================================================
// K2a: score histogram over a strided sample of rows (exact when stride=1
// and the sample is every row).  One CTA = (sample chunk, query tile);
// per-tile histograms live in shared memory, flushed with global atomics.
// ============================================================================
struct Sum4 { uint32_t lo, hi; };  // u16x2: queries (0,2) and (1,3) of a lane

template <int MPAD, int QTX = default_qt(MPAD)>
__device__ __forceinline__ Sum4 lut_sum(const uint8_t* L, uint32_t w0, uint32_t w1) {
  // L = tile base + lic * 4 (generic addressing; used off the hot path)
  using G = ScanGeom<MPAD, QTX>;
  Sum4 s{0u, 0u};
#pragma unroll
  for (int j = 0; j < MPAD; ++j) {
    const uint32_t w = j < 4 ? w0 : w1;
    const uint32_t idx = (w >> (8 * (j & 3))) & 0xFFu;
    const uint32_t v = lds32(L + (j / G::SPR) * 65536 + (idx << 8) + (j % G::SPR) * G::ROWB);
    s.lo += v & 0x00FF00FFu;
    s.hi += __byte_perm(v, 0u, 0x4341u);
  }
  return s;
}

// a * b + c as an integer multiply-add: with b an opaque runtime 1 the
// add is issued on the FMA pipe (IMAD) instead of the saturated ALU pipe.
__device__ __forceinline__ uint32_t fma_add(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// Hot-path variant: base = 64-KB aligned shared address | lic * 4.
template <int MPAD, int QTX = default_qt(MPAD)>
__device__ __forceinline__ Sum4 lut_sum_fast(uint32_t base, uint32_t w0, uint32_t w1, uint32_t one) {
  using G = ScanGeom<MPAD, QTX>;
  Sum4 s{0u, 0u};
#pragma unroll
  for (int j = 0; j < MPAD; ++j) {
    const uint32_t w = j < 4 ? w0 : w1;
    // result bytes: [base.b0 | (j%SPR)*ROWB, w.b(j&3), base.b2, base.b3]
    const uint32_t a = __byte_perm(w, base + (j % G::SPR) * G::ROWB, 0x7604u | ((j & 3) << 4));
    uint32_t v;
    if (j / G::SPR == 0) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    else asm volatile("ld.shared.u32 %0, [%1+65536];" : "=r"(v) : "r"(a));
    if (j == 0) {
      s.lo = v & 0x00FF00FFu;
      s.hi = __byte_perm(v, 0u, 0x4341u);
    } else {
      s.lo = fma_add(v & 0x00FF00FFu, one, s.lo);
      s.hi = fma_add(__byte_perm(v, 0u, 0x4341u), one, s.hi);
    }
  }
  return s;
}

// Fast variant for 7-bit (clamped) tiles, MPAD = 4: add the words of
// subspaces (0,1) and (2,3) first (bytes <= 254, no carries), then split the
// two pair sums.
template <int QTX = 128>
__device__ __forceinline__ Sum4 lut_sum_fast7(uint32_t base, uint32_t w, uint32_t one) {
  using G = ScanGeom<4, QTX>;
  uint32_t v[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t a = __byte_perm(w, base + (j % G::SPR) * G::ROWB, 0x7604u | ((j & 3) << 4));
    if (j / G::SPR == 0) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v[j]) : "r"(a));
    else asm volatile("ld.shared.u32 %0, [%1+65536];" : "=r"(v[j]) : "r"(a));
  }
  const uint32_t p01 = fma_add(v[0], one, v[1]), p23 = fma_add(v[2], one, v[3]);
  Sum4 s;
  s.lo = fma_add(p01 & 0x00FF00FFu, one, p23 & 0x00FF00FFu);
  s.hi = fma_add(__byte_perm(p01, 0u, 0x4341u), one, __byte_perm(p23, 0u, 0x4341u));
  return s;
}

// QT = 64 geometries (CPW = 2): the two half-warps read rows of different
// codes, and a subspace's 64-B slot sits in the same 16 banks of every row,
// so unrotated lookups of the two halves always collide (2-way).  Half-warp 1
// visits the subspaces of each 64-KB table in the order 1, 2, 3, 0 (sums are
// order-free), which puts the two halves in opposite bank halves: rb[j] /
// rs[j] = the lane's base (+ offset) and byte selector of its j-th lookup.
template <int MPAD>
__device__ __forceinline__ Sum4 lut_sum_rot(const uint32_t* rb, const uint32_t* rs, uint32_t w0, uint32_t w1,
                                            uint32_t one) {
  Sum4 s{0u, 0u};
#pragma unroll
  for (int j = 0; j < MPAD; ++j) {
    const uint32_t a = __byte_perm(j < 4 ? w0 : w1, rb[j & 3], rs[j & 3]);
    uint32_t v;
    if (j < 4) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    else asm volatile("ld.shared.u32 %0, [%1+65536];" : "=r"(v) : "r"(a));
    if (j == 0) {
      s.lo = v & 0x00FF00FFu;
      s.hi = __byte_perm(v, 0u, 0x4341u);
    } else {
      s.lo = fma_add(v & 0x00FF00FFu, one, s.lo);
      s.hi = fma_add(__byte_perm(v, 0u, 0x4341u), one, s.hi);
    }
  }
  return s;
}
// MPAD = 8 over 7-bit (clamped, <= 127) tiles: the eight entries added as
// four byte pair sums (<= 254, no carries), then widened once.
__device__ __forceinline__ Sum4 lut_sum_rot7_8(const uint32_t* rb, const uint32_t* rs, uint32_t w0, uint32_t w1,
                                               uint32_t one) {
  uint32_t v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t a = __byte_perm(j < 4 ? w0 : w1, rb[j & 3], rs[j & 3]);
    if (j < 4) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v[j]) : "r"(a));
    else asm volatile("ld.shared.u32 %0, [%1+65536];" : "=r"(v[j]) : "r"(a));
  }
  const uint32_t p0 = fma_add(v[0], one, v[1]), p1 = fma_add(v[2], one, v[3]);
  const uint32_t p2 = fma_add(v[4], one, v[5]), p3 = fma_add(v[6], one, v[7]);
  Sum4 s;
  s.lo = fma_add(p0 & 0x00FF00FFu, one, p1 & 0x00FF00FFu) + fma_add(p2 & 0x00FF00FFu, one, p3 & 0x00FF00FFu);
  s.hi = fma_add(__byte_perm(p0, 0u, 0x4341u), one, __byte_perm(p1, 0u, 0x4341u)) +
         fma_add(__byte_perm(p2, 0u, 0x4341u), one, __byte_perm(p3, 0u, 0x4341u));
  return s;
}
__device__ __forceinline__ Sum4 lut_sum_rot7(const uint32_t* rb, const uint32_t* rs, uint32_t w, uint32_t one) {
  uint32_t v[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t a = __byte_perm(w, rb[j], rs[j]);
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v[j]) : "r"(a));
  }
  const uint32_t p01 = fma_add(v[0], one, v[1]), p23 = fma_add(v[2], one, v[3]);
  Sum4 s;
  s.lo = fma_add(p01 & 0x00FF00FFu, one, p23 & 0x00FF00FFu);
  s.hi = fma_add(__byte_perm(p01, 0u, 0x4341u), one, __byte_perm(p23, 0u, 0x4341u));
  return s;
}

// 128-bit shared loads of the wide loop (hi: + 64 KB, subspaces 2/3)
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 lds128_hi(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4+65536];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a));
  return v;
}

// Wide loop, one code word w: byte sums of the four subspace entries for
// the lane's 16 queries (4 words x 4 bytes).  b0 = lane base (64-KB aligned
// LUT | chunk part * 16), b1 = b0 + 128 (odd subspaces).
__device__ __forceinline__ void wide_sums(uint32_t w, uint32_t b0, uint32_t b1, uint32_t one, uint32_t t[4]) {
  const uint4 A0 = lds128(__byte_perm(w, b0, 0x7604u));
  const uint4 A1 = lds128(__byte_perm(w, b1, 0x7614u));
  const uint4 A2 = lds128_hi(__byte_perm(w, b0, 0x7624u));
  const uint4 A3 = lds128_hi(__byte_perm(w, b1, 0x7634u));
  t[0] = fma_add(A3.x, one, A0.x + A1.x + A2.x);
  t[1] = fma_add(A3.y, one, A0.y + A1.y + A2.y);
  t[2] = fma_add(A3.z, one, A0.z + A1.z + A2.z);
  t[3] = fma_add(A3.w, one, A0.w + A1.w + A2.w);
}

// per word: bit 7 of byte b clear <=> query b of the word hits
template <int MODE>
__device__ __forceinline__ uint32_t wide_u(uint32_t t, uint32_t c, uint32_t one) {
  if constexpr (MODE == kModeWide5) return t;  // bias folded into the table
  else return t | fma_add(t & 0x7F7F7F7Fu, one, c);
}

// score of lane query qsel (0..3) from the packed sums
__device__ __forceinline__ uint32_t sum_of(Sum4 s, int qsel) {
  const uint32_t w = (qsel & 1) ? s.hi : s.lo;
  return (qsel & 2) ? (w >> 16) : (w & 0xFFFFu);
}

// Histogram counters are u16 pairs inside u32 words; a CTA handles at most
// kHistRowsPerCta rows so no counter can wrap.
constexpr int64_t kHistRowsPerCta = 65535;

template <int MPAD, int NT, int QTX = default_qt(MPAD)>
__global__ void __launch_bounds__(NT, 1)
    k_scan_hist(const uint8_t* __restrict__ plane, int64_t stride, int64_t n_samp,
                int64_t samp_per_cta, const uint8_t* __restrict__ lut,
                const int* __restrict__ tile_list, uint32_t* __restrict__ hist,
                const int64_t* __restrict__ tile_row0, const int64_t* __restrict__ tile_nsamp,
                const int* __restrict__ slot_query) {
  // slot_query (ivf): counts go straight to the histogram row of the slot's
  // query (hist is then [nq][256]) instead of a per-slot row
  using G = ScanGeom<MPAD, QTX>;
  extern __shared__ __align__(16) uint8_t smem[];
  uint8_t* slut = smem;
  uint32_t* sh = reinterpret_cast<uint32_t*>(smem + G::LUT_BYTES);  // [QT][128] u16 pairs
  __shared__ __align__(8) uint64_t lut_bar;
  const int tile = tile_list ? tile_list[blockIdx.y] : blockIdx.y;
  if (threadIdx.x == 0) {  // the 128-KB tile by one TMA bulk copy while the counters are cleared
    mbar_init(&lut_bar, 1);
    mbar_expect_tx(&lut_bar, G::LUT_BYTES);
    bulk_g2s(slut, lut + (int64_t)tile * G::LUT_BYTES, G::LUT_BYTES, &lut_bar);
  }
  for (int i = threadIdx.x; i < G::QT * 128; i += NT) sh[i] = 0;
  __syncthreads();
  mbar_wait(&lut_bar, 0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lic = lane % G::LPC, half = lane / G::LPC;
  const uint8_t* L = slut + lic * 4;
  // rows sampled: row0 + s * stride for s in [0, nsamp) (per tile for ivf lists)
  const int64_t row0 = tile_row0 ? tile_row0[tile] : 0;
  const int64_t nsamp_t = tile_nsamp ? tile_nsamp[tile] : n_samp;
  const int64_t s0 = (int64_t)blockIdx.x * samp_per_cta;
  const int64_t s1 = min(nsamp_t, s0 + samp_per_cta);
  auto bump = [&](int qq, uint32_t score) {
    if (score < 255u) atomicAdd(sh + qq * 128 + (score >> 1), 1u << (16 * (score & 1)));
  };
  for (int64_t g = s0 + (int64_t)warp * 32; g < s1; g += (int64_t)NT) {
    const int64_t my = g + lane;
    uint32_t w0 = 0, w1 = 0;
    if (my < s1) {
      const uint8_t* p = plane + (row0 + my * stride) * MPAD;
      w0 = *reinterpret_cast<const uint32_t*>(p);
      if (MPAD == 8) w1 = *reinterpret_cast<const uint32_t*>(p + 4);
    }
    const int cnt = (int)min((int64_t)32, s1 - g);
    for (int k = 0; k < 32; k += G::CPW) {
      const int src_lane = k + half;
      const uint32_t c0 = __shfl_sync(0xffffffffu, w0, src_lane);
      const uint32_t c1 = __shfl_sync(0xffffffffu, w1, src_lane);
      if (src_lane < cnt) {
        const Sum4 sm = lut_sum<MPAD, QTX>(L, c0, c1);
#pragma unroll
        for (int qs = 0; qs < 4; ++qs) bump(4 * lic + qs, sum_of(sm, qs));
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G::QT * 128; i += NT) {
    const uint32_t v = sh[i];
    const int qq = i / 128, b = (i % 128) * 2;
    if (!v) continue;
    int64_t row = (int64_t)tile * G::QT + qq;
    if (slot_query) {
      row = slot_query[row];
      if (row < 0) continue;  // padding slot
    }
    uint32_t* gh = hist + row * 256;
    if (v & 0xFFFFu) atomicAdd(gh + b, v & 0xFFFFu);
    if (v >> 16) atomicAdd(gh + b + 1, v >> 16);
  }
}

// ============================================================================
// K2b: the first-pass scan.  One CTA holds the 8-bit tables of QT queries in
// shared memory (128 KB) and streams a contiguous range of code rows:
// each warp pulls 512-B chunks of the low-byte plane with 128-bit
// non-allocating loads (double-buffered through registers), re-reads them as
// warp-uniform 128-bit shared loads, and every lane sums the table entries of
// its four queries for each row with MPAD conflict-free 32-bit LDS (one row
// of one table = one 128-B line read by the 32 lanes), split into two u16x2
// accumulators (queries 0,2 and 1,3) that never carry (sum <= 8*255 < 2^15).
// A row is emitted for a query iff its raw sum <= guard (then score = raw
// sum < 255), tested with one subtract per accumulator:
//   G = (0x8000 + B0) | (0x8000 + B2) << 16;  hit = bit 15 / 31 of (G - s).
// ============================================================================
struct EmitArgs {
  const uint8_t* plane;
  int64_t row_begin, row_end;   // scanned rows [row_begin, row_end)
  int64_t rows_per_cta;
  const uint8_t* lut;
  const uint16_t* gword;        // [tiles*QT] guard words (0x8000+B or 0x7F7F)
  const int* tile_list;         // optional blockIdx.y -> tile
  const int* slot_query;        // optional slot -> emit list (ivf); else slot
  const int* slot_probe;        // optional slot -> probe index (ivf)
  uint32_t* emit_cnt;
  uint64_t* emit;
  uint32_t cap;
  unsigned* unit_counter;       // zeroed before launch (persistent scheduling)
  const int* unit_tile;         // optional per-unit tile (ivf); else u / units_per_tile
  const int* n_units_dev = nullptr;  // optional: the unit count in device memory (device-built ivf plan)
  const int64_t* unit_r0;       // optional per-unit row range (ivf)
  const int64_t* unit_r1;
  uint32_t one;                 // = 1 (opaque to the compiler, see fma_add)
  const int* tile_fast = nullptr;  // optional per-tile mode (kMode*, see k_build_lut)
  unsigned long long* n_wide = nullptr;  // optional: units scanned by the wide loop
  int runs = 0;                 // rows sorted by (subspace 0, 1) low bytes: reuse their sums
  const int* chunk_list = nullptr;  // optional per-tile lists of 128-row chunks to scan (run filter)
  const int* list_len = nullptr;    //   [tiles] list lengths (device); list of tile t at t * list_stride
  const int* list_next = nullptr;   //   [tiles] chunks handed out so far (zeroed before the launch)
  int64_t list_stride = 0;
  int n_units;                  // tiles * units_per_tile
  int units_per_tile;
  int emit32 = 0;               // 4-byte records (pack_emit32) instead of pack_emit
  unsigned long long* n_lut = nullptr;  // optional: LUT tile loads (bulk copies of G::LUT_BYTES)
  const int* live = nullptr;    // optional: queries left to this scan (0: every query took the direct scan)
};

// Persistent scan.  Work unit = (query tile, contiguous row range); CTAs
// (one per SM, 32 warps) pull units from a global counter, so the grid never
// has a partial last wave.  Per unit the CTA loads the tile's 8-bit tables
// (128 KB) into shared memory once and its warps stream the unit's rows.
//
// Hit staging: a warp appends the rows that pass a guard to a private
// shared-memory buffer (positions from ballot/popc, no atomics) and flushes
// it when it may overflow or at the end of the unit: per-query counts in
// shared memory, ONE global atomicAdd per query present in the buffer to
// reserve space in that query's emit list, then the stores.  The common path
// is 4 LDS + ~11 ALU per code and one warp vote per 4 codes.
constexpr int kWarpBuf = 256;  // staged hits per warp (1 KB of 4-byte entries, flushed at least once per chunk)
constexpr uint32_t kLutShared = 0x10000;  // LUT at shared address 64 KB

// Shared layout: [stage | hit buffers] below 64 KB, LUT in [64 KB, 192 KB),
// per-warp hit counters above it.
template <int MPAD, int NT>
__host__ __device__ constexpr int emit_low_bytes() { return (NT / 32) * (32 * 16 + kWarpBuf * 4); }
// (QT-independent)
constexpr int kLaneQ = 8;  // lane-private hit records per chunk (u16 each)
template <int MPAD, int NT, int QTX = default_qt(MPAD)>
__host__ __device__ constexpr int emit_smem_bytes() {
  return (int)kLutShared + ScanGeom<MPAD, QTX>::LUT_BYTES + (NT / 32) * ScanGeom<MPAD, QTX>::QT * 4 +
         (NT / 32) * kLaneQ * 32 * 2;
}

template <int MPAD, int NT, int QTX = default_qt(MPAD)>
__global__ void __launch_bounds__(NT, 1) k_scan_emit(EmitArgs a) {
  using G = ScanGeom<MPAD, QTX>;
  constexpr int NW = NT / 32;
  if (a.live && *a.live == 0) return;
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ int s_unit;
  __shared__ int s_next;  // unit mode: the unit's next unclaimed chunk (warps balance within a unit)
  __shared__ __align__(8) uint64_t lut_bar;  // completion of the LUT bulk copy
  uint32_t lut_phase = 0;
  const uint32_t dyn = (uint32_t)__cvta_generic_to_shared(smem);
  if (dyn + emit_low_bytes<MPAD, NT>() > kLutShared) __trap();  // layout invariant
  if (threadIdx.x == 0) mbar_init(&lut_bar, 1);
  uint8_t* slut = smem + (kLutShared - dyn);
  uint4* stage = reinterpret_cast<uint4*>(smem);
  uint32_t* hbuf_all = reinterpret_cast<uint32_t*>(smem + NW * 32 * 16);
  uint32_t* hcnt_all = reinterpret_cast<uint32_t*>(slut + G::LUT_BYTES);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lic = lane % G::LPC, half = lane / G::LPC;
  const uint32_t lbase = kLutShared | (uint32_t)(lic * 4);
  uint32_t rot_b[4], rot_s[4];  // CPW = 2: rotated subspace order of this half-warp (lut_sum_rot)
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int jr = (j + (G::CPW == 2 ? half : 0)) & 3;
    rot_b[j] = lbase + (uint32_t)((jr % G::SPR) * G::ROWB);
    rot_s[j] = 0x7604u | ((uint32_t)jr << 4);
  }
  uint4* wst = stage + warp * 32;
  uint32_t* hbuf = hbuf_all + warp * kWarpBuf;
  uint32_t* hcnt = hcnt_all + warp * G::QT;
  uint16_t* lq = reinterpret_cast<uint16_t*>(hcnt_all + NW * G::QT) + warp * kLaneQ * 32 + lane;
  uint16_t* cq = reinterpret_cast<uint16_t*>(hcnt_all + NW * G::QT) + warp * kLaneQ * 32;  // wide drain (128)
  const uint32_t lt = (1u << lane) - 1u;
  const uint32_t one = a.one, mone = 0u - a.one;  // opaque 1 / -1 (see fma_add)
  auto lut_sum_any = [&](uint32_t w0, uint32_t w1) -> Sum4 {  // the lane's sums of one code (any geometry)
    if constexpr (G::CPW == 2) return lut_sum_rot<MPAD>(rot_b, rot_s, w0, w1, one);
    else return lut_sum_fast<MPAD, QTX>(lbase, w0, w1, one);
  };
  int cur_tile = -1;
  bool first_unit = true;
  for (;;) {
    __syncthreads();  // previous unit finished by every warp
    if (threadIdx.x == 0) {
      if (a.chunk_list) {
        // list mode, dynamic: start on a tile in proportion to the list
        // lengths, then move to the tile with the most chunks left
        int nt = a.n_units, pick = -1;
        if (first_unit) {
          int64_t tot = 0;
          for (int t = 0; t < nt; ++t) tot += a.list_len[t];
          const int64_t target = (int64_t)blockIdx.x * tot / gridDim.x;
          int64_t cum = 0;
          for (int t = 0; t < nt && pick < 0; ++t) {
            cum += a.list_len[t];
            if (cum > target) pick = t;
          }
        } else {
          int best = 0;
          for (int t = 0; t < nt; ++t) {
            const int left = a.list_len[t] - *((volatile int*)a.list_next + t);
            if (left > best) { best = left; pick = t; }
          }
        }
        s_unit = pick;
      } else {
        s_unit = (int)atomicAdd(a.unit_counter, 1u);
        s_next = NW;  // chunks 0 .. NW-1 go to warps 0 .. NW-1
      }
    }
    __syncthreads();
    first_unit = false;
    const int u = s_unit;
    if (a.chunk_list ? u < 0 : u >= (a.n_units_dev ? *a.n_units_dev : a.n_units)) break;
    int tile;
    int64_t r0, r1;
    if (a.chunk_list) {
      tile = u;
      r0 = 0;
      r1 = a.list_len[tile];
    } else if (a.unit_tile) {
      tile = a.unit_tile[u];
      r0 = a.unit_r0[u];
      r1 = a.unit_r1[u];
    } else {
      // tile-minor order: CTAs running at the same time cover all tiles of
      // the same rows (plane rows re-read from L2, emit counters of every
      // query tile shared out instead of one tile's at a time)
      const int ntl = a.n_units / a.units_per_tile;
      const int tix = u % ntl;
      const int64_t chunk_u = u / ntl;
      tile = a.tile_list ? a.tile_list[tix] : tix;
      r0 = a.row_begin + chunk_u * a.rows_per_cta;
      r1 = min(a.row_end, r0 + a.rows_per_cta);
    }
    if (tile != cur_tile) {
      // every warp is past the previous unit (barrier above): one thread
      // moves the 128-KB tile with a TMA bulk copy, all wait on the mbarrier
      if (threadIdx.x == 0) {
        if (a.n_lut) atomicAdd(a.n_lut, 1ull);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&lut_bar, G::LUT_BYTES);
        bulk_g2s(slut, a.lut + (int64_t)tile * G::LUT_BYTES, G::LUT_BYTES, &lut_bar);
      }
      // warp 0 reconverges before spinning: lanes 1-31 polling the barrier
      // must not be scheduled ahead of lane 0's copy issue (a layout-dependent
      // hang otherwise, seen on m = 1 models)
      __syncwarp();
      mbar_wait(&lut_bar, lut_phase);
      lut_phase ^= 1u;
      cur_tile = tile;
    }
    const int tmode = a.tile_fast != nullptr ? a.tile_fast[tile] : kModeGeneric;
    const bool fast_tile = tmode == kMode7;
    const bool wide = MPAD == 4 && G::QT == 128 && (tmode == kModeWide5 || tmode == kModeWide6);
    const int q0 = tile * G::QT + 4 * lic;
    const uint32_t glo = (uint32_t)a.gword[q0] | ((uint32_t)a.gword[q0 + 2] << 16);
    const uint32_t ghi = (uint32_t)a.gword[q0 + 1] | ((uint32_t)a.gword[q0 + 3] << 16);
    // wide loop: lane = (quarter qd: code stream, part cp: queries 16cp..16cp+15)
    const int qd = lane >> 3, cp = lane & 7;
    const uint32_t wb0 = kLutShared | (uint32_t)(cp << 4), wb1 = wb0 + 128u;
    uint32_t cw0 = 0, cw1 = 0, cw2 = 0, cw3 = 0;  // per-query bias C, word k byte b = query 16cp+4k+b
    uint32_t kprev = 0x10000u, bs0 = 0, bs1 = 0, bs2 = 0, bs3 = 0;  // run state (sorted rows): key, 0+1 sums
    if (wide) {
      if (a.n_wide && threadIdx.x == 0) atomicAdd(a.n_wide, 1ull);
      const uint16_t* gq = a.gword + tile * G::QT + 16 * cp;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        cw0 |= wide_bias(gq[b]) << (8 * b);
        cw1 |= wide_bias(gq[4 + b]) << (8 * b);
        cw2 |= wide_bias(gq[8 + b]) << (8 * b);
        cw3 |= wide_bias(gq[12 + b]) << (8 * b);
      }
    }
    // Logical range [r0, r1); loads start at the 512-B aligned row r0a and
    // rows outside the range are never emitted.
    if (r0 >= r1) continue;
    // list mode: [r0, r1) indexes the tile's chunk list, rows are absolute
    const int* clist = a.chunk_list ? a.chunk_list + tile * a.list_stride : nullptr;
    const int64_t r0a = clist ? 0 : (r0 & ~(int64_t)(G::CHUNK_ROWS - 1));
    const int64_t nchunks = clist ? r1 - r0 : (r1 - r0a + G::CHUNK_ROWS - 1) / G::CHUNK_ROWS;
    if (clist) { r0 = a.row_begin; r1 = a.row_end; }
    // next chunk of this warp: strided, or (list mode) pulled from the
    // tile's global counter so chunks of uneven cost balance across warps/CTAs
    auto next_chunk = [&](int64_t cprev) -> int64_t {
      int v = 0;
      if (!clist) {  // unit mode: claimed from the CTA's shared counter
        if (lane == 0) v = atomicAdd(&s_next, 1);
        return (int64_t)__shfl_sync(0xffffffffu, v, 0);
      }
      if (lane == 0) v = atomicAdd(const_cast<int*>(a.list_next) + tile, 1);
      return (int64_t)__shfl_sync(0xffffffffu, v, 0);
    };
    int64_t c = clist ? next_chunk(0) : warp;
    if (c >= nchunks) continue;
    int wc = 0;  // staged hits (warp-uniform)
    auto chunk_row = [&](int64_t ci) -> int64_t {
      return clist ? (int64_t)clist[ci] * G::CHUNK_ROWS : r0a + ci * G::CHUNK_ROWS;
    };
    auto chunk_ptr = [&](int64_t ci) {
      return reinterpret_cast<const uint4*>(a.plane + chunk_row(ci) * MPAD) + lane;
    };
    // entry (4 B): row in the current chunk (7 b) | local slot << 7 | score << 14;
    // the buffer is flushed before the chunk changes (cur_rb = the chunk's first row)
    int64_t cur_rb = 0;
    auto flush = [&]() {
      for (int s = lane; s < G::QT; s += 32) hcnt[s] = 0;
      __syncwarp();
      for (int i = lane; i < wc; i += 32) atomicAdd(hcnt + ((hbuf[i] >> 7) & 0x7F), 1u);
      __syncwarp();
      {  // per-query reservations: all of the lane's atomics in flight at once
        constexpr int SL = G::QT / 32;
        uint32_t base[SL];
#pragma unroll
        for (int k = 0; k < SL; ++k) {
          const int s = lane + 32 * k;
          const uint32_t n = hcnt[s];
          base[k] = 0u;
          if (n) {
            const int slot = tile * G::QT + s;
            const int qe = a.slot_query ? a.slot_query[slot] : slot;
            base[k] = atomicAdd(a.emit_cnt + qe, n);
          }
        }
#pragma unroll
        for (int k = 0; k < SL; ++k) hcnt[lane + 32 * k] = base[k];
      }
      __syncwarp();
      for (int i = lane; i < wc; i += 32) {
        const uint32_t e = hbuf[i];
        const int s = (int)((e >> 7) & 0x7F);
        const uint32_t pos = atomicAdd(hcnt + s, 1u);
        const int slot = tile * G::QT + s;
        const int qe = a.slot_query ? a.slot_query[slot] : slot;
        const uint32_t probe = a.slot_probe ? (uint32_t)a.slot_probe[slot] : 0u;
        if (pos < a.cap) {
          if (a.emit32)
            reinterpret_cast<uint32_t*>(a.emit)[(int64_t)qe * a.cap + pos] =
                pack_emit32(cur_rb + (int64_t)(e & 0x7F), e >> 14);
          else
            a.emit[(int64_t)qe * a.cap + pos] = pack_emit(cur_rb + (int64_t)(e & 0x7F), probe, e >> 14);
        }
      }
      __syncwarp();
      wc = 0;
    };
    // Stage hits.  hm bit 4k+qs = hit of lane query qs on code k (row
    // offset roff0 + k from r0a).  One ballot round per hit per lane.
    auto stage_hits = [&](uint32_t hm, Sum4 sa, Sum4 sb, Sum4 sc2, Sum4 sd, uint32_t roff0) {
      for (;;) {
        const bool has = hm != 0u;
        const uint32_t bal = __ballot_sync(0xffffffffu, has);
        if (!bal) break;
        if (wc + 32 > kWarpBuf) flush();
        if (has) {
          const int b = __ffs(hm) - 1;
          hm &= hm - 1u;
          const int k = b >> 2, qs = b & 3;
          const Sum4 sk = k == 0 ? sa : (k == 1 ? sb : (k == 2 ? sc2 : sd));
          hbuf[wc + __popc(bal & lt)] = (roff0 + k) | ((uint32_t)(4 * lic + qs) << 7) | (sum_of(sk, qs) << 14);
        }
        wc += __popc(bal);
      }
    };
    // hit bits of one code from (guard - sum): qs0 lo.15, qs1 hi.15, qs2 lo.31, qs3 hi.31
    auto bits_x = [](uint32_t xl, uint32_t xh) -> uint32_t {
      return ((xl >> 15) & 1u) | ((xh >> 14) & 2u) | ((xl >> 29) & 4u) | ((xh >> 28) & 8u);
    };
    // The (rare) hit path of the inner loop only appends a 16-bit record
    // (i, code, query) to a lane-private shared queue; the records are
    // turned into emit entries once per 128-code chunk (drain below).
    int lcnt = 0;
    auto record = [&](uint32_t xl, uint32_t xh, int i, int k) {
      uint32_t hm = bits_x(xl, xh);
      do {
        const int qs = __ffs(hm) - 1;
        hm &= hm - 1u;
        if (lcnt < kLaneQ) lq[lcnt * 32] = (uint16_t)((i << 4) | (k << 2) | qs);
        ++lcnt;
      } while (hm);
    };
    uint4 nxt = ldg_stream(chunk_ptr(c));
    int64_t cn = c;
    for (; c < nchunks; c = cn) {
      __syncwarp();
      wst[lane] = nxt;
      __syncwarp();
      cn = next_chunk(c);
      if (cn < nchunks) nxt = ldg_stream(chunk_ptr(cn));
      const int64_t rb = chunk_row(c);
      // rows of this chunk outside [r0, r1) only at the unit's two ends
      const bool edge = rb < r0 || rb + G::CHUNK_ROWS > r1;
      const uint32_t lo = edge ? (uint32_t)max((int64_t)0, r0 - rb) : 0u;
      const uint32_t hi = edge ? (uint32_t)min((int64_t)G::CHUNK_ROWS, r1 - rb) : (uint32_t)G::CHUNK_ROWS;
      cur_rb = rb;
      if constexpr (MPAD == 4 && G::QT == 128) {
        if (wide) {
          // Wide loop: quarter qd scans rows 32qd .. 32qd+31 of the chunk,
          // one row per step; each lane sums its 16 queries with 4 x LDS.128
          // (4 codes per warp step, conflict-free: the 8 lanes of a quarter
          // read the 8 16-B parts of one 128-B table row).  A step with a hit
          // only appends its step index to a lane-private u8 queue.
          auto wide_chunk = [&](auto md, auto rn) {
            constexpr int MODE = decltype(md)::value;
            const uint32_t* wsw = reinterpret_cast<const uint32_t*>(wst);
            constexpr bool RUNS = decltype(rn)::value;
            uint32_t smask = 0u;  // bit i: step i had a hit (lane-private, never overflows)
#pragma unroll 2
            for (int i4 = 0; i4 < 8; ++i4) {
              const uint4 cv = wst[qd * 8 + i4];
              const uint32_t cws[4] = {cv.x, cv.y, cv.z, cv.w};
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                uint32_t t[4];
                if constexpr (RUNS) {
                  // sorted rows: subspace 0/1 part reloaded only when the
                  // (g0, g1) key of the quarter's row changes
                  const uint32_t w = cws[u];
                  if ((w & 0xFFFFu) != kprev) {
                    const uint4 A0 = lds128(__byte_perm(w, wb0, 0x7604u));
                    const uint4 A1 = lds128(__byte_perm(w, wb1, 0x7614u));
                    bs0 = A0.x + A1.x; bs1 = A0.y + A1.y; bs2 = A0.z + A1.z; bs3 = A0.w + A1.w;
                    kprev = w & 0xFFFFu;
                  }
                  const uint4 A2 = lds128_hi(__byte_perm(w, wb0, 0x7624u));
                  const uint4 A3 = lds128_hi(__byte_perm(w, wb1, 0x7634u));
                  t[0] = bs0 + A2.x + A3.x; t[1] = bs1 + A2.y + A3.y;
                  t[2] = bs2 + A2.z + A3.z; t[3] = bs3 + A2.w + A3.w;
                } else {
                  wide_sums(cws[u], wb0, wb1, one, t);
                }
                const uint32_t all = wide_u<MODE>(t[0], cw0, one) & wide_u<MODE>(t[1], cw1, one) &
                                     wide_u<MODE>(t[2], cw2, one) & wide_u<MODE>(t[3], cw3, one);
                smask |= (uint32_t)((~all & 0x80808080u) != 0u) << (4 * i4 + u);
              }
            }
            if (!__any_sync(0xffffffffu, smask != 0u)) return;
            // Drain: the warp's (lane, step) records are compacted (up to 4
            // per lane per pass, <= 128 per pass) and spread over the lanes;
            // each recomputes its step's sums for the recording lane's 16
            // queries and stages the hits.
            const uint32_t cwk[4] = {cw0, cw1, cw2, cw3};
            for (;;) {
              // up to kLaneQ records per lane per pass (the cq capacity is kLaneQ * 32);
              // usually every record of the chunk goes in one pass
              uint32_t sel = smask, rest = 0u;
              if (__popc(smask) > kLaneQ) {
                sel = 0u;
                rest = smask;
#pragma unroll
                for (int k = 0; k < kLaneQ; ++k) { const uint32_t bit = rest & (0u - rest); sel |= bit; rest ^= bit; }
              }
              const int nsel = __popc(sel);
              int off = nsel;  // inclusive scan over lanes
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, off, o);
                if (lane >= o) off += v;
              }
              const int total = __shfl_sync(0xffffffffu, off, 31);
              if (total == 0) break;
              off -= nsel;
              for (uint32_t tt = sel; tt; tt &= tt - 1u) cq[off++] = (uint16_t)((lane << 5) | (__ffs(tt) - 1));
              smask = rest;
              __syncwarp();
              for (int base = 0; base < total; base += 32) {
                const bool has = base + lane < total;
                const uint32_t rec = has ? cq[base + lane] : 0u;
                const int src = (int)(rec >> 5), i = (int)(rec & 31u);
                const int sq = src >> 3, sp = src & 7;
                uint32_t c4[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) c4[k] = __shfl_sync(0xffffffffu, cwk[k], src);
                uint32_t hm = 0u, t[4] = {0u, 0u, 0u, 0u};
                const uint32_t r = 32u * (uint32_t)sq + (uint32_t)i;
                if (has) {
                  const uint32_t sb0 = kLutShared | (uint32_t)(sp << 4);
                  wide_sums(wsw[32 * sq + i], sb0, sb0 + 128u, one, t);
#pragma unroll
                  for (int k = 0; k < 4; ++k) {
                    const uint32_t hb = ~wide_u<MODE>(t[k], c4[k], one) & 0x80808080u;
                    // bits 7, 15, 23, 31 -> 28..31 in one multiply (the shifted copies never overlap)
                    hm |= ((hb * 0x00204081u) >> 28) << (4 * k);
                  }
                  if (edge && !(r >= lo && r < hi)) hm = 0u;
                }
                // stage: one warp prefix sum, then every lane writes its hits
                const int nh = __popc(hm);
                int incl = nh;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                  const int v = __shfl_up_sync(0xffffffffu, incl, o);
                  if (lane >= o) incl += v;
                }
                const int tot = __shfl_sync(0xffffffffu, incl, 31);
                if (tot > 0) {
                  if (wc + tot > kWarpBuf) flush();
                  int o = wc + incl - nh;
                  const int lim = min(kWarpBuf, wc + tot);  // (tot > kWarpBuf: rest below)
                  uint32_t hr = hm;
                  while (hr && o < lim) {
                    const int b = __ffs(hr) - 1;
                    hr &= hr - 1u;
                    const int k = b >> 2, sh = 8 * (b & 3);
                    const uint32_t tw = k == 0 ? t[0] : (k == 1 ? t[1] : (k == 2 ? t[2] : t[3]));
                    uint32_t sc = (tw >> sh) & 0xFFu;
                    if (MODE == kModeWide5) {
                      const uint32_t ck = k == 0 ? c4[0] : (k == 1 ? c4[1] : (k == 2 ? c4[2] : c4[3]));
                      sc -= (ck >> sh) & 0xFFu;
                    }
                    hbuf[o++] = r | ((uint32_t)(16 * sp + b) << 7) | (sc << 14);
                  }
                  wc = lim;
                  // more hits than one buffer holds (<= 512): the rest, one ballot round each
                  for (;;) {
                    const bool hh = hr != 0u;
                    const uint32_t bal = __ballot_sync(0xffffffffu, hh);
                    if (!bal) break;
                    if (wc + 32 > kWarpBuf) flush();
                    if (hh) {
                      const int b = __ffs(hr) - 1;
                      hr &= hr - 1u;
                      const int k = b >> 2, sh = 8 * (b & 3);
                      const uint32_t tw = k == 0 ? t[0] : (k == 1 ? t[1] : (k == 2 ? t[2] : t[3]));
                      uint32_t sc = (tw >> sh) & 0xFFu;
                      if (MODE == kModeWide5) {
                        const uint32_t ck = k == 0 ? c4[0] : (k == 1 ? c4[1] : (k == 2 ? c4[2] : c4[3]));
                        sc -= (ck >> sh) & 0xFFu;
                      }
                      hbuf[wc + __popc(bal & lt)] = r | ((uint32_t)(16 * sp + b) << 7) | (sc << 14);
                    }
                    wc += __popc(bal);
                  }
                }
              }
              __syncwarp();
            }
          };
          if (a.runs) {
            if (tmode == kModeWide5) wide_chunk(std::integral_constant<int, kModeWide5>(), std::true_type());
            else wide_chunk(std::integral_constant<int, kModeWide6>(), std::true_type());
          } else {
            if (tmode == kModeWide5) wide_chunk(std::integral_constant<int, kModeWide5>(), std::false_type());
            else wide_chunk(std::integral_constant<int, kModeWide6>(), std::false_type());
          }
          if (wc > 0) flush();  // entries are chunk-relative
          continue;
        }
      }
      // the lane's code k (< G::CPL) of the 16-B plane group v and its row in the chunk:
      // (4, 128) all lanes read the group's 4 codes; (4, 64) half-warps read 2 codes each;
      // MPAD = 8 half-warps read one 8-byte code each
      auto wsel = [&](const uint4 v, int k, uint32_t& w0, uint32_t& w1) {
        if constexpr (MPAD == 8) {
          w0 = half ? v.z : v.x;
          w1 = half ? v.w : v.y;
        } else {
          const int c = half * G::CPL + k;
          w0 = c == 0 ? v.x : (c == 1 ? v.y : (c == 2 ? v.z : v.w));
          w1 = 0u;
        }
      };
      auto rowof = [&](int i, int k) -> uint32_t { return (uint32_t)((16 / MPAD) * i + half * G::CPL + k); };
      auto group4 = [&](const uint4 v, int i, auto fast7) {
        Sum4 s0, s1, s2, s3;
        if constexpr (decltype(fast7)::value) {
          s0 = lut_sum_fast7<QTX>(lbase, v.x, one); s1 = lut_sum_fast7<QTX>(lbase, v.y, one);
          s2 = lut_sum_fast7<QTX>(lbase, v.z, one); s3 = lut_sum_fast7<QTX>(lbase, v.w, one);
        } else {
          s0 = lut_sum_fast<MPAD, QTX>(lbase, v.x, 0, one); s1 = lut_sum_fast<MPAD, QTX>(lbase, v.y, 0, one);
          s2 = lut_sum_fast<MPAD, QTX>(lbase, v.z, 0, one); s3 = lut_sum_fast<MPAD, QTX>(lbase, v.w, 0, one);
        }
        const uint32_t xl0 = fma_add(s0.lo, mone, glo), xh0 = fma_add(s0.hi, mone, ghi);
        const uint32_t xl1 = fma_add(s1.lo, mone, glo), xh1 = fma_add(s1.hi, mone, ghi);
        const uint32_t xl2 = fma_add(s2.lo, mone, glo), xh2 = fma_add(s2.hi, mone, ghi);
        const uint32_t xl3 = fma_add(s3.lo, mone, glo), xh3 = fma_add(s3.hi, mone, ghi);
        if ((xl0 | xh0) & 0x80008000u) record(xl0, xh0, i, 0);
        if ((xl1 | xh1) & 0x80008000u) record(xl1, xh1, i, 1);
        if ((xl2 | xh2) & 0x80008000u) record(xl2, xh2, i, 2);
        if ((xl3 | xh3) & 0x80008000u) record(xl3, xh3, i, 3);
      };
      auto group2 = [&](const uint4 v, int i, auto fast7) {  // (4, 64): this half-warp's two codes
        const uint32_t wa = half ? v.z : v.x, wb = half ? v.w : v.y;
        Sum4 s0, s1;
        if constexpr (decltype(fast7)::value) {
          s0 = lut_sum_rot7(rot_b, rot_s, wa, one); s1 = lut_sum_rot7(rot_b, rot_s, wb, one);
        } else {
          s0 = lut_sum_rot<MPAD>(rot_b, rot_s, wa, 0, one); s1 = lut_sum_rot<MPAD>(rot_b, rot_s, wb, 0, one);
        }
        const uint32_t xl0 = fma_add(s0.lo, mone, glo), xh0 = fma_add(s0.hi, mone, ghi);
        const uint32_t xl1 = fma_add(s1.lo, mone, glo), xh1 = fma_add(s1.hi, mone, ghi);
        if ((xl0 | xh0) & 0x80008000u) record(xl0, xh0, i, 0);
        if ((xl1 | xh1) & 0x80008000u) record(xl1, xh1, i, 1);
      };
      if constexpr (MPAD == 4 && G::CPL == 4) {
        if (fast_tile) {
#pragma unroll 2
          for (int i = 0; i < 32; ++i) group4(wst[i], i, std::integral_constant<bool, true>());
        } else {
#pragma unroll 2
          for (int i = 0; i < 32; ++i) group4(wst[i], i, std::integral_constant<bool, false>());
        }
      } else if constexpr (MPAD == 4) {
        if (fast_tile) {
#pragma unroll 2
          for (int i = 0; i < 32; ++i) group2(wst[i], i, std::integral_constant<bool, true>());
        } else {
#pragma unroll 2
          for (int i = 0; i < 32; ++i) group2(wst[i], i, std::integral_constant<bool, false>());
        }
      } else {
        auto group1 = [&](const uint4 v, int i, auto fast7) {  // MPAD = 8: this half-warp's code
          uint32_t w0, w1;
          wsel(v, 0, w0, w1);
          Sum4 s0;
          if constexpr (decltype(fast7)::value) s0 = lut_sum_rot7_8(rot_b, rot_s, w0, w1, one);
          else s0 = lut_sum_any(w0, w1);
          const uint32_t xl0 = fma_add(s0.lo, mone, glo), xh0 = fma_add(s0.hi, mone, ghi);
          if ((xl0 | xh0) & 0x80008000u) record(xl0, xh0, i, 0);
        };
        if (G::CPW == 2 && fast_tile) {
#pragma unroll 2
          for (int i = 0; i < 32; ++i) group1(wst[i], i, std::integral_constant<bool, true>());
        } else {
#pragma unroll 2
          for (int i = 0; i < 32; ++i) group1(wst[i], i, std::integral_constant<bool, false>());
        }
      }
      // drain: records -> emit entries (scores recomputed from the staged codes)
      if (__any_sync(0xffffffffu, lcnt > 0)) {
        if (__any_sync(0xffffffffu, lcnt > kLaneQ)) {
          // a lane overflowed its queue (degenerate data): redo the whole
          // chunk with warp-wide staging (exact, just slower)
          for (int i = 0; i < 32; ++i) {
            const uint4 v = wst[i];
            for (int k = 0; k < G::CPL; ++k) {
              uint32_t w0, w1;
              wsel(v, k, w0, w1);
              const uint32_t r = rowof(i, k);
              const Sum4 sm = lut_sum_any(w0, w1);
              uint32_t hm = bits_x(glo - sm.lo, ghi - sm.hi);
              if (edge && !(r >= lo && r < hi)) hm = 0u;
              stage_hits(hm, sm, sm, sm, sm, r);
            }
          }
        } else {
          const int maxc = __reduce_max_sync(0xffffffffu, (unsigned)lcnt);
          for (int e = 0; e < maxc; ++e) {
            bool has = e < lcnt;
            uint32_t sc = 0, roff = 0, slot = 0;
            if (has) {
              const uint32_t rec = lq[e * 32];
              const int i = (int)(rec >> 4), k = (int)((rec >> 2) & 3), qs = (int)(rec & 3);
              uint32_t w0, w1;
              wsel(wst[i], k, w0, w1);
              const uint32_t r = rowof(i, k);
              has = !edge || (r >= lo && r < hi);
              sc = sum_of(lut_sum_any(w0, w1), qs);
              roff = r;
              slot = 4 * lic + qs;
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, has);
            if (wc + 32 > kWarpBuf) flush();
            if (has) hbuf[wc + __popc(bal & lt)] = roff | (slot << 7) | (sc << 14);
            wc += __popc(bal);
          }
        }
        lcnt = 0;
      }
      if (wc > 0) flush();  // entries are chunk-relative
    }
    if (wc > 0) flush();
  }
}

// ============================================================================
// Guard selection from (sample or exact) histograms.  One thread per slot.
//   exact: B = min{b <= 254 : cum[b] >= r2}, else 254  (the true b*)
//   sample of S rows out of N: lambda = r2*S/N expected sample hits below
//   b*; B = min{b : cum_s[b] >= lambda + 3 sqrt(lambda) + 4}, else 254.
// A guard that proves too tight is detected by K3 and redone exactly.
// ============================================================================
constexpr int kGuardSlotsPerCta = 4;  // k_guard: one warp per slot
__global__ void __launch_bounds__(32 * kGuardSlotsPerCta)
    k_guard(const uint32_t* __restrict__ hist, int nslot, int r2, double lambda, int exact,
            const uint8_t* __restrict__ only, uint16_t* __restrict__ guard_b, uint16_t* __restrict__ gword,
            const double* __restrict__ lambda_s) {
  // lane l holds bins 8l .. 8l+7: lane-local running sums, a warp scan of
  // the lane totals, then the first bin whose cumulative count reaches the
  // target (bin 255 never counts: B <= 254) — guard_of_hist
  const int s = blockIdx.x * kGuardSlotsPerCta + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (s >= nslot) return;
  if (only && !only[s]) return;
  const double lam = lambda_s ? lambda_s[s] : lambda;
  const int B = guard_of_hist(hist + (int64_t)s * 256, lane, r2, lam, exact || lam < 0.0);  // lambda < 0: exact histogram
  if (lane == 0) {
    guard_b[s] = (uint16_t)B;
    gword[s] = (uint16_t)(0x8000 + B);
  }
}

// ============================================================================
// K3: b* per query from the emitted scores (every emitted score <= guard, so
// the histogram below the guard is exact).  flags: 1 = guard too tight
// (cum[guard] < r2 with guard < 254: redo with the exact histogram),
// 2 = emit buffer overflow.  When hist_out is given (sharded search) the
// local histogram is exported instead and b* is decided after the
// all-reduce.
// ============================================================================
template <int NT>
__global__ void __launch_bounds__(NT)
    k_threshold(const uint64_t* __restrict__ emit, const uint32_t* __restrict__ emit_cnt,
                uint32_t cap, const uint16_t* __restrict__ guard_b, int r2,
                const uint8_t* __restrict__ only, int32_t* __restrict__ bstar,
                int64_t* __restrict__ ncand, uint8_t* __restrict__ flags,
                int32_t* __restrict__ hist_out, unsigned long long* __restrict__ n_emitted, int emit32,
                const uint32_t* __restrict__ scan_hist = nullptr,
                const uint16_t* __restrict__ direct_gword = nullptr) {
  // per-warp sub-histograms (scores cluster in a few bins: 8x less shared
  // atomic contention), emit lists read with 16-byte loads, two in flight
  constexpr int NW = NT / 32;
  __shared__ uint32_t hw[NW][256];
  __shared__ uint32_t h[256];
  const int q = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  if (only && !only[q]) return;
  const uint32_t n = emit_cnt[q];
  if (n > cap) {
    if (tid == 0) { flags[q] = 2; bstar[q] = -1; }  // (-1: refine nothing until redone)
    if (hist_out)  // sharded: this shard's histogram is unknown, export zeros (the query is redone)
      for (int i = tid; i < 256; i += NT) hist_out[(int64_t)q * 256 + i] = 0;
    return;
  }
  if (n_emitted && tid == 0) atomicAdd(n_emitted, (unsigned long long)n);
  // the direct scan counted its hits by score (DirectArgs::hist): no pass over the emit list of a
  // query it scanned (all of them, or with direct_gword those k_key_select marked 0x7F7F)
  if (scan_hist && (!direct_gword || direct_gword[q] == (uint16_t)0x7F7Fu)) {
    for (int b = tid; b < 256; b += NT) h[b] = scan_hist[(int64_t)q * 256 + b];
  } else {
  for (int i = tid; i < NW * 256; i += NT) (&hw[0][0])[i] = 0;
  __syncthreads();
  uint32_t* hm = hw[tid >> 5];
  if (emit32) {
    const uint32_t* e = reinterpret_cast<const uint32_t*>(emit) + (int64_t)q * cap;
    uint32_t done = 0;
    if ((reinterpret_cast<uintptr_t>(e) & 15) == 0) {
      const uint4* e4 = reinterpret_cast<const uint4*>(e);
      const uint32_t n4 = n / 4;
      auto add4 = [&](uint4 v) {
        atomicAdd(hm + (v.x >> kRow32Bits), 1u); atomicAdd(hm + (v.y >> kRow32Bits), 1u);
        atomicAdd(hm + (v.z >> kRow32Bits), 1u); atomicAdd(hm + (v.w >> kRow32Bits), 1u);
      };
      for (uint32_t i = tid; i < n4; i += 2 * NT) {
        const uint4 v0 = __ldg(e4 + i);
        const bool has1 = i + NT < n4;
        uint4 v1 = make_uint4(0u, 0u, 0u, 0u);
        if (has1) v1 = __ldg(e4 + i + NT);
        add4(v0);
        if (has1) add4(v1);
      }
      done = n4 * 4;
    }
    for (uint32_t i = done + tid; i < n; i += NT) atomicAdd(hm + (e[i] >> kRow32Bits), 1u);
  } else {
    const uint64_t* e = emit + (int64_t)q * cap;
    for (uint32_t i = tid; i < n; i += NT) atomicAdd(hm + emit_score(e[i]), 1u);
  }
  __syncthreads();
  for (int b = tid; b < 256; b += NT) {
    uint32_t v = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) v += hw[w][b];
    h[b] = v;
  }
  }  // !scan_hist
  __syncthreads();
  if (hist_out) {
    for (int i = tid; i < 256; i += NT) hist_out[(int64_t)q * 256 + i] = (int32_t)h[i];
    if (tid == 0) flags[q] = 0;
    return;
  }
  if (tid < 32) {
    // b* = first b <= B with cum[b] >= r2 (warp scan: lane l holds bins 8l .. 8l+7)
    const int B = guard_b[q];
    int64_t v[8], tot = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      v[i] = 8 * lane + i <= B ? (int64_t)h[8 * lane + i] : 0;
      tot += v[i];
    }
    int64_t incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t x = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += x;
    }
    int64_t cum = incl - tot, at = 0;
    int first = 8;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      cum += v[i];
      if (first == 8 && 8 * lane + i <= B && cum >= r2) { first = i; at = cum; }
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, first < 8);
    const int64_t all = __shfl_sync(0xffffffffu, incl, 31);
    if (bal) {
      const int src = __ffs(bal) - 1;
      const int f = __shfl_sync(0xffffffffu, first, src);
      const int64_t c = __shfl_sync(0xffffffffu, at, src);
      if (lane == 0) { bstar[q] = 8 * src + f; ncand[q] = c; flags[q] = 0; }
    } else if (lane == 0) {
      if (B >= 254) {
        bstar[q] = 254; ncand[q] = all; flags[q] = 0;
      } else {
        flags[q] = 1;
        bstar[q] = -1;
      }
    }
  }
}

// b* from a (globally summed) candidate histogram; sharded search.
__global__ void k_bstar_from_hist(const int32_t* __restrict__ hist, const uint16_t* __restrict__ guard_b,
                                  int nq, int r2, int32_t* __restrict__ bstar,
                                  int64_t* __restrict__ ncand, uint8_t* __restrict__ flags) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const int32_t* h = hist + (int64_t)q * 256;
  const int B = guard_b[q];
  int64_t cum = 0;
  int bs = -1;
  for (int b = 0; b <= B; ++b) {
    cum += h[b];
    if (cum >= r2) { bs = b; break; }
  }
  const bool over = flags[q] == 2;  // this shard's emit list overflowed in the scan: keep the flag
  if (bs >= 0) { bstar[q] = over ? -1 : bs; ncand[q] = cum; flags[q] = over ? 2 : 0; }
  else if (B >= 254) { bstar[q] = over ? -1 : 254; ncand[q] = cum; flags[q] = over ? 2 : 0; }
  else { flags[q] = 1; bstar[q] = -1; }
}

// Exact top-r of the union of n_parts per-shard top-r lists (each sorted
// by (dist, id), padded with (+inf, -1)), i.e. ResultSet.from_arrays over the
// concatenation (search.py:115-124) / shard.merge_topr: the rank of element
// (g, p) in the union is p plus, for every other list, the number of its
// elements ordered before it (binary search), with padding last and ties
// between paddings broken by (list, position).  Elements of rank < r are
// written; one CTA per query, no shared-memory limit on n_parts * r.
__device__ __forceinline__ bool merge_before(double da, int64_t ia, int ga, int pa, double db, int64_t ib, int gb,
                                             int pb) {
  const int64_t ka = ia < 0 ? INT64_MAX : ia, kb = ib < 0 ? INT64_MAX : ib;
  if (da != db) return da < db;
  if (ka != kb) return ka < kb;
  if (ga != gb) return ga < gb;
  return pa < pb;
}

__global__ void __launch_bounds__(256) k_merge_topr(const double* __restrict__ pd, const int64_t* __restrict__ pi,
                                                    int n_parts, int nq, int r, double* __restrict__ out_d,
                                                    int64_t* __restrict__ out_i) {
  const int q = blockIdx.x;
  const int64_t stride = (int64_t)nq * r;  // parts are (n_parts, nq, r)
  for (int e = threadIdx.x; e < n_parts * r; e += blockDim.x) {
    const int g = e / r, p = e % r;
    const double d = pd[g * stride + (int64_t)q * r + p];
    const int64_t id = pi[g * stride + (int64_t)q * r + p];
    int rank = p;
    for (int h = 0; h < n_parts && rank < r; ++h) {
      if (h == g) continue;
      const double* hd = pd + h * stride + (int64_t)q * r;
      const int64_t* hi = pi + h * stride + (int64_t)q * r;
      int lo = 0, up = r;  // first position of list h not before (d, id, g, p)
      while (lo < up) {
        const int mid = (lo + up) >> 1;
        if (merge_before(hd[mid], hi[mid], h, mid, d, id, g, p)) lo = mid + 1;
        else up = mid;
      }
      rank += lo;
    }
    if (rank < r) {
      out_d[(int64_t)q * r + rank] = id < 0 ? INFINITY : d;
      out_i[(int64_t)q * r + rank] = id;
    }
  }
}

// ============================================================================
// K5: full-codebook tables, exact (row_sq_dists, search.py:16-25).
//
// Tables are stored group-major: entry (q, j, c) with c = ibar * kbar + g
// lives at ((q * m + j) * kbar + g) * gsize + ibar  (gsize = k / kbar), so
// the members of one derived group are contiguous.
//
// k_group_tables (derived search) is the GPU form of LazyTables
// (twopass.py:220-251): a candidate's score s <= b* <= 254 is a sum of
// non-negative 8-bit entries, so every subspace entry satisfies
// q8[j][c_j mod kbar] <= b*; only groups with q8 <= b* can ever be gathered.
// One CTA per (group, subspace) stages the group's gsize codebook rows in
// shared memory once and computes entries for exactly the queries of the
// batch where that group is active.  Entries are bit-identical to eager
// tables (same pairwise kernel), so distances are bitwise the reference's.
//
// k_full_tables (conventional search, debug seam) computes every entry.
// ============================================================================
__host__ __device__ __forceinline__ int64_t table_index(int q, int j, uint32_t c, int m, int kbar,
                                                        int bbar, int gsize) {
  return (((int64_t)q * m + j) * kbar + (c & (kbar - 1))) * gsize + (c >> bbar);
}

struct GroupTablesArgs {
  const float* cb; const float* y; int ystride;
  const uint8_t* q8; const int32_t* bstar;
  const int32_t* slack = nullptr;  // [nq][m] sum over the other subspaces of their smallest entry (k_entry_slack)
  int nq, m, k, kbar, bbar, dsub;
  float* tables;
  unsigned long long* n_entries;
  unsigned long long negzero2 = kNegZero2;  // runtime (-0, -0) pair for sqdiff2 (see dpq_device.cuh)
};

// slack[q][j] = sum over subspaces i != j of min_g q8[q][i][g].  A candidate
// (score <= b*) whose sub-code of subspace j lies in group g has
// q8[q][j][g] <= b* - slack[q][j], so only those groups need exact entries.
// One warp per query.
__global__ void __launch_bounds__(128) k_entry_slack(const uint8_t* __restrict__ q8, int nq, int m, int kbar,
                                                     int32_t* __restrict__ slack) {
  const int q = blockIdx.x * 4 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (q >= nq) return;
  const uint8_t* e = q8 + (int64_t)q * m * kbar;
  int mn[8], sum = 0;
  for (int j = 0; j < m && j < 8; ++j) {
    unsigned v = 255u;
    for (int g = lane; g < kbar; g += 32) v = min(v, (unsigned)e[j * kbar + g]);
    mn[j] = (int)__reduce_min_sync(0xffffffffu, v);
    sum += mn[j];
  }
  if (lane == 0)
    for (int j = 0; j < m && j < 8; ++j) slack[q * m + j] = sum - mn[j];
}

// Register-row variant (DSUB = 32): thread ib holds codebook row ib of the
// group in registers and loops over the group's active queries, whose
// sub-vectors are staged 32 at a time in shared memory.  Same association
// order as pw_block / pw_sqdist_v8 (8 running sums, pairwise combine).
template <int DSUB>
__global__ void __launch_bounds__(256) k_group_tables_reg(GroupTablesArgs a) {
  extern __shared__ __align__(16) float gsm[];
  float* ys = gsm;                                      // [32][DSUB]
  int* act = reinterpret_cast<int*>(gsm + 32 * DSUB);   // [nq]
  __shared__ int nact;
  const int g = blockIdx.x, j = blockIdx.y, tid = threadIdx.x;
  const int gsize = a.k / a.kbar;
  if (tid == 0) nact = 0;
  __syncthreads();
  // blockIdx.z of gridDim.z CTAs per group: queries q = z (mod gridDim.z)
  for (int q = blockIdx.z + tid * gridDim.z; q < a.nq; q += 256 * gridDim.z)
    if ((int)a.q8[((int64_t)q * a.m + j) * a.kbar + g] <= a.bstar[q] - (a.slack ? a.slack[q * a.m + j] : 0))
      act[atomicAdd(&nact, 1)] = q;
  __syncthreads();
  const int n = nact;
  if (n == 0) return;  // (no codebook rows loaded for a group no query needs)
  for (int ib0 = 0; ib0 < gsize; ib0 += 256) {
    const int ib = ib0 + tid;
    f32x2_t c2[DSUB / 2];  // the codebook row as lane pairs
    const f32x2_t z2 = a.negzero2;
    if (ib < gsize) {
      const float4* src = reinterpret_cast<const float4*>(a.cb + (((int64_t)j * a.k) + (int64_t)ib * a.kbar + g) * DSUB);
#pragma unroll
      for (int i = 0; i < DSUB / 4; ++i) {
        const float4 v = __ldg(src + i);
        c2[2 * i] = pack2(v.x, v.y);
        c2[2 * i + 1] = pack2(v.z, v.w);
      }
    }
    for (int base = 0; base < n; base += 32) {
      const int nb = min(32, n - base);
      __syncthreads();
      for (int e = tid; e < nb * DSUB; e += 256) {
        const int qi = act[base + e / DSUB];
        ys[e] = a.y[(int64_t)qi * a.ystride + j * DSUB + e % DSUB];
      }
      __syncthreads();
      if (ib < gsize) {
        for (int t = 0; t < nb; ++t) {
          const ulonglong2* y2 = reinterpret_cast<const ulonglong2*>(ys + t * DSUB);
          f32x2_t r[4];
#pragma unroll
          for (int i = 0; i < DSUB / 8; ++i) {  // 8 elements = 4 lane pairs (running sums r0..r7)
            const ulonglong2 p = y2[2 * i], q = y2[2 * i + 1];
            const f32x2_t yv[4] = {p.x, p.y, q.x, q.y};
#pragma unroll
            for (int l = 0; l < 4; ++l) {
              const f32x2_t sd = sqdiff2(c2[4 * i + l], yv[l], z2);
              r[l] = i == 0 ? sd : add2(r[l], sd);
            }
          }
          const float v = pw_combine2(r);
          a.tables[(((int64_t)act[base + t] * a.m + j) * a.kbar + g) * gsize + ib] = v;
        }
      }
    }
  }
  if (a.n_entries && tid == 0) atomicAdd(a.n_entries, (unsigned long long)n * gsize);
}

template <int DSUB>
__global__ void __launch_bounds__(256) k_group_tables(GroupTablesArgs a) {
  extern __shared__ __align__(16) float tile[];  // [gsize][ld]
  __shared__ int nact;
  const int g = blockIdx.x, j = blockIdx.y;
  const int dsub = DSUB > 0 ? DSUB : a.dsub;
  // DSUB > 0 or 8 | dsub <= 128: rows padded to 16-B multiples + 4 floats
  // (conflict-free float4 reads across consecutive rows, paired-FP32 path);
  // otherwise +1 float
  const bool v8 = DSUB > 0 || ((dsub & 7) == 0 && dsub <= 128);
  const int gsize = a.k / a.kbar, ld = DSUB > 0 ? DSUB + 4 : (v8 ? dsub + 4 : dsub + 1);
  int* act = reinterpret_cast<int*>(tile + gsize * ld);
  if (threadIdx.x == 0) nact = 0;
  for (int e = threadIdx.x; e < gsize * dsub; e += 256) {
    const int ib = e / dsub, t = e - ib * dsub;
    tile[ib * ld + t] = a.cb[(((int64_t)j * a.k) + (int64_t)ib * a.kbar + g) * dsub + t];
  }
  __syncthreads();
  for (int q = threadIdx.x; q < a.nq; q += 256)
    if ((int)a.q8[((int64_t)q * a.m + j) * a.kbar + g] <= a.bstar[q] - (a.slack ? a.slack[q * a.m + j] : 0))
      act[atomicAdd(&nact, 1)] = q;
  __syncthreads();
  const int n = nact;
  for (int p = threadIdx.x; p < n * gsize; p += 256) {
    const int qi = act[p / gsize], ib = p % gsize;
    const float* yq = a.y + (int64_t)qi * a.ystride + j * dsub;
    const float* row = tile + ib * ld;
    float v;
    if constexpr (DSUB > 0) {
      v = pw_sqdist_v8(row, yq, DSUB);  // both operands 16-B aligned
    } else if (v8 && (reinterpret_cast<uintptr_t>(yq) & 15) == 0) {
      v = pw_sqdist_v8_x2(row, yq, dsub, a.negzero2);  // e.g. config 5: dsub = 120
    } else {
      v = pw_sqdist(row, yq, dsub);
    }
    a.tables[(((int64_t)qi * a.m + j) * a.kbar + g) * gsize + ib] = v;
  }
  if (a.n_entries && threadIdx.x == 0) atomicAdd(a.n_entries, (unsigned long long)n * gsize);
}

__global__ void __launch_bounds__(256)
    k_full_tables(const float* __restrict__ y, const float* __restrict__ cb, int m, int k, int kbar,
                  int bbar, int dsub, int group_major, float* __restrict__ out) {
  extern __shared__ float ysub[];
  const int q = blockIdx.z, j = blockIdx.y;
  for (int t = threadIdx.x; t < dsub; t += 256) ysub[t] = y[((int64_t)q * m + j) * dsub + t];
  __syncthreads();
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (i < k) {
    const float v = pw_sqdist(cb + ((int64_t)j * k + i) * dsub, ysub, dsub);
    const int64_t o = group_major ? table_index(q, j, (uint32_t)i, m, kbar, bbar, k / kbar)
                                  : ((int64_t)q * m + j) * k + i;
    out[o] = v;
  }
}

// ============================================================================
// K6: refine + exact top-r.  One CTA per query.  Every candidate's distance
// is the f64 sum, subspace order, of its m full-table entries, each entry
// computed on the fly with the same pairwise kernel as compute_tables (so
// it is bit-identical to the lazily filled table of twopass.py:220-251
// without materialising the table).  Survivors of the running threshold
// (strictly better (dist,id) than the current r-th best) are collected in a
// shared-memory buffer that is bitonic-sorted and truncated to r whenever it
// could overflow.
// Source of candidates:
//   MODE_EMIT: emit list entries with score <= b*  (derived search)
//   MODE_ALL : every row of [0, n_rows)            (conventional, tables)
// ============================================================================
// MODE_EMIT_APPROX: tables are the tensor-core approximations of
// dpq_tctab.cu; entry (q, j, c) is within g (||y'_qj|| + ||c'_jc||)^2 of
// numpy's, so a candidate's approximate distance a is within E = the sum of
// its m entry bounds of the exact one d.  Pass 0 ranks the upper bounds
// a + E and takes U = the r-th smallest (>= r candidates have d <= U, so the
// exact r-th distance D_r <= U); pass 1 recomputes exactly (numpy entries,
// entry_dist) every candidate with a - E <= U — which includes every exact
// top-r member (d <= D_r) — and keeps the exact top-r.
enum { MODE_EMIT = 0, MODE_ALL = 1, MODE_EMIT_TABLE = 2, MODE_EMIT_APPROX = 3, MODE_EMIT_TABLE32 = 4 };
// MODE_EMIT_TABLE32: MODE_EMIT_TABLE over 4-byte emit records (flat PQ 4x16 shards of < 2^24 rows);
// only the software-pipelined loop is instantiated.

struct RefineArgs {
  const uint64_t* emit; const uint32_t* emit_cnt; uint32_t cap;
  const int32_t* bstar;
  int64_t n_rows;            // MODE_ALL
  const void* codes; int code_bytes; int m; int k; int dsub; int kbar; int bbar;
  const float* cb;           // [m][k][dsub]
  const float* tables;       // MODE_ALL / MODE_EMIT_TABLE: group-major tables
  const float* y;            // [nq][ystride] query / per-probe residuals
  int ystride;               // floats per query in y (d, or ma*d for ivf)
  const int64_t* row_ids;    // optional row -> id (ivf sorted_ids)
  int64_t id_base;
  int r;
  double* out_d; int64_t* out_i;
  unsigned long long* n_refined;
  const int* order = nullptr;  // optional CTA -> query (heaviest emit lists first)
  int y_in_smem = 1;           // stage the query's y block in shared memory (else read it from global)
  const double* ny = nullptr;     // MODE_EMIT_APPROX: (nq, m) ||y'|| (centred query sub-vectors)
  const float* cnorm = nullptr;   //   (m, k) ||c'|| in group-major entry order
  double gamma = 0.0;             //   entry bound coefficient
  unsigned long long* n_exact = nullptr;  // MODE_EMIT_APPROX: candidates recomputed exactly
  int emit32 = 0;                 // emit lists hold 4-byte records (pack_emit32)
};

// Dynamic shared-memory budget of one refine CTA (buffer + staged y block).
constexpr size_t kRefineSmemMax = 220 * 1024;

// Query order for the refine launch: descending emitted count (coarse
// counting sort, one CTA), so the longest lists start first and the short
// ones fill in behind them (LPT scheduling over the CTA slots).
__global__ void __launch_bounds__(1024) k_order_by_count(const uint32_t* __restrict__ emit_cnt, int nq,
                                                         uint32_t cap, int* __restrict__ order) {
  __shared__ int cnt[1025];
  __shared__ unsigned mx;
  const int tid = threadIdx.x;
  if (tid == 0) mx = 0;
  for (int i = tid; i < 1025; i += 1024) cnt[i] = 0;
  __syncthreads();
  for (int q = tid; q < nq; q += 1024) atomicMax(&mx, min(emit_cnt[q], cap));
  __syncthreads();
  int shift = 0;
  while ((mx >> shift) >= 1024u) ++shift;
  auto key = [&](int q) { return 1023 - (int)(min(emit_cnt[q], cap) >> shift); };  // descending
  for (int q = tid; q < nq; q += 1024) atomicAdd(&cnt[key(q) + 1], 1);
  __syncthreads();
  if (tid == 0)
    for (int i = 1; i < 1025; ++i) cnt[i] += cnt[i - 1];
  __syncthreads();
  for (int q = tid; q < nq; q += 1024) order[atomicAdd(&cnt[key(q)], 1)] = q;
}

// Bitonic sort of the first P (power of two) entries of the buffer.
template <int NT>
__device__ void sort_pairs(uint64_t* keys, int64_t* ids, int P) {
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < P / 2; t += NT) {
        const int i = 2 * t - (t & (stride - 1));
        const int j = i + stride;
        const bool asc = (i & size) == 0;
        const uint64_t ki = keys[i], kj = keys[j];
        const int64_t ii = ids[i], ij = ids[j];
        const bool sw = asc ? pair_less(kj, ij, ki, ii) : pair_less(ki, ii, kj, ij);
        if (sw) { keys[i] = kj; keys[j] = ki; ids[i] = ij; ids[j] = ii; }
      }
      __syncthreads();
    }
  }
}

// Radix select of the r smallest (key, id) pairs among buffer[0, f)
// (keys: non-negative doubles as u64, ids unique), r < f <= NT * EPT.
// 8-bit digit passes over the key bits that vary within the buffer, stopping
// as soon as the target's bucket holds one element; remaining key ties are
// broken by id.  The r kept pairs are compacted to [0, r) (unordered) and
// (thr_k, thr_i) is set to the r-th pair.  Replaces a full bitonic sort of
// the buffer: ~EPT shared loads per pass instead of two per stage.
struct SelShared {
  uint32_t hist[256];
  uint64_t red_k[32];
  int64_t red_i[32];
  uint64_t pfx, K;
  int64_t I;
  int bits, need, done, cnt;
};

template <int NT, int EPT>
__device__ void select_r(uint64_t* keys, int64_t* ids, int f, int r, SelShared& S, uint64_t& thr_k,
                         int64_t& thr_i) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint64_t k[EPT];
  int64_t v[EPT];
  uint64_t mn = ~0ull, mx = 0ull;
#pragma unroll
  for (int e = 0; e < EPT; ++e) {
    const int i = tid + e * NT;
    k[e] = i < f ? keys[i] : ~0ull;
    v[e] = i < f ? ids[i] : INT64_MAX;
    if (i < f) { mn = min(mn, k[e]); mx = max(mx, k[e]); }
  }
  // block min / max of the keys
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, (uint64_t)__shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, (uint64_t)__shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (lane == 0) { S.red_k[warp] = mn; S.red_i[warp] = (int64_t)mx; }
  __syncthreads();
  if (tid == 0) {
    uint64_t a = ~0ull, b = 0ull;
    for (int w = 0; w < NT / 32; ++w) { a = min(a, S.red_k[w]); b = max(b, (uint64_t)S.red_i[w]); }
    const int bits = a == b ? 0 : 64 - __clzll((long long)(a ^ b));
    S.bits = bits;
    S.pfx = bits == 64 ? 0ull : (a >> bits) << bits;
    S.need = r;
    S.done = 0;
  }
  __syncthreads();
  // digit passes
  for (;;) {
    const int bits = S.bits;
    if (bits == 0 || S.done) break;
    const int w = min(8, bits), sft = bits - w;
    const uint64_t pfx = S.pfx;
    for (int i = tid; i < 256; i += NT) S.hist[i] = 0;
    __syncthreads();
#pragma unroll
    for (int e = 0; e < EPT; ++e)
      if (tid + e * NT < f && (bits == 64 || (k[e] >> bits) == (pfx >> bits)))
        atomicAdd(&S.hist[(uint32_t)(k[e] >> sft) & ((1u << w) - 1u)], 1u);
    __syncthreads();
    if (warp == 0) {
      // the need-th element's digit: warp prefix sum over 8 bins per lane
      const int need = S.need, nb = 1 << w;
      uint32_t ls = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) ls += lane * 8 + i < nb ? S.hist[lane * 8 + i] : 0u;
      uint32_t incl = ls;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const uint32_t reach = __ballot_sync(0xffffffffu, incl >= (uint32_t)need);
      const int L = __ffs(reach) - 1;  // first lane whose prefix reaches need (exists: need <= total)
      if (lane == L) {
        uint32_t below = incl - ls;
        int d = lane * 8;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint32_t hb = S.hist[lane * 8 + i];
          if (below + hb >= (uint32_t)need) { d = lane * 8 + i; break; }
          below += hb;
        }
        S.need = need - (int)below;
        S.pfx = (bits == 64 ? 0ull : pfx) | ((uint64_t)d << sft);
        S.bits = sft;
        S.done = S.hist[d] == 1u;  // the target is the only element of its bucket
        S.cnt = 0;
      }
    }
    __syncthreads();
  }
  // resolve the target pair (K, I): unique element of the bucket, or the
  // need-th smallest id among the elements whose key equals the prefix
  const int bits = S.bits;
  const uint64_t pfx = S.pfx;
  if (tid == 0) { S.cnt = 0; S.I = INT64_MAX; }
  __syncthreads();
  if (S.done) {
#pragma unroll
    for (int e = 0; e < EPT; ++e)
      if (tid + e * NT < f && (bits == 64 || (k[e] >> bits) == (pfx >> bits))) { S.K = k[e]; S.I = v[e]; }
  } else {
    // all remaining keys equal pfx; ties by id (rare): rank ids among them
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      if (tid + e * NT < f && k[e] == pfx) {
        int rank = 0;
        for (int j = 0; j < f; ++j) rank += (keys[j] == pfx && ids[j] < v[e]) ? 1 : 0;
        if (rank == S.need - 1) { S.K = pfx; S.I = v[e]; }
      }
    }
  }
  __syncthreads();
  const uint64_t K = S.K;
  const int64_t I = S.I;
  // compact the kept pairs (registers -> [0, r))
#pragma unroll
  for (int e = 0; e < EPT; ++e) {
    if (tid + e * NT < f && !pair_less(K, I, k[e], v[e])) {  // (k, v) <= (K, I)
      const int p = atomicAdd(&S.cnt, 1);
      keys[p] = k[e];
      ids[p] = v[e];
    }
  }
  if (tid == 0) { thr_k = K; thr_i = I; }
  __syncthreads();
}

template <int DSUB>
__device__ __forceinline__ float entry_dist(const float* cbrow, const float* ys, int dsub) {
  if constexpr (DSUB > 0) return pw_sqdist_fixed<DSUB>(cbrow, ys);
  else return pw_sqdist(cbrow, ys, dsub);
}

template <int BUF, int NT, int MODE, int DSUB>
#ifndef DPQ_REFINE_MINB
#define DPQ_REFINE_MINB 4  // CTAs per SM the register budget is sized for (5: 48 regs, spills since the pipelined gathers)
#endif
__global__ void __launch_bounds__(NT, MODE == MODE_EMIT_APPROX ? 3 : DPQ_REFINE_MINB) k_refine_topk(RefineArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem);
  int64_t* ids = reinterpret_cast<int64_t*>(keys + BUF);
  float* ys_s = reinterpret_cast<float*>(ids + BUF);
  __shared__ int cnt3[3];  // insert counters, round r uses cnt3[r % 3] (one barrier per round)
  __shared__ uint64_t thr_k;
  __shared__ int64_t thr_i;
  __shared__ unsigned nref;
  const int q = a.order ? a.order[blockIdx.x] : blockIdx.x;
  // query / per-probe residual block: staged in shared memory when it fits
  // (launch_refine_buf), else read through L1/L2 (ivf with a large ma * d)
  const float* ys = a.y_in_smem ? ys_s : a.y + (int64_t)q * a.ystride;
  if (a.y_in_smem)
    for (int i = threadIdx.x; i < a.ystride; i += NT) ys_s[i] = a.y[(int64_t)q * a.ystride + i];
  if (threadIdx.x == 0) { cnt3[0] = cnt3[1] = cnt3[2] = 0; thr_k = ~0ull; thr_i = INT64_MAX; nref = 0; }
  __syncthreads();
  const int d = a.m * a.dsub;
  int64_t ntot;
  int bs = 254;
  const uint64_t* e = nullptr;
  const uint32_t* e32 = nullptr;
  if (MODE != MODE_ALL) {
    ntot = min(a.emit_cnt[q], a.cap);
    bs = a.bstar[q];
    e = a.emit + (int64_t)q * a.cap;
    e32 = reinterpret_cast<const uint32_t*>(a.emit) + (int64_t)q * a.cap;
  } else {
    ntot = a.n_rows;
  }
  unsigned my_ref = 0;
  const float* tq = a.tables ? a.tables + (int64_t)q * a.m * a.k : nullptr;
  // candidate -> (key, id); false when it is not a candidate (score > b*)
  // row -> id (sorted flat rows / ivf lists: row_ids), looked up only for a
  // candidate that ties the threshold distance or enters the buffer
  auto id_of = [&](int64_t row) -> int64_t { return a.row_ids ? a.row_ids[row] : a.id_base + row; };
  // v: the candidate's emit entry (prefetched one round ahead)
  int pass = 0;                 // MODE_EMIT_APPROX: 0 = approximate ranking, 1 = exact re-rank
  double tau = 0.0;             //   pass-1 filter on the approximate distance
  unsigned my_exact = 0;
  auto eval = [&](int64_t idx, uint64_t v, uint64_t& key, int64_t& id) -> bool {
    int64_t row;
    uint32_t probe = 0;
    if (MODE != MODE_ALL) {
      if ((int)emit_score(v) > bs) return false;
      row = emit_row(v);
      probe = emit_probe(v);
    } else {
      row = idx;
    }
    if (MODE != MODE_EMIT_APPROX || pass == 0) ++my_ref;
    double dist = 0.0;
    const float* yq = ys + (int64_t)probe * d;
    double E = 0.0;  // MODE_EMIT_APPROX: bound on |approx - exact| of this candidate
    auto ebound = [&](int j, uint32_t c) {
      const int64_t ej = (int64_t)j * a.k + ((c & (uint32_t)(a.kbar - 1)) * (uint32_t)(a.k >> a.bbar) + (c >> a.bbar));
      const double s = a.ny[(int64_t)q * a.m + j] + (double)__ldg(a.cnorm + ej);
      E += a.gamma * s * s;
    };
    if ((MODE == MODE_EMIT_TABLE || MODE == MODE_EMIT_APPROX) && a.code_bytes == 2 && a.m == 4) {
      // one 8-byte code load, four independent table gathers with 32-bit
      // offsets inside this query's table block (m * k floats)
      const uint2 v = *reinterpret_cast<const uint2*>((const uint16_t*)a.codes + row * 4);
      const uint32_t kmask = (uint32_t)a.kbar - 1u, gs = (uint32_t)(a.k >> a.bbar);
      auto off = [&](uint32_t j, uint32_t c) { return ((j << a.bbar) + (c & kmask)) * gs + (c >> a.bbar); };
      const float t0 = __ldg(tq + off(0, v.x & 0xFFFFu));
      const float t1 = __ldg(tq + off(1, v.x >> 16));
      const float t2 = __ldg(tq + off(2, v.y & 0xFFFFu));
      const float t3 = __ldg(tq + off(3, v.y >> 16));
      dist = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(dist, (double)t0), (double)t1), (double)t2), (double)t3);
      if (MODE == MODE_EMIT_APPROX) {
        ebound(0, v.x & 0xFFFFu); ebound(1, v.x >> 16); ebound(2, v.y & 0xFFFFu); ebound(3, v.y >> 16);
      }
    } else {
      for (int j = 0; j < a.m; ++j) {
        const uint32_t c = code_at(a.codes, a.code_bytes, row * a.m + j);
        float t;
        if (MODE != MODE_EMIT) t = __ldg(a.tables + table_index(q, j, c, a.m, a.kbar, a.bbar, a.k / a.kbar));
        else t = entry_dist<DSUB>(a.cb + ((int64_t)j * a.k + c) * a.dsub, yq + j * a.dsub, a.dsub);
        dist = __dadd_rn(dist, (double)t);
        if (MODE == MODE_EMIT_APPROX) ebound(j, c);
      }
    }
    if (MODE == MODE_EMIT_APPROX) E = E * (1.0 + 1e-9) + fabs(dist) * 1e-12;  // (f64 sums themselves)
    if (MODE == MODE_EMIT_APPROX && pass == 0) dist = dist + E;  // rank by the upper bound
    if (MODE == MODE_EMIT_APPROX && pass == 1) {  // exact re-rank of the candidates inside the margin
      if (!(dist - E <= tau)) return false;
      ++my_exact;
      dist = 0.0;
      for (int j = 0; j < a.m; ++j) {
        const uint32_t c = code_at(a.codes, a.code_bytes, row * a.m + j);
        dist = __dadd_rn(dist, (double)entry_dist<DSUB>(a.cb + ((int64_t)j * a.k + c) * a.dsub, yq + j * a.dsub,
                                                        a.dsub));
      }
    }
    key = (uint64_t)__double_as_longlong(dist);
    id = row;  // (a row until id_of)
    return true;
  };
#ifndef DPQ_REFINE_U
#define DPQ_REFINE_U 2
#endif
  constexpr int U = DPQ_REFINE_U;  // candidates per thread per round (independent gather chains)
  auto pow2_at_least = [](int v) { int p = 2; while (p < v) p <<= 1; return p; };
  uint64_t ev[U];
  auto load_e = [&](int64_t base) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t idx = base + (int64_t)u * NT + threadIdx.x;
      // (MODE_EMIT_TABLE: 4-byte records only reach the piped loop, see dpq_flat_create)
      ev[u] = (MODE != MODE_ALL && idx < ntot)
                  ? ((MODE != MODE_EMIT_TABLE && MODE != MODE_EMIT_TABLE32 && a.emit32) ? widen_emit32(e32[idx]) : e[idx])
                  : 0ull;
    }
  };
  int fb = 0;   // buffer fill before this round (same value in every thread)
  int rnd = 0;  // round index mod 3
  // Buffer entries may hold a row tagged kDeferId instead of its id (the
  // piped loop defers the row -> id gather of sorted flat rows until the id
  // matters): resolved before any sort / select / output.
  constexpr int64_t kDeferId = (int64_t)1 << 62;
  auto resolve_ids = [&](int f) {
    if (!a.row_ids) return;
    for (int i = threadIdx.x; i < f; i += NT) {
      const int64_t v = ids[i];
      if (v & kDeferId) ids[i] = a.row_ids[v & ~kDeferId];
    }
    __syncthreads();
  };
  // one round's survivors into the buffer; sort / select once it fills
  auto commit = [&](const bool* keep, const uint64_t* key, const int64_t* id) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (keep[u]) {
        const int p = fb + atomicAdd(&cnt3[rnd], 1);
        keys[p] = key[u];
        ids[p] = id[u];
      }
    }
    __syncthreads();
    // every thread reads this round's counter after the barrier; the counter
    // of round + 2 (last read before this barrier) is cleared for reuse
    const int f = fb + cnt3[rnd];
    if (threadIdx.x == 0) cnt3[rnd == 0 ? 2 : rnd - 1] = 0;
    fb = f;
    // sort + truncate once the buffer is half full (the next round adds at
    // most U * NT <= BUF / 2 entries): early, small sorts tighten the
    // threshold sooner than waiting for a full buffer
    if (f >= BUF - U * NT || (f >= 2 * a.r && f >= (BUF - U * NT) / 2 && thr_k == ~0ull)) {
      resolve_ids(f);
      if (BUF == NT * 4 && f > a.r) {
        // keep the r smallest (unordered) and set the threshold: radix select
        __shared__ SelShared sel;
        select_r<NT, BUF / NT>(keys, ids, f, a.r, sel, thr_k, thr_i);
        fb = a.r;
      } else {
        const int P = pow2_at_least(f);
        for (int i = f + threadIdx.x; i < P; i += NT) { keys[i] = ~0ull; ids[i] = INT64_MAX; }
        __syncthreads();
        sort_pairs<NT>(keys, ids, P);
        fb = min(f, a.r);
        if (threadIdx.x == 0 && fb == a.r) { thr_k = keys[fb - 1]; thr_i = ids[fb - 1]; }
        __syncthreads();
      }
    }
  };
  constexpr int NPASS = MODE == MODE_EMIT_APPROX ? 2 : 1;
  bool piped = false;
#ifndef DPQ_REFINE_PIPE
#define DPQ_REFINE_PIPE 1
#endif
  if constexpr ((MODE == MODE_EMIT_TABLE && DPQ_REFINE_PIPE) || MODE == MODE_EMIT_TABLE32) {
    if (MODE == MODE_EMIT_TABLE32 || (a.code_bytes == 2 && a.m == 4)) {
      // Software-pipelined gathers (flat PQ 4x16, the configs[1-3] shape):
      // emit entries are loaded two rounds ahead and the candidates' codes
      // one round ahead, so a round waits on one dependent gather (its
      // table entries) instead of the emit -> code -> table chain.
      piped = true;
      const uint32_t kmask = (uint32_t)a.kbar - 1u, gs = (uint32_t)(a.k >> a.bbar);
      auto off = [&](uint32_t j, uint32_t c) { return ((j << a.bbar) + (c & kmask)) * gs + (c >> a.bbar); };
      // k = 65536, kbar = 256: entry (j, c) sits at j << 16 | (c & 255) << 8 | c >> 8, one byte permute
      const bool k16 = a.k == 65536 && a.bbar == 8;
      const uint2* codes2 = reinterpret_cast<const uint2*>(a.codes);
      // one loop per record width (disjoint register live ranges)
      auto piped_loop = [&](auto w32_tag) {
        constexpr bool W32 = decltype(w32_tag)::value;
        using RT = std::conditional_t<W32, uint32_t, uint64_t>;
        const RT* ep = reinterpret_cast<const RT*>(W32 ? (const void*)e32 : (const void*)e);
        auto rrow = [](RT v) -> int64_t {
          if constexpr (W32) return (int64_t)(v & ((1u << kRow32Bits) - 1u));
          else return emit_row(v);
        };
        auto rscore = [](RT v) -> int {
          if constexpr (W32) return (int)(v >> kRow32Bits);
          else return (int)emit_score(v);
        };
        auto valid = [&](RT v, int64_t idx) { return idx < ntot && rscore(v) <= bs; };
        auto ld_e = [&](int64_t idx) -> RT { return idx < ntot ? ep[idx] : (RT)0; };
        RT e0[U], e1[U];
        uint2 c0[U];
        const int64_t step = (int64_t)U * NT;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t i0 = (int64_t)u * NT + threadIdx.x;
          e0[u] = ld_e(i0);
          e1[u] = ld_e(i0 + step);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t i0 = (int64_t)u * NT + threadIdx.x;
          c0[u] = valid(e0[u], i0) ? __ldg(codes2 + rrow(e0[u])) : make_uint2(0u, 0u);
        }
        for (int64_t base = 0; base < ntot; base += step, rnd = rnd == 2 ? 0 : rnd + 1) {
          uint2 cn[U];
          RT en[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int64_t i1 = base + step + (int64_t)u * NT + threadIdx.x;
            cn[u] = valid(e1[u], i1) ? __ldg(codes2 + rrow(e1[u])) : make_uint2(0u, 0u);
            en[u] = ld_e(i1 + step);
          }
          uint64_t key[U];
          int64_t id[U];
          bool keep[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int64_t i0 = base + (int64_t)u * NT + threadIdx.x;
            keep[u] = valid(e0[u], i0);
            if (keep[u]) {
              ++my_ref;
              const uint2 v = c0[u];
              uint32_t o0, o1, o2, o3;
              if (k16) {
                o0 = __byte_perm(v.x, 0u, 0x5401u); o1 = __byte_perm(v.x, 1u, 0x5423u);
                o2 = __byte_perm(v.y, 2u, 0x5401u); o3 = __byte_perm(v.y, 3u, 0x5423u);
              } else {
                o0 = off(0, v.x & 0xFFFFu); o1 = off(1, v.x >> 16); o2 = off(2, v.y & 0xFFFFu); o3 = off(3, v.y >> 16);
              }
              const float t0 = __ldg(tq + o0);
              const float t1 = __ldg(tq + o1);
              const float t2 = __ldg(tq + o2);
              const float t3 = __ldg(tq + o3);
              const double dist =
                  __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(0.0, (double)t0), (double)t1), (double)t2), (double)t3);
              key[u] = (uint64_t)__double_as_longlong(dist);
              if (key[u] < thr_k) {  // kept whatever its id: the row -> id gather waits until it matters
                id[u] = a.row_ids ? (rrow(e0[u]) | kDeferId) : a.id_base + rrow(e0[u]);
              } else if (key[u] == thr_k) {
                id[u] = id_of(rrow(e0[u]));
                keep[u] = id[u] < thr_i;
              } else {
                keep[u] = false;
              }
            }
          }
          commit(keep, key, id);
#pragma unroll
          for (int u = 0; u < U; ++u) { e0[u] = e1[u]; c0[u] = cn[u]; e1[u] = en[u]; }
        }
      };
      if constexpr (MODE == MODE_EMIT_TABLE32) piped_loop(std::true_type());
      else piped_loop(std::false_type());
    }
  }
  for (pass = 0; pass < NPASS && !piped && MODE != MODE_EMIT_TABLE32; ++pass) {
  if (pass == 1) {
    const int P = pow2_at_least(fb);
    for (int i = fb + threadIdx.x; i < P; i += NT) { keys[i] = ~0ull; ids[i] = INT64_MAX; }
    __syncthreads();
    sort_pairs<NT>(keys, ids, P);
    // U = r-th smallest upper bound a + E (all candidates pass when fewer than r)
    tau = fb >= a.r ? __longlong_as_double((long long)keys[a.r - 1]) : INFINITY;
    __syncthreads();
    if (threadIdx.x == 0) { cnt3[0] = cnt3[1] = cnt3[2] = 0; thr_k = ~0ull; thr_i = INT64_MAX; }
    __syncthreads();
    fb = 0;
    rnd = 0;
  }
  load_e(0);
  for (int64_t base = 0; base < ntot; base += (int64_t)U * NT, rnd = rnd == 2 ? 0 : rnd + 1) {
    uint64_t key[U], cur[U];
    int64_t id[U];
    bool keep[U];
#pragma unroll
    for (int u = 0; u < U; ++u) cur[u] = ev[u];
    load_e(base + (int64_t)U * NT);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t idx = base + (int64_t)u * NT + threadIdx.x;
      keep[u] = idx < ntot && eval(idx, cur[u], key[u], id[u]) && key[u] <= thr_k;
      if (keep[u]) {
        id[u] = id_of(id[u]);
        keep[u] = pair_less(key[u], id[u], thr_k, thr_i);
      }
    }
    commit(keep, key, id);
  }
  }  // pass
  const int f = fb;
  resolve_ids(f);
  const int P = pow2_at_least(f);
  for (int i = f + threadIdx.x; i < P; i += NT) { keys[i] = ~0ull; ids[i] = INT64_MAX; }
  __syncthreads();
  sort_pairs<NT>(keys, ids, P);
  const int got = min(f, a.r);
  for (int i = threadIdx.x; i < a.r; i += NT) {
    const int64_t o = (int64_t)q * a.r + i;
    if (i < got) {
      a.out_d[o] = __longlong_as_double((long long)keys[i]);
      a.out_i[o] = ids[i];
    } else {
      a.out_d[o] = INFINITY;
      a.out_i[o] = -1;
    }
  }
  if (a.n_refined) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my_ref += __shfl_xor_sync(0xffffffffu, my_ref, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&nref, my_ref);
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(a.n_refined, (unsigned long long)nref);
  }
  if (MODE == MODE_EMIT_APPROX && a.n_exact) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my_exact += __shfl_xor_sync(0xffffffffu, my_exact, o);
    if ((threadIdx.x & 31) == 0 && my_exact) atomicAdd(a.n_exact, (unsigned long long)my_exact);
  }
}

}  // namespace dpq
