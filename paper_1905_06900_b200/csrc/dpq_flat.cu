// dpq_flat.cu — flat-index orchestration of the derived two-pass search and
// the conventional single-pass search on one GPU, plus the C ABI for them.
//
// Batch pipeline (one stream, inputs already in HBM):
//   K1 k_small_tables -> K2a k_scan_hist (row sample) -> k_guard
//   -> K2b k_scan_emit -> K3 k_threshold -> [rare: exact redo] -> K6 refine
// The only host synchronisation per batch is the 1-byte-per-query flag read
// after K3 (guard too tight / emit overflow), which decides whether the
// exact redo runs.
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <omp.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/dpq.h"
#include "dpq_impl.h"
#include "dpq_kernels.cuh"

namespace dpq {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
const char* last_error() { return g_last_error.c_str(); }

#define DPQ_CUDA(call)                                                          \
  do {                                                                          \
    cudaError_t e_ = (call);                                                    \
    if (e_ != cudaSuccess) {                                                    \
      set_error(std::string(#call) + ": " + cudaGetErrorString(e_) + " (" +     \
                __FILE__ + ":" + std::to_string(__LINE__) + ")");               \
      return DPQ_ERR_CUDA;                                                      \
    }                                                                           \
  } while (0)

#define DPQ_LAUNCHED(h)                                                         \
  do {                                                                          \
    cudaError_t e_ = cudaGetLastError();                                        \
    if (e_ != cudaSuccess) {                                                    \
      set_error(std::string("kernel launch: ") + cudaGetErrorString(e_) + " (" + \
                __FILE__ + ":" + std::to_string(__LINE__) + ")");               \
      return DPQ_ERR_CUDA;                                                      \
    }                                                                           \
    (h)->counters[0]++;                                                         \
  } while (0)

// DPQ_DEBUG_ERR=1: report (and clear) a CUDA error left pending by an unchecked call.
static void dbg_pending(const char* where) {
  static const bool on = getenv("DPQ_DEBUG_ERR") != nullptr;
  if (!on) return;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fprintf(stderr, "[dpq] pending CUDA error at %s: %s\n", where, cudaGetErrorString(e));
}

#define DPQ_TRY(expr)            \
  do {                           \
    int rc_ = (expr);            \
    if (rc_ != DPQ_OK) return rc_; \
  } while (0)

static constexpr int kScanThreads = 1024;
#ifndef DPQ_EMIT_THREADS
#define DPQ_EMIT_THREADS 1024
#endif
static constexpr int kEmitThreads = DPQ_EMIT_THREADS;  // (512 x 128 registers measured slower)
#ifndef DPQ_TOP_THREADS
#define DPQ_TOP_THREADS 256  // threads of a refine CTA (A/B: 512 with DPQ_REFINE_MINB=2)
#endif
static constexpr int kTopThreads = DPQ_TOP_THREADS;

static uint64_t g_alloc_epoch = 0;  // bumped by every device (re)allocation (invalidates captured graphs)

template <typename T>
static int dmalloc(T** p, size_t count) {
  ++g_alloc_epoch;
  if (*p) { cudaFree(*p); *p = nullptr; }
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error(std::string("cudaMalloc(") + std::to_string(count * sizeof(T)) + " B): " + cudaGetErrorString(e));
    *p = nullptr;
    return DPQ_ERR_NOMEM;
  }
  return DPQ_OK;
}
template <class T>
static int hmalloc(T** p, size_t count) {
  if (*p) { cudaFreeHost(*p); *p = nullptr; }
  if (count == 0) count = 1;
  cudaError_t e = cudaMallocHost((void**)p, count * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error(std::string("cudaMallocHost: ") + cudaGetErrorString(e));
    *p = nullptr;
    return DPQ_ERR_NOMEM;
  }
  return DPQ_OK;
}

// Static + dynamic shared memory above 48 KB needs a per-(device, kernel)
// attribute.  The largest dynamic size set so far is cached per (device,
// kernel) and recorded only after the call succeeds, so a failed request
// (too large) never masks a later valid one.  Called before every launch
// with dynamic shared memory.
static int set_smem_impl(int device, const void* kern, size_t bytes) {
  if (bytes == 0) return DPQ_OK;
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_pair(device, kern);
  const auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return DPQ_OK;
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("dynamic shared memory of " + std::to_string(bytes) + " B not available: " + cudaGetErrorString(e));
    return DPQ_ERR_ARG;
  }
  done[key] = bytes;
  return DPQ_OK;
}
template <class K>
static int set_smem(const Index* h, K* kern, size_t bytes) {
  return set_smem_impl(h->device, reinterpret_cast<const void*>(kern), bytes);
}

// Queries per scan tile of this index (ScanGeom): flat m <= 4: 128, ivf m <= 4: 64 (h->qt), m = 8: 64.
static inline int qt_of(const Index* h) { return h->qt; }
static inline int tiles_of(int nslot, const Index* h) { return (nslot + qt_of(h) - 1) / qt_of(h); }

// Slot-indexed arrays (a slot = one query for flat, one (query, probe) of a
// query tile for ivf) are sized by nslot; query-indexed arrays (emit lists,
// thresholds, results) by nq (default: nq = nslot).
int ensure_ws(Index* h, int nslot, int r, int ystride, int nq) {
  Workspace& w = h->ws;
  if (nq < 0) nq = nslot;
  const int qt = qt_of(h);
  if (nslot > w.qb || ystride > w.ystride || nq > w.qn) {
    const int qb = std::max(nslot, w.qb);
    const int qn = std::max(nq, w.qn);
    const int ys = std::max(ystride, w.ystride);
    const int tiles = (qb + qt - 1) / qt;
    const size_t mk = (size_t)h->m * h->kbar;
    DPQ_TRY(dmalloc(&w.y, (size_t)std::max(qb, qn) * ys));
    DPQ_TRY(dmalloc(&w.small, (size_t)qb * mk));
    DPQ_TRY(dmalloc(&w.q8, (size_t)qb * mk));
    DPQ_TRY(dmalloc(&w.qmin, (size_t)qb));
    DPQ_TRY(dmalloc(&w.qmax, (size_t)qb));
    DPQ_TRY(dmalloc(&w.bounds, (size_t)qb * 2));
    DPQ_TRY(dmalloc(&w.lut, (size_t)tiles * h->mpad * 256 * (qt / 4) * 4));  // u8, 4 per word
    DPQ_TRY(dmalloc(&w.hist, (size_t)std::max(tiles * qt, qn) * 256));
    DPQ_TRY(dmalloc(&w.hist_i, (size_t)qn * 256));
    DPQ_TRY(dmalloc(&w.guard_b, (size_t)std::max(tiles * qt, qn)));
    DPQ_TRY(dmalloc(&w.gword, (size_t)std::max(tiles * qt, qn)));
    DPQ_TRY(dmalloc(&w.gword_p, (size_t)tiles * qt));
    DPQ_TRY(dmalloc(&w.bstar, (size_t)qn));
    DPQ_TRY(dmalloc(&w.ncand, (size_t)qn));
    DPQ_TRY(dmalloc(&w.flags, (size_t)qn));
    DPQ_TRY(dmalloc(&w.only, (size_t)std::max(tiles * qt, qn)));
    DPQ_TRY(dmalloc(&w.tile_list, (size_t)tiles));
    DPQ_TRY(dmalloc(&w.order, (size_t)qn));
    DPQ_TRY(dmalloc(&w.cluster, (size_t)qb));
    DPQ_TRY(dmalloc(&w.tile_fast, (size_t)tiles));
    if (!w.counter) DPQ_TRY(dmalloc(&w.counter, 4));
    DPQ_TRY(dmalloc(&w.slot_query, (size_t)tiles * qt));
    DPQ_TRY(dmalloc(&w.slot_probe, (size_t)tiles * qt));
    DPQ_TRY(dmalloc(&w.slot_pre_off, (size_t)tiles * qt));
    DPQ_TRY(dmalloc(&w.slot_pre_len, (size_t)tiles * qt));
    DPQ_TRY(hmalloc(&w.h_y, (size_t)std::max(qb, qn) * ys));
    DPQ_TRY(hmalloc(&w.h_flags, (size_t)qn));
    DPQ_TRY(hmalloc(&w.h_cnt, (size_t)qn));
    w.qb = qb;
    w.qn = qn;
    w.ystride = ys;
    w.qcap_emit = 0;  // emit buffers re-sized below
    w.h_out_elems = 0;
  }
  if (w.qcap_emit < w.qn || w.emit == nullptr) {
    if (w.cap == 0 && h->cap0 > 0) w.cap = (uint32_t)h->cap0;
    if (w.cap == 0) {
      // flat: ~n/64 rows emitted per query at most on the bench data (19.5k
      // of 10M); growth (grow_emit) covers outliers, so cap the first guess
      int64_t c = std::min<int64_t>(h->n / 64, (int64_t)1 << 20);
      c = std::max<int64_t>(c, 16384);
      c = std::min<int64_t>(c, std::max<int64_t>(h->n, 1));
      int64_t p2 = 1;
      while (p2 < c) p2 <<= 1;
      w.cap = (uint32_t)std::min<int64_t>(p2, (int64_t)1 << 31);
    }
    DPQ_TRY(dmalloc(&w.emit_cnt, (size_t)w.qn));
    DPQ_TRY(dmalloc(&w.emit, (size_t)w.qn * w.cap));
    w.qcap_emit = w.qn;
  }
  if (r > w.rcap || w.h_out_elems < (size_t)w.qn * std::max(r, w.rcap)) {
    const int rc = std::max(r, w.rcap);
    DPQ_TRY(dmalloc(&w.out_d, (size_t)w.qn * rc));
    DPQ_TRY(dmalloc(&w.out_i, (size_t)w.qn * rc));
    DPQ_TRY(hmalloc(&w.h_d, (size_t)w.qn * rc));
    DPQ_TRY(hmalloc(&w.h_i, (size_t)w.qn * rc));
    w.rcap = rc;
    w.h_out_elems = (size_t)w.qn * rc;
  }
  return DPQ_OK;
}

static int grow_emit(Index* h, uint32_t need) {
  Workspace& w = h->ws;
  uint64_t c = w.cap;
  while (c < need) c <<= 1;
  c = std::min<uint64_t>(c, (uint64_t)1 << 31);
  w.cap = (uint32_t)c;
  DPQ_TRY(dmalloc(&w.emit, (size_t)w.qcap_emit * w.cap));
  return DPQ_OK;
}

static inline void ev_rec(Index* h, int i) {
  if (h->timing) cudaEventRecord(h->ev[i], h->stream);
}
static inline float ev_ms(Index* h, int a, int b) {
  float ms = 0.f;
  if (h->timing) cudaEventElapsedTime(&ms, h->ev[a], h->ev[b]);
  return ms;
}

// Fork / join: work enqueued on h->side between fork_side(h, i) and
// join_side(h, i) runs concurrently with h->stream's (graph capture records
// the two branches; eager runs overlap them the same way).
static int fork_side(Index* h, int i) {
  DPQ_CUDA(cudaEventRecord(h->fk[2 * i], h->stream));
  DPQ_CUDA(cudaStreamWaitEvent(h->side, h->fk[2 * i], 0));
  return DPQ_OK;
}
static int join_side(Index* h, int i) {
  DPQ_CUDA(cudaEventRecord(h->fk[2 * i + 1], h->side));
  DPQ_CUDA(cudaStreamWaitEvent(h->stream, h->fk[2 * i + 1], 0));
  return DPQ_OK;
}

// ---------------------------------------------------------------------------
// Launch helpers (template dispatch on MPAD)
// ---------------------------------------------------------------------------
static int num_sms(Index* h);

template <int MPAD, int QTX>
static int launch_hist_t(Index* h, int ntiles, const int* tile_list, int64_t stride,
                         int64_t nsamp, const uint8_t* plane, const int64_t* tile_row0 = nullptr,
                         const int64_t* tile_nsamp = nullptr, const int* slot_query = nullptr,
                         uint32_t* hist_out = nullptr) {
  using G = ScanGeom<MPAD, QTX>;
  const size_t smem = G::LUT_BYTES + (size_t)G::QT * 128 * 4;
  DPQ_TRY(set_smem(h, k_scan_hist<MPAD, kScanThreads, QTX>, smem));
  // one CTA per SM (the 128-KB LUT tile + counters fill its shared memory):
  // chunks per tile so the grid is a single wave
  int chunks = (int)std::max<int64_t>(1, std::min<int64_t>(num_sms(h) / ntiles, (nsamp + 511) / 512));
  int64_t per = (nsamp + chunks - 1) / chunks;
  per = (per + 31) / 32 * 32;
  per = std::min<int64_t>(per, kHistRowsPerCta / 32 * 32);  // u16 counters never wrap
  chunks = (int)((nsamp + per - 1) / per);
  if (chunks < 1) chunks = 1;
  dim3 grid(chunks, ntiles);
  k_scan_hist<MPAD, kScanThreads, QTX><<<grid, kScanThreads, smem, h->stream>>>(
      plane, stride, nsamp, per, h->ws.lut, tile_list, hist_out ? hist_out : h->ws.hist, tile_row0, tile_nsamp,
      slot_query);
  DPQ_LAUNCHED(h);
  return DPQ_OK;
}

// nsamp = samples per tile (the max when tile_nsamp is given per tile)
// slot_query / hist_out (ivf): per-query histograms [nq][256] directly
static int launch_hist(Index* h, int ntiles, const int* tile_list, int64_t stride, int64_t nsamp,
                       const uint8_t* plane, const int64_t* tile_row0 = nullptr,
                       const int64_t* tile_nsamp = nullptr, const int* slot_query = nullptr,
                       uint32_t* hist_out = nullptr) {
  if (ntiles < 1 || nsamp < 1) return DPQ_OK;
  if (h->mpad == 8)
    return launch_hist_t<8, 64>(h, ntiles, tile_list, stride, nsamp, plane, tile_row0, tile_nsamp, slot_query,
                                hist_out);
  if (h->qt == 64)
    return launch_hist_t<4, 64>(h, ntiles, tile_list, stride, nsamp, plane, tile_row0, tile_nsamp, slot_query,
                                hist_out);
  return launch_hist_t<4, 128>(h, ntiles, tile_list, stride, nsamp, plane, tile_row0, tile_nsamp, slot_query,
                               hist_out);
}

static int num_sms(Index* h) {
  if (!h->sms) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device) != cudaSuccess || sms < 1) sms = 148;
    h->sms = sms;
  }
  return h->sms;
}

template <int MPAD, int QTX>
static int launch_emit_t(Index* h, EmitArgs ea, int ntiles, int64_t rows) {
  using G = ScanGeom<MPAD, QTX>;
  constexpr int NW = kEmitThreads / 32;
  const size_t smem = emit_smem_bytes<MPAD, kEmitThreads, QTX>();
  DPQ_TRY(set_smem(h, k_scan_emit<MPAD, kEmitThreads, QTX>, smem));
  // Persistent CTAs (one per SM) pulling ~8 units each from a counter.
  const int sms = num_sms(h);
  ea.unit_counter = h->ws.counter;
  ea.one = 1u;
  ea.tile_fast = h->ws.tile_fast;
  ea.n_wide = h->d_nwide;
  ea.runs = h->rows_sorted ? 1 : 0;
  ea.n_lut = h->d_nrows + 2;
  if (ea.unit_tile) {  // caller-built units (ivf lists)
    if (ea.n_units < 1) return DPQ_OK;
    DPQ_CUDA(cudaMemsetAsync(h->ws.counter, 0, sizeof(unsigned), h->stream));
    k_scan_emit<MPAD, kEmitThreads, QTX><<<std::min(sms, ea.n_units), kEmitThreads, smem, h->stream>>>(ea);
    DPQ_LAUNCHED(h);
    return DPQ_OK;
  }
  if (ea.chunk_list) {  // run-filtered chunk lists, handed out dynamically (lengths on the device)
    ea.units_per_tile = 1;
    ea.n_units = ntiles;  // (list mode: the tile count)
    ea.rows_per_cta = 0;
    ea.list_next = h->ws.list_len + ntiles;
    DPQ_CUDA(cudaMemsetAsync(h->ws.list_len + ntiles, 0, (size_t)ntiles * sizeof(int), h->stream));
    k_scan_emit<MPAD, kEmitThreads, QTX><<<sms, kEmitThreads, smem, h->stream>>>(ea);
    DPQ_LAUNCHED(h);
    return DPQ_OK;
  }
  const int64_t min_rows = (int64_t)G::CHUNK_ROWS * NW;
  int64_t upt = std::max<int64_t>(1, (8LL * sms + ntiles - 1) / ntiles);  // ~8 units per CTA
  int64_t per = (rows + upt - 1) / upt;
  per = std::max(per, min_rows);
  per = (per + G::CHUNK_ROWS - 1) / G::CHUNK_ROWS * G::CHUNK_ROWS;
  upt = std::max<int64_t>(1, (rows + per - 1) / per);
  ea.rows_per_cta = per;
  ea.units_per_tile = (int)upt;
  ea.n_units = (int)(upt * ntiles);
  ea.unit_counter = h->ws.counter;
  ea.one = 1u;
  DPQ_CUDA(cudaMemsetAsync(h->ws.counter, 0, sizeof(unsigned), h->stream));
  const int grid = (int)std::min<int64_t>(sms, ea.n_units);
  k_scan_emit<MPAD, kEmitThreads, QTX><<<grid, kEmitThreads, smem, h->stream>>>(ea);
  DPQ_LAUNCHED(h);
  return DPQ_OK;
}

static int launch_emit(Index* h, EmitArgs ea, int ntiles, int64_t rows) {
  if (h->mpad == 8) return launch_emit_t<8, 64>(h, ea, ntiles, rows);
  if (h->qt == 64) return launch_emit_t<4, 64>(h, ea, ntiles, rows);
  return launch_emit_t<4, 128>(h, ea, ntiles, rows);
}

template <int BUF, int MODE>
static int launch_refine_buf(Index* h, const RefineArgs& ra, int nq) {
  // the query's residual block (ystride floats) is staged in shared memory
  // when it fits next to the buffer; otherwise it is read from global/L2
  // (ivf with a large ma * d)
  const size_t buf_bytes = (size_t)BUF * 16;
  RefineArgs rb = ra;
  static const int ysm_env = getenv("DPQ_REFINE_YSMEM") ? atoi(getenv("DPQ_REFINE_YSMEM")) : -1;
  // stage the block when it fits and is small (a query's full ivf residual block, ma * d floats, is
  // mostly probes without candidates: read it through L1/L2 instead)
  const size_t ymax = ysm_env >= 0 ? (ysm_env ? kRefineSmemMax : 0) : (size_t)8192;
  rb.y_in_smem = buf_bytes + (size_t)ra.ystride * 4 <= kRefineSmemMax && (size_t)ra.ystride * 4 <= ymax ? 1 : 0;
  const size_t smem = buf_bytes + (rb.y_in_smem ? (size_t)ra.ystride * 4 : 0);
  auto go = [&](auto kern) -> int {
    DPQ_TRY(set_smem(h, kern, smem));
    kern<<<nq, kTopThreads, smem, h->stream>>>(rb);
    return DPQ_OK;
  };
  if (MODE != MODE_EMIT && MODE != MODE_EMIT_APPROX) DPQ_TRY(go(k_refine_topk<BUF, kTopThreads, MODE, 0>));
  else if (ra.dsub == 32) DPQ_TRY(go(k_refine_topk<BUF, kTopThreads, MODE, 32>));
  else if (ra.dsub == 120) DPQ_TRY(go(k_refine_topk<BUF, kTopThreads, MODE, 120>));
  else DPQ_TRY(go(k_refine_topk<BUF, kTopThreads, MODE, 0>));
  DPQ_LAUNCHED(h);
  return DPQ_OK;
}

template <int MODE>
static int launch_refine(Index* h, const RefineArgs& ra, int nq) {
  const int need = ra.r + DPQ_REFINE_U * kTopThreads;  // DPQ_REFINE_U candidates per thread per round
  if (need <= 1024) return launch_refine_buf<1024, MODE>(h, ra, nq);
  if (need <= 2048) return launch_refine_buf<2048, MODE>(h, ra, nq);
  if (need <= 4096) return launch_refine_buf<4096, MODE>(h, ra, nq);
  if (need <= 8192) return launch_refine_buf<8192, MODE>(h, ra, nq);
  set_error("r=" + std::to_string(ra.r) + " exceeds the device top-r limit (7680)");
  return DPQ_ERR_ARG;
}

// ---------------------------------------------------------------------------
// K1 for nslot slots whose queries are already in ws.y.
// ---------------------------------------------------------------------------
int build_lut(Index* h, int nslot, const uint16_t* gword, const int* slot_query = nullptr,
              const int* slot_live = nullptr, const int* live = nullptr);
// K1 over nslot slots (or only the n_list slots of slot_list) and, with lut,
// the scan-layout LUT tiles of all nslot slots (slot_live: padding slots < 0).
int run_small_tables(Index* h, int nslot, const void* prefix, int64_t npre,
                     const int64_t* pre_off, const int64_t* pre_len, const double* bounds_in,
                     bool export_debug, const float* y_slots, const int* slot_list = nullptr,
                     int n_list = 0, bool lut = true, const int* slot_live = nullptr,
                     const int* y_sq = nullptr, const int* y_sp = nullptr, int y_ma = 0) {
  Workspace& w = h->ws;
  TablesArgs ta;
  ta.y = y_slots ? y_slots : w.y;
  ta.y_sq = y_sq; ta.y_sp = y_sp; ta.y_ma = y_ma;
  ta.dcb = h->dcb;
  ta.m = h->m; ta.kbar = h->kbar; ta.dsub = h->dsub; ta.mask = h->mask;
  ta.prefix = prefix; ta.code_bytes = h->code_bytes; ta.npre = npre;
  ta.prefix_off = pre_off; ta.prefix_len = pre_len; ta.bounds_in = bounds_in;
  ta.nslot = nslot;
  ta.small_out = export_debug ? w.small : nullptr;
  ta.q8_out = w.q8;  // read by k_group_tables
  ta.qmin_out = w.qmin; ta.qmax_out = w.qmax;
  ta.lut = w.lut; ta.mpad = h->mpad; ta.qt = qt_of(h);
  ta.cluster = (!pre_off && h->m >= 2) ? w.cluster : nullptr;  // flat: slot clustering keys
  const size_t smem = (size_t)(h->d + h->m * h->kbar) * 4 + (size_t)h->m * h->kbar + 16;
  ta.slot_list = slot_list;
  const int nlaunch = slot_list ? n_list : nslot;
  const char* ms_env = getenv("DPQ_MS_MIN");  // many-slot K1 from this slot count (default 256; test hook)
  const int ms_min = ms_env ? atoi(ms_env) : 256;
  const char* spc_env = getenv("DPQ_MS_SPC");  // slots per CTA of the many-slot K1 (2, 4 or 8)
  // 4 slots per CTA at flat batch sizes (1024 queries: 256 CTAs, tables 59 -> 48 us), 8 for IVF slot counts
  const int spc = spc_env ? atoi(spc_env) : (nlaunch >= 8192 ? 8 : 4);
  const bool many = nlaunch >= ms_min && (h->dsub & 7) == 0 && h->dsub <= 128;
  if (nlaunch > 0 && many) {  // IVF-size slot counts: spc slots per CTA
    auto go = [&](auto kern, int S) -> int {
      const size_t smem_ms = (size_t)S * (h->d + h->m * h->kbar) * 4;
      DPQ_TRY(set_smem(h, kern, smem_ms));
      kern<<<(nlaunch + S - 1) / S, 256, smem_ms, h->stream>>>(ta, nlaunch);
      return DPQ_OK;
    };
    if (spc == 2) DPQ_TRY(go(k_small_tables_ms<2>, 2));
    else if (spc == 4) DPQ_TRY(go(k_small_tables_ms<4>, 4));
    else DPQ_TRY(go(k_small_tables_ms<8>, 8));
    DPQ_LAUNCHED(h);
  } else if (nlaunch > 0) {
    DPQ_TRY(set_smem(h, k_small_tables, smem));
    k_small_tables<<<nlaunch, 256, smem, h->stream>>>(ta);
    DPQ_LAUNCHED(h);
  }
  return lut ? build_lut(h, nslot, nullptr, nullptr, slot_live) : DPQ_OK;
}

// Scan-layout LUT tiles from ws.q8; with gword (guards known) tiles whose
// guards are all <= 126 are clamped to 7-bit entries and flagged fast.
int build_lut(Index* h, int nslot, const uint16_t* gword, const int* slot_query, const int* slot_live,
              const int* live) {
  Workspace& w = h->ws;
  const int ntiles = tiles_of(nslot, h);
  int* tf = w.tile_fast;  // reset to 0 when gword is null (unclamped LUT)
  const dim3 grid((unsigned)ntiles, (unsigned)h->mpad);
  if (h->mpad == 8)
    k_build_lut<8, 64><<<grid, 256, 0, h->stream>>>(w.q8, nslot, h->m, h->kbar, w.lut, ntiles, gword, tf, h->wide,
                                                    slot_query, slot_live, live);
  else if (h->qt == 64)
    k_build_lut<4, 64><<<grid, 256, 0, h->stream>>>(w.q8, nslot, h->m, h->kbar, w.lut, ntiles, gword, tf, h->wide,
                                                    slot_query, slot_live, live);
  else
    k_build_lut<4, 128><<<grid, 256, 0, h->stream>>>(w.q8, nslot, h->m, h->kbar, w.lut, ntiles, gword, tf, h->wide,
                                                     slot_query, slot_live, live);
  DPQ_LAUNCHED(h);
  return DPQ_OK;
}

// ---------------------------------------------------------------------------
// First pass for a flat batch (slots = queries): guard, scan, b*.  Handles
// the rare exact redo and emit overflow.  On return ws.bstar / emit are
// valid for every query of the batch.
// ---------------------------------------------------------------------------
// Flat scan preparation once the guards are known (ws.gword by query):
// query slots clustered into tiles (k_sort_slots), clamped LUT tiles, and
// with sorted rows the run-filtered chunk lists.  Shared by the single-GPU
// first pass and the sharded scan (dpq_shard_scan).
struct ScanPlan {
  bool sorted = false, list = false, direct = false;
  bool skip_tiles = false;      // (single-GPU speculative first pass only) tile kernels not launched
  bool scan_hist = false;       // (with skip_tiles) the direct scan counts its hits by score into ws.hist for K3
  const uint32_t* hist = nullptr;  // when set, k_key_select computes the guard itself (k_guard's rule)
  int r2 = 0, exact = 0;
  double lambda = 0.0;
  int item_cap = 0;
  const uint16_t* gw = nullptr;
  const int* slot_q = nullptr;
};

int plan_flat_scan(Index* h, int nb, ScanPlan& sp) {
  Workspace& w = h->ws;
  const int tiles = tiles_of(nb, h);
  sp.list = h->rows_sorted && h->run_filter && h->m >= 2 && h->n > 0;
  // query tiles clustered by guard class and nearest (g0, g1): feeds the
  // wide loop (MPAD 4) and makes the per-tile run filter selective
  sp.sorted = h->sort_slots && nb > 1 && (h->mpad == 4 ? h->wide != 0 : sp.list);
  if (sp.list && (w.list_tiles < tiles || w.list_chunks < h->n_chunks)) {
    DPQ_TRY(dmalloc(&w.pot, (size_t)tiles * 65536));
    DPQ_TRY(dmalloc(&w.chunk_list, (size_t)tiles * h->n_chunks));
    DPQ_TRY(dmalloc(&w.list_len, (size_t)tiles * 2));  // lengths | handed-out counters
    w.list_tiles = tiles;
    w.list_chunks = h->n_chunks;
  }
  sp.gw = sp.sorted ? w.gword_p : w.gword;
  sp.slot_q = sp.sorted ? w.slot_query : nullptr;
  // queries with few (g0, g1) keys under their guard are scanned one by one (k_scan_direct)
  sp.direct = sp.list && h->direct && h->key_start && nb <= kDirMaxBatch;
  if (sp.direct) {
    // budget: on average n / 64 rows per query (beyond that the tile scan, which shares one pass over the
    // rows between 128 queries, is cheaper), never less than 192 items per query
    const int64_t per_q = std::max<int64_t>(192, h->n / ((int64_t)kDirSeg * 64) + 64);
    sp.item_cap = h->direct_items > 0 ? h->direct_items
                                      : (int)std::min<int64_t>((int64_t)1 << 26, std::max<int64_t>(4096, per_q * nb));
    if (w.dir_items_cap < sp.item_cap) {
      DPQ_TRY(dmalloc(&w.dir_items, (size_t)sp.item_cap));
      w.dir_items_cap = sp.item_cap;
    }
    if (!w.dir_state) DPQ_TRY(dmalloc(&w.dir_state, 4));
    if (!w.h_tileq) DPQ_TRY(hmalloc(&w.h_tileq, 1));
    if (h->gt_slack && h->m <= 8 && w.slack_cap < nb * h->m) {
      DPQ_TRY(dmalloc(&w.slack, (size_t)nb * h->m));
      w.slack_cap = nb * h->m;
    }
  }
  return DPQ_OK;
}

static bool scan_hist_on(const Index* h) { return h->scan_hist >= 0 ? h->scan_hist != 0 : !h->emit32; }

int prepare_flat_scan(Index* h, int nb, const ScanPlan& sp) {
  Workspace& w = h->ws;
  const int qt = qt_of(h);
  const int tiles = tiles_of(nb, h);
  const int* live = nullptr;  // direct scan: the tile kernels return at once when no query is left to them
  if (sp.direct) {
    DPQ_CUDA(cudaMemsetAsync(w.dir_state, 0, 4 * sizeof(int), h->stream));
    KeySelArgs ka;
    ka.q8 = w.q8; ka.m = h->m; ka.kbar = h->kbar; ka.guard_b = w.guard_b; ka.gword = w.gword;
    ka.key_start = h->key_start; ka.items = w.dir_items; ka.state = w.dir_state;
    ka.item_cap = sp.item_cap; ka.item_qcap = std::max(64, sp.item_cap / 8); ka.pair_cap = 16384;
    ka.n_rows = h->d_nrows;
    ka.hist = sp.hist; ka.r2 = sp.r2; ka.exact = sp.exact; ka.lambda = sp.lambda;
    ka.skip_tiles = sp.skip_tiles ? 1 : 0;
    ka.zero_hist = (sp.scan_hist && sp.hist) ? 1 : 0;
    if (h->gt_slack && h->m <= 8) ka.slack = w.slack;
    k_key_select<<<nb, 256, 0, h->stream>>>(ka, nb);
    DPQ_LAUNCHED(h);
    w.slack_ready = ka.slack != nullptr;
    live = w.dir_state + 1;
    if (sp.skip_tiles) return DPQ_OK;  // no tile kernels at all (see Index::tile_skip)
  } else {
    w.slack_ready = false;
  }
  if (sp.sorted) {
    k_sort_slots<<<1, 1024, 0, h->stream>>>(w.gword, h->m >= 2 ? w.cluster : nullptr, nb, tiles * qt,
                                            w.slot_query, w.gword_p, live);
    DPQ_LAUNCHED(h);
  }
  if (sp.list) {
    // the LUT tiles (side branch) and the run filter (main) both follow the slot order only
    DPQ_TRY(fork_side(h, 0));
    cudaStream_t main_stream = h->stream;
    h->stream = h->side;
    const int rc = build_lut(h, nb, sp.gw, sp.slot_q, nullptr, live);  // clamped tiles (modes 5/6/7) where the guards allow
    h->stream = main_stream;
    DPQ_TRY(rc);
  } else {
    DPQ_TRY(build_lut(h, nb, sp.gw, sp.slot_q, nullptr, live));
  }
  if (sp.list) {  // run filter: per tile, the chunks whose (g0, g1) keys can reach a guard
    DPQ_CUDA(cudaMemsetAsync(w.list_len, 0, (size_t)tiles * 4, h->stream));
    k_run_potential<<<dim3(256 / kRunG0, tiles), 256, (size_t)qt * 64 * 4 + kRunG0 * qt * 4, h->stream>>>(
        w.q8, h->m, h->kbar, sp.slot_q, sp.gw, qt, nb, w.pot, live);
    DPQ_LAUNCHED(h);
    k_chunk_list<<<dim3((unsigned)((h->n_chunks + 256 * kChunkPerThread - 1) / (256 * kChunkPerThread)), tiles), 256, 0,
                   h->stream>>>(
        h->chunk_keys, (int)h->n_chunks, 512 / h->mpad, w.pot, w.chunk_list, w.list_len, h->n, nb, qt, h->d_nrows,
        live);
    DPQ_LAUNCHED(h);
    DPQ_TRY(join_side(h, 0));
  }
  return DPQ_OK;
}

// The direct scan of the queries k_key_select took (after launch_emit: both
// append to the emit lists with atomics, in any order).
int launch_direct(Index* h, const ScanPlan& sp) {
  if (!sp.direct) return DPQ_OK;
  Workspace& w = h->ws;
  DirectArgs da;
  da.plane = h->plane; da.q8 = w.q8; da.m = h->m; da.kbar = h->kbar; da.guard_b = w.guard_b;
  da.items = w.dir_items; da.state = w.dir_state; da.item_cap = sp.item_cap;
  da.emit_cnt = w.emit_cnt; da.emit = w.emit; da.cap = w.cap;
  da.hist = sp.scan_hist ? w.hist : nullptr;
  // one wave of resident CTAs, items strided over their warps
  auto go = [&](auto kern, int slot) -> int {
    static int per_sm[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (!per_sm[slot]) {
      int nb = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, 256, 0) != cudaSuccess || nb < 1) nb = 4;
      per_sm[slot] = nb;
    }
    kern<<<per_sm[slot] * num_sms(h), 256, 0, h->stream>>>(da);
    return DPQ_OK;
  };
  if (da.hist) {
    if (h->mpad == 8) {
      if (h->emit32) go(k_scan_direct<8, true, true>, 4);
      else go(k_scan_direct<8, false, true>, 5);
    } else {
      if (h->emit32) go(k_scan_direct<4, true, true>, 6);
      else go(k_scan_direct<4, false, true>, 7);
    }
  } else if (h->mpad == 8) {
    if (h->emit32) go(k_scan_direct<8, true>, 0);
    else go(k_scan_direct<8, false>, 1);
  } else {
    if (h->emit32) go(k_scan_direct<4, true>, 2);
    else go(k_scan_direct<4, false>, 3);
  }
  DPQ_LAUNCHED(h);
  return DPQ_OK;
}

void plan_emit_args(Index* h, const ScanPlan& sp, EmitArgs& ea) {
  ea.gword = sp.gw;
  ea.live = sp.direct ? h->ws.dir_state + 1 : nullptr;
  ea.slot_query = sp.slot_q;
  ea.chunk_list = sp.list ? h->ws.chunk_list : nullptr;
  ea.list_len = h->ws.list_len;
  ea.list_stride = h->n_chunks;
}

static int flat_first_pass(Index* h, int nb, int r2) {
  if (h->order_forked) {  // (a previous first pass that did not reach its refine)
    h->order_forked = false;
    DPQ_TRY(join_side(h, 1));
  }
  Workspace& w = h->ws;
  const int qt = qt_of(h);
  const int tiles = tiles_of(nb, h);
  // guard words of padding slots never hit: 0x7F7F < 0x8000
  DPQ_CUDA(cudaMemsetAsync(w.gword, 0x7F, (size_t)tiles * qt * 2, h->stream));
  DPQ_CUDA(cudaMemsetAsync(w.hist, 0, (size_t)tiles * qt * 256 * 4, h->stream));
  const int64_t n = h->n;
  const bool exact = n <= h->exact_limit;
  const int64_t nsamp = exact ? n : std::min<int64_t>(n, h->sample);
  const int64_t stride = exact ? 1 : n / nsamp;
  DPQ_TRY(launch_hist(h, tiles, nullptr, stride, nsamp, h->plane));
  const double lambda = (double)r2 * (double)nsamp / (double)std::max<int64_t>(n, 1);
  ScanPlan sp;
  DPQ_TRY(plan_flat_scan(h, nb, sp));
  h->dir_batch = sp.direct;
  if (sp.direct) {  // k_key_select computes the guard itself
    sp.hist = w.hist; sp.r2 = r2; sp.exact = exact ? 1 : 0; sp.lambda = lambda;
    sp.skip_tiles = h->tile_skip && h->tile_skip_ok && !h->no_spec && nb > 1;
    sp.scan_hist = sp.skip_tiles && scan_hist_on(h);  // every emitted record then comes from k_scan_direct
  } else {
    k_guard<<<(nb + kGuardSlotsPerCta - 1) / kGuardSlotsPerCta, 32 * kGuardSlotsPerCta, 0, h->stream>>>(w.hist, nb, r2, lambda, exact ? 1 : 0, nullptr,
                                                      w.guard_b, w.gword, nullptr);
    DPQ_LAUNCHED(h);
  }
  auto sort_and_build = [&]() -> int { return prepare_flat_scan(h, nb, sp); };
  DPQ_TRY(sort_and_build());
  sp.hist = nullptr;  // (an exact redo below sets its guards with k_guard)
  ev_rec(h, 2);
  bool first = true;
  for (int attempt = 0; attempt < 8; ++attempt) {
    DPQ_CUDA(cudaMemsetAsync(w.emit_cnt, 0, (size_t)nb * 4, h->stream));
    EmitArgs ea;
    ea.plane = h->plane; ea.row_begin = 0; ea.row_end = n; ea.rows_per_cta = 0;
    ea.lut = w.lut; ea.tile_list = nullptr; ea.slot_probe = nullptr;
    plan_emit_args(h, sp, ea);
    ea.unit_tile = nullptr; ea.unit_r0 = nullptr; ea.unit_r1 = nullptr;
    ea.emit_cnt = w.emit_cnt; ea.emit = w.emit; ea.cap = w.cap; ea.emit32 = (int)h->emit32;
    if (!sp.skip_tiles) DPQ_TRY(launch_emit(h, ea, tiles, n));
    DPQ_TRY(launch_direct(h, sp));
    if (!sp.list) {  // (list mode: counted on the device)
      h->counters[2] += (int64_t)nb * n;
      h->plane_rows += (int64_t)tiles * n;
    }
    if (first) ev_rec(h, 3);
    if (!h->no_spec && nb > 1 && attempt == 0) {
      // the refine order (heaviest emit lists first) needs only the emit
      // counts: computed on the side branch while K3 runs
      DPQ_TRY(fork_side(h, 1));
      k_order_by_count<<<1, 1024, 0, h->side>>>(w.emit_cnt, nb, w.cap, w.order);
      DPQ_LAUNCHED(h);
      h->order_forked = true;
    }
    k_threshold<256><<<nb, 256, 0, h->stream>>>(w.emit, w.emit_cnt, w.cap, w.guard_b, r2, nullptr,
                                                w.bstar, w.ncand, w.flags, nullptr, h->d_nemit, (int)h->emit32,
                                                (sp.scan_hist && attempt == 0) ? w.hist : nullptr);
    DPQ_LAUNCHED(h);
    if (first) ev_rec(h, 4);
    first = false;
    DPQ_CUDA(cudaMemcpyAsync(w.h_flags, w.flags, nb, cudaMemcpyDeviceToHost, h->stream));
    if (sp.direct && attempt == 0)
      DPQ_CUDA(cudaMemcpyAsync(w.h_tileq, w.dir_state + 1, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    if (!h->no_spec) {
      // speculative: the batch goes on (flagged queries have b* = -1 and
      // refine nothing); the caller checks h_flags after its final sync and
      // redoes the batch without speculation if any query was flagged
      h->spec_nb = nb;
      return DPQ_OK;
    }
    DPQ_CUDA(cudaStreamSynchronize(h->stream));
    bool any_exact = false, any_over = false;
    for (int q = 0; q < nb; ++q) {
      any_exact |= w.h_flags[q] == 1;
      any_over |= w.h_flags[q] == 2;
    }
    if (!any_exact && !any_over) return DPQ_OK;
    h->counters[4]++;
    if (any_over) {
      DPQ_CUDA(cudaMemcpyAsync(w.h_cnt, w.emit_cnt, (size_t)nb * 4, cudaMemcpyDeviceToHost, h->stream));
      DPQ_CUDA(cudaStreamSynchronize(h->stream));
      uint32_t need = 0;
      for (int q = 0; q < nb; ++q)
        if (w.h_flags[q] == 2) need = std::max(need, w.h_cnt[q]);
      if ((size_t)w.qcap_emit * need * 8 > h->emit_budget && nb > 1) return 100;  // split batch
      DPQ_TRY(grow_emit(h, need));
    }
    if (any_exact) {
      // exact histogram for every tile holding a flagged query
      std::vector<int> tl;
      for (int t = 0; t < tiles; ++t) {
        bool f = false;
        for (int q = t * qt; q < std::min(nb, (t + 1) * qt); ++q) f |= w.h_flags[q] == 1;
        if (f) tl.push_back(t);
      }
      for (int q = 0; q < nb; ++q) w.h_flags[q] = w.h_flags[q] == 1;
      DPQ_CUDA(cudaMemcpyAsync(w.only, w.h_flags, nb, cudaMemcpyHostToDevice, h->stream));
      DPQ_CUDA(cudaMemcpyAsync(w.tile_list, tl.data(), tl.size() * sizeof(int), cudaMemcpyHostToDevice,
                               h->stream));
      DPQ_CUDA(cudaMemsetAsync(w.hist, 0, (size_t)tiles * qt * 256 * 4, h->stream));
      DPQ_TRY(build_lut(h, nb, nullptr));  // exact histogram needs unclamped entries
      DPQ_TRY(launch_hist(h, (int)tl.size(), w.tile_list, 1, n, h->plane));
      k_guard<<<(nb + kGuardSlotsPerCta - 1) / kGuardSlotsPerCta, 32 * kGuardSlotsPerCta, 0, h->stream>>>(w.hist, nb, r2, 0.0, 1, w.only, w.guard_b, w.gword,
                                                        nullptr);
      DPQ_LAUNCHED(h);
      DPQ_TRY(sort_and_build());
      DPQ_CUDA(cudaStreamSynchronize(h->stream));
    }
  }
  set_error("first pass did not converge");
  return DPQ_ERR_CUDA;
}

static RefineArgs make_refine_args(Index* h, int r) {
  Workspace& w = h->ws;
  RefineArgs ra;
  ra.emit = w.emit; ra.emit_cnt = w.emit_cnt; ra.cap = w.cap; ra.bstar = w.bstar; ra.emit32 = (int)h->emit32;
  ra.n_rows = h->n;
  ra.codes = h->codes; ra.code_bytes = h->code_bytes; ra.m = h->m; ra.k = h->k; ra.dsub = h->dsub;
  ra.kbar = h->kbar; ra.bbar = h->bbar;
  ra.cb = h->cb; ra.tables = w.tables; ra.y = w.y; ra.ystride = h->d;
  ra.row_ids = h->sorted_ids; ra.id_base = h->id_base; ra.r = r;  // sorted flat rows -> ids
  ra.out_d = w.out_d; ra.out_i = w.out_i; ra.n_refined = h->d_nref;
  if (h->host_out) {  // pinned host memory is device-addressable (UVA): results cross PCIe as CTAs finish
    ra.out_d = w.h_d;
    ra.out_i = w.h_i;
  } else if (h->dev_out_d) {
    ra.out_d = h->dev_out_d;
    ra.out_i = h->dev_out_i;
  }
  return ra;
}

static int ensure_tables(Index* h, int nq) {
  Workspace& w = h->ws;
  const int64_t need = (int64_t)nq * h->m * h->k;
  if (need > w.tables_elems) {
    DPQ_TRY(dmalloc(&w.tables, (size_t)need));
    w.tables_elems = need;
  }
  return DPQ_OK;
}

static bool group_tables_fit(Index* h, int nq) {
  const size_t smem = (size_t)(h->k / h->kbar) * (h->dsub + 4) * 4 + (size_t)nq * 4;
  return smem <= 200 * 1024;
}

// Group-lazy exact tables for the batch (after K3 set ws.bstar).
int run_group_tables(Index* h, int nq, int ystride) {
  Workspace& w = h->ws;
  DPQ_TRY(ensure_tables(h, nq));
  GroupTablesArgs ga;
  ga.cb = h->cb; ga.y = w.y; ga.ystride = ystride; ga.q8 = w.q8; ga.bstar = w.bstar;
  ga.nq = nq; ga.m = h->m; ga.k = h->k; ga.kbar = h->kbar; ga.bbar = h->bbar; ga.dsub = h->dsub;
  ga.tables = w.tables; ga.n_entries = h->d_nent;
  if (h->m <= 8 && h->gt_slack) {  // tighter activity test: the other subspaces' smallest entries count too
    if (w.slack_cap < nq * h->m) {
      DPQ_TRY(dmalloc(&w.slack, (size_t)nq * h->m));
      w.slack_cap = nq * h->m;
    }
    if (!w.slack_ready) {  // (else k_key_select wrote this batch's slack)
      k_entry_slack<<<(nq + 3) / 4, 128, 0, h->stream>>>(w.q8, nq, h->m, h->kbar, w.slack);
      DPQ_LAUNCHED(h);
    }
    w.slack_ready = false;
    ga.slack = w.slack;
  }
  const int gsize = h->k / h->kbar;
  const int ld = ((h->dsub & 7) == 0 && h->dsub <= 128) ? h->dsub + 4 : h->dsub + 1;  // k_group_tables rows
  const size_t smem = (size_t)gsize * ld * 4 + (size_t)nq * 4;
  dim3 grid(h->kbar, h->m);
  if (h->dsub == 32) {
    const size_t sm2 = (size_t)32 * 32 * 4 + (size_t)nq * 4;
    DPQ_TRY(set_smem(h, k_group_tables_reg<32>, sm2));
#ifndef DPQ_K5_SPLIT
#define DPQ_K5_SPLIT 2  // CTAs per (group, subspace): the busiest groups bound K5 (A/B: 1 -> 2 saves ~10 us)
#endif
    k_group_tables_reg<32><<<dim3(grid.x, grid.y, DPQ_K5_SPLIT), 256, sm2, h->stream>>>(ga);
  } else {
    DPQ_TRY(set_smem(h, k_group_tables<0>, smem));
    k_group_tables<0><<<grid, 256, smem, h->stream>>>(ga);
  }
  DPQ_LAUNCHED(h);
  return DPQ_OK;
}

// Tensor-core full tables (dpq_tctab.cu) instead of the lazy exact group
// tables: used where the lazy builder's CUDA-core work is large (dsub >= 64,
// e.g. BASELINE configs[4]: 8 x 65536 x 120), or forced by DPQ_TC_TABLES.
// Auto: large sub-vectors, unless the candidate fraction is small (r2 / n <=
// 1 / 4096): then the slack-tightened lazy tables touch so few groups (configs[4]:
// 7.6k of 524k entries per query) that they beat the full GEMM by far.
static bool use_tc_tables(Index* h, int r2) {
  const bool few = h->gt_slack && r2 > 0 && (int64_t)r2 * 4096 <= h->n;
  const int mode = h->use_tc >= 0 ? h->use_tc : ((h->dsub >= 64 && !few) ? 1 : 0);
  return mode != 0 && tct_supported(h->m, h->k, h->kbar, h->dsub);
}

static int ensure_tct(Index* h) {
  if (h->tct) return DPQ_OK;
  return tct_prepare(h->device, h->cb, h->m, h->k, h->kbar, h->dsub, h->stream, &h->tct);
}

// Approximate full tables of nq query rows y (device, row stride ystride)
// into ws.tables (group-major) with their error bounds in tct_eps.
int run_tc_tables(Index* h, int nq, const float* y, int64_t ystride) {
  DPQ_TRY(ensure_tct(h));
  DPQ_TRY(ensure_tables(h, nq));
  if ((int64_t)nq * h->m > h->tct_eps_cap) {
    DPQ_TRY(dmalloc(&h->tct_eps, (size_t)nq * h->m));
    DPQ_TRY(dmalloc(&h->tct_ny, (size_t)nq * h->m));
    h->tct_eps_cap = (int64_t)nq * h->m;
  }
  DPQ_TRY(tct_build(h->tct, y, ystride, nq, h->ws.tables, h->tct_eps, h->tct_ny, h->tc_eps_scale, h->stream));
  h->counters[0]++;
  return DPQ_OK;
}

// One flat derived batch: queries already in ws.y (nb rows), results into
// ws.out_d / ws.out_i.  Returns 100 when the batch must be split.
static int flat_derived_batch_body(Index* h, int nb, int r, int r2);

// One flat derived batch.  The speculative pipeline (no host decision until
// the flags come back with the results) is captured once per (batch size,
// r, r2, allocation epoch) into a CUDA graph and replayed: one launch instead
// of ~20 kernel launches and memsets per batch.  The first call with a new
// configuration runs eagerly (it sizes every buffer), the second captures.
static int flat_derived_batch(Index* h, int nb, int r, int r2) {
  if (use_tc_tables(h, r2)) DPQ_TRY(ensure_tct(h));  // (synchronous, never inside a graph capture)
  const bool graphable = h->use_graph && !h->timing && !h->no_spec;
  if (!graphable) return flat_derived_batch_body(h, nb, r, r2);
  BatchGraph& G = h->graph;
  const bool same = G.nb == nb && G.r == r && G.r2 == r2 && G.host_out == (int)h->host_out &&
                    G.tile_skip == h->tile_skip && G.dev_out == (const void*)h->dev_out_d &&
                    G.epoch == g_alloc_epoch;
  if (G.exec && same) {
    DPQ_CUDA(cudaGraphLaunch(G.exec, h->stream));
    for (int i = 0; i < 8; ++i) h->counters[i] += G.counters[i];
    h->spec_nb = nb;
    return DPQ_OK;
  }
  if (!same || !G.warm) {  // eager run; capture on the next call with this configuration
    if (G.exec) { cudaGraphExecDestroy(G.exec); G.exec = nullptr; }
    const int rc = flat_derived_batch_body(h, nb, r, r2);
    G.nb = nb; G.r = r; G.r2 = r2; G.host_out = (int)h->host_out; G.tile_skip = h->tile_skip; G.dev_out = h->dev_out_d; G.epoch = g_alloc_epoch; G.warm = rc == DPQ_OK;
    return rc;
  }
  int64_t c0[8];
  for (int i = 0; i < 8; ++i) c0[i] = h->counters[i];
  DPQ_CUDA(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
  const int rc = flat_derived_batch_body(h, nb, r, r2);
  cudaGraph_t graph = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(h->stream, &graph);
  if (rc != DPQ_OK || ce != cudaSuccess || G.epoch != g_alloc_epoch) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    G.warm = false;
    h->use_graph = 0;  // something in the pipeline is not capturable: stay eager
    return flat_derived_batch_body(h, nb, r, r2);
  }
  for (int i = 0; i < 8; ++i) G.counters[i] = h->counters[i] - c0[i];
  const cudaError_t ie = cudaGraphInstantiate(&G.exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ie != cudaSuccess) {
    cudaGetLastError();
    G.exec = nullptr;
    h->use_graph = 0;
    return flat_derived_batch_body(h, nb, r, r2);
  }
  DPQ_CUDA(cudaGraphLaunch(G.exec, h->stream));
  h->spec_nb = nb;
  return DPQ_OK;
}

static int flat_derived_batch_body(Index* h, int nb, int r, int r2) {
  ev_rec(h, 0);
  const int64_t npre = std::min<int64_t>(r2, h->n_prefix);
  DPQ_TRY(run_small_tables(h, nb, h->prefix, npre, nullptr, nullptr, nullptr, false, nullptr));
  ev_rec(h, 1);
  int rc = flat_first_pass(h, nb, r2);
  if (rc != DPQ_OK) return rc;
  ev_rec(h, 5);
  RefineArgs ra = make_refine_args(h, r);
  if (h->order_forked) {  // computed on the side branch during K3
    h->order_forked = false;
    DPQ_TRY(join_side(h, 1));
    ra.order = h->ws.order;
  } else if (nb > 1) {  // heaviest emit lists first
    k_order_by_count<<<1, 1024, 0, h->stream>>>(h->ws.emit_cnt, nb, h->ws.cap, h->ws.order);
    DPQ_LAUNCHED(h);
    ra.order = h->ws.order;
  }
  if (use_tc_tables(h, r2)) {  // tensor-core full tables + exact re-rank of the margin set
    DPQ_TRY(run_tc_tables(h, nb, h->ws.y, h->d));
    ra.tables = h->ws.tables;
    ra.ny = h->tct_ny;
    ra.cnorm = tct_cnorm(h->tct);
    ra.gamma = tct_gamma(h->tct, h->tc_eps_scale);
    ra.n_exact = h->d_nrows + 3;
    DPQ_TRY(launch_refine<MODE_EMIT_APPROX>(h, ra, nb));
  } else if (group_tables_fit(h, nb)) {
    DPQ_TRY(run_group_tables(h, nb, h->d));
    ra.tables = h->ws.tables;  // (re)allocated by run_group_tables
    DPQ_TRY(h->emit32 ? launch_refine<MODE_EMIT_TABLE32>(h, ra, nb) : launch_refine<MODE_EMIT_TABLE>(h, ra, nb));
  } else {
    DPQ_TRY(launch_refine<MODE_EMIT>(h, ra, nb));  // entries computed per candidate
  }
  ev_rec(h, 6);
  h->counters[1] += nb;
  if (h->timing) {
    DPQ_CUDA(cudaEventSynchronize(h->ev[6]));
    h->phase_ms[PH_TABLES] = ev_ms(h, 0, 1);
    h->phase_ms[PH_GUARD] = ev_ms(h, 1, 2);
    h->phase_ms[PH_SCAN] = ev_ms(h, 2, 3);
    h->phase_ms[PH_THRESH] = ev_ms(h, 3, 4);
    h->phase_ms[PH_FALLBACK] = ev_ms(h, 4, 5);
    h->phase_ms[PH_REFINE] = ev_ms(h, 5, 6);
    h->phase_ms[PH_TOTAL] = ev_ms(h, 0, 6);
  }
  return DPQ_OK;
}

static int flat_conventional_batch(Index* h, int nb, int r) {
  Workspace& w = h->ws;
  ev_rec(h, 0);
  DPQ_TRY(ensure_tables(h, nb));
  dim3 grid((h->k + 255) / 256, h->m, nb);  // NB: make_refine_args below reads ws.tables
  k_full_tables<<<grid, 256, h->dsub * 4, h->stream>>>(w.y, h->cb, h->m, h->k, h->kbar, h->bbar, h->dsub, 1,
                                                       w.tables);
  DPQ_LAUNCHED(h);
  ev_rec(h, 1);
  RefineArgs ra = make_refine_args(h, r);
  DPQ_TRY(launch_refine<MODE_ALL>(h, ra, nb));
  ev_rec(h, 2);
  h->counters[1] += nb;
  if (h->timing) {
    DPQ_CUDA(cudaEventSynchronize(h->ev[2]));
    h->phase_ms[PH_TABLES] = ev_ms(h, 0, 1);
    h->phase_ms[PH_SCAN] = ev_ms(h, 1, 2);
    h->phase_ms[PH_REFINE] = 0.f;
    h->phase_ms[PH_TOTAL] = ev_ms(h, 0, 2);
  }
  return DPQ_OK;
}

// Generic host-buffer driver: splits nq into batches, stages through pinned
// memory, calls `batch(nb)` and copies results back.
// Host staging copies (queries in, results out) split over a few OpenMP
// threads: one thread moves ~20 GB/s, a 1024-query batch is ~2 MB.
static void par_memcpy2(void* d0, const void* s0, size_t b0, void* d1, const void* s1, size_t b1) {
  constexpr size_t kMin = 256 << 10;
  const size_t tot = b0 + b1;
  if (tot < kMin) { memcpy(d0, s0, b0); if (b1) memcpy(d1, s1, b1); return; }
  const int nt = (int)std::min<size_t>(8, tot / (kMin / 2));
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int t = 0; t < nt; ++t) {  // thread t copies bytes [a, b) of the concatenation
    const size_t a = tot * t / nt, b = tot * (t + 1) / nt;
    if (a < b0) memcpy((char*)d0 + a, (const char*)s0 + a, std::min(b, b0) - a);
    if (b > b0) {
      const size_t a1 = std::max(a, b0) - b0, e1 = b - b0;
      memcpy((char*)d1 + a1, (const char*)s1 + a1, e1 - a1);
    }
  }
}
static void par_memcpy(void* dst, const void* src, size_t bytes) { par_memcpy2(dst, src, bytes, nullptr, nullptr, 0); }

// The staging copy of a float32 query batch with the finiteness scan of
// check_array riding on it (each thread scans the slice it just copied, still
// in its cache): returns true when a NaN or +-inf was seen.
static bool par_memcpy_check_f32(float* dst, const float* src, size_t n) {
  constexpr size_t kMin = 64 << 10;  // floats (256 KB)
  const int nt = n < kMin ? 1 : (int)std::min<size_t>(8, n / (kMin / 2));
  uint32_t special = 0;
#pragma omp parallel for num_threads(nt) schedule(static) reduction(| : special)
  for (int t = 0; t < nt; ++t) {
    const size_t a = n * t / nt, b = n * (t + 1) / nt;
    memcpy(dst + a, src + a, (b - a) * 4);
    const uint32_t* w = reinterpret_cast<const uint32_t*>(dst + a);
    uint32_t s = 0;
    for (size_t i = 0; i < b - a; ++i) s |= (uint32_t)((w[i] & 0x7F800000u) == 0x7F800000u);
    special |= s;
  }
  return special != 0;
}

// Wait for the stream, then copy the staged results to the caller's buffers.
// The threads touch their slice of the destination pages while the GPU still
// works (first-touch faults of freshly allocated numpy results cost ~70 us
// per 1.6 MB), then spin until the stream is done and copy — no OpenMP
// sleep/wake latency after a ~1 ms wait.
static cudaError_t sync_copy_out(cudaStream_t st, void* d0, const void* s0, size_t b0, void* d1, const void* s1,
                                 size_t b1) {
  const size_t tot = b0 + b1;
  const int nt = tot < (256u << 10) ? 1 : (int)std::min<size_t>(8, tot / (128u << 10));
  std::atomic<int> state{0};  // 0 wait, 1 copy, 2 error
  cudaError_t err = cudaSuccess;
#pragma omp parallel num_threads(nt)
  {
    const int t = omp_get_thread_num(), T = omp_get_num_threads();
    const size_t a = tot * t / T, b = tot * (t + 1) / T;
    auto dst = [&](size_t o) -> volatile char* {
      return o < b0 ? (volatile char*)d0 + o : (volatile char*)d1 + (o - b0);
    };
    for (size_t o = a; o < b; o = (o | 4095) + 1) *dst(o) = 0;
    if (t == 0) {
      err = cudaStreamSynchronize(st);
      state.store(err == cudaSuccess ? 1 : 2, std::memory_order_release);
    } else {
      while (state.load(std::memory_order_acquire) == 0) __builtin_ia32_pause();
    }
    if (state.load(std::memory_order_acquire) == 1) {
      if (a < b0) memcpy((char*)d0 + a, (const char*)s0 + a, std::min(b, b0) - a);
      if (b > b0) {
        const size_t a1 = std::max(a, b0) - b0, e1 = b - b0;
        memcpy((char*)d1 + a1, (const char*)s1 + a1, e1 - a1);
      }
    }
  }
  return err;
}

// After a stream sync: did the last speculative first pass flag a query?
// (clears the pending state either way)
static bool spec_failed(Index* h) {
  const int nb = h->spec_nb;
  h->spec_nb = 0;
  bool failed = false;
  for (int q = 0; q < nb && !failed; ++q) failed = h->ws.h_flags[q] != 0;
  if (nb > 0 && h->dir_batch && h->ws.h_tileq) {  // adaptive tile-kernel skipping (Index::tile_skip)
    if (h->tile_skip) {
      if (failed) { h->tile_skip = 0; h->skip_streak = 0; }
    } else if (!failed && *h->ws.h_tileq == 0) {
      if (++h->skip_streak >= 2) h->tile_skip = 1;
    } else {
      h->skip_streak = 0;
    }
  }
  return failed;
}

template <class F>
static int host_driver(Index* h, const float* y, int64_t nq, int r, int batch_limit, double* dists,
                       int64_t* ids, double* phase_us, F&& batch) {
  struct HostOutReset {  // host_out is set per batch below; cleared on every exit
    Index* h;
    ~HostOutReset() { h->host_out = false; }
  } host_out_reset{h};
  int bsz = std::max(1, std::min<int>(h->batch, batch_limit));
  int64_t q0 = 0;
  static const bool trace = getenv("DPQ_HOST_TRACE") != nullptr;  // per-segment host timings (stderr)
  auto now = []() { return std::chrono::duration<double, std::micro>(
                        std::chrono::steady_clock::now().time_since_epoch()).count(); };
  double t_0 = trace ? now() : 0.0, t_in = 0, t_enq = 0, t_sync = 0;
  while (q0 < nq) {
    const int nb = (int)std::min<int64_t>(bsz, nq - q0);
    DPQ_TRY(ensure_ws(h, nb, r, h->d, -1));
    Workspace& w = h->ws;
    if (h->direct_copy) {
      if (h->check_finite && dpq_all_finite(y + q0 * h->d, (int64_t)nb * h->d) != 0) {
        set_error("non-finite query value");
        return DPQ_ERR_ARG;
      }
      DPQ_CUDA(cudaMemcpyAsync(w.y, y + q0 * h->d, (size_t)nb * h->d * 4, cudaMemcpyHostToDevice, h->stream));
    } else {
      if (h->check_finite) {
        if (par_memcpy_check_f32(w.h_y, y + q0 * h->d, (size_t)nb * h->d)) {
          // (earlier batches' results may already be in the caller's buffers: the caller raises)
          cudaStreamSynchronize(h->stream);
          set_error("non-finite query value");
          return DPQ_ERR_ARG;
        }
      } else {
        par_memcpy(w.h_y, y + q0 * h->d, (size_t)nb * h->d * 4);
      }
      DPQ_CUDA(cudaMemcpyAsync(w.y, w.h_y, (size_t)nb * h->d * 4, cudaMemcpyHostToDevice, h->stream));
    }
    const bool want_t = phase_us != nullptr;
    const bool old_t = h->timing;
    if (want_t) h->timing = true;
    if (trace) t_in = now();
    h->host_out = r > 0 && !h->direct_copy;
    int rc = batch(nb);
    if (trace) t_enq = now();
    h->timing = old_t;
    if (rc == 100) {  // split
      bsz = std::max(1, nb / 2);
      continue;
    }
    if (rc != DPQ_OK) return rc;
    bool redo = false;
  copy_out:
    if (r > 0 && h->direct_copy) {
      DPQ_CUDA(cudaMemcpyAsync(dists + q0 * r, w.out_d, (size_t)nb * r * 8, cudaMemcpyDeviceToHost, h->stream));
      DPQ_CUDA(cudaMemcpyAsync(ids + q0 * r, w.out_i, (size_t)nb * r * 8, cudaMemcpyDeviceToHost, h->stream));
      DPQ_CUDA(cudaStreamSynchronize(h->stream));
    } else if (r > 0) {  // results already in w.h_d / w.h_i (host_out)
      const cudaError_t ce = sync_copy_out(h->stream, dists + q0 * r, w.h_d, (size_t)nb * r * 8, ids + q0 * r,
                                           w.h_i, (size_t)nb * r * 8);
      if (ce != cudaSuccess) { h->host_out = false; DPQ_CUDA(ce); }
    } else {
      DPQ_CUDA(cudaStreamSynchronize(h->stream));
    }
    if (trace) t_sync = now();
    if (!redo && spec_failed(h)) {  // a speculative batch had a flagged query: redo it exactly
      redo = true;
      h->no_spec = true;
      rc = batch(nb);
      h->no_spec = false;
      if (rc == 100) { bsz = std::max(1, nb / 2); continue; }
      if (rc != DPQ_OK) return rc;
      goto copy_out;
    }
    if (trace) {
      const double t_out = now();
      fprintf(stderr, "[dpq host] in %.1f us | enqueue %.1f us | wait %.1f us | out %.1f us | total %.1f us\n",
              t_in - t_0, t_enq - t_in, t_sync - t_enq, t_out - t_sync, t_out - t_0);
      t_0 = t_out;
    }
    if (want_t) {
      const double per = 1000.0 / nb;  // ms per batch -> us per query
      for (int i = 0; i < nb; ++i) {
        double* t = phase_us + (q0 + i) * 4;
        t[0] = 0.0;  // flat: nothing to probe (flat.py:75-80)
        t[1] = h->phase_ms[PH_TABLES] * per;
        t[2] = (h->phase_ms[PH_GUARD] + h->phase_ms[PH_SCAN] + h->phase_ms[PH_THRESH] +
                h->phase_ms[PH_FALLBACK]) * per;
        t[3] = h->phase_ms[PH_REFINE] * per;
      }
    }
    q0 += nb;
  }
  return DPQ_OK;
}

static int make_plane(Index* h);
static void ivf_free(Index* h);

}  // namespace dpq

using namespace dpq;

// ============================================================================
// Plane construction and index lifetime
// ============================================================================
namespace dpq {

__global__ void k_make_plane(const void* codes, int code_bytes, int64_t n, int m, int mask, int mpad,
                             uint8_t* plane) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  uint8_t b[8];
  for (int j = 0; j < mpad; ++j)
    b[j] = j < m ? (uint8_t)(code_at(codes, code_bytes, row * m + j) & mask) : (uint8_t)0;
  for (int j = 0; j < mpad; ++j) plane[row * mpad + j] = b[j];
}

// Flat row order.  The index keeps its rows sorted (stably) by the low bytes
// of subspaces 0 and 1, so runs of consecutive rows share those two 8-bit
// table rows and the wide scan loop gathers only subspaces 2 and 3 per row.
// sorted_ids[row] = id_base + original row (ids and (dist, id) ties are the
// reference's); the original codes stay as the qmax prefix (first r2 rows in
// insertion order, twopass.py:76-84).
__global__ void k_row_keys(const void* codes, int code_bytes, int64_t n, int m, int mask, uint32_t* keys,
                           int32_t* rows) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = ((code_at(codes, code_bytes, i * m) & mask) << 8) | (code_at(codes, code_bytes, i * m + 1) & mask);
  rows[i] = (int32_t)i;
}
// key range [first row, last row] of every scan chunk (512 B of plane: 128 rows at MPAD 4, 64 at 8)
__global__ void k_chunk_keys(const uint32_t* skeys, int64_t n, int64_t nchunks, int cr, uint32_t* chunk_keys) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  const int64_t a = c * cr, b = std::min<int64_t>(a + cr - 1, n - 1);
  chunk_keys[c] = skeys[a] | (skeys[b] << 16);
}
__global__ void k_gather_rows(const uint8_t* codes, int row_bytes, int64_t n, const int32_t* perm, int64_t id_base,
                              uint8_t* out, int64_t* ids) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t src = perm[i];
  for (int b = 0; b < row_bytes; ++b) out[i * row_bytes + b] = codes[src * row_bytes + b];
  ids[i] = id_base + src;
}

// Unit seams: adc_low_batch (twopass.py:99-106) of every row for a batch of
// queries, written in original row order (scores[q * n + original row]).
__global__ void k_low_scores(const void* codes, int code_bytes, int64_t n, int m, int kbar, const uint8_t* q8,
                             const int64_t* sorted_ids, int64_t id_base, uint8_t* scores) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int q = blockIdx.y;
  if (row >= n) return;
  uint32_t acc = 0;
  for (int j = 0; j < m; ++j)
    acc += q8[((int64_t)q * m + j) * kbar + (code_at(codes, code_bytes, row * m + j) & (uint32_t)(kbar - 1))];
  const int64_t orig = sorted_ids ? sorted_ids[row] - id_base : row;
  scores[(int64_t)q * n + orig] = (uint8_t)min(acc, 255u);
}

// Emit entries of query q -> (score << 56 | id) for candidates (score <= b*,
// i.e. the rows the refine walk takes, twopass.py:295-302), ~0 otherwise.
__global__ void k_emit_keys(uint64_t* emit, const uint32_t* emit_cnt, uint32_t cap, const int32_t* bstar,
                            const int64_t* sorted_ids, int64_t id_base) {
  const int q = blockIdx.x;
  const uint32_t n = min(emit_cnt[q], cap);
  const int bs = bstar[q];
  uint64_t* e = emit + (int64_t)q * cap;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    const uint64_t v = e[i];
    const uint32_t sc = emit_score(v);
    const int64_t row = emit_row(v);
    const int64_t id = sorted_ids ? sorted_ids[row] : id_base + row;
    e[i] = ((int)sc <= bs && sc < 255u) ? (((uint64_t)sc << 56) | (uint64_t)id) : ~0ull;
  }
}

static int sort_rows(Index* h) {
  const int64_t n = h->n;
  uint32_t *k0 = nullptr, *k1 = nullptr;
  int32_t *r0 = nullptr, *r1 = nullptr;
  uint8_t* tmp = nullptr;
  uint8_t* sorted = nullptr;
  size_t tbytes = 0;
  auto cleanup = [&]() { cudaFree(k0); cudaFree(k1); cudaFree(r0); cudaFree(r1); cudaFree(tmp); };
  int rc = DPQ_OK;
  if ((rc = dmalloc(&k0, (size_t)n)) || (rc = dmalloc(&k1, (size_t)n)) || (rc = dmalloc(&r0, (size_t)n)) ||
      (rc = dmalloc(&r1, (size_t)n))) { cleanup(); return rc; }
  const unsigned blocks = (unsigned)((n + 255) / 256);
  {
    dbg_pending("sort_rows entry");
    cudaGetLastError();  // an error left pending by someone else's unchecked call is not this sort's (cub returns it)
    k_row_keys<<<blocks, 256, 0, h->stream>>>(h->codes, h->code_bytes, n, h->m, h->mask, k0, r0);
    const cudaError_t e1 = cudaGetLastError();
    const cudaError_t e2 = cub::DeviceRadixSort::SortPairs(nullptr, tbytes, k0, k1, r0, r1, (int)n, 0, 16, h->stream);
    if (e1 != cudaSuccess || e2 != cudaSuccess) {
      cleanup();
      set_error(std::string("row sort setup failed: keys '") + cudaGetErrorString(e1) + "', sort size '" +
                cudaGetErrorString(e2) + "', n = " + std::to_string(n));
      return DPQ_ERR_CUDA;
    }
  }
  if ((rc = dmalloc(&tmp, tbytes))) { cleanup(); return rc; }
  {
    const cudaError_t e = cub::DeviceRadixSort::SortPairs(tmp, tbytes, k0, k1, r0, r1, (int)n, 0, 16, h->stream);
    if (e != cudaSuccess) {
      cleanup();
      set_error(std::string("row sort failed: ") + cudaGetErrorString(e) + " (n = " + std::to_string(n) +
                ", temp bytes " + std::to_string(tbytes) + ")");
      return DPQ_ERR_CUDA;
    }
  }
  const int row_bytes = h->m * h->code_bytes;
  if ((rc = dmalloc(&sorted, (size_t)n * row_bytes + 16)) || (rc = dmalloc(&h->sorted_ids, (size_t)n))) {
    cudaFree(sorted); cleanup(); return rc;
  }
  k_gather_rows<<<blocks, 256, 0, h->stream>>>((const uint8_t*)h->codes, row_bytes, n, r1, h->id_base, sorted,
                                               h->sorted_ids);
  const int cr = 512 / h->mpad;  // rows per scan chunk
  h->n_chunks = (n + cr - 1) / cr;
  if ((rc = dmalloc(&h->chunk_keys, (size_t)h->n_chunks))) { cudaFree(sorted); cleanup(); return rc; }
  k_chunk_keys<<<(unsigned)((h->n_chunks + 255) / 256), 256, 0, h->stream>>>(k1, n, h->n_chunks, cr, h->chunk_keys);
  if (n < ((int64_t)1 << 32) - 2 * kDirSeg) {  // (direct scan items hold 32-bit rows)
    if ((rc = dmalloc(&h->key_start, (size_t)65537))) { cudaFree(sorted); cleanup(); return rc; }
    k_key_starts<<<(unsigned)((n + 1 + 255) / 256), 256, 0, h->stream>>>(k1, n, h->key_start);
  }
  {
    cudaError_t e = cudaStreamSynchronize(h->stream);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) {
      cleanup(); set_error(std::string("row sort failed (sync): ") + cudaGetErrorString(e)); return DPQ_ERR_CUDA;
    }
  }
  cleanup();
  if (h->prefix == h->codes) {  // original order stays as the qmax prefix
    h->own_prefix = true;
  } else {
    cudaFree(h->codes);
  }
  h->codes = sorted;
  h->rows_sorted = true;
  return DPQ_OK;
}

static int make_plane(Index* h) {
  const int64_t pad_rows = ((h->n + 127) / 128) * 128 + 128;
  h->n_pad = pad_rows;
  DPQ_TRY(dmalloc(&h->plane, (size_t)pad_rows * h->mpad));
  DPQ_CUDA(cudaMemsetAsync(h->plane, 0, (size_t)pad_rows * h->mpad, h->stream));
  if (h->n > 0) {
    k_make_plane<<<(unsigned)((h->n + 255) / 256), 256, 0, h->stream>>>(h->codes, h->code_bytes, h->n, h->m,
                                                                         h->mask, h->mpad, h->plane);
    DPQ_LAUNCHED(h);
  }
  return DPQ_OK;
}

int index_common_init(Index* h, int device, int m, int k, int kbar, int dsub, const float* codebooks,
                      const float* derived, int code_bytes) {
  if (m < 1 || m > 8) { set_error("m must be in [1, 8] for the device path"); return DPQ_ERR_ARG; }
  if (k < 1 || k > 65536) { set_error("k must be in [1, 65536]"); return DPQ_ERR_ARG; }
  if (kbar < 1 || kbar > 256 || (kbar & (kbar - 1))) {
    set_error("kbar must be a power of two <= 256 for the device path"); return DPQ_ERR_ARG;
  }
  if (dsub < 1) { set_error("dsub must be >= 1"); return DPQ_ERR_ARG; }
  if (code_bytes != 1 && code_bytes != 2) { set_error("code_bytes must be 1 or 2"); return DPQ_ERR_ARG; }
  h->device = device;
  DPQ_CUDA(cudaSetDevice(device));
  h->m = m; h->k = k; h->kbar = kbar; h->dsub = dsub; h->d = m * dsub; h->mask = kbar - 1;
  h->bbar = 0;
  while ((1 << h->bbar) < kbar) ++h->bbar;
  if (k % kbar) { set_error("k must be a multiple of kbar"); return DPQ_ERR_ARG; }
  h->mpad = m <= 4 ? 4 : 8;
  h->qt = h->mpad == 4 ? 128 : 64;
  h->code_bytes = code_bytes;
  if (const char* e = getenv("DPQ_GUARD_SAMPLE")) h->sample = std::max<int64_t>(1, atoll(e));
  if (const char* e = getenv("DPQ_EXACT_LIMIT")) h->exact_limit = std::max<int64_t>(0, atoll(e));
  if (const char* e = getenv("DPQ_EMIT_CAP")) h->cap0 = std::max<int64_t>(1, atoll(e));
  if (const char* e = getenv("DPQ_SCAN_WIDE")) h->wide = atoi(e) != 0;
  if (const char* e = getenv("DPQ_SORT_SLOTS")) h->sort_slots = atoi(e) != 0;
  if (const char* e = getenv("DPQ_SORT_ROWS")) h->sort_rows = atoi(e) != 0;
  if (const char* e = getenv("DPQ_RUN_FILTER")) h->run_filter = atoi(e) != 0;
  if (const char* e = getenv("DPQ_DIRECT")) h->direct = atoi(e) != 0;
  if (const char* e = getenv("DPQ_GT_SLACK")) h->gt_slack = atoi(e) != 0;
  if (const char* e = getenv("DPQ_TILE_SKIP")) h->tile_skip_ok = atoi(e) != 0;
  if (const char* e = getenv("DPQ_SCAN_HIST")) h->scan_hist = atoi(e) != 0;
  if (const char* e = getenv("DPQ_DIRECT_ITEMS")) h->direct_items = std::max(0, atoi(e));
  if (const char* e = getenv("DPQ_DIRECT_COPY")) h->direct_copy = atoi(e) != 0;
  if (const char* e = getenv("DPQ_SPECULATE")) h->no_spec = atoi(e) == 0;
  if (const char* e = getenv("DPQ_GRAPH")) h->use_graph = atoi(e) != 0;
  if (const char* e = getenv("DPQ_TC_TABLES")) h->use_tc = atoi(e);
  if (const char* e = getenv("DPQ_TC_EPS_SCALE")) h->tc_eps_scale = atof(e);
  DPQ_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  h->own_stream = true;
  for (int i = 0; i < 8; ++i) DPQ_CUDA(cudaEventCreate(&h->ev[i]));
  DPQ_CUDA(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
  for (int i = 0; i < 4; ++i) DPQ_CUDA(cudaEventCreateWithFlags(&h->fk[i], cudaEventDisableTiming));
  DPQ_TRY(dmalloc(&h->cb, (size_t)m * k * dsub));
  DPQ_TRY(dmalloc(&h->dcb, (size_t)m * kbar * dsub));
  DPQ_TRY(dmalloc(&h->d_nref, 1));
  DPQ_TRY(dmalloc(&h->d_nemit, 1));
  DPQ_TRY(dmalloc(&h->d_nent, 1));
  DPQ_TRY(dmalloc(&h->d_nwide, 1));
  DPQ_TRY(dmalloc(&h->d_nrows, 8));  // query-rows, plane rows, LUT tile loads (scan), exact re-ranks, probe exact d2
  DPQ_CUDA(cudaMemset(h->d_nrows, 0, 64));
  DPQ_CUDA(cudaMemset(h->d_nent, 0, 8));
  DPQ_CUDA(cudaMemset(h->d_nwide, 0, 8));
  DPQ_CUDA(cudaMemcpy(h->cb, codebooks, (size_t)m * k * dsub * 4, cudaMemcpyHostToDevice));
  DPQ_CUDA(cudaMemcpy(h->dcb, derived, (size_t)m * kbar * dsub * 4, cudaMemcpyHostToDevice));
  DPQ_CUDA(cudaMemset(h->d_nref, 0, 8));
  DPQ_CUDA(cudaMemset(h->d_nemit, 0, 8));
  return DPQ_OK;
}

void index_free(Index* h) {
  if (!h) return;
  dbg_pending("index_free entry");
  cudaSetDevice(h->device);
  ivf_free(h);
  dbg_pending("after ivf_free");
  if (h->stream) cudaStreamSynchronize(h->stream);
  tct_free(h->tct);
  if (h->tct_eps) cudaFree(h->tct_eps);
  if (h->tct_ny) cudaFree(h->tct_ny);
  if (h->graph.exec) cudaGraphExecDestroy(h->graph.exec);
  Workspace& w = h->ws;
  void* dev[] = {h->cb, h->dcb, h->codes, h->plane, h->own_prefix ? h->prefix : nullptr, h->centers,
                 h->offsets, h->sorted_ids, h->d_nref, h->d_nemit, h->d_nent, h->d_nwide, h->d_nrows, h->chunk_keys, h->key_start, w.dir_items, w.dir_state, w.slack, w.pot, w.chunk_list, w.list_len, w.y, w.small, w.q8, w.qmin, w.qmax, w.bounds,
                 w.lut, w.hist, w.hist_i, w.guard_b, w.gword, w.gword_p, w.emit_cnt, w.emit, w.bstar, w.ncand,
                 w.flags, w.only, w.tile_list, w.order, w.cluster, w.out_d, w.out_i, w.tables, w.slot_query, w.slot_probe,
                 w.slot_pre_off, w.slot_pre_len, w.counter, w.tile_fast};
  dbg_pending("index_free before frees");
  for (void* p : dev)
    if (p) {
      cudaFree(p);
      dbg_pending("index_free cudaFree");
    }
  void* host[] = {w.h_y, w.h_d, w.h_i, w.h_flags, w.h_cnt, w.h_tileq};
  for (void* p : host)
    if (p) cudaFreeHost(p);
  for (int i = 0; i < 8; ++i)
    if (h->ev[i]) cudaEventDestroy(h->ev[i]);
  for (int i = 0; i < 4; ++i)
    if (h->fk[i]) cudaEventDestroy(h->fk[i]);
  if (h->side) cudaStreamDestroy(h->side);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  dbg_pending("index_free exit");
  delete h;
}

}  // namespace dpq

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

const char* dpq_last_error(void) { return dpq::last_error(); }
int dpq_abi_version(void) { return 2; }
int dpq_all_finite(const float* x, int64_t n) {
  if (!x || n <= 0) return 0;
  const uint32_t* b = reinterpret_cast<const uint32_t*>(x);
  uint32_t any_special = 0;  // vectorizable: exponent all ones; a few threads above 256 KB
  const int nt = n < (64 << 10) ? 1 : (int)std::min<int64_t>(8, n / (32 << 10));
#pragma omp parallel for num_threads(nt) reduction(| : any_special) schedule(static)
  for (int64_t i = 0; i < n; ++i) any_special |= (uint32_t)((b[i] & 0x7F800000u) == 0x7F800000u);
  if (!any_special) return 0;
  for (int64_t i = 0; i < n; ++i)
    if ((b[i] & 0x7F800000u) == 0x7F800000u && (b[i] & 0x007FFFFFu)) return 1;
  return 2;
}

// quantizer.rotate (quantizer.py:235-239) of many rows in the reference's
// call shapes through the caller's CBLAS: (1, d) @ R per row is numpy's
// sgemv (RowMajor, Trans), a (g, d) @ R block (g >= 2) numpy's sgemm
// (RowMajor, NoTrans, NoTrans); identical calls, so identical bits, run on
// a few OpenMP threads.
typedef void (*sgemv_lp64_t)(int, int, int, int, float, const float*, int, const float*, int, float, float*, int);
typedef void (*sgemm_lp64_t)(int, int, int, int, int, int, float, const float*, int, const float*, int, float, float*,
                             int);
typedef void (*sgemv_ilp64_t)(int, int, int64_t, int64_t, float, const float*, int64_t, const float*, int64_t, float,
                              float*, int64_t);
typedef void (*sgemm_ilp64_t)(int, int, int, int64_t, int64_t, int64_t, float, const float*, int64_t, const float*,
                              int64_t, float, float*, int64_t);
int dpq_rotate_rows(const float* x, int64_t n, int64_t rows_per_call, int d, const float* rotation, float* out,
                    void* sgemv, void* sgemm, int ilp64, int threads) {
  if (n < 0 || d < 1 || rows_per_call < 1 || (n > 0 && (!x || !rotation || !out)) || n % rows_per_call) {
    set_error("dpq_rotate_rows: bad arguments"); return DPQ_ERR_ARG;
  }
  if ((rows_per_call == 1 && !sgemv) || (rows_per_call > 1 && !sgemm)) {
    set_error("dpq_rotate_rows: missing BLAS entry point"); return DPQ_ERR_ARG;
  }
  const int64_t calls = n / rows_per_call;
  const int g = (int)rows_per_call;
  const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(threads > 0 ? threads : 8, calls / 16));
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int64_t c = 0; c < calls; ++c) {
    const float* a = x + c * g * d;
    float* o = out + c * g * d;
    if (g == 1) {
      if (ilp64) ((sgemv_ilp64_t)sgemv)(101, 112, d, d, 1.f, rotation, d, a, 1, 0.f, o, 1);
      else ((sgemv_lp64_t)sgemv)(101, 112, d, d, 1.f, rotation, d, a, 1, 0.f, o, 1);
    } else {
      if (ilp64) ((sgemm_ilp64_t)sgemm)(101, 111, 111, g, d, d, 1.f, a, d, rotation, d, 0.f, o, d);
      else ((sgemm_lp64_t)sgemm)(101, 111, 111, g, d, d, 1.f, a, d, rotation, d, 0.f, o, d);
    }
  }
  return DPQ_OK;
}

int dpq_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int dpq_flat_create(int device, int m, int k, int kbar, int dsub, const float* codebooks,
                    const float* derived_codebooks, const void* codes, int code_bytes, int64_t n,
                    int64_t id_base, const void* prefix_codes, int64_t n_prefix, dpq_index_t** out) {
  if (!out || !codebooks || !derived_codebooks || (n > 0 && !codes) || n < 0) {
    set_error("null pointer or negative size");
    return DPQ_ERR_ARG;
  }
  if (n >= ((int64_t)1 << kRowBits)) { set_error("too many rows for one index shard"); return DPQ_ERR_ARG; }
  dbg_pending("flat_create entry");
  Index* h = new Index();
  h->kind = KIND_FLAT;
  int rc = index_common_init(h, device, m, k, kbar, dsub, codebooks, derived_codebooks, code_bytes);
  if (rc != DPQ_OK) { index_free(h); return rc; }
  h->n = n;
  h->id_base = id_base;
  const size_t cbytes = (size_t)n * m * code_bytes;
  if ((rc = dmalloc((uint8_t**)&h->codes, cbytes + 16)) != DPQ_OK) { index_free(h); return rc; }
  if (n > 0 && cudaMemcpy(h->codes, codes, cbytes, cudaMemcpyDefault) != cudaSuccess) {
    set_error("codes upload failed"); index_free(h); return DPQ_ERR_CUDA;
  }
  if (prefix_codes && n_prefix > 0) {
    const size_t pb = (size_t)n_prefix * m * code_bytes;
    if ((rc = dmalloc((uint8_t**)&h->prefix, pb)) != DPQ_OK) { index_free(h); return rc; }
    if (cudaMemcpy(h->prefix, prefix_codes, pb, cudaMemcpyDefault) != cudaSuccess) {
      set_error("prefix upload failed"); index_free(h); return DPQ_ERR_CUDA;
    }
    h->own_prefix = true;
    h->n_prefix = n_prefix;
  } else {
    h->prefix = h->codes;
    h->n_prefix = n;
  }
  // compact 4-byte emit records when every shard row fits in 24 bits, for the PQ 4x16 layout whose
  // table refine is the software-pipelined loop (DPQ_EMIT32=0: 8-byte records)
  h->emit32 = n < ((int64_t)1 << kRow32Bits) && m == 4 && code_bytes == 2 &&
              !(getenv("DPQ_EMIT32") && atoi(getenv("DPQ_EMIT32")) == 0);
  if (h->sort_rows && m >= 2 && n > 1 && n < ((int64_t)1 << 31) &&
      (rc = sort_rows(h)) != DPQ_OK) { index_free(h); return rc; }
  // optimistic start: the first batch already runs without the tile kernels (a query that needs them
  // gets the batch redone with them and switches the mode off)
  h->tile_skip = (h->direct && h->key_start && h->tile_skip_ok) ? 1 : 0;
  if ((rc = make_plane(h)) != DPQ_OK) { index_free(h); return rc; }
  if (cudaStreamSynchronize(h->stream) != cudaSuccess) {
    set_error("index build failed"); index_free(h); return DPQ_ERR_CUDA;
  }
  *out = reinterpret_cast<dpq_index_t*>(h);
  return DPQ_OK;
}

void dpq_destroy(dpq_index_t* index) { index_free(reinterpret_cast<Index*>(index)); }

int dpq_set_stream(dpq_index_t* index, void* stream) {
  Index* h = reinterpret_cast<Index*>(index);
  if (!h) { set_error("null index"); return DPQ_ERR_ARG; }
  cudaSetDevice(h->device);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  if (stream) {
    h->stream = (cudaStream_t)stream;
    h->own_stream = false;
  } else {
    DPQ_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    h->own_stream = true;
  }
  return DPQ_OK;
}

int dpq_set_batch(dpq_index_t* index, int batch) {
  Index* h = reinterpret_cast<Index*>(index);
  if (!h || batch < 1) { set_error("bad batch"); return DPQ_ERR_ARG; }
  h->batch = batch;
  return DPQ_OK;
}

int dpq_set_check_finite(dpq_index_t* index, int enabled) {
  Index* h = reinterpret_cast<Index*>(index);
  if (!h) { set_error("null index"); return DPQ_ERR_ARG; }
  h->check_finite = enabled != 0;
  return DPQ_OK;
}

int dpq_set_timing(dpq_index_t* index, int enabled) {
  Index* h = reinterpret_cast<Index*>(index);
  if (!h) { set_error("null index"); return DPQ_ERR_ARG; }
  h->timing = enabled != 0;
  return DPQ_OK;
}

static int check_search(Index* h, int64_t nq, int r, int r2, bool derived) {
  if (!h) { set_error("null index"); return DPQ_ERR_ARG; }
  if (nq < 0 || r < 1) { set_error("need nq >= 0 and r >= 1"); return DPQ_ERR_ARG; }
  if (derived && (r2 < 1 || r > r2)) { set_error("need 1 <= r <= r2"); return DPQ_ERR_ARG; }
  if (derived && h->n_prefix < 1 && h->kind == KIND_FLAT) {
    set_error("need at least one code to estimate qmax"); return DPQ_ERR_ARG;
  }
  cudaSetDevice(h->device);
  return DPQ_OK;
}

int dpq_flat_search_derived(dpq_index_t* index, const float* yr, int64_t nq, int r, int r2, int capped,
                            double* dists, int64_t* ids, double* phase_us) {
  (void)capped;
  Index* h = reinterpret_cast<Index*>(index);
  DPQ_TRY(check_search(h, nq, r, r2, true));
  if (h->kind != KIND_FLAT) { set_error("not a flat index"); return DPQ_ERR_STATE; }
  return host_driver(h, yr, nq, r, 1 << 30, dists, ids, phase_us,
                     [&](int nb) { return flat_derived_batch(h, nb, r, r2); });
}

int dpq_flat_search_derived_dev(dpq_index_t* index, const float* yr, int64_t nq, int r, int r2, double* dists,
                                int64_t* ids) {
  Index* h = reinterpret_cast<Index*>(index);
  DPQ_TRY(check_search(h, nq, r, r2, true));
  if (h->kind != KIND_FLAT) { set_error("not a flat index"); return DPQ_ERR_STATE; }
  int bsz = h->batch;
  int64_t q0 = 0;
  struct DevOutReset {  // (cleared on every exit)
    Index* h;
    ~DevOutReset() { h->dev_out_d = nullptr; h->dev_out_i = nullptr; }
  } dev_out_reset{h};
  while (q0 < nq) {
    const int nb = (int)std::min<int64_t>(bsz, nq - q0);
    DPQ_TRY(ensure_ws(h, nb, r, h->d, -1));
    Workspace& w = h->ws;
    DPQ_CUDA(cudaMemcpyAsync(w.y, yr + q0 * h->d, (size_t)nb * h->d * 4, cudaMemcpyDeviceToDevice, h->stream));
    // a call that is one batch: the refine writes into the caller's buffers (the graph is keyed on them)
    const bool direct_out = q0 == 0 && nb == nq;
    h->dev_out_d = direct_out ? dists : nullptr;
    h->dev_out_i = direct_out ? ids : nullptr;
    int rc = flat_derived_batch(h, nb, r, r2);
    if (rc == 100) { bsz = std::max(1, nb / 2); continue; }
    if (rc != DPQ_OK) return rc;
    if (h->spec_nb) {
      DPQ_CUDA(cudaStreamSynchronize(h->stream));
      if (spec_failed(h)) {
        h->no_spec = true;
        rc = flat_derived_batch(h, nb, r, r2);
        h->no_spec = false;
        if (rc == 100) { bsz = std::max(1, nb / 2); continue; }
        if (rc != DPQ_OK) return rc;
      }
    }
    if (!direct_out) {
      DPQ_CUDA(cudaMemcpyAsync(dists + q0 * r, w.out_d, (size_t)nb * r * 8, cudaMemcpyDeviceToDevice, h->stream));
      DPQ_CUDA(cudaMemcpyAsync(ids + q0 * r, w.out_i, (size_t)nb * r * 8, cudaMemcpyDeviceToDevice, h->stream));
    }
    q0 += nb;
  }
  DPQ_CUDA(cudaStreamSynchronize(h->stream));
  return DPQ_OK;
}

int dpq_flat_search_conventional(dpq_index_t* index, const float* yr, int64_t nq, int r, double* dists,
                                 int64_t* ids, double* phase_us) {
  Index* h = reinterpret_cast<Index*>(index);
  DPQ_TRY(check_search(h, nq, r, r, false));
  if (h->kind != KIND_FLAT) { set_error("not a flat index"); return DPQ_ERR_STATE; }
  // full tables are m*k floats per query: keep the batch's tables <= 1 GB
  const int lim = (int)std::max<int64_t>(1, ((int64_t)1 << 28) / ((int64_t)h->m * h->k));
  return host_driver(h, yr, nq, r, lim, dists, ids, phase_us,
                     [&](int nb) { return flat_conventional_batch(h, nb, r); });
}

int dpq_debug_quantize_tables(dpq_index_t* index, const float* yr, int64_t nq, int r2, float* small, uint8_t* q,
                              double* qmin, double* qmax) {
  Index* h = reinterpret_cast<Index*>(index);
  DPQ_TRY(check_search(h, nq, 1, r2, true));
  const int64_t mk = (int64_t)h->m * h->kbar;
  for (int64_t q0 = 0; q0 < nq; q0 += h->batch) {
    const int nb = (int)std::min<int64_t>(h->batch, nq - q0);
    DPQ_TRY(ensure_ws(h, nb, 1, h->d, -1));
    Workspace& w = h->ws;
    DPQ_CUDA(cudaMemcpyAsync(w.y, yr + q0 * h->d, (size_t)nb * h->d * 4, cudaMemcpyHostToDevice, h->stream));
    DPQ_TRY(run_small_tables(h, nb, h->prefix, std::min<int64_t>(r2, h->n_prefix), nullptr, nullptr, nullptr,
                             true, nullptr));
    DPQ_CUDA(cudaMemcpyAsync(small + q0 * mk, w.small, (size_t)nb * mk * 4, cudaMemcpyDeviceToHost, h->stream));
    DPQ_CUDA(cudaMemcpyAsync(q + q0 * mk, w.q8, (size_t)nb * mk, cudaMemcpyDeviceToHost, h->stream));
    DPQ_CUDA(cudaMemcpyAsync(qmin + q0, w.qmin, (size_t)nb * 8, cudaMemcpyDeviceToHost, h->stream));
    DPQ_CUDA(cudaMemcpyAsync(qmax + q0, w.qmax, (size_t)nb * 8, cudaMemcpyDeviceToHost, h->stream));
    DPQ_CUDA(cudaStreamSynchronize(h->stream));
  }
  return DPQ_OK;
}

int dpq_debug_candidates(dpq_index_t* index, const float* yr, int64_t nq, int r2, int32_t* bstar,
                         int64_t* ncand) {
  Index* h = reinterpret_cast<Index*>(index);
  DPQ_TRY(check_search(h, nq, 1, r2, true));
  if (h->kind != KIND_FLAT) { set_error("not a flat index"); return DPQ_ERR_STATE; }
  for (int64_t q0 = 0; q0 < nq; q0 += h->batch) {
    const int nb = (int)std::min<int64_t>(h->batch, nq - q0);
    DPQ_TRY(ensure_ws(h, nb, 1, h->d, -1));
    Workspace& w = h->ws;
    DPQ_CUDA(cudaMemcpyAsync(w.y, yr + q0 * h->d, (size_t)nb * h->d * 4, cudaMemcpyHostToDevice, h->stream));
    DPQ_TRY(run_small_tables(h, nb, h->prefix, std::min<int64_t>(r2, h->n_prefix), nullptr, nullptr, nullptr,
                             false, nullptr));
    const bool ns = h->no_spec;
    h->no_spec = true;  // exact b* needed right here
    int rc = flat_first_pass(h, nb, r2);
    h->no_spec = ns;
    if (rc == 100) { set_error("debug_candidates: emit budget exceeded, use a smaller batch"); return DPQ_ERR_NOMEM; }
    if (rc != DPQ_OK) return rc;
    DPQ_CUDA(cudaMemcpyAsync(bstar + q0, w.bstar, (size_t)nb * 4, cudaMemcpyDeviceToHost, h->stream));
    DPQ_CUDA(cudaMemcpyAsync(ncand + q0, w.ncand, (size_t)nb * 8, cudaMemcpyDeviceToHost, h->stream));
    DPQ_CUDA(cudaStreamSynchronize(h->stream));
  }
  return DPQ_OK;
}

int dpq_debug_full_tables(dpq_index_t* index, const float* yr, int64_t nq, float* tables) {
  Index* h = reinterpret_cast<Index*>(index);
  DPQ_TRY(check_search(h, nq, 1, 1, false));
  const int64_t per = (int64_t)h->m * h->k;
  for (int64_t q0 = 0; q0 < nq; ++q0) {
    DPQ_TRY(ensure_ws(h, 1, 1, h->d, -1));
    Workspace& w = h->ws;
    if (per > w.tables_elems) {
      DPQ_TRY(dmalloc(&w.tables, (size_t)per));
      w.tables_elems = per;
    }
    DPQ_CUDA(cudaMemcpyAsync(w.y, yr + q0 * h->d, (size_t)h->d * 4, cudaMemcpyHostToDevice, h->stream));
    dim3 grid((h->k + 255) / 256, h->m, 1);
    k_full_tables<<<grid, 256, h->dsub * 4, h->stream>>>(w.y, h->cb, h->m, h->k, h->kbar, h->bbar, h->dsub, 0,
                                                         w.tables);
    DPQ_LAUNCHED(h);
    DPQ_CUDA(cudaMemcpyAsync(tables + q0 * per, w.tables, (size_t)per * 4, cudaMemcpyDeviceToHost, h->stream));
    DPQ_CUDA(cudaStreamSynchronize(h->stream));
  }
  return DPQ_OK;
}

int dpq_debug_low_scores(dpq_index_t* index, const float* yr, int64_t nq, int r2, uint8_t* scores) {
  Index* h = reinterpret_cast<Index*>(index);
  DPQ_TRY(check_search(h, nq, 1, r2, true));
  if (h->kind != KIND_FLAT) { set_error("not a flat index"); return DPQ_ERR_STATE; }
  if (nq > 0 && !scores) { set_error("null scores"); return DPQ_ERR_ARG; }
  const int bq = (int)std::max<int64_t>(1, std::min<int64_t>(h->batch, ((int64_t)1 << 30) / std::max<int64_t>(1, h->n)));
  uint8_t* d_scores = nullptr;
  DPQ_TRY(dmalloc(&d_scores, (size_t)bq * std::max<int64_t>(1, h->n)));
  int rc = DPQ_OK;
  for (int64_t q0 = 0; q0 < nq && rc == DPQ_OK; q0 += bq) {
    const int nb = (int)std::min<int64_t>(bq, nq - q0);
    if ((rc = ensure_ws(h, nb, 1, h->d, -1)) != DPQ_OK) break;
    Workspace& w = h->ws;
    if (cudaMemcpyAsync(w.y, yr + q0 * h->d, (size_t)nb * h->d * 4, cudaMemcpyHostToDevice, h->stream) != cudaSuccess) {
      rc = DPQ_ERR_CUDA; set_error("query upload failed"); break;
    }
    if ((rc = run_small_tables(h, nb, h->prefix, std::min<int64_t>(r2, h->n_prefix), nullptr, nullptr, nullptr,
                               false, nullptr, nullptr, 0, false)) != DPQ_OK) break;
    if (h->n > 0) {
      k_low_scores<<<dim3((unsigned)((h->n + 255) / 256), (unsigned)nb), 256, 0, h->stream>>>(
          h->codes, h->code_bytes, h->n, h->m, h->kbar, w.q8, h->rows_sorted ? h->sorted_ids : nullptr, h->id_base,
          d_scores);
      if (cudaGetLastError() != cudaSuccess) { rc = DPQ_ERR_CUDA; set_error("k_low_scores launch failed"); break; }
      h->counters[0]++;
      if (cudaMemcpyAsync(scores + q0 * h->n, d_scores, (size_t)nb * h->n, cudaMemcpyDeviceToHost, h->stream) !=
              cudaSuccess ||
          cudaStreamSynchronize(h->stream) != cudaSuccess) {
        rc = DPQ_ERR_CUDA; set_error("low scores download failed"); break;
      }
    }
  }
  cudaFree(d_scores);
  return rc;
}

int dpq_debug_candidate_ids(dpq_index_t* index, const float* yr, int64_t nq, int r2, int64_t cap, int64_t* ids,
                            uint8_t* scores, int64_t* counts) {
  Index* h = reinterpret_cast<Index*>(index);
  DPQ_TRY(check_search(h, nq, 1, r2, true));
  if (h->kind != KIND_FLAT) { set_error("not a flat index"); return DPQ_ERR_STATE; }
  if (cap < 0 || (nq > 0 && (!counts || (cap > 0 && !ids)))) { set_error("bad candidate buffers"); return DPQ_ERR_ARG; }
  std::vector<uint64_t> keys;
  std::vector<uint32_t> cnt;
  std::vector<int32_t> bs;
  for (int64_t q0 = 0; q0 < nq; q0 += h->batch) {
    const int nb = (int)std::min<int64_t>(h->batch, nq - q0);
    DPQ_TRY(ensure_ws(h, nb, 1, h->d, -1));
    Workspace& w = h->ws;
    DPQ_CUDA(cudaMemcpyAsync(w.y, yr + q0 * h->d, (size_t)nb * h->d * 4, cudaMemcpyHostToDevice, h->stream));
    DPQ_TRY(run_small_tables(h, nb, h->prefix, std::min<int64_t>(r2, h->n_prefix), nullptr, nullptr, nullptr,
                             false, nullptr));
    const bool ns = h->no_spec, e32 = h->emit32;
    h->no_spec = true;  // exact b* needed right here
    h->emit32 = false;  // k_emit_keys rewrites 8-byte records in place
    int rc = flat_first_pass(h, nb, r2);
    h->no_spec = ns;
    h->emit32 = e32;
    if (rc == 100) { set_error("debug_candidate_ids: emit budget exceeded, use a smaller batch"); return DPQ_ERR_NOMEM; }
    if (rc != DPQ_OK) return rc;
    // emit entries -> (score << 56 | id) in place, ~0 for non-candidates
    k_emit_keys<<<nb, 256, 0, h->stream>>>(w.emit, w.emit_cnt, w.cap, w.bstar, h->rows_sorted ? h->sorted_ids : nullptr,
                                           h->id_base);
    DPQ_LAUNCHED(h);
    cnt.resize(nb);
    bs.resize(nb);
    DPQ_CUDA(cudaMemcpyAsync(cnt.data(), w.emit_cnt, (size_t)nb * 4, cudaMemcpyDeviceToHost, h->stream));
    DPQ_CUDA(cudaMemcpyAsync(bs.data(), w.bstar, (size_t)nb * 4, cudaMemcpyDeviceToHost, h->stream));
    DPQ_CUDA(cudaStreamSynchronize(h->stream));
    for (int q = 0; q < nb; ++q) {
      const uint32_t c = std::min(cnt[q], w.cap);
      keys.resize(c);
      if (c) DPQ_CUDA(cudaMemcpy(keys.data(), w.emit + (int64_t)q * w.cap, (size_t)c * 8, cudaMemcpyDeviceToHost));
      keys.erase(std::remove(keys.begin(), keys.end(), ~0ull), keys.end());
      std::sort(keys.begin(), keys.end());  // (score, id): the bucket walk order
      const int64_t gq = q0 + q;
      counts[gq] = (int64_t)keys.size();
      const int64_t nw = std::min<int64_t>(cap, (int64_t)keys.size());
      for (int64_t i = 0; i < nw; ++i) {
        ids[gq * cap + i] = (int64_t)(keys[i] & kRowMask);
        if (scores) scores[gq * cap + i] = (uint8_t)(keys[i] >> 56);
      }
    }
  }
  return DPQ_OK;
}

int dpq_debug_tc_tables(dpq_index_t* index, const float* yr, int64_t nq, float* tables, double* eps) {
  Index* h = reinterpret_cast<Index*>(index);
  DPQ_TRY(check_search(h, nq, 1, 1, false));
  if (!tct_supported(h->m, h->k, h->kbar, h->dsub)) { set_error("unsupported shape for tensor-core tables"); return DPQ_ERR_ARG; }
  if (nq > 0 && (!tables || !eps)) { set_error("null output"); return DPQ_ERR_ARG; }
  const int64_t per = (int64_t)h->m * h->k;
  const int gsize = h->k / h->kbar;
  std::vector<float> gm;
  const int bq = std::max(1, std::min(h->batch, 256));
  for (int64_t q0 = 0; q0 < nq; q0 += bq) {
    const int nb = (int)std::min<int64_t>(bq, nq - q0);
    DPQ_TRY(ensure_ws(h, nb, 1, h->d, -1));
    Workspace& w = h->ws;
    DPQ_CUDA(cudaMemcpyAsync(w.y, yr + q0 * h->d, (size_t)nb * h->d * 4, cudaMemcpyHostToDevice, h->stream));
    DPQ_TRY(run_tc_tables(h, nb, w.y, h->d));
    gm.resize((size_t)nb * per);
    DPQ_CUDA(cudaMemcpyAsync(gm.data(), w.tables, (size_t)nb * per * 4, cudaMemcpyDeviceToHost, h->stream));
    DPQ_CUDA(cudaMemcpyAsync(eps + q0 * h->m, h->tct_eps, (size_t)nb * h->m * 8, cudaMemcpyDeviceToHost, h->stream));
    DPQ_CUDA(cudaStreamSynchronize(h->stream));
    for (int q = 0; q < nb; ++q)  // group-major -> centroid order
      for (int j = 0; j < h->m; ++j)
        for (int c = 0; c < h->k; ++c)
          tables[(q0 + q) * per + (int64_t)j * h->k + c] =
              gm[(size_t)q * per + (size_t)j * h->k + (size_t)(c & h->mask) * gsize + (c >> h->bbar)];
  }
  return DPQ_OK;
}

int dpq_last_phase_ms(dpq_index_t* index, float* ms7) {
  Index* h = reinterpret_cast<Index*>(index);
  if (!h || !ms7) { set_error("null argument"); return DPQ_ERR_ARG; }
  for (int i = 0; i < PH_N; ++i) ms7[i] = h->phase_ms[i];
  return DPQ_OK;
}

int dpq_counters_ex(dpq_index_t* index, int64_t* out, int n) {
  Index* h = reinterpret_cast<Index*>(index);
  if (!h || !out || n < 0) { set_error("null argument"); return DPQ_ERR_ARG; }
  int64_t base[8];
  DPQ_TRY(dpq_counters(index, base));
  unsigned long long dv[8] = {};
  DPQ_CUDA(cudaMemcpy(dv, h->d_nrows, sizeof(dv), cudaMemcpyDeviceToHost));
  const int64_t all[kCountersEx] = {base[0], base[1], base[2], base[3], base[4], base[5], base[6], base[7],
                                    (int64_t)dv[1] + h->plane_rows, (int64_t)dv[2], (int64_t)dv[3],
                                    (int64_t)dv[4]};
  for (int i = 0; i < n; ++i) out[i] = i < kCountersEx ? all[i] : 0;
  return DPQ_OK;
}

int dpq_counters(dpq_index_t* index, int64_t* out8) {
  Index* h = reinterpret_cast<Index*>(index);
  if (!h || !out8) { set_error("null argument"); return DPQ_ERR_ARG; }
  unsigned long long nref = 0, nemit = 0, nent = 0, nwide = 0, nrows = 0;
  cudaSetDevice(h->device);
  DPQ_CUDA(cudaMemcpy(&nref, h->d_nref, 8, cudaMemcpyDeviceToHost));
  DPQ_CUDA(cudaMemcpy(&nemit, h->d_nemit, 8, cudaMemcpyDeviceToHost));
  DPQ_CUDA(cudaMemcpy(&nent, h->d_nent, 8, cudaMemcpyDeviceToHost));
  DPQ_CUDA(cudaMemcpy(&nwide, h->d_nwide, 8, cudaMemcpyDeviceToHost));
  DPQ_CUDA(cudaMemcpy(&nrows, h->d_nrows, 8, cudaMemcpyDeviceToHost));
  h->counters[3] = (int64_t)nref;
  h->counters[5] = (int64_t)nemit;
  h->counters[6] = (int64_t)nent;
  h->counters[7] = (int64_t)nwide;
  for (int i = 0; i < 8; ++i) out8[i] = h->counters[i];
  out8[2] += (int64_t)nrows;
  return DPQ_OK;
}

}  // extern "C"

#include "dpq_ivf.cuh"
