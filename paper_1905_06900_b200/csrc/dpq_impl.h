// dpq_impl.h — host-side state of a libdpq index handle (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

namespace dpq {

void set_error(const std::string& msg);

// tensor-core full tables (dpq_tctab.cu)
bool tct_supported(int m, int k, int kbar, int dsub);
int tct_prepare(int device, const float* cb, int m, int k, int kbar, int dsub, cudaStream_t stream, void** out);
int tct_build(void* t, const float* y, int64_t ystride, int nq, float* tables, double* eps, double* ny,
              double eps_scale, cudaStream_t stream);
double tct_gamma(void* t, double eps_scale);
int tct_argmin(void* t, const float* x, int64_t ldx, int64_t n, int32_t* codes, unsigned long long* scratch,
               cudaStream_t stream);
const float* tct_cnorm(void* t);
void tct_free(void* t);

enum Kind { KIND_FLAT = 0, KIND_IVF = 1 };

// Phase slots of dpq_last_phase_ms.
constexpr int kCountersEx = 12;  // dpq_counters_ex

enum Phase { PH_TABLES = 0, PH_GUARD, PH_SCAN, PH_THRESH, PH_REFINE, PH_FALLBACK, PH_TOTAL, PH_N };

// Per-batch device workspace, grown on demand.
struct Workspace {
  int qb = 0;             // slot capacity
  int qn = 0;             // query capacity
  int rcap = 0;           // result columns capacity
  uint32_t cap = 0;       // emit capacity per query
  int qcap_emit = 0;      // queries the emit buffer is sized for
  float* y = nullptr;     // [qb][ystride]
  int ystride = 0;
  float* small = nullptr;     // [qb][m][kbar]
  uint8_t* q8 = nullptr;      // [qb][m][kbar]
  double* qmin = nullptr;
  double* qmax = nullptr;
  double* bounds = nullptr;   // [qb][2]
  uint8_t* lut = nullptr;     // [tiles][mpad][256][qt] u8
  uint32_t* hist = nullptr;   // [tiles*qt][256]
  int32_t* hist_i = nullptr;  // [qb][256] (sharded exchange)
  uint16_t* guard_b = nullptr;
  uint16_t* gword = nullptr;
  int* order = nullptr;         // refine CTA -> query
  uint16_t* cluster = nullptr;  // per slot: g0* << 8 | g1* (flat slot clustering)
  uint16_t* gword_p = nullptr;  // guard words in sorted-slot order (flat)
  uint8_t* pot = nullptr;       // run filter: [tiles][65536] key has potential
  int* chunk_list = nullptr;    // [tiles][n_chunks] chunks to scan
  int* list_len = nullptr;      // [tiles]
  int32_t* slack = nullptr;     // [qb][m] group-table activity slack (k_entry_slack / k_key_select)
  int slack_cap = 0;
  bool slack_ready = false;     // this batch's slack was written by k_key_select
  int* h_tileq = nullptr;       // pinned: queries the last first pass left to the tile scan (dir_state[1])
  uint2* dir_items = nullptr;   // direct scan work items (k_key_select)
  int dir_items_cap = 0;
  int* dir_state = nullptr;     // [0] items reserved, [1] queries left to the tile scan
  int list_tiles = 0;
  int64_t list_chunks = 0;
  uint32_t* emit_cnt = nullptr;
  uint64_t* emit = nullptr;
  int32_t* bstar = nullptr;
  int64_t* ncand = nullptr;
  uint8_t* flags = nullptr;
  uint8_t* only = nullptr;
  int* tile_list = nullptr;
  int* tile_fast = nullptr;     // per tile: LUT clamped to 7-bit entries
  unsigned* counter = nullptr;  // persistent-scan unit counter
  double* out_d = nullptr;
  int64_t* out_i = nullptr;
  float* tables = nullptr;    // conventional full tables
  int64_t tables_elems = 0;
  // ivf slot maps
  int* slot_query = nullptr;
  int* slot_probe = nullptr;
  int64_t* slot_pre_off = nullptr;
  int64_t* slot_pre_len = nullptr;
  // pinned host staging
  float* h_y = nullptr;
  double* h_d = nullptr;
  int64_t* h_i = nullptr;
  uint8_t* h_flags = nullptr;
  uint32_t* h_cnt = nullptr;
  size_t h_y_bytes = 0, h_out_elems = 0;
};

struct BatchGraph {
  cudaGraphExec_t exec = nullptr;
  int nb = -1, r = -1, r2 = -1, host_out = -1, tile_skip = -1;
  const void* dev_out = nullptr;  // device-API calls: the caller's result buffer the refine writes into
  uint64_t epoch = 0;
  bool warm = false;
  int64_t counters[8] = {};  // host counter increments of one captured batch
};

struct Index {
  int device = 0;
  int kind = KIND_FLAT;
  int m = 0, k = 0, kbar = 0, bbar = 0, dsub = 0, d = 0, mask = 0, mpad = 4, code_bytes = 2;
  int64_t n = 0, n_pad = 0, id_base = 0;
  float* cb = nullptr;      // [m][k][dsub]
  float* dcb = nullptr;     // [m][kbar][dsub]
  void* codes = nullptr;    // [n][m]
  uint8_t* plane = nullptr; // [n_pad][mpad]
  void* prefix = nullptr;   // flat qmax prefix rows
  int64_t n_prefix = 0;
  bool own_prefix = false;
  // ivf
  int n_cells = 0;
  float* centers = nullptr;       // [K][d]
  int64_t* offsets = nullptr;     // device [K+1]
  std::vector<int64_t> h_offsets; // host copy
  int64_t* sorted_ids = nullptr;  // [n]
  void* ivf_state = nullptr;      // IvfBuffers (dpq_ivf.cuh)
  // ivf list-split shard (dpq_ivf_set_shard): this handle holds a slice of
  // every inverted list; bounds and sampling follow the GLOBAL lists
  bool ivf_shard = false;
  std::vector<int64_t> g_offsets;  // (K+1) global list offsets
  std::vector<int64_t> g_pre_off;  // (K+1) offsets of each list's prefix rows in g_prefix
  void* g_prefix = nullptr;        // device: first min(P, len) rows of every global list (qmax, ivf.py:205-217)
  int64_t g_pre_rows = 0;          // P
  // execution
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int batch = 1024;
  bool timing = false;
  bool check_finite = false;  // dpq_set_check_finite: host query batches scanned while they are staged
  cudaEvent_t ev[8] = {};
  cudaStream_t side = nullptr;  // fork/join branch of the batch (independent kernels overlap)
  cudaEvent_t fk[4] = {};       // fork / join events of the two branch points
  // The direct scan counts its hits by score for K3, which then skips its pass over those queries'
  // emit lists.  -1 = auto: on for 8-byte emit records (shards of 2^24 rows or more, where the lists
  // outgrow L2: configs[2] K3 0.31 -> 0.01 ms, scan 0.75 -> 0.90), off for 4-byte records (configs[1]:
  // K3 24 -> 10 us, scan 80 -> 100 us).  env DPQ_SCAN_HIST=0/1 forces it.
  int scan_hist = -1;
  bool order_forked = false;    // k_order_by_count already enqueued on `side` (speculative first pass)
  float phase_ms[PH_N] = {};
  int64_t counters[8] = {};  // launches, queries, rows scanned, refined, fallbacks, emitted, table entries, wide units
  unsigned long long* d_nref = nullptr;
  unsigned long long* d_nemit = nullptr;
  unsigned long long* d_nent = nullptr;   // lazily computed table entries
  unsigned long long* d_nwide = nullptr;  // scan units run by the wide loop
  unsigned long long* d_nrows = nullptr;  // [8]: query-rows (list mode), plane rows (list mode), LUT loads, exact re-ranks, probe exact d2
  int64_t plane_rows = 0;                 // plane rows read by the scan (non-list mode, host-counted)
  size_t emit_budget = (size_t)16 << 30;  // bytes for emit buffers
  // guard sampling (env DPQ_GUARD_SAMPLE / DPQ_EXACT_LIMIT / DPQ_EMIT_CAP
  // override them so tests can force the exact-redo and overflow paths)
  int64_t sample = 16384;
  int64_t exact_limit = 65536;
  int64_t cap0 = 0;
  bool host_out = false;  // host API: the refine writes results straight into the pinned staging buffers
  double* dev_out_d = nullptr;  // device API, single-batch call: the refine writes straight into the caller's
  int64_t* dev_out_i = nullptr; //   device buffers (no copy after the batch)
  int wide = 1;       // wide scan tiles (env DPQ_SCAN_WIDE=0 disables)
  int sort_slots = 1; // flat: order query tiles by guard (env DPQ_SORT_SLOTS=0)
  int sort_rows = 1;  // flat: rows sorted by (g0, g1) at build (env DPQ_SORT_ROWS=0)
  bool rows_sorted = false;
  bool no_spec = false;  // first pass waits for its flags (no speculative refine)
  int use_graph = 1;     // replay speculative batches as a CUDA graph (env DPQ_GRAPH=0 disables)
  BatchGraph graph;
  int spec_nb = 0;       // flags of a speculative first pass still to check
  int sms = 0;           // SM count of the device (cached)
  int direct_copy = 0;  // host API: copy straight from/to the caller's (pageable) buffers (env DPQ_DIRECT_COPY)
  int run_filter = 1;  // flat sorted rows: scan only chunks whose keys can reach a guard (env DPQ_RUN_FILTER=0)
  uint32_t* chunk_keys = nullptr;  // [n_chunks] first | last key << 16 of each 128-row chunk
  uint32_t* key_start = nullptr;   // [65537] first row of every (g0, g1) key (sorted flat rows)
  int direct = 1;          // per-query direct scan of the few (g0, g1) runs a query can hit (env DPQ_DIRECT=0 disables)
  // Adaptive: after batches in which every query took the direct scan the tile kernels are not even
  // launched (a query that needs them makes K3 flag the batch, which is redone with them).
  int tile_skip = 0;       // current mode (starts on for indexes with a direct scan, dpq_flat_create)
  int skip_streak = 0;     // consecutive all-direct speculative batches
  int tile_skip_ok = 1;    // env DPQ_TILE_SKIP=0 disables
  bool dir_batch = false;  // the last first pass ran k_key_select (h_tileq is valid after its sync)
  int gt_slack = 1;        // group-table activity test tightened by the other subspaces' minima (env DPQ_GT_SLACK=0)
  int direct_items = 0;    // work-item budget per batch (env DPQ_DIRECT_ITEMS; 0: 192 per query)
  int64_t n_chunks = 0;
  // tensor-core full tables (dpq_tctab.cu): prepared operand, per-batch
  // entry error bounds, mode (-1 auto: dsub >= 64; env DPQ_TC_TABLES=0/1)
  void* tct = nullptr;
  double* tct_eps = nullptr;  // (nq, m) per-(query, subspace) bounds
  double* tct_ny = nullptr;   // (nq, m) ||y'||
  int64_t tct_eps_cap = 0;
  int use_tc = -1;
  bool emit32 = false;        // 4-byte emit records (flat, n < 2^24)
  int qt = 0;                 // queries per scan tile (set at creation from mpad; ivf m <= 4: 64)
  bool ivf_dev_plan = true;   // env DPQ_IVF_DEVPLAN=0: the host-built ivf plan
  int probe_tc = 1;           // env DPQ_PROBE_TC at creation: 0 f64 probe, 1 tensor cores for K >= 1024, 2 always
  double tc_eps_scale = 1.0;  // env DPQ_TC_EPS_SCALE (tests: tighten to force more exact re-ranks)
  Workspace ws;
  // sharded-search state between dpq_shard_* calls
  int shard_nq = 0;
  int64_t shard_samp = 0;
  int shard_ma = 0;          // ivf shard: probes of the current batch
  int64_t shard_stride = 1;  // ivf shard: sampling stride of the current batch (1 = exact)
};

}  // namespace dpq
