// dpq_container.cu — model/index containers straight to the device (SURVEY
// §8f rank 4).
//
// Replaces the bulk half of derivedpq.vecio.load_model (vecio.py:156-198):
// the container's array bytes are read from the file by a few host threads
// into pinned buffers and copied to HBM while the next piece is read; the
// per-array checksum the container header records (zlib CRC-32, vecio.py:
// 141,188-192) is computed ON THE DEVICE over the bytes that arrived there, so
// a 16-GB index never takes a host CRC pass; and the structural checks of
// validate() that touch the bulk arrays (code range, flat.py:112-118;
// inverted lists partition the database and agree with cell_of,
// ivf.py:280-292) run as device reductions.  The JSON header is parsed by the
// Python mirror (paper_1905_06900_b200/container.py), which passes the array
// byte ranges here.
//
// Device CRC-32 (reflected, poly 0xEDB88320, zlib conventions).  The CRC is
// linear over GF(2): with A_n = "advance the register over n zero bytes" and
// raw(M) = the register after M from 0,
//   raw(M1 || M2) = A_|M2|(raw(M1)) ^ raw(M2),
//   zlib(M)       = ~(A_|M|(0xFFFFFFFF) ^ raw(M)).
// A CTA owns 256-KB chunks; thread t reads the 16-byte words at 16 t + 4096 g
// (g = 0..63: perfectly coalesced 128-bit loads) and absorbs each 4-byte
// word with the byte-sliced table of A_4, then jumps the register over the
// 4084 bytes other threads own with the table of A_4084 — so every thread
// carries "its words, zeros elsewhere".  The last word of each thread only
// advances A_4, leaving thread t's register positioned 16 (255 - t) bytes
// before the chunk end; a shuffle tree with A_{16 2^k} (then A_512 across
// warps) folds them into the chunk's raw CRC at the chunk end, which one
// thread advances to the end of the array and XORs into the array's
// accumulator.  A ragged tail (< 256 KB) is copied into a zero-padded
// scratch chunk and un-padded with A_{(2^32-1) - z} = A_z^{-1} (x has order
// 2^32 - 1 modulo the CRC-32 polynomial).  Cost: one shared-memory table
// lookup per byte — 2-4 TB/s on a B200, far above PCIe / page-cache rates.

#include <cuda_runtime.h>
#include <fcntl.h>
#include <omp.h>
#include <stdint.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <mutex>
#include <string>
#include <vector>

#include "dpq.h"
#include "dpq_impl.h"

namespace dpq {
namespace crc {

constexpr int kThreads = 256;
constexpr int kGroupBytes = 16;
constexpr int kStride = kThreads * kGroupBytes;  // 4096 bytes between one thread's words
constexpr int kGroups = 64;
constexpr int64_t kChunk = (int64_t)kStride * kGroups;  // 256 KB per CTA iteration
constexpr uint32_t kOrder = 0xFFFFFFFFu;                // multiplicative order of x mod P

struct Tables {
  uint32_t t4[4][256];    // A_4, byte-sliced: A_4(v) = ^_k t4[k][byte k of v]
  uint32_t tj[4][256];    // A_{kStride - 12}
  uint32_t tree[5][32];   // A_{16 * 2^k} as 32 columns (k = 0..4)
  uint32_t w512[32];      // A_512
  uint32_t pow2[32][32];  // A_{2^i}
};

// ---------------------------------------------------------- host algebra --
using Mat = std::vector<uint32_t>;  // 32 columns: M(1 << b)

static uint32_t apply_h(const Mat& m, uint32_t v) {
  uint32_t r = 0;
  for (int b = 0; b < 32; ++b)
    if ((v >> b) & 1u) r ^= m[b];
  return r;
}

static Mat mul_h(const Mat& a, const Mat& b) {  // a o b
  Mat r(32);
  for (int i = 0; i < 32; ++i) r[i] = apply_h(a, b[i]);
  return r;
}

static Mat adv_h(const std::vector<Mat>& pw, uint64_t n) {
  Mat r(32);
  for (int b = 0; b < 32; ++b) r[b] = 1u << b;
  n %= kOrder;
  for (int i = 0; n; ++i, n >>= 1)
    if (n & 1) r = mul_h(pw[i], r);
  return r;
}

static void build(Tables* t) {
  uint32_t byte_tab[256];
  for (uint32_t i = 0; i < 256; ++i) {
    uint32_t c = i;
    for (int j = 0; j < 8; ++j) c = (c >> 1) ^ ((c & 1u) ? 0xEDB88320u : 0u);
    byte_tab[i] = c;
  }
  Mat a1(32);
  for (int b = 0; b < 32; ++b) {
    const uint32_t v = 1u << b;
    a1[b] = (v >> 8) ^ byte_tab[v & 0xFFu];  // one zero byte
  }
  std::vector<Mat> pw{a1};
  for (int i = 1; i < 32; ++i) pw.push_back(mul_h(pw.back(), pw.back()));
  for (int i = 0; i < 32; ++i) std::copy(pw[i].begin(), pw[i].end(), t->pow2[i]);
  const Mat a4 = adv_h(pw, 4), aj = adv_h(pw, kStride - 12);
  for (int k = 0; k < 4; ++k)
    for (uint32_t b = 0; b < 256; ++b) {
      t->t4[k][b] = apply_h(a4, b << (8 * k));
      t->tj[k][b] = apply_h(aj, b << (8 * k));
    }
  for (int k = 0; k < 5; ++k) {
    const Mat m = adv_h(pw, (uint64_t)16 << k);
    std::copy(m.begin(), m.end(), t->tree[k]);
  }
  const Mat m512 = adv_h(pw, 512);
  std::copy(m512.begin(), m512.end(), t->w512);
}

// Per-device copy of the tables (built once per process).
static const Tables* device_tables(int device) {
  static std::mutex mu;
  static std::vector<Tables*> per_dev;
  static Tables host;
  static bool built = false;
  std::lock_guard<std::mutex> lock(mu);
  if (!built) {
    build(&host);
    built = true;
  }
  if ((int)per_dev.size() <= device) per_dev.resize(device + 1, nullptr);
  if (!per_dev[device]) {
    Tables* d = nullptr;
    if (cudaMalloc(&d, sizeof(Tables)) != cudaSuccess) return nullptr;
    if (cudaMemcpy(d, &host, sizeof(Tables), cudaMemcpyHostToDevice) != cudaSuccess) {
      cudaFree(d);
      return nullptr;
    }
    per_dev[device] = d;
  }
  return per_dev[device];
}

// --------------------------------------------------------------- device --
__device__ __forceinline__ uint32_t apply_m(const uint32_t* __restrict__ m, uint32_t v) {
  uint32_t r = 0;
#pragma unroll
  for (int b = 0; b < 32; ++b) r ^= m[b] & (0u - ((v >> b) & 1u));
  return r;
}

__device__ __forceinline__ uint32_t advance(const uint32_t (*pow2)[32], uint32_t v, uint64_t n) {
  n %= kOrder;
  for (int i = 0; n; ++i, n >>= 1)
    if (n & 1) v = apply_m(pow2[i], v);
  return v;
}

__device__ __forceinline__ uint32_t sliced(const uint32_t (*t)[256], uint32_t v) {
  return t[0][v & 0xFFu] ^ t[1][(v >> 8) & 0xFFu] ^ t[2][(v >> 16) & 0xFFu] ^ t[3][v >> 24];
}

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// Raw CRC of `nchunks` full 256-KB chunks starting at p (16-B aligned),
// each advanced to the message end (`after` bytes follow the last chunk) and
// XOR-ed into *acc.
__global__ void __launch_bounds__(kThreads) k_crc_chunks(const uint4* __restrict__ p, int64_t nchunks,
                                                         uint64_t after, const Tables* __restrict__ tab,
                                                         uint32_t* __restrict__ acc) {
  __shared__ uint32_t t4[4][256], tj[4][256], tree[5][32], w512[32], pow2[32][32];
  __shared__ uint32_t wv[kThreads / 32];
  for (int i = threadIdx.x; i < 1024; i += kThreads) {
    (&t4[0][0])[i] = (&tab->t4[0][0])[i];
    (&tj[0][0])[i] = (&tab->tj[0][0])[i];
    (&pow2[0][0])[i] = (&tab->pow2[0][0])[i];
  }
  for (int i = threadIdx.x; i < 160; i += kThreads) (&tree[0][0])[i] = (&tab->tree[0][0])[i];
  if (threadIdx.x < 32) w512[threadIdx.x] = tab->w512[threadIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const uint4* q = p + c * (kChunk / 16) + threadIdx.x;
    uint32_t s = 0;
#pragma unroll 8
    for (int g = 0; g < kGroups - 1; ++g) {
      const uint4 w = ld_stream(q + g * kThreads);
      s = sliced(t4, s ^ w.x);
      s = sliced(t4, s ^ w.y);
      s = sliced(t4, s ^ w.z);
      s = sliced(tj, s ^ w.w);
    }
    {
      const uint4 w = ld_stream(q + (kGroups - 1) * kThreads);
      s = sliced(t4, s ^ w.x);
      s = sliced(t4, s ^ w.y);
      s = sliced(t4, s ^ w.z);
      s = sliced(t4, s ^ w.w);
    }
    // thread t sits 16 (255 - t) bytes before the chunk end: fold to lane 31
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, s, 1 << k);
      const int mask = (2 << k) - 1;
      const uint32_t moved = apply_m(tree[k], o);
      if ((lane & mask) == mask) s ^= moved;
    }
    if (lane == 31) wv[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t v = wv[0];
      for (int w = 1; w < kThreads / 32; ++w) v = apply_m(w512, v) ^ wv[w];
      v = advance(pow2, v, (uint64_t)(nchunks - 1 - c) * kChunk + after);
      atomicXor(acc, v);
    }
    __syncthreads();
  }
}

// zlib value from the accumulators: acc[0] = raw CRC of the full chunks,
// acc[1] = raw CRC of the zero-padded tail chunk (z padding bytes).
__global__ void k_crc_final(const uint32_t* __restrict__ acc, uint64_t len, uint64_t z,
                            const Tables* __restrict__ tab, uint32_t* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  uint32_t raw = acc[0] ^ advance(tab->pow2, acc[1], (uint64_t)kOrder - (z % kOrder));
  *out = ~(advance(tab->pow2, 0xFFFFFFFFu, len) ^ raw);
}

// zlib CRC-32 of a device buffer into *out_dev (device), enqueued on `st`.
// scratch: kChunk bytes + 2 u32 accumulators (device).
static int crc32_enqueue(int device, const uint8_t* data, uint64_t len, uint8_t* scratch, uint32_t* acc2,
                         uint32_t* out_dev, cudaStream_t st) {
  const Tables* tab = device_tables(device);
  if (!tab) {
    set_error("CRC table upload failed");
    return DPQ_ERR_CUDA;
  }
  if (((uintptr_t)data & 15u) != 0) {
    set_error("CRC input must be 16-byte aligned");
    return DPQ_ERR_ARG;
  }
  const int64_t full = (int64_t)(len / kChunk);
  const uint64_t tail = len - (uint64_t)full * kChunk;
  if (cudaMemsetAsync(acc2, 0, 8, st) != cudaSuccess) goto fail;
  if (full > 0) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int grid = (int)std::min<int64_t>(full, (int64_t)sms * 6);
    k_crc_chunks<<<grid, kThreads, 0, st>>>(reinterpret_cast<const uint4*>(data), full, tail, tab, acc2);
  }
  if (tail > 0) {
    if (cudaMemsetAsync(scratch + tail, 0, kChunk - tail, st) != cudaSuccess ||
        cudaMemcpyAsync(scratch, data + (uint64_t)full * kChunk, tail, cudaMemcpyDefault, st) != cudaSuccess)
      goto fail;
    k_crc_chunks<<<1, kThreads, 0, st>>>(reinterpret_cast<const uint4*>(scratch), 1, 0, tab, acc2 + 1);
  }
  k_crc_final<<<1, 32, 0, st>>>(acc2, len, tail ? (uint64_t)kChunk - tail : 0, tab, out_dev);
  if (cudaGetLastError() != cudaSuccess) goto fail;
  return DPQ_OK;
fail:
  set_error(std::string("device CRC-32: ") + cudaGetErrorString(cudaGetLastError()));
  return DPQ_ERR_CUDA;
}

}  // namespace crc

// ----------------------------------------------------- device validation --
template <typename T>
__global__ void k_codes_max(const T* __restrict__ c, int64_t n, unsigned* __restrict__ out) {
  unsigned mx = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    mx = max(mx, (unsigned)c[i]);
  for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, mx);
}

// seen[id] = 1 for every in-range id; out-of-range ids counted in bad[0].
__global__ void k_perm_mark(const int64_t* __restrict__ ids, int64_t n, uint8_t* __restrict__ seen,
                            unsigned long long* __restrict__ bad) {
  unsigned long long b = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = ids[i];
    if (v < 0 || v >= n) ++b;
    else seen[v] = 1;
  }
  for (int o = 16; o; o >>= 1) b += __shfl_xor_sync(0xFFFFFFFFu, b, o);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(bad, b);
}

// rows never marked (a missing id means another one repeats) into bad[1].
__global__ void k_perm_holes(const uint8_t* __restrict__ seen, int64_t n, unsigned long long* __restrict__ bad) {
  unsigned long long b = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b += seen[i] == 0;
  for (int o = 16; o; o >>= 1) b += __shfl_xor_sync(0xFFFFFFFFu, b, o);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(bad + 1, b);
}

// counts[c] = |{i : cell_of[i] == c}| (shared-memory privatised when K fits);
// out-of-range cells into bad[0].
__global__ void k_bincount(const int32_t* __restrict__ cell, int64_t n, int K, unsigned long long* __restrict__ counts,
                           unsigned long long* __restrict__ bad) {
  extern __shared__ unsigned sh[];
  const bool priv = K <= 12288;
  if (priv)
    for (int i = threadIdx.x; i < K; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  unsigned long long b = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = cell[i];
    if (c < 0 || c >= K) ++b;
    else if (priv) atomicAdd(&sh[c], 1u);
    else atomicAdd(&counts[c], 1ull);
  }
  for (int o = 16; o; o >>= 1) b += __shfl_xor_sync(0xFFFFFFFFu, b, o);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(bad, b);
  __syncthreads();
  if (priv)
    for (int i = threadIdx.x; i < K; i += blockDim.x)
      if (sh[i]) atomicAdd(&counts[i], (unsigned long long)sh[i]);
}

static int grid_for(int device, int64_t n) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sms * 8));
}

}  // namespace dpq

using namespace dpq;

namespace {

struct DevAllocs {  // freed on scope exit unless released
  std::vector<void*> p;
  int device = 0;
  ~DevAllocs() {
    cudaSetDevice(device);
    for (void* x : p) cudaFree(x);
  }
};

#define CK(call)                                                                                   \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess) {                                                                       \
      set_error(std::string(#call) + ": " + cudaGetErrorString(e_));                               \
      return DPQ_ERR_CUDA;                                                                         \
    }                                                                                              \
  } while (0)

}  // namespace

extern "C" {

int dpq_crc32_dev(int device, const void* data, int64_t len, uint32_t* crc) {
  if (len < 0 || (len > 0 && !data) || !crc) {
    set_error("bad CRC arguments");
    return DPQ_ERR_ARG;
  }
  CK(cudaSetDevice(device));
  DevAllocs tmp;
  tmp.device = device;
  uint8_t* scratch = nullptr;
  uint32_t* acc = nullptr;
  CK(cudaMalloc(&scratch, crc::kChunk));
  tmp.p.push_back(scratch);
  CK(cudaMalloc(&acc, 16));
  tmp.p.push_back(acc);
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  int rc = crc::crc32_enqueue(device, static_cast<const uint8_t*>(data), (uint64_t)len, scratch, acc, acc + 2, st);
  if (rc == DPQ_OK && cudaMemcpyAsync(crc, acc + 2, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess) rc = DPQ_ERR_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess && rc == DPQ_OK) {
    set_error("device CRC-32 failed");
    rc = DPQ_ERR_CUDA;
  }
  cudaStreamDestroy(st);
  return rc;
}

int dpq_container_read(int device, const char* path, int n_arrays, const int64_t* offsets, const int64_t* nbytes,
                       int verify, int threads, void** dev_out, uint32_t* crc_out, double* stats4) {
  if (!path || n_arrays < 0 || (n_arrays > 0 && (!offsets || !nbytes || !dev_out || (verify && !crc_out)))) {
    set_error("bad container arguments");
    return DPQ_ERR_ARG;
  }
  for (int a = 0; a < n_arrays; ++a)
    if (offsets[a] < 0 || nbytes[a] < 0) {
      set_error("negative array range");
      return DPQ_ERR_ARG;
    }
  const auto t0 = std::chrono::steady_clock::now();
  CK(cudaSetDevice(device));
  const int fd = open(path, O_RDONLY);
  if (fd < 0) {
    set_error(std::string("cannot open ") + path);
    return DPQ_ERR_ARG;
  }
  struct Closer {
    int fd;
    ~Closer() { close(fd); }
  } closer{fd};
  struct stat sb;
  if (fstat(fd, &sb) != 0) {
    set_error("fstat failed");
    return DPQ_ERR_ARG;
  }
  for (int a = 0; a < n_arrays; ++a)
    if (offsets[a] + nbytes[a] > (int64_t)sb.st_size) {
      set_error("array " + std::to_string(a) + " runs past the end of the file");
      return DPQ_ERR_ARG;
    }
  if (threads < 1) threads = 1;
  DevAllocs out;  // released to the caller on success
  out.device = device;
  DevAllocs tmp;
  tmp.device = device;
  constexpr size_t kPiece = (size_t)64 << 20;
  uint8_t* pinned[2] = {nullptr, nullptr};
  struct PinnedFree {
    uint8_t** p;
    ~PinnedFree() {
      for (int i = 0; i < 2; ++i)
        if (p[i]) cudaFreeHost(p[i]);
    }
  } pf{pinned};
  CK(cudaHostAlloc((void**)&pinned[0], kPiece, cudaHostAllocDefault));
  CK(cudaHostAlloc((void**)&pinned[1], kPiece, cudaHostAllocDefault));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamFree {
    cudaStream_t s;
    cudaEvent_t e[4];
    ~StreamFree() {
      for (auto x : e)
        if (x) cudaEventDestroy(x);
      cudaStreamDestroy(s);
    }
  } sf{st, {nullptr, nullptr, nullptr, nullptr}};
  CK(cudaEventCreateWithFlags(&sf.e[0], cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&sf.e[1], cudaEventDisableTiming));
  uint8_t* scratch = nullptr;
  uint32_t* acc = nullptr;
  if (verify) {
    CK(cudaMalloc(&scratch, crc::kChunk));
    tmp.p.push_back(scratch);
    CK(cudaMalloc(&acc, (size_t)std::max(n_arrays, 1) * 16));
    tmp.p.push_back(acc);
  }
  double read_s = 0.0;
  int64_t total = 0;
  int cur = 0;
  bool pending[2] = {false, false};
  for (int a = 0; a < n_arrays; ++a) {
    uint8_t* d = nullptr;
    CK(cudaMalloc(&d, (size_t)std::max<int64_t>(nbytes[a], 16)));
    out.p.push_back(d);
    for (int64_t pos = 0; pos < nbytes[a]; pos += kPiece) {
      const int64_t len = std::min<int64_t>((int64_t)kPiece, nbytes[a] - pos);
      if (pending[cur]) CK(cudaEventSynchronize(sf.e[cur]));  // the copy out of this buffer is done
      const auto r0 = std::chrono::steady_clock::now();
      const int64_t part = (len + threads - 1) / threads;
      int bad = 0;
#pragma omp parallel for num_threads(threads) reduction(+ : bad)
      for (int t = 0; t < threads; ++t) {
        int64_t o = t * part, e = std::min<int64_t>(len, o + part);
        while (o < e) {
          const ssize_t got = pread(fd, pinned[cur] + o, (size_t)(e - o), (off_t)(offsets[a] + pos + o));
          if (got <= 0) {
            ++bad;
            break;
          }
          o += got;
        }
      }
      read_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - r0).count();
      if (bad) {
        set_error("read failed inside array " + std::to_string(a));
        return DPQ_ERR_ARG;
      }
      CK(cudaMemcpyAsync(d + pos, pinned[cur], (size_t)len, cudaMemcpyHostToDevice, st));
      CK(cudaEventRecord(sf.e[cur], st));
      pending[cur] = true;
      cur ^= 1;
      total += len;
    }
    if (verify) {
      int rc = crc::crc32_enqueue(device, d, (uint64_t)nbytes[a], scratch, acc + 4 * a, acc + 4 * a + 2, st);
      if (rc != DPQ_OK) return rc;
    }
  }
  CK(cudaStreamSynchronize(st));
  if (verify) {
    std::vector<uint32_t> h((size_t)std::max(n_arrays, 1) * 4);
    CK(cudaMemcpy(h.data(), acc, h.size() * 4, cudaMemcpyDeviceToHost));
    for (int a = 0; a < n_arrays; ++a) crc_out[a] = h[4 * a + 2];
  }
  for (int a = 0; a < n_arrays; ++a) dev_out[a] = out.p[a];
  out.p.clear();
  if (stats4) {
    stats4[0] = (double)total;
    stats4[1] = read_s;
    stats4[2] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    stats4[3] = (double)n_arrays;
  }
  return DPQ_OK;
}

int dpq_dev_free(int device, void* p) {
  if (!p) return DPQ_OK;
  CK(cudaSetDevice(device));
  CK(cudaFree(p));
  return DPQ_OK;
}

int dpq_dev_download(int device, const void* src, int64_t nbytes, void* dst) {
  if (nbytes < 0 || (nbytes > 0 && (!src || !dst))) {
    set_error("bad download arguments");
    return DPQ_ERR_ARG;
  }
  CK(cudaSetDevice(device));
  if (nbytes) CK(cudaMemcpy(dst, src, (size_t)nbytes, cudaMemcpyDeviceToHost));
  return DPQ_OK;
}

int dpq_dev_codes_max(int device, const void* codes, int64_t count, int code_bytes, int64_t* out_max) {
  if (count < 0 || (count > 0 && !codes) || !out_max || (code_bytes != 1 && code_bytes != 2)) {
    set_error("bad code-range arguments");
    return DPQ_ERR_ARG;
  }
  CK(cudaSetDevice(device));
  unsigned* d = nullptr;
  CK(cudaMalloc(&d, 4));
  DevAllocs tmp;
  tmp.device = device;
  tmp.p.push_back(d);
  CK(cudaMemset(d, 0, 4));
  if (count > 0) {
    const int g = grid_for(device, count);
    if (code_bytes == 1) k_codes_max<uint8_t><<<g, 256>>>(static_cast<const uint8_t*>(codes), count, d);
    else k_codes_max<uint16_t><<<g, 256>>>(static_cast<const uint16_t*>(codes), count, d);
    CK(cudaGetLastError());
  }
  unsigned h = 0;
  CK(cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost));
  *out_max = count > 0 ? (int64_t)h : -1;
  return DPQ_OK;
}

int dpq_dev_check_permutation(int device, const int64_t* ids, int64_t n, int64_t* out2) {
  if (n < 0 || (n > 0 && !ids) || !out2) {
    set_error("bad permutation arguments");
    return DPQ_ERR_ARG;
  }
  CK(cudaSetDevice(device));
  out2[0] = out2[1] = 0;
  if (n == 0) return DPQ_OK;
  DevAllocs tmp;
  tmp.device = device;
  uint8_t* seen = nullptr;
  unsigned long long* bad = nullptr;
  CK(cudaMalloc(&seen, (size_t)n));
  tmp.p.push_back(seen);
  CK(cudaMalloc(&bad, 16));
  tmp.p.push_back(bad);
  CK(cudaMemset(seen, 0, (size_t)n));
  CK(cudaMemset(bad, 0, 16));
  const int g = grid_for(device, n);
  k_perm_mark<<<g, 256>>>(ids, n, seen, bad);
  k_perm_holes<<<g, 256>>>(seen, n, bad);
  CK(cudaGetLastError());
  unsigned long long h[2];
  CK(cudaMemcpy(h, bad, 16, cudaMemcpyDeviceToHost));
  out2[0] = (int64_t)h[0];
  out2[1] = (int64_t)h[1];
  return DPQ_OK;
}

int dpq_dev_bincount(int device, const int32_t* cells, int64_t n, int n_cells, int64_t* counts, int64_t* n_bad) {
  if (n < 0 || n_cells < 1 || (n > 0 && !cells) || !counts || !n_bad) {
    set_error("bad bincount arguments");
    return DPQ_ERR_ARG;
  }
  CK(cudaSetDevice(device));
  DevAllocs tmp;
  tmp.device = device;
  unsigned long long* d = nullptr;
  CK(cudaMalloc(&d, ((size_t)n_cells + 1) * 8));
  tmp.p.push_back(d);
  CK(cudaMemset(d, 0, ((size_t)n_cells + 1) * 8));
  if (n > 0) {
    const size_t smem = n_cells <= 12288 ? (size_t)n_cells * 4 : 0;
    k_bincount<<<grid_for(device, n), 256, smem>>>(cells, n, n_cells, d, d + n_cells);
    CK(cudaGetLastError());
  }
  std::vector<unsigned long long> h((size_t)n_cells + 1);
  CK(cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost));
  for (int c = 0; c < n_cells; ++c) counts[c] = (int64_t)h[c];
  *n_bad = (int64_t)h[n_cells];
  return DPQ_OK;
}

}  // extern "C"
