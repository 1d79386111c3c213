// dpq_tctab.cu — full-codebook distance tables on the 5th-generation tensor
// cores (tcgen05 + TMEM, kind::tf32), sm_100a.  north_star (i).
//
// Replaces compute_tables(yr, codebooks_) (search.py:28-48) — the m x k
// table of ||y_j - c_jc||^2 per query — as one GEMM-shaped contraction per
// subspace with cached centroid norms:
//
//   T~[q, j, c] = ||c'||^2 - 2 y'.c' + ||y'||^2,   y' = y_j - mu_j, c' = c - mu_j
//
// (mu_j = the subspace's codebook mean, so the norms stay small), computed
// 3xTF32 as in dpq_encode.cu: y' = y_hi + y_lo, -2c' = hi + lo split at tf32
// precision, ||c'||^2 (f64) split into three tf32 pieces folded in by one
// extra MMA against a constant "ones" block, ||y'||^2 added in the epilogue.
//
// These entries are NOT numpy's bits (the reference sums (c - y)^2 pairwise
// in f32): every entry carries a rigorous error bound eps[q, j] (written
// next to the tables), and the refine that consumes them (k_refine_topk,
// MODE_EMIT_APPROX) re-ranks exactly: it finds the r-th smallest approximate
// distance A_r, then recomputes the exact numpy entries of every candidate
// whose approximate distance is <= A_r + 2 * sum_j eps[q, j] — a set that
// provably contains the exact top-r — so results stay bit-identical to the
// reference.
//
// Layout: tables are written group-major, exactly where the lazy exact
// builder (k_group_tables) puts them: entry e = g * gsize + ibar of
// subspace j (centroid c = ibar * kbar + g) at (q * m + j) * k + e.  One
// N = 256 tile covers entries [256 t, 256 t + 256), so a tile row is 1 KB of
// contiguous output.  The centroid operand is prepared once per index in
// K-chunks of 16 f32 (SWIZZLE_64B, K-major): per tile and chunk
// [hi 16 KB | lo 16 KB], then an 8-KB norm block.
//
// Kernel (persistent, one CTA per SM, 10 warps; same roles as the encoder):
//   warp 0     TMA producer: chunk-by-chunk cp.async.bulk into a 2-stage ring
//   warp 1     TMEM allocator + MMA issuer: per tile 2 k-steps x (hi.hi,
//              hi.lo[, lo.hi]) per chunk + the norm MMA, M = 128, N = 256,
//              into a double-buffered TMEM accumulator (2 x 256 columns)
//   warps 2-9  stage the unit's 128 query rows (y' hi/lo, ||y'||^2, eps),
//              then drain TMEM (tcgen05.ld, 32 columns at a time), add
//              ||y'||^2 and store the tile's rows (128 B per thread per load).
// A unit is (subspace j, range of tiles, block of 128 queries); query blocks
// vary fastest, so the CTAs running together stream the same centroid tiles
// (L2 reuse of the operand across query blocks).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>

#include "../../include/dpq.h"
#include "dpq_impl.h"

namespace dpq {
namespace tct {

constexpr int BN = 256;                     // entries per tile (MMA N)
constexpr int BM = 128;                     // queries per block (MMA M)
constexpr int KCH = 16;                     // f32 per K-chunk (64-B rows, SWIZZLE_64B)
constexpr int KC_MAX = 8;                   // dsub <= 128
constexpr int CH_B = BN * 64;               // 16 KB: one chunk of 256 centroid rows (hi or lo)
constexpr int CH_A = BM * 64;               // 8 KB: one chunk of 128 query rows (hi or lo)
constexpr int NORMB = BN * 32;              // 8 KB: 256 rows x 8 f32, no swizzle (core matrices)
constexpr int NORMB_A = BM * 32;            // 4 KB: the constant "ones" A block
constexpr int STAGE_B = 2 * CH_B;           // 32 KB ring slot (a chunk's hi + lo, or a norm block)
constexpr int STAGES = 2;
constexpr int kThreads = 320;
constexpr int kEpiWarps = 8;
constexpr int OFF_A = 0;                             // KC_MAX x (hi 8 KB | lo 8 KB) = 128 KB
constexpr int OFF_B = OFF_A + KC_MAX * 2 * CH_A;     // 131072
constexpr int OFF_ONES = OFF_B + STAGES * STAGE_B;   // +65536
constexpr int OFF_YN = OFF_ONES + NORMB_A;           // ||y'||^2 of the block's rows (f32)
constexpr int OFF_BAR = OFF_YN + BM * 4;
constexpr int SMEM_BYTES = OFF_BAR + 256 + 1024;     // + alignment slack
constexpr uint32_t kTmemCols = 512;
constexpr float kPadNorm = 1.2676506e30f;

__host__ __device__ constexpr int tile_bytes(int kc) { return kc * STAGE_B + NORMB; }

// Byte offset of (row r, 16-B chunk ch < 4) in a SWIZZLE_64B K-major atom
// stack: 8-row groups of 512 B, chunk index XOR bits 1-2 of the row.
__host__ __device__ constexpr int sw64(int r, int ch) {
  return (r >> 3) * 512 + (r & 7) * 64 + ((ch ^ ((r >> 1) & 3)) << 4);
}
__host__ __device__ constexpr int nrm(int r, int e) {
  return (r >> 3) * 256 + (e >> 2) * 128 + (r & 7) * 16 + (e & 3) * 4;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
// Bounded wait: a protocol bug traps (a CUDA error) instead of hanging the GPU.
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok = 0;
  for (uint64_t spin = 0;; ++spin) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(su32(b)), "r"(parity)
        : "memory");
    if (ok) return;
    if (spin > (1ull << 26)) __trap();
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(b))
      : "memory");
}
// UMMA shared-memory descriptors (sm_100: version bits [46,48) = 1)
__device__ __forceinline__ uint64_t desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;           // LBO (unused for swizzled K-major)
  d |= (uint64_t)(512 >> 4) << 32;  // SBO: 8-row groups 512 B apart
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;           // SWIZZLE_64B
  return d;
}
__device__ __forceinline__ uint64_t desc_plain(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(128 >> 4) << 16;  // LBO: K halves 128 B apart
  d |= (uint64_t)(256 >> 4) << 32;  // SBO: 8-row groups 256 B apart
  d |= (uint64_t)1 << 46;
  return d;
}
// kind::tf32, D f32, A/B tf32 K-major, M = 128, N = 256
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b))
               : "memory");
}
__device__ __forceinline__ void tc_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// ---- operand preparation (once per index) ----------------------------------
// mu[j][t] = mean over the k centroids of subspace j (f64 sum, f32 result).
__global__ void k_tct_mean(const float* __restrict__ cb, int k, int dsub, float* __restrict__ mu) {
  const int j = blockIdx.x, t = blockIdx.y;
  __shared__ double red[256];
  double s = 0.0;
  for (int c = threadIdx.x; c < k; c += 256) s += (double)cb[((int64_t)j * k + c) * dsub + t];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) mu[j * dsub + t] = (float)(red[0] / (double)k);
}

// Centroid operand: one thread per (subspace, padded group-major entry e).
// Also R[j] = max_c ||c'|| (f64 bits, atomic max of the non-negative value).
__global__ void k_tct_prep(const float* __restrict__ cb, const float* __restrict__ mu, int m, int k, int kbar,
                           int dsub, int kc, int nt, uint8_t* __restrict__ img, unsigned long long* __restrict__ rmax,
                           float* __restrict__ cnorm) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t kp = (int64_t)nt * BN;
  if (gid >= (int64_t)m * kp) return;
  const int j = (int)(gid / kp), e = (int)(gid % kp), t = e / BN, r = e % BN;
  const int gsize = k / kbar;
  const bool live = e < k;
  const int c = live ? (e % gsize) * kbar + e / gsize : 0;  // centroid of group-major entry e
  uint8_t* blk = img + ((int64_t)j * nt + t) * tile_bytes(kc);
  double n2 = 0.0;
  for (int ck = 0; ck < kc; ++ck) {
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
      float hi[4], lo[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int dd = ck * KCH + q4 * 4 + u;
        const float v = (live && dd < dsub) ? __fsub_rn(cb[((int64_t)j * k + c) * dsub + dd], mu[j * dsub + dd]) : 0.f;
        n2 += (double)v * (double)v;
        const float w = -2.f * v;  // exact
        hi[u] = tf32_rna(w);
        lo[u] = w - hi[u];         // exact in f32
      }
      *reinterpret_cast<float4*>(blk + ck * STAGE_B + sw64(r, q4)) = make_float4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<float4*>(blk + ck * STAGE_B + CH_B + sw64(r, q4)) = make_float4(lo[0], lo[1], lo[2], lo[3]);
    }
  }
  float p[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (live) {
    const float a = tf32_rna((float)n2);
    const double r1 = n2 - (double)a;
    const float b = tf32_rna((float)r1);
    const float cc = tf32_rna((float)(r1 - (double)b));
    p[0] = a; p[1] = b; p[2] = cc;
    atomicMax(rmax + j, (unsigned long long)__double_as_longlong(sqrt(n2)));
    cnorm[(int64_t)j * k + e] = __double2float_ru(sqrt(n2));  // ||c'|| rounded up, group-major entry order
  } else {
    p[0] = kPadNorm;
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) *reinterpret_cast<float*>(blk + kc * STAGE_B + nrm(r, u)) = p[u];
}

struct Args {
  const float* y;       // (nq, ystride) f32 queries (rotated), subspace j at columns [j*dsub, ...)
  int64_t ystride;
  int nq, m, k, dsub, kc, nt;
  const uint8_t* img;   // (m, nt, tile_bytes) centroid operand
  const float* mu;      // (m, dsub)
  const double* rmax;   // (m)
  float* tables;        // (nq, m, k) group-major
  double* eps;          // (nq, m) entry error bounds (with the subspace's largest ||c'||)
  double* ny;           // (nq, m) ||y'|| (optional: per-entry bounds gamma (||y'|| + ||c'||)^2)
  unsigned long long* argmin = nullptr;  // encoder mode (kbar = 1 operand): per (row, j) min of
                                         // (ordered ||c'||^2 - 2 y'.c', c); no tables written
  double gamma;         // error-bound coefficient (see tct_build)
  int ntr, tpr, nqb;    // tile ranges, tiles per range, query blocks
  int64_t units;        // m * ntr * nqb
};

__global__ void __launch_bounds__(kThreads, 1) k_tct_gemm(Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm + OFF_A;
  uint8_t* sB = sm + OFF_B;
  uint8_t* sOnes = sm + OFF_ONES;
  float* sYn = reinterpret_cast<float*>(sm + OFF_YN);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + OFF_BAR);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint64_t* afull = tempty + 2;      // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(afull + 1);
  volatile uint32_t* aflag = tmem_slot + 1;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { bar_init(&full[s], 1); bar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { bar_init(&tfull[b], 1); bar_init(&tempty[b], kEpiWarps); }
    bar_init(afull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (warp >= 2) {  // constant "ones" A operand of the norm MMA: rows (1, 1, 1, 0, ...)
    for (int i = threadIdx.x - 64; i < BM * 8; i += kEpiWarps * 32) {
      const int r = i >> 3, e = i & 7;
      *reinterpret_cast<float*>(sOnes + nrm(r, e)) = e < 3 ? 1.f : 0.f;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  const uint32_t tmem = *tmem_slot;
  const int kc = a.kc;
  const int tb = tile_bytes(kc);
  auto unit_of = [&](int64_t u, int& j, int& t0, int& t1, int& qb) {
    qb = (int)(u % a.nqb);
    const int tr = (int)((u / a.nqb) % a.ntr);
    j = (int)(u / ((int64_t)a.nqb * a.ntr));
    t0 = tr * a.tpr;
    t1 = min(a.nt, t0 + a.tpr);
  };

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer --
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      for (int64_t u = blockIdx.x; u < a.units; u += gridDim.x) {
        int j, t0, t1, qb;
        unit_of(u, j, t0, t1, qb);
        for (int t = t0; t < t1; ++t) {
          const uint8_t* g = a.img + ((int64_t)j * a.nt + t) * tb;
          for (int c = 0; c <= kc; ++c) {  // kc chunks, then the norm block
            const uint32_t bytes = c < kc ? STAGE_B : NORMB;
            bar_wait(&empty[stage], phase ^ 1);
            bar_expect_tx(&full[stage], bytes);
            bulk_g2s(sB + stage * STAGE_B, g + (int64_t)c * STAGE_B, bytes, &full[stage]);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // -------------------------------------------------------- MMA issuer --
    if (lane == 0) {
      uint32_t stage = 0, phase = 0, uphase = 0;
      uint64_t acc_t = 0;
      const uint32_t sA32 = su32(sA), sB32 = su32(sB), sOnes32 = su32(sOnes);
      for (int64_t u = blockIdx.x; u < a.units; u += gridDim.x) {
        int j, t0, t1, qb;
        unit_of(u, j, t0, t1, qb);
        bar_wait(afull, uphase);
        uphase ^= 1;
        const bool three = *aflag != 0;
        for (int t = t0; t < t1; ++t, ++acc_t) {
          const uint32_t buf = (uint32_t)(acc_t & 1), ap = (uint32_t)((acc_t >> 1) & 1);
          const uint32_t d = tmem + buf * BN;
          bar_wait(&tempty[buf], ap ^ 1);
          for (int c = 0; c < kc; ++c) {
            bar_wait(&full[stage], phase);
            tc_after_sync();
            const uint32_t bb = sB32 + stage * STAGE_B;
            const uint32_t ab = sA32 + c * 2 * CH_A;
#pragma unroll
            for (int s = 0; s < 2; ++s) {  // two k8 steps per 64-B row
              mma_tf32(d, desc_sw64(ab + s * 32), desc_sw64(bb + s * 32), (c | s) != 0);  // y_hi . hi
              mma_tf32(d, desc_sw64(ab + s * 32), desc_sw64(bb + CH_B + s * 32), 1);      // y_hi . lo
              if (three) mma_tf32(d, desc_sw64(ab + CH_A + s * 32), desc_sw64(bb + s * 32), 1);  // y_lo . hi
            }
            mma_commit(&empty[stage]);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          bar_wait(&full[stage], phase);  // norm block: + ||c'||^2
          tc_after_sync();
          mma_tf32(d, desc_plain(sOnes32), desc_plain(sB32 + stage * STAGE_B), 1);
          mma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
          mma_commit(&tfull[buf]);
        }
      }
    }
  } else {
    // ------------------------------------------------ staging + epilogue --
    const int et = threadIdx.x - 64;   // 0..255
    const int q4 = warp & 3;           // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;  // column half of each tile it drains
    const int row = q4 * 32 + lane;
    uint64_t acc_t = 0;
    for (int64_t u = blockIdx.x; u < a.units; u += gridDim.x) {
      int j, t0, t1, qb;
      unit_of(u, j, t0, t1, qb);
      {  // stage y' hi/lo of the block's 128 queries (the previous unit's MMAs are all complete)
        int any_lo = 0;
        if (et < BM) {
          const int64_t gq = (int64_t)qb * BM + et;
          const bool live = gq < a.nq;
          const float* src = a.y + gq * a.ystride + (int64_t)j * a.dsub;
          float yn = 0.f;
          double n2 = 0.0;
          for (int c = 0; c < kc; ++c) {
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
              float hi[4], lo[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int dd = c * KCH + ch * 4 + e;
                const float v = (live && dd < a.dsub) ? __fsub_rn(src[dd], a.mu[j * a.dsub + dd]) : 0.f;
                yn = __fadd_rn(yn, __fmul_rn(v, v));
                n2 += (double)v * (double)v;
                hi[e] = tf32_rna(v);
                lo[e] = v - hi[e];
                any_lo |= lo[e] != 0.f;
              }
              *reinterpret_cast<float4*>(sA + c * 2 * CH_A + sw64(et, ch)) = make_float4(hi[0], hi[1], hi[2], hi[3]);
              *reinterpret_cast<float4*>(sA + c * 2 * CH_A + CH_A + sw64(et, ch)) =
                  make_float4(lo[0], lo[1], lo[2], lo[3]);
            }
          }
          sYn[et] = yn;
          if (live && t0 == 0 && a.eps) {  // entry error bound of (query, subspace): once per (j, query block)
            const double s = sqrt(n2) + a.rmax[j];
            a.eps[gq * a.m + j] = a.gamma * s * s;
            if (a.ny) a.ny[gq * a.m + j] = sqrt(n2);
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        int any;
        asm volatile(
            "{\n\t.reg .pred p, q;\n\t"
            "setp.ne.s32 p, %1, 0;\n\t"
            "bar.red.or.pred q, 1, 256, p;\n\t"
            "selp.s32 %0, 1, 0, q;\n}"
            : "=r"(any)
            : "r"(any_lo)
            : "memory");
        if (et == 0) {
          *aflag = (uint32_t)any;
          bar_arrive(afull);
        }
      }
      const int64_t gq = (int64_t)qb * BM + row;
      const float yn = sYn[row];
      float* out = a.argmin ? nullptr : a.tables + (gq * a.m + j) * (int64_t)a.k;
      float best = INFINITY;  // encoder mode: running (min, first centroid) of this row's half
      int bidx = 0;
      for (int t = t0; t < t1; ++t, ++acc_t) {
        const uint32_t buf = (uint32_t)(acc_t & 1), ap = (uint32_t)((acc_t >> 1) & 1);
        bar_wait(&tfull[buf], ap);
        tc_after_sync();
        const uint32_t base = tmem + ((uint32_t)(q4 * 32) << 16) + buf * BN + half * (BN / 2);
#pragma unroll 1
        for (int ch = 0; ch < BN / 64; ++ch) {
          float v[32];
          tmem_ld32(base + ch * 32, v);
          const int e0 = t * BN + half * (BN / 2) + ch * 32;
          if (a.argmin) {  // pad entries (e >= k) carry a 2^100 norm: they never win
            float mn = v[0];
#pragma unroll
            for (int i = 1; i < 32; ++i) mn = fminf(mn, v[i]);
            if (mn < best) {  // first column holding the chunk minimum (lowest index on ties)
              int f = 31;
#pragma unroll
              for (int i = 31; i >= 0; --i) f = v[i] == mn ? i : f;
              best = mn;
              bidx = e0 + f;
            }
            continue;
          }
          if (gq < a.nq && e0 + 32 <= a.k) {
            float4* o = reinterpret_cast<float4*>(out + e0);
#pragma unroll
            for (int i = 0; i < 8; ++i)
              o[i] = make_float4(__fadd_rn(v[4 * i], yn), __fadd_rn(v[4 * i + 1], yn), __fadd_rn(v[4 * i + 2], yn),
                                 __fadd_rn(v[4 * i + 3], yn));
          } else if (gq < a.nq) {
            for (int i = 0; i < 32 && e0 + i < a.k; ++i) out[e0 + i] = __fadd_rn(v[i], yn);
          }
        }
        tc_before_sync();
        __syncwarp();
        if (lane == 0) bar_arrive(&tempty[buf]);
      }
      if (a.argmin && gq < a.nq) {  // (min value, then lowest centroid) across halves, ranges and CTAs
        uint32_t u = __float_as_uint(best);
        u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);  // order-preserving float -> u32
        atomicMin(a.argmin + gq * a.m + j, ((unsigned long long)u << 32) | (unsigned)bidx);
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");  // sYn / sA reuse by the next unit
    }
  }
  tc_before_sync();
  __syncthreads();
  if (warp == 1) {
    tc_after_sync();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
  }
}

}  // namespace tct

// Per-index prepared operand of the tensor-core table builder.
struct TcTables {
  int m = 0, k = 0, kbar = 0, dsub = 0, kc = 0, nt = 0;
  uint8_t* img = nullptr;
  float* mu = nullptr;
  double* rmax = nullptr;
  float* cnorm = nullptr;  // (m, k) ||c'|| in group-major entry order, rounded up
  int sms = 148;
};

#define TCT_CUDA(call)                                                                                  \
  do {                                                                                                  \
    cudaError_t e_ = (call);                                                                            \
    if (e_ != cudaSuccess) {                                                                            \
      set_error(std::string(#call) + ": " + cudaGetErrorString(e_) + " (dpq_tctab.cu:" +               \
                std::to_string(__LINE__) + ")");                                                        \
      return DPQ_ERR_CUDA;                                                                              \
    }                                                                                                   \
  } while (0)

bool tct_supported(int m, int k, int kbar, int dsub) {
  return m >= 1 && dsub >= 1 && dsub <= tct::KC_MAX * tct::KCH && k % 4 == 0 && kbar >= 1 && k % kbar == 0;
}

void tct_free(void* p) {
  TcTables* t = reinterpret_cast<TcTables*>(p);
  if (!t) return;
  cudaFree(t->img);
  cudaFree(t->mu);
  cudaFree(t->rmax);
  cudaFree(t->cnorm);
  delete t;
}

// Prepare the centroid operand of an index (codebooks cb (m, k, dsub) f32 on
// the device).  Synchronous on `stream`.
int tct_prepare(int device, const float* cb, int m, int k, int kbar, int dsub, cudaStream_t stream, void** out) {
  if (!tct_supported(m, k, kbar, dsub)) {
    set_error("tensor-core tables: unsupported shape (need dsub <= 128, 4 | k)");
    return DPQ_ERR_ARG;
  }
  TcTables* t = new TcTables();
  t->m = m; t->k = k; t->kbar = kbar; t->dsub = dsub;
  t->kc = (dsub + tct::KCH - 1) / tct::KCH;
  t->nt = (k + tct::BN - 1) / tct::BN;
  auto fail = [&](int rc) { tct_free(t); return rc; };
  cudaDeviceGetAttribute(&t->sms, cudaDevAttrMultiProcessorCount, device);
  if (cudaMalloc(&t->img, (size_t)m * t->nt * tct::tile_bytes(t->kc)) != cudaSuccess ||
      cudaMalloc(&t->mu, (size_t)m * dsub * 4) != cudaSuccess || cudaMalloc(&t->rmax, (size_t)m * 8) != cudaSuccess ||
      cudaMalloc(&t->cnorm, (size_t)m * k * 4) != cudaSuccess) {
    cudaGetLastError();
    set_error("tensor-core tables: operand allocation failed");
    return fail(DPQ_ERR_NOMEM);
  }
  if (cudaMemsetAsync(t->rmax, 0, (size_t)m * 8, stream) != cudaSuccess) return fail(DPQ_ERR_CUDA);
  tct::k_tct_mean<<<dim3(m, dsub), 256, 0, stream>>>(cb, k, dsub, t->mu);
  const int64_t tot = (int64_t)m * t->nt * tct::BN;
  tct::k_tct_prep<<<(unsigned)((tot + 255) / 256), 256, 0, stream>>>(
      cb, t->mu, m, k, kbar, dsub, t->kc, t->nt, t->img, reinterpret_cast<unsigned long long*>(t->rmax), t->cnorm);
  if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(stream) != cudaSuccess) {
    set_error("tensor-core tables: operand preparation failed");
    return fail(DPQ_ERR_CUDA);
  }
  if (cudaFuncSetAttribute(tct::k_tct_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, tct::SMEM_BYTES) !=
      cudaSuccess) {
    cudaGetLastError();
    set_error("tensor-core tables: shared memory attribute");
    return fail(DPQ_ERR_CUDA);
  }
  *out = t;
  return DPQ_OK;
}

// Approximate full tables of nq queries y (device, row stride ystride
// floats) into tables (nq, m, k) group-major, and per (query, subspace) the
// entry error bound eps (nq, m):  |T~ - T_numpy| <= eps.
//
// Bound (f64), per entry: |T~ - T| <= gamma * (||y'|| + ||c'||)^2 (the
// refine uses this with the stored ||y'|| (ny) and ||c'|| (tct_cnorm));
// eps = gamma * (||y'|| + max_c ||c'||)^2 bounds a whole (query, subspace); with
//   gamma = (4 * Kp + 64) * 2^-23,  Kp = 16 * ceil(dsub / 16):
// the 3xTF32 GEMM accumulates 3 Kp + 3 products in f32 (each add <= 2^-23
// relative to the running magnitude <= (||y'|| + ||c'||)^2, allowing
// truncation), the dropped lo.lo term is <= 2^-22 |y'||c'|, ||y'||^2 adds Kp
// roundings, the centring y - mu, c - mu one rounding per component, and
// numpy's own pairwise sum <= (Kp / 8 + 8) 2^-24 of the same magnitude.
double tct_gamma(void* p, double eps_scale) {
  const TcTables* t = reinterpret_cast<const TcTables*>(p);
  return eps_scale * (4.0 * t->kc * tct::KCH + 64.0) * std::ldexp(1.0, -23);
}
const float* tct_cnorm(void* p) { return reinterpret_cast<const TcTables*>(p)->cnorm; }

int tct_build(void* p, const float* y, int64_t ystride, int nq, float* tables, double* eps, double* ny,
              double eps_scale, cudaStream_t stream) {
  TcTables* t = reinterpret_cast<TcTables*>(p);
  if (!t) { set_error("tensor-core tables not prepared"); return DPQ_ERR_STATE; }
  if (nq <= 0) return DPQ_OK;
  tct::Args a;
  a.y = y; a.ystride = ystride; a.nq = nq; a.m = t->m; a.k = t->k; a.dsub = t->dsub; a.kc = t->kc; a.nt = t->nt;
  a.img = t->img; a.mu = t->mu; a.rmax = t->rmax; a.tables = tables; a.eps = eps; a.ny = ny;
  a.gamma = tct_gamma(p, eps_scale);
  a.nqb = (nq + tct::BM - 1) / tct::BM;
  const int64_t base = (int64_t)t->m * a.nqb;
  a.ntr = (int)std::max<int64_t>(1, std::min<int64_t>(t->nt, (4LL * t->sms + base - 1) / base));
  a.tpr = (t->nt + a.ntr - 1) / a.ntr;
  a.ntr = (t->nt + a.tpr - 1) / a.tpr;
  a.units = base * a.ntr;
  const int grid = (int)std::min<int64_t>(a.units, t->sms);
  tct::k_tct_gemm<<<grid, tct::kThreads, tct::SMEM_BYTES, stream>>>(a);
  TCT_CUDA(cudaGetLastError());
  return DPQ_OK;
}

__global__ void k_tct_codes(const unsigned long long* __restrict__ packed, int64_t n, int32_t* __restrict__ codes) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) codes[i] = (int32_t)(packed[i] & 0xFFFFFFFFull);
}

// Nearest centroid per (row, subspace) of x (n rows, row stride ldx floats):
// the tensor-core GEMM in encoder mode (operand prepared with kbar = 1, so
// entry = centroid index), argmin with ties to the lowest index
// (clustering.py:53-77).  scratch: n * m u64.
int tct_argmin(void* p, const float* x, int64_t ldx, int64_t n, int32_t* codes, unsigned long long* scratch,
               cudaStream_t stream) {
  TcTables* t = reinterpret_cast<TcTables*>(p);
  if (!t || t->kbar != 1) { set_error("tensor-core encoder operand not prepared"); return DPQ_ERR_STATE; }
  if (n <= 0) return DPQ_OK;
  TCT_CUDA(cudaMemsetAsync(scratch, 0xFF, (size_t)n * t->m * 8, stream));
  for (int64_t s0 = 0; s0 < n; s0 += (int64_t)1 << 30) {  // (nq is an int)
    const int nq = (int)std::min<int64_t>(n - s0, (int64_t)1 << 30);
    tct::Args a;
    a.y = x + s0 * ldx; a.ystride = ldx; a.nq = nq; a.m = t->m; a.k = t->k; a.dsub = t->dsub; a.kc = t->kc;
    a.nt = t->nt; a.img = t->img; a.mu = t->mu; a.rmax = t->rmax; a.tables = nullptr; a.eps = nullptr;
    a.ny = nullptr; a.argmin = scratch + s0 * t->m; a.gamma = 0.0;
    a.nqb = (nq + tct::BM - 1) / tct::BM;
    const int64_t base = (int64_t)t->m * a.nqb;
    a.ntr = (int)std::max<int64_t>(1, std::min<int64_t>(t->nt, (4LL * t->sms + base - 1) / base));
    a.tpr = (t->nt + a.ntr - 1) / a.ntr;
    a.ntr = (t->nt + a.tpr - 1) / a.tpr;
    a.units = base * a.ntr;
    const int grid = (int)std::min<int64_t>(a.units, t->sms);
    tct::k_tct_gemm<<<grid, tct::kThreads, tct::SMEM_BYTES, stream>>>(a);
    TCT_CUDA(cudaGetLastError());
  }
  const int64_t tot = n * t->m;
  k_tct_codes<<<(unsigned)((tot + 255) / 256), 256, 0, stream>>>(scratch, tot, codes);
  TCT_CUDA(cudaGetLastError());
  return DPQ_OK;
}

}  // namespace dpq
