// dpq_encode.cu — nearest-centroid encoding on the 5th-generation tensor
// cores (tcgen05 + TMEM), sm_100a.
//
// Replaces ProductQuantizer._encode_with (quantizer.py:75-83) ->
// nearest_centroids (clustering.py:53-77): for every row i and subspace j,
//   code[i, j] = argmin_c ||x_ij - C_j[c]||^2, ties to the lowest index.
// The reference computes d2 = ||c||^2 (f64) - 2 * (x . c) with an f32 BLAS
// GEMM for the cross term; here the same quantity (minus the row constant
// ||x||^2, which does not move the argmin) is one fused GEMM + row-argmin:
//
//   D[i, c] = x_hi . (-2c)_hi + x_hi . (-2c)_lo + x_lo . (-2c)_hi
//             + 1 . n1 + 1 . n2 + 1 . n3          (kind::tf32, f32 in TMEM)
//
// "3xTF32": x = x_hi + x_lo and -2c = hi + lo split at tf32 precision
// (cvt.rna.tf32), ||c||^2 (computed in f64) split into three tf32 pieces, so
// D carries ~fp32 accuracy like the reference's sgemm.  When every x of a
// row block is tf32-exact (e.g. SIFT's integer components) the x_lo MMAs are
// skipped; they would add exact zeros.  Near-ties (|D - D_best| at the f32
// rounding level) may resolve differently from the reference's BLAS, which
// is itself BLAS-build dependent.
//
// Kernel structure (persistent, one CTA per SM, 10 warps):
//   warp 0     TMA producer: cp.async.bulk of pre-swizzled centroid tiles
//              (256 centroids x [hi 128 B | lo 128 B | norm 32 B] = 72 KB)
//              into a 2-stage smem ring (full/empty mbarriers)
//   warp 1     TMEM allocator + MMA issuer (one elected thread): per tile,
//              9 or 13 tcgen05.mma (M=128, N=256, K=8) into a double-buffered
//              TMEM accumulator (2 x 256 columns)
//   warps 2-9  epilogue: 4 lane quarters x 2 column halves; tcgen05.ld 32
//              columns at a time, running (min, first index) per row, the two
//              halves merged per unit; they also stage the next unit's 128
//              query rows (x_hi/x_lo, SWIZZLE_128B) in smem.
// A unit is (subspace j, 128 consecutive rows); CTAs sweep units so that the
// CTAs running at any moment share one subspace's 18 MB centroid operand in
// L2.  (N = 128 tiles with 2 row blocks measured 1.23x slower: the single
// issuing thread pays ~100-200 cycles per MMA, so fewer, wider MMAs win.)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>

#include "../../include/dpq.h"
#include "dpq_impl.h"

namespace dpq {
namespace enc {

constexpr int BN = 256;                    // centroids per tile (MMA N)
constexpr int BM = 128;                    // rows per row block (MMA M)
constexpr int RB = 1;                      // row blocks per unit
constexpr int STAGES = 2;
constexpr int ATOM = BN * 128;             // 32 KB: 256 centroid rows x 32 f32, SWIZZLE_128B K-major
constexpr int ATOM_A = BM * 128;           // 16 KB: 128 query rows
constexpr int NORMB = BN * 32;             // 8 KB: 256 rows x 8 f32, no swizzle (core matrices)
constexpr int NORMB_A = BM * 32;           // 4 KB: the constant "ones" A block
constexpr int TILE_B = 2 * ATOM + NORMB;   // 72 KB per centroid tile
constexpr int A_RB = 2 * ATOM_A;           // x_hi, x_lo of one row block
constexpr int kThreads = 320;
constexpr int kEpiWarps = 8;
// smem carve-up (offsets from a 1024-B aligned base)
constexpr int OFF_B = 0;
constexpr int OFF_A = OFF_B + STAGES * TILE_B;  // 147456
constexpr int OFF_ONES = OFF_A + RB * A_RB;     // +65536
constexpr int OFF_BAR = OFF_ONES + NORMB_A;     // +4096
constexpr int SMEM_BYTES = OFF_BAR + 256 + 1024;  // barriers + alignment slack
constexpr uint32_t kTmemCols = 512;
constexpr float kPadNorm = 1.2676506e30f;  // 2^100: padded centroids never win

// Byte offset of (row r, 16-B chunk ch) inside a SWIZZLE_128B K-major atom
// stack: 8-row groups of 1024 B, chunk index XOR (row mod 8).
__host__ __device__ constexpr int sw128(int r, int ch) {
  return (r >> 3) * 1024 + (r & 7) * 128 + ((ch ^ (r & 7)) << 4);
}
// Byte offset of (row r, element e < 8) in the un-swizzled K-major norm
// block: core matrices of 8 rows x 16 B; K halves 128 B apart (LBO), 8-row
// groups 256 B apart (SBO).
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

// UMMA shared-memory descriptors (sm_100: version bits [46,48) = 1).
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;            // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;  // SBO: 8-row groups 1024 B apart
  d |= (uint64_t)1 << 46;            // descriptor version (Blackwell)
  d |= (uint64_t)2 << 61;            // SWIZZLE_128B
  return d;
}
__device__ __forceinline__ uint64_t desc_plain(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(128 >> 4) << 16;  // LBO: K halves 128 B apart
  d |= (uint64_t)(256 >> 4) << 32;  // SBO: 8-row groups 256 B apart
  d |= (uint64_t)1 << 46;
  return d;                          // SWIZZLE_NONE
}
// Instruction descriptor: kind::tf32, D f32, A/B tf32 K-major, M=128, N=128.
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

// Centroid operand in its smem image, one 36-KB block per (subspace, tile):
// [(-2c)_hi  SWIZZLE_128B][(-2c)_lo SWIZZLE_128B][n1 n2 n3 0 0 0 0 0 plain].
// One thread per (subspace, padded centroid).
__global__ void k_enc_prep(const float* __restrict__ cb, int m, int k, int dsub, int nt, uint8_t* __restrict__ gB) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t kp = (int64_t)nt * BN;
  if (gid >= (int64_t)m * kp) return;
  const int j = (int)(gid / kp), c = (int)(gid % kp), t = c / BN, r = c % BN;
  uint8_t* blk = gB + ((int64_t)j * nt + t) * TILE_B;
  double n2 = 0.0;
  for (int ch = 0; ch < 8; ++ch) {
    float hi[4], lo[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int dd = ch * 4 + e;
      const float v = (c < k && dd < dsub) ? cb[((int64_t)j * k + c) * dsub + dd] : 0.f;
      n2 += (double)v * (double)v;
      const float w = -2.f * v;  // exact
      hi[e] = tf32_rna(w);
      lo[e] = w - hi[e];         // exact in f32
    }
    *reinterpret_cast<float4*>(blk + sw128(r, ch)) = make_float4(hi[0], hi[1], hi[2], hi[3]);
    *reinterpret_cast<float4*>(blk + ATOM + sw128(r, ch)) = make_float4(lo[0], lo[1], lo[2], lo[3]);
  }
  float p[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (c < k) {
    const float a = tf32_rna((float)n2);
    const double r1 = n2 - (double)a;
    const float b = tf32_rna((float)r1);
    const float cc = tf32_rna((float)(r1 - (double)b));
    p[0] = a; p[1] = b; p[2] = cc;
  } else {
    p[0] = kPadNorm;
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) *reinterpret_cast<float*>(blk + 2 * ATOM + nrm(r, e)) = p[e];
}

struct EncArgs {
  const float* x;      // (n, ldx) f32, subspace j at columns [j*dsub, (j+1)*dsub)
  int64_t ldx;
  int64_t n;
  int m, dsub, nt;     // nt = centroid tiles per subspace
  const uint8_t* gB;   // (m, nt, TILE_B) prepared centroid operand
  int32_t* codes;      // (n, m)
  int64_t units;       // m * ceil(n / 256)
  int64_t nblk;        // ceil(n / 256)
};

__global__ void __launch_bounds__(kThreads, 1) k_encode_tc(EncArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = sm + OFF_B;
  uint8_t* sA = sm + OFF_A;
  uint8_t* sOnes = sm + OFF_ONES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + OFF_BAR);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint64_t* afull = tempty + 2;       // [1]
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
  const int nt = a.nt;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer --
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      for (int64_t u = blockIdx.x; u < a.units; u += gridDim.x) {
        const int j = (int)(u / a.nblk);
        const uint8_t* g = a.gB + (int64_t)j * nt * TILE_B;
        for (int t = 0; t < nt; ++t) {
          bar_wait(&empty[stage], phase ^ 1);
          bar_expect_tx(&full[stage], TILE_B);
          bulk_g2s(sB + stage * TILE_B, g + (int64_t)t * TILE_B, TILE_B, &full[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
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
        bar_wait(afull, uphase);
        uphase ^= 1;
        const bool three = *aflag != 0;
        for (int t = 0; t < nt; ++t, ++acc_t) {
          const uint32_t buf = (uint32_t)(acc_t & 1), ap = (uint32_t)((acc_t >> 1) & 1);
          bar_wait(&tempty[buf], ap ^ 1);
          bar_wait(&full[stage], phase);
          tc_after_sync();
          const uint32_t bb = sB32 + stage * TILE_B;
#pragma unroll
          for (int rb = 0; rb < RB; ++rb) {
            const uint32_t d = tmem + buf * (RB * BN) + rb * BN;
            const uint32_t ab = sA32 + rb * A_RB;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)  // x_hi . (-2c)_hi
              mma_tf32(d, desc_sw128(ab + kk * 32), desc_sw128(bb + kk * 32), kk > 0);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)  // x_hi . (-2c)_lo
              mma_tf32(d, desc_sw128(ab + kk * 32), desc_sw128(bb + ATOM + kk * 32), 1);
            if (three) {
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)  // x_lo . (-2c)_hi
                mma_tf32(d, desc_sw128(ab + ATOM_A + kk * 32), desc_sw128(bb + kk * 32), 1);
            }
            mma_tf32(d, desc_plain(sOnes32), desc_plain(bb + 2 * ATOM), 1);  // + ||c||^2
          }
          mma_commit(&empty[stage]);
          mma_commit(&tfull[buf]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else {
    // ---------------------------------------------------------- epilogue --
    const int et = threadIdx.x - 64;        // 0..255
    const int q = warp & 3;                 // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;       // column half of each tile it scans
    const int rb = 0;
    const int row_in_blk = q * 32 + lane;
    __shared__ float hbest[BM];
    __shared__ int hidx[BM];
    uint64_t acc_t = 0;
    for (int64_t u = blockIdx.x; u < a.units; u += gridDim.x) {
      const int j = (int)(u / a.nblk);
      const int64_t r0 = (u % a.nblk) * (RB * BM);
      {  // stage x_hi / x_lo of rows r0 .. r0+127 (all MMAs of the previous unit are complete)
        const int64_t gr = et < BM ? r0 + et : a.n;  // threads 128..255 stage nothing
        const int rba = 0, rr = et & 127;
        uint8_t* dst = sA + rba * A_RB;
        int any_lo = 0;
        const float* src = a.x + gr * a.ldx + (int64_t)j * a.dsub;
        const bool vec = (a.dsub & 3) == 0 && ((reinterpret_cast<uintptr_t>(src) & 15) == 0);
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          float v[4];
          if (gr < a.n && vec && ch * 4 < a.dsub) {
            const float4 f = *reinterpret_cast<const float4*>(src + ch * 4);
            v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) v[e] = (gr < a.n && ch * 4 + e < a.dsub) ? src[ch * 4 + e] : 0.f;
          }
          float hi[4], lo[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            hi[e] = tf32_rna(v[e]);
            lo[e] = v[e] - hi[e];
            any_lo |= lo[e] != 0.f;
          }
          if (et < BM) *reinterpret_cast<float4*>(dst + sw128(rr, ch)) = make_float4(hi[0], hi[1], hi[2], hi[3]);
          if (et < BM) *reinterpret_cast<float4*>(dst + ATOM_A + sw128(rr, ch)) = make_float4(lo[0], lo[1], lo[2], lo[3]);
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
      float best = INFINITY;
      int bidx = 0;
      for (int t = 0; t < nt; ++t, ++acc_t) {
        const uint32_t buf = (uint32_t)(acc_t & 1), ap = (uint32_t)((acc_t >> 1) & 1);
        bar_wait(&tfull[buf], ap);
        tc_after_sync();
        const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + buf * (RB * BN) + rb * BN + half * (BN / 2);
#pragma unroll 1
        for (int ch = 0; ch < BN / 64; ++ch) {
          float v[32];
          tmem_ld32(base + ch * 32, v);
          float m8[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) m8[i] = fminf(fminf(v[4 * i], v[4 * i + 1]), fminf(v[4 * i + 2], v[4 * i + 3]));
          const float mn = fminf(fminf(fminf(m8[0], m8[1]), fminf(m8[2], m8[3])),
                                 fminf(fminf(m8[4], m8[5]), fminf(m8[6], m8[7])));
          if (mn < best) {  // first column holding the chunk minimum (lowest index on ties)
            int f = 31;
#pragma unroll
            for (int i = 31; i >= 0; --i) f = v[i] == mn ? i : f;
            best = mn;
            bidx = t * BN + half * (BN / 2) + ch * 32 + f;
          }
        }
        tc_before_sync();
        __syncwarp();
        if (lane == 0) bar_arrive(&tempty[buf]);
      }
      // merge the two column halves: (min value, then lowest index)
      if (half == 1) { hbest[row_in_blk] = best; hidx[row_in_blk] = bidx; }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (half == 0) {
        const float ob = hbest[row_in_blk];
        const int oi = hidx[row_in_blk];
        if (ob < best || (ob == best && oi < bidx)) { best = ob; bidx = oi; }
        const int64_t gr = r0 + row_in_blk;
        if (gr < a.n) a.codes[gr * a.m + j] = bidx;
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
    }
  }
  tc_before_sync();
  __syncthreads();
  if (warp == 1) {
    tc_after_sync();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
  }
}

__global__ void k_codes_u16(const int32_t* __restrict__ in, uint16_t* __restrict__ out, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (uint16_t)in[i];
}

}  // namespace enc

struct Encoder {
  int device = 0;
  int m = 0, k = 0, dsub = 0, nt = 0;
  uint8_t* gB = nullptr;
  // dsub > 32: the K-chunked tensor-core GEMM of dpq_tctab.cu in encoder mode
  void* tct = nullptr;
  unsigned long long* scratch = nullptr;
  int64_t scratch_rows = 0;
  cudaStream_t stream = nullptr;
  int sms = 0;
  // host-path staging
  float* d_x = nullptr;
  int32_t* d_codes = nullptr;
  uint16_t* d_u16 = nullptr;
  int64_t cap_rows = 0;
};

}  // namespace dpq

using dpq::Encoder;

#define ENC_CUDA(call)                                                                                  \
  do {                                                                                                  \
    cudaError_t e_ = (call);                                                                            \
    if (e_ != cudaSuccess) {                                                                            \
      dpq::set_error(std::string(#call) + ": " + cudaGetErrorString(e_) + " (dpq_encode.cu:" +          \
                     std::to_string(__LINE__) + ")");                                                   \
      return DPQ_ERR_CUDA;                                                                              \
    }                                                                                                   \
  } while (0)

extern "C" {

static int encoder_init(Encoder* e, const float* codebooks) {
  const int m = e->m, k = e->k, dsub = e->dsub;
  ENC_CUDA(cudaDeviceGetAttribute(&e->sms, cudaDevAttrMultiProcessorCount, e->device));
  ENC_CUDA(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
  float* d_cb = nullptr;
  const size_t cb_bytes = (size_t)m * k * dsub * sizeof(float);
  ENC_CUDA(cudaMalloc(&d_cb, cb_bytes));
  struct FreeCb {
    float* p;
    ~FreeCb() { cudaFree(p); }
  } free_cb{d_cb};
  ENC_CUDA(cudaMemcpyAsync(d_cb, codebooks, cb_bytes, cudaMemcpyHostToDevice, e->stream));
  if (dsub > 32)  // K-chunked tensor-core GEMM (dpq_tctab.cu), natural centroid order
    return dpq::tct_prepare(e->device, d_cb, m, k, 1, dsub, e->stream, &e->tct);
  ENC_CUDA(cudaMalloc(&e->gB, (size_t)m * e->nt * dpq::enc::TILE_B));
  const int64_t total = (int64_t)m * e->nt * dpq::enc::BN;
  dpq::enc::k_enc_prep<<<(unsigned)((total + 255) / 256), 256, 0, e->stream>>>(d_cb, m, k, dsub, e->nt, e->gB);
  ENC_CUDA(cudaGetLastError());
  ENC_CUDA(cudaStreamSynchronize(e->stream));
  ENC_CUDA(cudaFuncSetAttribute(dpq::enc::k_encode_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                dpq::enc::SMEM_BYTES));
  return DPQ_OK;
}

int dpq_encoder_create(int device, int m, int k, int dsub, const float* codebooks, dpq_encoder_t** out) {
  if (!out || !codebooks || m < 1 || k < 1 || dsub < 1) {
    dpq::set_error("dpq_encoder_create: invalid arguments");
    return DPQ_ERR_ARG;
  }
  if (dsub > 128 || k % 4) {
    dpq::set_error("dpq_encoder_create: the tensor-core encoder needs dsub <= 128 and 4 | k");
    return DPQ_ERR_ARG;
  }
  *out = nullptr;
  ENC_CUDA(cudaSetDevice(device));
  Encoder* e = new Encoder();
  e->device = device;
  e->m = m; e->k = k; e->dsub = dsub;
  e->nt = (k + dpq::enc::BN - 1) / dpq::enc::BN;
  const int rc = encoder_init(e, codebooks);
  if (rc != DPQ_OK) {  // no leak on a failed creation
    dpq_encoder_destroy(reinterpret_cast<dpq_encoder_t*>(e));
    return rc;
  }
  *out = reinterpret_cast<dpq_encoder_t*>(e);
  return DPQ_OK;
}

void dpq_encoder_destroy(dpq_encoder_t* enc) {
  Encoder* e = reinterpret_cast<Encoder*>(enc);
  if (!e) return;
  cudaSetDevice(e->device);
  if (e->stream) cudaStreamSynchronize(e->stream);
  cudaFree(e->gB);
  dpq::tct_free(e->tct);
  cudaFree(e->scratch);
  cudaFree(e->d_x);
  cudaFree(e->d_codes);
  cudaFree(e->d_u16);
  if (e->stream) cudaStreamDestroy(e->stream);
  delete e;
}

int dpq_encode_dev(dpq_encoder_t* enc, const float* x, int64_t n, int64_t ldx, int32_t* codes, void* stream) {
  Encoder* e = reinterpret_cast<Encoder*>(enc);
  if (!e || (n > 0 && (!x || !codes)) || n < 0 || ldx < (int64_t)e->m * e->dsub) {
    dpq::set_error("dpq_encode_dev: invalid arguments");
    return DPQ_ERR_ARG;
  }
  if (n == 0) return DPQ_OK;
  ENC_CUDA(cudaSetDevice(e->device));
  cudaStream_t st0 = stream ? reinterpret_cast<cudaStream_t>(stream) : e->stream;
  if (e->tct) {
    if (n > e->scratch_rows) {
      ENC_CUDA(cudaStreamSynchronize(st0));
      cudaFree(e->scratch);
      e->scratch = nullptr;
      e->scratch_rows = 0;
      ENC_CUDA(cudaMalloc(&e->scratch, (size_t)n * e->m * sizeof(unsigned long long)));
      e->scratch_rows = n;
    }
    return dpq::tct_argmin(e->tct, x, ldx, n, codes, e->scratch, st0);
  }
  dpq::enc::EncArgs a;
  a.x = x; a.ldx = ldx; a.n = n; a.m = e->m; a.dsub = e->dsub; a.nt = e->nt; a.gB = e->gB; a.codes = codes;
  a.nblk = (n + dpq::enc::RB * dpq::enc::BM - 1) / (dpq::enc::RB * dpq::enc::BM);
  a.units = a.nblk * e->m;
  const int grid = (int)std::min<int64_t>(a.units, e->sms);
  cudaStream_t st = stream ? reinterpret_cast<cudaStream_t>(stream) : e->stream;
  dpq::enc::k_encode_tc<<<grid, dpq::enc::kThreads, dpq::enc::SMEM_BYTES, st>>>(a);
  ENC_CUDA(cudaGetLastError());
  return DPQ_OK;
}

int dpq_encode(dpq_encoder_t* enc, const float* x, int64_t n, uint16_t* codes) {
  Encoder* e = reinterpret_cast<Encoder*>(enc);
  if (!e || n < 0 || (n > 0 && (!x || !codes))) {
    dpq::set_error("dpq_encode: invalid arguments");
    return DPQ_ERR_ARG;
  }
  if (e->k > 65536) {
    dpq::set_error("dpq_encode: uint16 codes need k <= 65536");
    return DPQ_ERR_ARG;
  }
  ENC_CUDA(cudaSetDevice(e->device));
  const int64_t d = (int64_t)e->m * e->dsub;
  const int64_t chunk = 1 << 20;
  if (e->cap_rows < std::min<int64_t>(n, chunk)) {
    cudaFree(e->d_x); cudaFree(e->d_codes); cudaFree(e->d_u16);
    e->d_x = nullptr; e->d_codes = nullptr; e->d_u16 = nullptr;
    e->cap_rows = std::min<int64_t>(n, chunk);
    ENC_CUDA(cudaMalloc(&e->d_x, (size_t)e->cap_rows * d * sizeof(float)));
    ENC_CUDA(cudaMalloc(&e->d_codes, (size_t)e->cap_rows * e->m * sizeof(int32_t)));
    ENC_CUDA(cudaMalloc(&e->d_u16, (size_t)e->cap_rows * e->m * sizeof(uint16_t)));
  }
  for (int64_t s = 0; s < n; s += chunk) {
    const int64_t c = std::min<int64_t>(chunk, n - s);
    ENC_CUDA(cudaMemcpyAsync(e->d_x, x + s * d, (size_t)c * d * sizeof(float), cudaMemcpyHostToDevice, e->stream));
    int rc = dpq_encode_dev(enc, e->d_x, c, d, e->d_codes, nullptr);
    if (rc != DPQ_OK) return rc;
    const int64_t tot = c * e->m;
    dpq::enc::k_codes_u16<<<(unsigned)((tot + 255) / 256), 256, 0, e->stream>>>(e->d_codes, e->d_u16, tot);
    ENC_CUDA(cudaGetLastError());
    ENC_CUDA(cudaMemcpyAsync(codes + s * e->m, e->d_u16, (size_t)tot * sizeof(uint16_t), cudaMemcpyDeviceToHost,
                             e->stream));
  }
  ENC_CUDA(cudaStreamSynchronize(e->stream));
  return DPQ_OK;
}

}  // extern "C"
