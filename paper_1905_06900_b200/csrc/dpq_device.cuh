// dpq_device.cuh — device helpers shared by the libdpq kernels (sm_100a).
//
// Exactness contract: every float operation that feeds a
// table entry, a quantized table or a refine distance uses an explicit
// round-to-nearest intrinsic (__fsub_rn/__fmul_rn/__fadd_rn, __dadd_rn, ...)
// so that no FMA contraction can change a bit; the library is additionally
// compiled with -fmad=false.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace dpq {

constexpr int kSaturated = 255;  // twopass.py:184 _SATURATED

// ---------------------------------------------------------------------------
// numpy float32 pairwise summation of squared differences.
//
// search.py:24-25 computes `diff = rows - v; (diff * diff).sum(axis=1)`.
// numpy reduces each contiguous float32 row with pairwise_sum (8 running
// accumulators, blocks of <=128, recursive halving above that); the model
// below was checked bit-for-bit against numpy 2.3.5 for every length 1..960
// (SURVEY Appendix A rule 1, re-verified by tests/test_oracle_numpy_model.py).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float sqdiff(float c, float y) {
  float d = __fsub_rn(c, y);
  return __fmul_rn(d, d);
}

// ---- paired FP32 (sm_100 FADD2 / FFMA2): two lanes of sqdiff / add per
// instruction, each lane rounded exactly like the scalar __fsub_rn /
// __fmul_rn / __fadd_rn.  The square is fma(d, d, z) with z = (-0, -0) a
// RUNTIME value (kernel argument): RN(d*d + -0) == RN(d*d) for every d, and
// since ptxas cannot prove z == -0 it cannot contract the following add into
// the square (with a literal -0 or a plain mul.rn it emits one FFMA2, which
// would change the rounding).
typedef unsigned long long f32x2_t;
constexpr unsigned long long kNegZero2 = 0x8000000080000000ull;
__device__ __forceinline__ f32x2_t pack2(float lo, float hi) {
  return (f32x2_t)__float_as_uint(lo) | ((f32x2_t)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ float lo2(f32x2_t v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float hi2(f32x2_t v) { return __uint_as_float((uint32_t)(v >> 32)); }
__device__ __forceinline__ f32x2_t sqdiff2(f32x2_t c, f32x2_t y, f32x2_t z) {
  f32x2_t d, q;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(c), "l"(y));
  asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(q) : "l"(d), "l"(z));
  return q;
}
__device__ __forceinline__ f32x2_t add2(f32x2_t a, f32x2_t b) {
  f32x2_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// pw_block / pw_sqdist_v8 association for 8 | n <= 128 with the 8 running
// sums held as 4 pairs (r0,r1) (r2,r3) (r4,r5) (r6,r7); c and y as pairs.
__device__ __forceinline__ float pw_combine2(const f32x2_t r[4]) {
  return __fadd_rn(__fadd_rn(__fadd_rn(lo2(r[0]), hi2(r[0])), __fadd_rn(lo2(r[1]), hi2(r[1]))),
                   __fadd_rn(__fadd_rn(lo2(r[2]), hi2(r[2])), __fadd_rn(lo2(r[3]), hi2(r[3]))));
}
// pw_sqdist_v8 (8 | n <= 128, 16-B aligned rows) on lane pairs
__device__ __forceinline__ float pw_sqdist_v8_x2(const float* __restrict__ c, const float* __restrict__ y, int n,
                                                 f32x2_t z2) {
  const ulonglong2* c2 = reinterpret_cast<const ulonglong2*>(c);
  const ulonglong2* y2 = reinterpret_cast<const ulonglong2*>(y);
  f32x2_t r[4];
  for (int i = 0; i < n / 8; ++i) {
    const ulonglong2 a = c2[2 * i], b = c2[2 * i + 1], p = y2[2 * i], q = y2[2 * i + 1];
    const f32x2_t v[4] = {sqdiff2(a.x, p.x, z2), sqdiff2(a.y, p.y, z2), sqdiff2(b.x, q.x, z2),
                          sqdiff2(b.y, q.y, z2)};
#pragma unroll
    for (int l = 0; l < 4; ++l) r[l] = (i == 0) ? v[l] : add2(r[l], v[l]);
  }
  return pw_combine2(r);
}

// n <= 128 block of the pairwise sum, c/y may be any address space.
__device__ __forceinline__ float pw_block(const float* __restrict__ c,
                                          const float* __restrict__ y, int n) {
  if (n < 8) {
    float res = -0.0f;
    for (int i = 0; i < n; ++i) res = __fadd_rn(res, sqdiff(c[i], y[i]));
    return res;
  }
  float r0 = sqdiff(c[0], y[0]), r1 = sqdiff(c[1], y[1]);
  float r2 = sqdiff(c[2], y[2]), r3 = sqdiff(c[3], y[3]);
  float r4 = sqdiff(c[4], y[4]), r5 = sqdiff(c[5], y[5]);
  float r6 = sqdiff(c[6], y[6]), r7 = sqdiff(c[7], y[7]);
  const int lim = n - (n & 7);
  for (int i = 8; i < lim; i += 8) {
    r0 = __fadd_rn(r0, sqdiff(c[i + 0], y[i + 0]));
    r1 = __fadd_rn(r1, sqdiff(c[i + 1], y[i + 1]));
    r2 = __fadd_rn(r2, sqdiff(c[i + 2], y[i + 2]));
    r3 = __fadd_rn(r3, sqdiff(c[i + 3], y[i + 3]));
    r4 = __fadd_rn(r4, sqdiff(c[i + 4], y[i + 4]));
    r5 = __fadd_rn(r5, sqdiff(c[i + 5], y[i + 5]));
    r6 = __fadd_rn(r6, sqdiff(c[i + 6], y[i + 6]));
    r7 = __fadd_rn(r7, sqdiff(c[i + 7], y[i + 7]));
  }
  float res = __fadd_rn(__fadd_rn(__fadd_rn(r0, r1), __fadd_rn(r2, r3)),
                        __fadd_rn(__fadd_rn(r4, r5), __fadd_rn(r6, r7)));
  for (int i = lim; i < n; ++i) res = __fadd_rn(res, sqdiff(c[i], y[i]));
  return res;
}

// Full model including the recursive split for n > 128 (iterative, explicit
// stack: at most log2(n/128) levels; 960-d / m=1 needs 3).
__device__ __noinline__ float pw_sqdist_long(const float* __restrict__ c,
                                             const float* __restrict__ y,
                                             int n) {
  // Recursion pw(a,n) = pw(a,n2) + pw(a+n2,n-n2), evaluated depth-first with
  // results combined in the same association order.
  struct Frame { int off, n, state; float left; };
  Frame st[24];
  int sp = 0;
  st[0] = {0, n, 0, 0.f};
  float ret = 0.f;
  while (sp >= 0) {
    Frame& f = st[sp];
    if (f.n <= 128) {
      ret = pw_block(c + f.off, y + f.off, f.n);
      --sp;
      continue;
    }
    int n2 = f.n / 2;
    n2 -= n2 % 8;
    if (f.state == 0) {
      f.state = 1;
      st[sp + 1] = {f.off, n2, 0, 0.f};
      ++sp;
    } else if (f.state == 1) {
      f.left = ret;
      f.state = 2;
      st[sp + 1] = {f.off + n2, f.n - n2, 0, 0.f};
      ++sp;
    } else {
      ret = __fadd_rn(f.left, ret);
      --sp;
    }
  }
  return ret;
}

__device__ __forceinline__ float pw_sqdist(const float* __restrict__ c,
                                           const float* __restrict__ y,
                                           int n) {
  return n <= 128 ? pw_block(c, y, n) : pw_sqdist_long(c, y, n);
}

// Runtime n with 8 | n <= 128 and 16-B aligned rows: same association
// order as pw_block, 128-bit loads for both operands.
__device__ __forceinline__ float pw_sqdist_v8(const float* __restrict__ c, const float* __restrict__ y, int n) {
  const float4* c4 = reinterpret_cast<const float4*>(c);
  const float4* y4 = reinterpret_cast<const float4*>(y);
  float r[8];
  for (int i = 0; i < n / 8; ++i) {
    const float4 a = c4[2 * i], b = c4[2 * i + 1];
    const float4 p = y4[2 * i], q = y4[2 * i + 1];
    const float v[8] = {sqdiff(a.x, p.x), sqdiff(a.y, p.y), sqdiff(a.z, p.z), sqdiff(a.w, p.w),
                        sqdiff(b.x, q.x), sqdiff(b.y, q.y), sqdiff(b.z, q.z), sqdiff(b.w, q.w)};
#pragma unroll
    for (int l = 0; l < 8; ++l) r[l] = (i == 0) ? v[l] : __fadd_rn(r[l], v[l]);
  }
  return __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                   __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
}

// Compile-time dsub specialisation (dsub % 4 == 0, <= 128): codebook row
// fetched with 128-bit loads, same association order as pw_block.
template <int DSUB>
__device__ __forceinline__ float pw_sqdist_fixed(const float* __restrict__ c,
                                                 const float* __restrict__ y) {
  static_assert(DSUB % 8 == 0 && DSUB <= 128, "fixed path needs 8 | dsub <= 128");
  float r[8];
  const float4* c4 = reinterpret_cast<const float4*>(c);
#pragma unroll
  for (int i = 0; i < DSUB / 8; ++i) {
    float4 a = __ldg(c4 + 2 * i);
    float4 b = __ldg(c4 + 2 * i + 1);
    float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int l = 0; l < 8; ++l) {
      float s = sqdiff(v[l], y[8 * i + l]);
      r[l] = (i == 0) ? s : __fadd_rn(r[l], s);
    }
  }
  return __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                   __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
}

// ---------------------------------------------------------------------------
// 8-bit quantization, twopass.py:50-60 (quantize_with_bounds):
//   q = clip(floor((D - qmin) * (255 / (qmax - qmin))), 0, 254)  in f64
//   q = 255 where D > qmax, compared in float32 (NEP 50 weak scalar).
// scale is 255.0/(qmax-qmin) computed once in f64 by the caller.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint8_t quantize_entry(float d, double qmin,
                                                  double scale, float qmaxf) {
  double v = floor(__dmul_rn(__dsub_rn((double)d, qmin), scale));
  v = v < 0.0 ? 0.0 : (v > 254.0 ? 254.0 : v);
  uint8_t q = (uint8_t)v;
  if (d > qmaxf) q = (uint8_t)kSaturated;
  return q;
}

__device__ __forceinline__ uint32_t code_at(const void* codes, int code_bytes,
                                            int64_t idx) {
  return code_bytes == 2 ? (uint32_t)((const uint16_t*)codes)[idx]
                         : (uint32_t)((const uint8_t*)codes)[idx];
}

// Warp/block reductions ------------------------------------------------------
__device__ __forceinline__ float warp_min_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// (dist, id) ordering of search.py:73-88: ascending distance, ties to the
// lower id.  Distances are non-negative doubles, so their bit patterns order
// like unsigned integers.
__device__ __forceinline__ bool pair_less(uint64_t ka, int64_t ia, uint64_t kb,
                                          int64_t ib) {
  return ka < kb || (ka == kb && ia < ib);
}

}  // namespace dpq
