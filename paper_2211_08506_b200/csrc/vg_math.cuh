// vg_math.cuh — the scalar numerics of the voxel-mass tables, shared verbatim
// between the sm_100a kernels and a host build used only for conformance
// tests (vg_exp_f32_host / vg_erf_f32_host in the C-ABI).
//
// Every operation is written as an explicitly-rounded IEEE op so that nvcc
// can never contract a multiply and an add into an FMA (and the host build is
// compiled with -ffp-contract=off). The op sequence restates, bit for bit:
//
//   * numpy's float32 SIMD exp (AVX2/AVX512 dispatch of numpy >= 1.20; the
//     reference pins numpy>=1.24, pkg/pyproject.toml:10-13; 2.3.5 measured):
//     Cody-Waite reduction x = k*ln2 + r with ln2 split hi/lo, a Remez
//     (5,2) rational approximation of exp(r), then an exact 2^k scaling.
//     Conformance: all 2^32 float32 inputs bit-identical to np.exp (float32)
//     on an AVX512_SKX host (tests/test_math_host.py, `pytest --runslow`).
//   * the Bürmann-series erf of the reference, /root/reference/pkg/src/
//     voxgrid/kernels.py:43-56 (_erf_core), in its exact fp32 op order.
//   * the fp64 edge arguments, kernels.py:131-136 / :252-254 (+ periodic
//     images :247-251), rounded once to fp32 (kernels.py:142, :257).
#pragma once

#include <stdint.h>

#if defined(__CUDACC__)
#define VG_HD __host__ __device__ __forceinline__
#else
#define VG_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define VG_FMUL(a, b) __fmul_rn((a), (b))
#define VG_FADD(a, b) __fadd_rn((a), (b))
#define VG_FSUB(a, b) __fsub_rn((a), (b))
#define VG_FDIV(a, b) __fdiv_rn((a), (b))
#define VG_FSQRT(a) __fsqrt_rn((a))
#define VG_FFMA(a, b, c) __fmaf_rn((a), (b), (c))
#define VG_FRINT(a) rintf((a))
#define VG_DMUL(a, b) __dmul_rn((a), (b))
#define VG_DADD(a, b) __dadd_rn((a), (b))
#define VG_D2F(a) __double2float_rn((a))
#define VG_LDEXP1(k) __int_as_float((int)(((k) + 127) << 23))
#else
#include <math.h>
#include <string.h>
#define VG_FMUL(a, b) ((float)(a) * (float)(b))
#define VG_FADD(a, b) ((float)(a) + (float)(b))
#define VG_FSUB(a, b) ((float)(a) - (float)(b))
#define VG_FDIV(a, b) ((float)(a) / (float)(b))
#define VG_FSQRT(a) sqrtf((a))
#define VG_FFMA(a, b, c) fmaf((a), (b), (c))
#define VG_FRINT(a) rintf((a))
#define VG_DMUL(a, b) ((double)(a) * (double)(b))
#define VG_DADD(a, b) ((double)(a) + (double)(b))
#define VG_D2F(a) ((float)(a))
static inline float vg_pow2_normal_host(int k) {
  uint32_t bits = (uint32_t)(k + 127) << 23;
  float f;
  memcpy(&f, &bits, sizeof f);
  return f;
}
#define VG_LDEXP1(k) vg_pow2_normal_host((k))
#endif

// ---- numpy float32 exp -----------------------------------------------------
// Constants of the published algorithm (Cody-Waite split of ln2, Remez
// coefficients of the (5,2) rational, overflow/underflow limits).
#define VG_EXP_XMAX 88.72283935546875f
#define VG_EXP_XMIN -103.97208404541015625f
#define VG_LOG2E 1.442695040888963407359924681001892137f
#define VG_LN2_HI -6.93145752e-1f
#define VG_LN2_LO -1.42860677e-6f
#define VG_EXP_P0 9.999999999980870924916e-01f
#define VG_EXP_P1 7.257664613233124478488e-01f
#define VG_EXP_P2 2.473615434895520810817e-01f
#define VG_EXP_P3 5.114512081637298353406e-02f
#define VG_EXP_P4 6.757896990527504603057e-03f
#define VG_EXP_P5 5.082762527590693718096e-04f
#define VG_EXP_Q0 1.0f
#define VG_EXP_Q1 -2.742335390411667452936e-01f
#define VG_EXP_Q2 2.159509375685829852307e-02f

VG_HD float vg_exp_f32(float x) {
  if (x != x) return x;                      // NaN propagates
  if (x > VG_EXP_XMAX) return __builtin_huge_valf();
  if (x < VG_EXP_XMIN) return 0.0f;
  const float kq = VG_FRINT(VG_FMUL(x, VG_LOG2E));  // round-half-even
  float r = VG_FFMA(kq, VG_LN2_HI, x);
  r = VG_FFMA(kq, VG_LN2_LO, r);
  r = VG_FFMA(kq, 0.0f, r);                  // third Cody-Waite term is 0
  float num = VG_FFMA(VG_EXP_P5, r, VG_EXP_P4);
  num = VG_FFMA(num, r, VG_EXP_P3);
  num = VG_FFMA(num, r, VG_EXP_P2);
  num = VG_FFMA(num, r, VG_EXP_P1);
  num = VG_FFMA(num, r, VG_EXP_P0);
  float den = VG_FFMA(VG_EXP_Q2, r, VG_EXP_Q1);
  den = VG_FFMA(den, r, VG_EXP_Q0);
  const float poly = VG_FDIV(num, den);
  const int k = (int)kq;
  // poly * 2^k with a single rounding (scalef semantics). 2^k is built from
  // normal powers only; the split keeps each factor representable and the
  // first product exact.
  if (k > 127) return VG_FMUL(VG_FMUL(poly, 2.0f), VG_LDEXP1(k - 1));
  if (k >= -126) return VG_FMUL(poly, VG_LDEXP1(k));
  return VG_FMUL(VG_FMUL(poly, VG_LDEXP1(-64)), VG_LDEXP1(k + 64));
}

// ---- Bürmann erf, kernels.py:49-56 -------------------------------------------
// fl32 constants: A = 2/sqrt(pi), c1 = 31/200, c2 = 341/8000 (kernels.py:43-46)
#define VG_ERF_A 0x1.20dd76p+0f   /* np.float32(2/sqrt(pi)) */
#define VG_ERF_C1 0x1.3d70a4p-3f   /* np.float32(31/200) */
#define VG_ERF_C2 0x1.5d2f1ap-5f   /* np.float32(341/8000) */

VG_HD float vg_erf_f32(float t) {
  const float u = vg_exp_f32(-VG_FMUL(t, t));
  const float w = VG_FDIV(u, VG_FADD(1.0f, VG_FSQRT(VG_FSUB(1.0f, u))));
  const float q = VG_FMUL(VG_FMUL(VG_ERF_A, u), VG_FSUB(VG_ERF_C1, VG_FMUL(VG_ERF_C2, u)));
  const float res = VG_FSUB(VG_FMUL(w, VG_FADD(1.0f, q)), q);
  const float v = VG_FSUB(1.0f, res);
  // np.sign: +1 / -1 / +0 (for +-0); sign * v with v >= 0
  return (t > 0.0f) ? v : ((t < 0.0f) ? -v : VG_FMUL(0.0f, v));
}

// Saturation: for every float32 t >= VG_TSAT, vg_erf_f32(t) == 1.0f exactly
// (and -1.0f for t <= -VG_TSAT, by odd symmetry); VG_TSAT is the successor of
// the largest t with E(t) < 1 (exhaustive scan, tests/test_native_cpu.py).
#define VG_TSAT 0x1.01a2a2p+2f

// vg_erf_f32 for |t| < VG_TSAT (or NaN): there x = -t*t lies in (-16.3, 0],
// so numpy's exp never reaches its NaN / overflow / underflow branches and
// k = rint(x*log2e) is in [-24, 0], a normal power of two: the same ops with
// the range checks dropped, hence bit-identical on that domain.
VG_HD float vg_erf_core_f32(float t) {
  const float x = -VG_FMUL(t, t);
  const float kq = VG_FRINT(VG_FMUL(x, VG_LOG2E));
  float r = VG_FFMA(kq, VG_LN2_HI, x);
  r = VG_FFMA(kq, VG_LN2_LO, r);
  r = VG_FFMA(kq, 0.0f, r);
  float num = VG_FFMA(VG_EXP_P5, r, VG_EXP_P4);
  num = VG_FFMA(num, r, VG_EXP_P3);
  num = VG_FFMA(num, r, VG_EXP_P2);
  num = VG_FFMA(num, r, VG_EXP_P1);
  num = VG_FFMA(num, r, VG_EXP_P0);
  float den = VG_FFMA(VG_EXP_Q2, r, VG_EXP_Q1);
  den = VG_FFMA(den, r, VG_EXP_Q0);
  const float u = VG_FMUL(VG_FDIV(num, den), VG_LDEXP1((int)kq));
  const float w = VG_FDIV(u, VG_FADD(1.0f, VG_FSQRT(VG_FSUB(1.0f, u))));
  const float q = VG_FMUL(VG_FMUL(VG_ERF_A, u), VG_FSUB(VG_ERF_C1, VG_FMUL(VG_ERF_C2, u)));
  const float res = VG_FSUB(VG_FMUL(w, VG_FADD(1.0f, q)), q);
  const float v = VG_FSUB(1.0f, res);
  return (t > 0.0f) ? v : ((t < 0.0f) ? -v : VG_FMUL(0.0f, v));
}

// E(t) with the saturated tails answered without evaluating the series.
VG_HD float vg_erf_sat_f32(float t) {
  if (t >= VG_TSAT) return 1.0f;
  if (t <= -VG_TSAT) return -1.0f;
  return vg_erf_core_f32(t);
}

// ---- fp64 edge argument, kernels.py:252-254 (open) / :247-251 (periodic) ----
// open axis:      t_e = fl32( ((o - mu) + delta*e) * s ),  rel = o - mu
// periodic image: t_e = fl32( (-p + delta*e) * s ),        rel = -p
// In both cases the caller passes `rel` (fp64) and the edge index e.
VG_HD float vg_edge_arg(double rel, double delta, int e, double scale) {
  return VG_D2F(VG_DMUL(VG_DADD(rel, VG_DMUL(delta, (double)e)), scale));
}
