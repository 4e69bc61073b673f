// vg_reversal.cu — sm_100a kernels for grid reversal.
//
// The reversal (reference reversal.py) descends the grid-space MSE from seed
// coordinates; every iteration regenerates candidate grids (the hot path,
// vg_generate_f32) and needs
//   * the loss  _mse (reversal.py:256-258): mean((regen - ref)^2) in fp64 —
//     vg_mse_f64 does G candidate grids at once, two-pass fixed-order
//     reduction (deterministic);
//   * the analytic gradient _gradient_from_diff (reversal.py:271-306):
//     per atom and axis, 2/N * sum over the support block of
//     (regen - ref) * f_x[i] f_y[j] f_z[k] in fp64, where the axis' factor is
//     the derivative table (axis_gradient, kernels.py:277-296, built on
//     erf_approx_derivative, kernels.py:73-98) and the other two are the value
//     tables — vg_loss_gradient_f64, one CTA per atom, tables in shared memory.
// Bits follow the reference where it matters for the path (value tables are
// the K1 numerics); the fp64 sums and float32 expm1 of the derivative are
// tolerance-level (row f2).

#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>

#include "../../include/voxgrid_b200.h"
#include "vg_device.cuh"
#include "vg_math.cuh"

#define VG_API extern "C" __attribute__((visibility("default")))

// error plumbing lives in vg_kernels.cu
extern "C" int vg_internal_set_error(int code, const char* msg);

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kMseBlocks = 296;     // partial sums per grid (2 x 148 SMs)
constexpr int kMseThreads = 256;
constexpr int kGradThreads = 512;
constexpr int kGradMaxAxis = 1024;  // per-axis table length staged in shared memory

int fail(int code, const char* what, cudaError_t e) {
  char buf[256];
  snprintf(buf, sizeof buf, "%s: %s", what, cudaGetErrorString(e));
  return vg_internal_set_error(code, buf);
}

__device__ double block_reduce_f64(double v, double* red) {
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(kFull, v, off);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < nw; ++w) t += red[w];
  return t;  // thread 0
}

// pass 1: partial[g * kMseBlocks + blk] = sum over a fixed voxel range
__global__ void __launch_bounds__(kMseThreads) vg_mse_partial_kernel(const float* __restrict__ ref,
                                                                     const float* __restrict__ grids,
                                                                     int64_t n, int per_ref,
                                                                     double* partial) {
  __shared__ double red[kMseThreads / 32];
  const int g = blockIdx.y;
  ref += (int64_t)(g / per_ref) * n;   // grids g*per_ref .. share reference g/per_ref
  const int64_t per = (n + kMseBlocks - 1) / kMseBlocks;
  const int64_t lo = (int64_t)blockIdx.x * per, hi = min(n, lo + per);
  const float* gr = grids + (int64_t)g * n;
  double acc = 0.0;
  for (int64_t v = lo + threadIdx.x; v < hi; v += blockDim.x) {
    const double d = (double)__ldg(gr + v) - (double)__ldg(ref + v);
    acc = __dadd_rn(acc, __dmul_rn(d, d));
  }
  const double t = block_reduce_f64(acc, red);
  if (threadIdx.x == 0) partial[(int64_t)g * kMseBlocks + blockIdx.x] = t;
}

// pass 2: out[g] = (sum of partials in order) / n
__global__ void vg_mse_final_kernel(const double* partial, int64_t n, double* out) {
  __shared__ double red[32];
  const int g = blockIdx.x;
  double acc = 0.0;
  for (int b = threadIdx.x; b < kMseBlocks; b += blockDim.x) acc += partial[(int64_t)g * kMseBlocks + b];
  const double t = block_reduce_f64(acc, red);
  if (threadIdx.x == 0) out[g] = t / (double)n;
}

// Exact derivative of the Bürmann erf, op order of kernels.py:84-97 (fp32).
// expm1 is CUDA's (numpy's float32 expm1 may differ by an ulp: tolerance-level).
__device__ __forceinline__ float erf_deriv_f32(float t) {
  const float one = 1.0f;
  const float t2 = __fmul_rn(t, t);
  const float u = vg_exp_f32(-t2);
  const float phi = (t2 == 0.0f) ? one : __fdiv_rn(-expm1f(-t2), t2);
  const float sp = __fsqrt_rn(phi);
  const float poly = __fadd_rn(one, __fmul_rn(__fmul_rn(VG_ERF_A, u), __fsub_rn(VG_ERF_C1, __fmul_rn(VG_ERF_C2, u))));
  const float dpoly = __fmul_rn(VG_ERF_A, __fsub_rn(VG_ERF_C1, __fmul_rn(__fmul_rn(2.0f, VG_ERF_C2), u)));
  const float inner = __fsub_rn(__fdiv_rn(poly, sp), __fmul_rn(__fmul_rn(__fmul_rn(2.0f, t2), sp), dpoly));
  return __fmul_rn(u, inner);
}

struct GradParams {
  const int64_t* offsets;   // molecule b owns atoms [offsets[b], offsets[b+1]); refs/regens per molecule
  int64_t n_mol;
  int64_t grid_stride;      // C*H*W*D floats between molecules' grids
  const double* xyz;
  const int32_t* channel;
  const float* ref;
  const float* regen;
  double* grad;
  double origin[3], delta[3];
  double scale;     // 1/(sigma*sqrt(2))
  float gscale;     // fl32(0.5/(sigma*sqrt(2)))
  double inv_n2;    // 2/N
  int n[3];         // voxels along x, y, z  (W, H, D)
  int H, W, D, C;
};

// One CTA per atom: value + derivative tables of its 3 axes in shared memory,
// then per axis the fp64 block sum over (derivative support on that axis) x
// (value supports on the other two), reversal.py:255-275.
__global__ void __launch_bounds__(kGradThreads) vg_grad_kernel(const __grid_constant__ GradParams p) {
  __shared__ float val[3][kGradMaxAxis];
  __shared__ float der[3][kGradMaxAxis];
  __shared__ float edge_e[kGradMaxAxis + 1];
  __shared__ float edge_d[kGradMaxAxis + 1];
  __shared__ int vsup[3][2], gsup[3][2];
  __shared__ double red[kGradThreads / 32];
  const int a = blockIdx.x;
  const int c = p.channel[a];
  int64_t mol = 0;   // the molecule owning atom a (largest b with offsets[b] <= a)
  if (p.n_mol > 1) {
    int64_t lo = 0, hi = p.n_mol - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (__ldg(p.offsets + mid) <= a) lo = mid; else hi = mid - 1;
    }
    mol = lo;
  }
  for (int ax = 0; ax < 3; ++ax) {
    const int n = p.n[ax];
    const double rel = __dsub_rn(p.origin[ax], p.xyz[a * 3 + ax]);
    __syncthreads();
    for (int e = threadIdx.x; e <= n; e += blockDim.x) {
      const float t = vg_edge_arg(rel, p.delta[ax], e, p.scale);
      edge_e[e] = vg_erf_f32(t);
      edge_d[e] = erf_deriv_f32(t);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
      val[ax][e] = __fmul_rn(0.5f, __fsub_rn(edge_e[e + 1], edge_e[e]));
      der[ax][e] = __fmul_rn(p.gscale, __fsub_rn(edge_d[e], edge_d[e + 1]));
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // supports: first/last nonzero, (0,0) if none
      int vlo = n, vhi = -1, glo = n, ghi = -1;
      for (int e = threadIdx.x; e < n; e += 32) {
        if (val[ax][e] != 0.0f) { vlo = min(vlo, e); vhi = max(vhi, e); }
        if (der[ax][e] != 0.0f) { glo = min(glo, e); ghi = max(ghi, e); }
      }
      for (int off = 16; off > 0; off >>= 1) {
        vlo = min(vlo, __shfl_xor_sync(kFull, vlo, off));
        vhi = max(vhi, __shfl_xor_sync(kFull, vhi, off));
        glo = min(glo, __shfl_xor_sync(kFull, glo, off));
        ghi = max(ghi, __shfl_xor_sync(kFull, ghi, off));
      }
      if (threadIdx.x == 0) {
        vsup[ax][0] = vhi < 0 ? 0 : vlo;
        vsup[ax][1] = vhi < 0 ? 0 : vhi + 1;
        gsup[ax][0] = ghi < 0 ? 0 : glo;
        gsup[ax][1] = ghi < 0 ? 0 : ghi + 1;
      }
    }
  }
  __syncthreads();
  // One pass over the union of the three axis boxes (derivative support on
  // the axis, value supports on the other two): each voxel's difference is
  // read once and feeds all three sums. Outside an axis' box one of its
  // factors is exactly +0, so the extra terms add nothing (d is finite).
  const int64_t slab = (int64_t)p.W * p.D;
  const float* ref_c = p.ref + mol * p.grid_stride + (int64_t)c * p.H * slab;
  const float* reg_c = p.regen + mol * p.grid_stride + (int64_t)c * p.H * slab;
  int lo[3], ext[3];
  bool empty = false;
  for (int q = 0; q < 3; ++q) {
    const bool v_ok = vsup[q][1] > vsup[q][0], g_ok = gsup[q][1] > gsup[q][0];
    empty = empty || !(v_ok || g_ok);
    const int l = !v_ok ? gsup[q][0] : (!g_ok ? vsup[q][0] : min(vsup[q][0], gsup[q][0]));
    const int h = !v_ok ? gsup[q][1] : (!g_ok ? vsup[q][1] : max(vsup[q][1], gsup[q][1]));
    lo[q] = l;
    ext[q] = h - l;
  }
  double acc[3] = {0.0, 0.0, 0.0};
  if (!empty) {
    const int nx = ext[0], ny = ext[1], nz = ext[2];
    const int total = nx * ny * nz;   // <= 1024^3 / 8 within one support box
    for (int v = threadIdx.x; v < total; v += blockDim.x) {
      const int r = v / nz;
      const int k = lo[2] + (v - r * nz);
      const int j = lo[1] + r / nx;
      const int i = lo[0] + (r - (r / nx) * nx);
      const int64_t off = (int64_t)j * slab + (int64_t)i * p.D + k;
      const double d = (double)reg_c[off] - (double)ref_c[off];
      const double vx = val[0][i], vy = val[1][j], vz = val[2][k];
      acc[0] += d * (double)der[0][i] * vy * vz;
      acc[1] += d * vx * (double)der[1][j] * vz;
      acc[2] += d * vx * vy * (double)der[2][k];
    }
  }
  for (int axis = 0; axis < 3; ++axis) {
    const double t = block_reduce_f64(acc[axis], red);
    if (threadIdx.x == 0) p.grad[a * 3 + axis] = p.inv_n2 * t;
  }
}

// --- device-resident descent (refine_coords, reversal.py:325-398) ----------
// One CTA per molecule k (batched reversal); molecule k's coordinates are
// [coff[k], coff[k+1]) (coff NULL: one molecule of n_coords), its G backoff
// candidates sit at cands[G*coff[k] + g*(coff[k+1]-coff[k]) + i] (the CSR
// order of the regeneration batch), its steps at steps[k*G + g].
__device__ __forceinline__ void coord_range(const int* coff, int n_coords, int k, int& lo, int& hi) {
  lo = coff != nullptr ? coff[k] : 0;
  hi = coff != nullptr ? coff[k + 1] : n_coords;
}

// The loop-top stop rules, then the backoff candidates.
__global__ void vg_descent_cand_kernel(vg_descent_state* states, const int* __restrict__ coff,
                                       int n_coords, const double* __restrict__ pos,
                                       const double* __restrict__ grad,
                                       const double* __restrict__ steps, double* __restrict__ cands,
                                       int G, long long max_iters, double tol) {
  __shared__ int any_nz;
  const int k = blockIdx.x;
  vg_descent_state* st = states + k;
  int lo, hi;
  coord_range(coff, n_coords, k, lo, hi);
  const int nc = hi - lo;
  if (threadIdx.x == 0) any_nz = 0;
  __syncthreads();
  if (st->done) return;   // uniform
  // `while iterations < max_iters`, `if current < tolerance: break`
  bool stop = st->iterations >= max_iters || st->current < tol;
  if (!stop) {
    bool nz = false;
    for (int i = threadIdx.x; i < nc; i += blockDim.x) nz = nz || grad[lo + i] != 0.0;
    if (nz) any_nz = 1;
  }
  __syncthreads();
  stop = stop || any_nz == 0;   // `if not np.any(grad): break`
  if (stop) {
    if (threadIdx.x == 0) st->done = 1;
    return;
  }
  double* out = cands + (size_t)G * lo;
  for (int i = threadIdx.x; i < G * nc; i += blockDim.x) {
    const int g = i / nc, q = i - g * nc;
    out[i] = __dsub_rn(pos[lo + q], __dmul_rn(steps[k * G + g], grad[lo + q]));  // pos - (step0*h)*grad
  }
}

// First candidate (in halving order) whose loss does not exceed the current
// one, else the smallest step; state update in the reference's order.
__global__ void vg_descent_select_kernel(vg_descent_state* states, const int* __restrict__ coff,
                                         int n_coords, const double* __restrict__ losses,
                                         const double* __restrict__ cands, int G, int patience,
                                         double* __restrict__ pos, double* __restrict__ best_pos) {
  const int k = blockIdx.x;
  vg_descent_state* st = states + k;
  int lo, hi;
  coord_range(coff, n_coords, k, lo, hi);
  const int nc = hi - lo;
  const bool done = st->done != 0;
  __syncthreads();
  if (done) {
    if (threadIdx.x == 0) st->moved = 0;
    return;
  }
  const double cur = st->current;
  const double* lk = losses + (size_t)k * G;
  int s = G - 1;
  bool ok_any = false;
  for (int g = 0; g < G; ++g) {
    if (lk[g] <= cur) {
      s = g;
      ok_any = true;
      break;
    }
  }
  const double next = lk[s];
  const bool better = next < st->best;
  const double* src = cands + (size_t)G * lo + (size_t)s * nc;
  for (int i = threadIdx.x; i < nc; i += blockDim.x) {
    const double v = src[i];
    pos[lo + i] = v;
    if (better) best_pos[lo + i] = v;
  }
  __syncthreads();   // every thread has read the state
  if (threadIdx.x == 0) {
    st->current = next;
    st->iterations += 1;
    st->forced = ok_any ? 0 : st->forced + 1;
    if (better) st->best = next;
    if (st->forced >= patience) {
      st->diverged = 1;
      st->done = 1;
    }
    st->sel = s;
    st->moved = 1;
  }
}

// regen[k] = grids[k*G + sel_k] after a step (grid-stride copy, blockIdx.y = k).
__global__ void vg_descent_regen_kernel(const vg_descent_state* states, const float* __restrict__ grids,
                                        float* __restrict__ regen, long long n, int G) {
  const int k = blockIdx.y;
  const vg_descent_state* st = states + k;
  if (!st->moved) return;
  const float* src = grids + ((long long)k * G + st->sel) * n;
  float* dst = regen + (long long)k * n;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

}  // namespace

namespace {

int descent_candidates(vg_descent_state* states, const int* coff, int n_mol, int n_coords,
                       const double* pos, const double* grad, const double* steps, double* cands,
                       int n_steps, int64_t max_iters, double tolerance, void* stream) {
  if (states == nullptr || pos == nullptr || grad == nullptr || steps == nullptr || cands == nullptr)
    return vg_internal_set_error(VG_ERR_INVALID, "vg_descent_candidates: NULL pointer");
  if (n_mol <= 0 || (coff == nullptr && n_coords <= 0) || n_steps <= 0)
    return vg_internal_set_error(VG_ERR_INVALID, "vg_descent_candidates: empty problem");
  vgdev::DeviceGuard guard(cands);
  vg_descent_cand_kernel<<<n_mol, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      states, coff, n_coords, pos, grad, steps, cands, n_steps, (long long)max_iters, tolerance);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? VG_OK : fail(VG_ERR_CUDA, "vg_descent_candidates", e);
}

int descent_select(vg_descent_state* states, const int* coff, int n_mol, int n_coords,
                   const double* losses, const double* cands, const float* grids, int n_steps,
                   int64_t n_voxels, int patience, double* pos, double* best_pos, float* regen,
                   void* stream) {
  if (states == nullptr || losses == nullptr || cands == nullptr || grids == nullptr ||
      pos == nullptr || best_pos == nullptr || regen == nullptr)
    return vg_internal_set_error(VG_ERR_INVALID, "vg_descent_select: NULL pointer");
  if (n_mol <= 0 || (coff == nullptr && n_coords <= 0) || n_steps <= 0 || n_voxels <= 0 ||
      patience < 1 || n_mol > 65535)
    return vg_internal_set_error(VG_ERR_INVALID, "vg_descent_select: bad sizes");
  vgdev::DeviceGuard guard(regen);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  vg_descent_select_kernel<<<n_mol, 128, 0, st>>>(states, coff, n_coords, losses, cands, n_steps,
                                                  patience, pos, best_pos);
  long long blocks = (n_voxels + 255) / 256;
  const long long cap = n_mol >= 64 ? 8 : 148 * 4 / n_mol + 1;
  if (blocks > cap) blocks = cap;
  vg_descent_regen_kernel<<<dim3((unsigned)blocks, (unsigned)n_mol), 256, 0, st>>>(
      states, grids, regen, (long long)n_voxels, n_steps);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? VG_OK : fail(VG_ERR_CUDA, "vg_descent_select", e);
}

}  // namespace

VG_API int vg_descent_candidates_f64(vg_descent_state* state, const double* pos, const double* grad,
                                     const double* steps, double* cands, int32_t n_coords,
                                     int32_t n_steps, int64_t max_iters, double tolerance,
                                     void* stream) {
  return descent_candidates(state, nullptr, 1, n_coords, pos, grad, steps, cands, n_steps,
                            max_iters, tolerance, stream);
}

VG_API int vg_descent_select_f64(vg_descent_state* state, const double* losses, const double* cands,
                                 const float* grids, int32_t n_coords, int32_t n_steps,
                                 int64_t n_voxels, int32_t patience, double* pos, double* best_pos,
                                 float* regen, void* stream) {
  return descent_select(state, nullptr, 1, n_coords, losses, cands, grids, n_steps, n_voxels,
                        patience, pos, best_pos, regen, stream);
}

VG_API int vg_descent_candidates_batch_f64(vg_descent_state* states, const int32_t* coord_offsets,
                                           int32_t n_molecules, const double* pos,
                                           const double* grad, const double* steps,
                                           double* cands, int32_t n_steps, int64_t max_iters,
                                           double tolerance, void* stream) {
  if (coord_offsets == nullptr)
    return vg_internal_set_error(VG_ERR_INVALID, "vg_descent_candidates_batch_f64: NULL offsets");
  return descent_candidates(states, coord_offsets, n_molecules, 0, pos, grad, steps, cands,
                            n_steps, max_iters, tolerance, stream);
}

VG_API int vg_descent_select_batch_f64(vg_descent_state* states, const int32_t* coord_offsets,
                                       int32_t n_molecules, const double* losses,
                                       const double* cands, const float* grids, int32_t n_steps,
                                       int64_t n_voxels, int32_t patience, double* pos,
                                       double* best_pos, float* regen, void* stream) {
  if (coord_offsets == nullptr)
    return vg_internal_set_error(VG_ERR_INVALID, "vg_descent_select_batch_f64: NULL offsets");
  return descent_select(states, coord_offsets, n_molecules, 0, losses, cands, grids, n_steps,
                        n_voxels, patience, pos, best_pos, regen, stream);
}

VG_API size_t vg_mse_workspace_bytes(int64_t n_voxels, int32_t n_grids) {
  (void)n_voxels;
  return (size_t)(n_grids > 0 ? n_grids : 0) * kMseBlocks * sizeof(double);
}

VG_API int vg_mse_grouped_f64(const float* refs, const float* grids, int64_t n_voxels,
                              int32_t n_grids, int32_t grids_per_ref, double* out, void* workspace,
                              size_t workspace_bytes, void* stream) {
  if (n_voxels <= 0 || n_grids < 0 || grids_per_ref < 1)
    return vg_internal_set_error(VG_ERR_INVALID,
                                 "vg_mse_f64: need n_voxels > 0, n_grids >= 0, grids_per_ref >= 1");
  if (n_grids == 0) return VG_OK;
  if (refs == nullptr || grids == nullptr || out == nullptr)
    return vg_internal_set_error(VG_ERR_INVALID, "vg_mse_f64: NULL pointer");
  if (workspace == nullptr || workspace_bytes < vg_mse_workspace_bytes(n_voxels, n_grids))
    return vg_internal_set_error(VG_ERR_WORKSPACE, "vg_mse_f64: workspace too small");
  if (n_grids > 65535) return vg_internal_set_error(VG_ERR_INVALID, "vg_mse_f64: too many grids");
  vgdev::DeviceGuard guard(out);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* partial = static_cast<double*>(workspace);
  vg_mse_partial_kernel<<<dim3(kMseBlocks, n_grids), kMseThreads, 0, st>>>(refs, grids, n_voxels,
                                                                            grids_per_ref, partial);
  vg_mse_final_kernel<<<n_grids, 256, 0, st>>>(partial, n_voxels, out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? VG_OK : fail(VG_ERR_CUDA, "vg_mse_f64", e);
}

VG_API int vg_mse_f64(const float* ref, const float* grids, int64_t n_voxels, int32_t n_grids,
                      double* out, void* workspace, size_t workspace_bytes, void* stream) {
  return vg_mse_grouped_f64(ref, grids, n_voxels, n_grids, n_grids > 0 ? n_grids : 1, out,
                            workspace, workspace_bytes, stream);
}

VG_API int vg_loss_gradient_f64(const vg_batch_desc* desc, const float* ref, const float* regen,
                                double* grad, void* stream) {
  if (desc == nullptr || ref == nullptr || regen == nullptr || grad == nullptr)
    return vg_internal_set_error(VG_ERR_INVALID, "vg_loss_gradient_f64: NULL pointer");
  const vg_batch_desc& d = *desc;
  if (d.n_atoms == 0) return VG_OK;
  if (d.periodic)
    return vg_internal_set_error(VG_ERR_INVALID,
                                 "reversal of periodic grids is not supported (open boundaries)");
  if (d.W > kGradMaxAxis || d.H > kGradMaxAxis || d.D > kGradMaxAxis)
    return vg_internal_set_error(VG_ERR_INVALID, "vg_loss_gradient_f64: axis longer than 1024");
  if (d.xyz == nullptr || d.channel == nullptr || !(d.scale > 0.0))
    return vg_internal_set_error(VG_ERR_INVALID, "vg_loss_gradient_f64: bad descriptor");
  if (d.n_molecules < 1 || (d.n_molecules > 1 && d.offsets == nullptr))
    return vg_internal_set_error(VG_ERR_INVALID, "vg_loss_gradient_f64: bad molecule count");
  vgdev::DeviceGuard guard(grad);
  GradParams p;
  memset(&p, 0, sizeof p);
  p.offsets = d.offsets;
  p.n_mol = d.n_molecules;
  p.grid_stride = (int64_t)d.C * d.H * d.W * d.D;
  p.xyz = d.xyz;
  p.channel = d.channel;
  p.ref = ref;
  p.regen = regen;
  p.grad = grad;
  for (int a = 0; a < 3; ++a) {
    p.origin[a] = d.origin[a];
    p.delta[a] = d.delta[a];
  }
  p.scale = d.scale;
  // fl32(0.5 / (sigma * sqrt(2))) = fl32(0.5 * scale) exactly (power-of-two factor)
  p.gscale = (float)(0.5 * d.scale);
  p.n[0] = d.W;
  p.n[1] = d.H;
  p.n[2] = d.D;
  p.H = d.H;
  p.W = d.W;
  p.D = d.D;
  p.C = d.C;
  p.inv_n2 = 2.0 / ((double)d.C * d.H * d.W * d.D);
  vg_grad_kernel<<<(unsigned)d.n_atoms, kGradThreads, 0, static_cast<cudaStream_t>(stream)>>>(p);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? VG_OK : fail(VG_ERR_CUDA, "vg_loss_gradient_f64", e);
}
