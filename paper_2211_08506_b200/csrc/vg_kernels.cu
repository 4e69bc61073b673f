// vg_kernels.cu — sm_100a kernels + C-ABI for batched Gaussian-density grids.
//
// Path replaced (reference /root/reference/pkg/src/voxgrid):
//   generate_batch   gridgen.py:173-221  -> vg_generate_f32
//   generate_grid    gridgen.py:130-153  -> vg_generate_f32 (B = 1)
//   splat_atom       gridgen.py:74-111   -> K3 vg_slab_kernel (per-voxel gather)
//   fused_axis_tables kernels.py:217-274 -> K1 vg_tables_kernel
//   erf_approx       kernels.py:49-70    -> vg_math.cuh / vg_erf_kernel
//
// Design:
//   K1  one warp per (atom, axis): n+1 edge erf values (shared endpoints,
//       kernels.py:256-262), masses 0.5*dE, optional threshold, exact support
//       [first nonzero, last nonzero+1) by warp ballots. Tables go to a global
//       workspace that K3 reads through L1/L2.
//   K3  one CTA per (molecule, channel, y-chunk, slot block). The CTA builds
//       the ordered list of candidate atoms of its channel whose y-support
//       meets the chunk (block-wide ordered compaction, no atomics), then for
//       every y-slab writes the (W x D) slab exactly once: each thread owns a
//       float4 of z-contiguous voxels, accumulates the candidates in input
//       order (fl32(acc + fl32(fl32(gy*gx)*gz)), gridgen.py:105-109) and
//       issues one coalesced 128-bit store. Warps whose rows miss an atom's
//       x-support skip it (a skipped term is exactly +0, so culling is exact).
//   No float atomics anywhere: output bits are independent of launch shape.

#include <cuda_runtime.h>

#include <atomic>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <unistd.h>   // environ

#include "../../include/voxgrid_b200.h"
#include "vg_device.cuh"
#include "vg_math.cuh"

#define VG_API extern "C" __attribute__((visibility("default")))

namespace {

thread_local char g_last_error[512] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof g_last_error, fmt, ap);
  va_end(ap);
  return code;
}

}  // namespace

// shared by the other translation units of the library (vg_reversal.cu)
extern "C" int vg_internal_set_error(int code, const char* msg) {
  return set_error(code, "%s", msg);
}

// K13, the one-launch path of small batches (vg_small.cu)
int vg_small_try(const vg_batch_desc* d, float* out, vg_mol_stats* stats, cudaStream_t st,
                 bool stats_zeroed, bool dry_run);

namespace {

int check_launch(const char* what) {
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return set_error(VG_ERR_CUDA, "%s: %s", what, cudaGetErrorString(err));
  return VG_OK;
}

constexpr unsigned kFull = 0xffffffffu;
constexpr int kTableThreads = 256;   // K1: 8 warps, one (atom, axis) each
#ifndef VG_LIST_CAP
#define VG_LIST_CAP 128
#endif
constexpr int kListCap = VG_LIST_CAP;  // K3: candidate segment capacity (staged candidates max)
constexpr int kFuseMeanAtoms = 64;   // K3: channel-fused CTAs up to this mean atom count
constexpr int kC0CapMax = 1536;      // K3 row kernel: level-0 candidates kept per CTA (max)
constexpr int kMaxCtaRows = 64;      // K3 row kernel: x rows per CTA (keeps staged rows short)
constexpr int kMaxThreads = 512;     // K3: threads per CTA (upper bound)
constexpr int kRowThreads = 512;     // K3 row kernel: threads per CTA (upper bound)
constexpr int kWsThreads = 256;      // K3W: consumer threads per CTA
#ifndef VG_ROW_MINB
#define VG_ROW_MINB 4   // K3 row kernel: resident 256-thread CTAs per SM the register budget
#endif                  // targets (64 registers; CTAs of up to 512 threads, 2 per SM)
#ifndef VG_ROW_MINB1
#define VG_ROW_MINB1 VG_ROW_MINB   // ... for one row step per CTA (M = 1)
#endif
#ifndef VG_WS_MINB
#define VG_WS_MINB 3    // K3W: resident persistent CTAs per SM the register budget targets
#endif
constexpr int row_minb(int m) {
  return (m == 1 ? VG_ROW_MINB1 : VG_ROW_MINB) * 256 / kRowThreads;
}
constexpr int64_t kTaskBytes = 262144;       // K3: output bytes per CTA (y-chunk sizing)
constexpr int64_t kFusedTaskBytes = 1048576; // ... per channel-fused CTA, all channels
constexpr int64_t kMinCtas = 148 * 8;         // K3: CTAs a launch should at least offer
constexpr int kMaxBins = 1024;                // K2: bins (channels x y-chunks) per molecule
constexpr int kBinWarps = 32;                 // K2: warps per molecule CTA
constexpr int kMaxAxis = 65535;      // supports are packed in 16 bits

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

__host__ __device__ inline int round_up4(int v) { return (v + 3) & ~3; }

// Tuning / test hooks (VG_* environment variables, read at every API call so
// that tests can switch code paths inside one process). One scan of environ
// per call copies the VG_* entries (a launch consults ~20 hooks; 20 getenv
// scans cost several microseconds of host time per batch).
constexpr int kEnvMax = 32, kEnvLen = 64;
struct EnvSnap {
  int n = 0;
  char kv[kEnvMax][kEnvLen];
};
thread_local EnvSnap g_env;

void refresh_env() {
  g_env.n = 0;
  for (char** e = environ; e != nullptr && *e != nullptr; ++e) {
    const char* v = *e;
    if (v[0] == 'V' && v[1] == 'G' && v[2] == '_' && g_env.n < kEnvMax) {
      strncpy(g_env.kv[g_env.n], v, kEnvLen - 1);
      g_env.kv[g_env.n][kEnvLen - 1] = '\0';
      ++g_env.n;
    }
  }
}

const char* env_get(const char* name) {
  const size_t len = strlen(name);
  for (int i = 0; i < g_env.n; ++i)
    if (strncmp(g_env.kv[i], name, len) == 0 && g_env.kv[i][len] == '=') return g_env.kv[i] + len + 1;
  return nullptr;
}

// The integer value of hook `name` if it is set, parses fully and lies in
// [lo, hi]; otherwise dflt.
int env_int(const char* name, int dflt, int lo, int hi) {
  const char* v = env_get(name);
  if (v == nullptr || *v == '\0') return dflt;
  char* end = nullptr;
  const long x = strtol(v, &end, 10);
  if (*end != '\0' || x < lo || x > hi) return dflt;
  return (int)x;
}

// ---------------------------------------------------------------------------
// K1: per-atom axis tables
// ---------------------------------------------------------------------------
struct TableParams {
  const int64_t* offsets;
  const double* xyz;
  const int32_t* channel;
  const double* mol_origin;
  const double* mol_delta;
  float* tbl[3];
  int32_t* supp;
  double origin[3];
  double delta[3];
  double scale;
  double tsat_over_s;   // t_sat / scale (window estimates)
  double inv_delta[3];  // 1 / delta (window estimates)
  int64_t n_atoms;
  int64_t n_molecules;
  int n[3];
  int row[3];
  int C;                // channels: atoms outside [0, C) are invalid
  float threshold;
  int has_threshold;
  int periodic;
};

// An atom the reference rejects with ValueError (gridgen.py:86-90, 114-119;
// core.py:190-199): channel outside [0, C) or a non-finite coordinate. K1
// gives it an empty support (so K2/K3 never touch it and it adds nothing to
// voxel_writes) and the channel marker -1, from which K3 flags its molecule
// (vg_mol_stats.voxel_writes < 0). Hosts validate first; this keeps device
// inputs memory-safe and their errors visible.
__device__ __forceinline__ bool atom_invalid(const TableParams& p, int64_t atom) {
  const int c = __ldg(p.channel + atom);
  const double x = __ldg(p.xyz + atom * 3), y = __ldg(p.xyz + atom * 3 + 1),
               z = __ldg(p.xyz + atom * 3 + 2);
  return (unsigned)c >= (unsigned)p.C || !isfinite(x) || !isfinite(y) || !isfinite(z);
}

// Python float `%` for a positive divisor (kernels.py:247): fmod is exact in
// IEEE arithmetic; the result takes the divisor's sign, +0 for exact zeros.
__device__ __forceinline__ double py_mod(double x, double y) {
  double r = fmod(x, y);
  if (r != 0.0) {
    if ((y < 0.0) != (r < 0.0)) r = __dadd_rn(r, y);
  } else {
    r = copysign(0.0, y);
  }
  return r;
}

// Largest b with offsets[b] <= atom: the molecule that owns `atom` (empty
// molecules share their offset with the next one and are skipped).
__device__ __forceinline__ int64_t owner_of(const int64_t* offsets, int64_t n_mol, int64_t atom) {
  int64_t lo = 0, hi = n_mol - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (__ldg(offsets + mid) <= atom) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// E(t_e) for one edge per lane, warp-uniform: the series runs only when some
// valid lane of the warp is unsaturated; otherwise each lane takes the exact
// saturated value vg_erf_sat_f32 would return (+-1). Invalid lanes give 0.
__device__ __forceinline__ float edge_erf_warp(bool valid, double rel, double d, int e, double s) {
  const float t = vg_edge_arg(rel, d, e, s);
  const bool live = valid && !(fabsf(t) >= VG_TSAT);
  float v = valid ? (t >= VG_TSAT ? 1.0f : -1.0f) : 0.0f;
  if (__any_sync(kFull, live) && valid) v = vg_erf_sat_f32(t);
  return v;
}

__global__ void __launch_bounds__(kTableThreads) vg_tables_kernel(TableParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * (kTableThreads / 32) + (threadIdx.x >> 5);
  if (gw >= p.n_atoms * 3) return;
  const int64_t atom = gw / 3;
  const int axis = (int)(gw - atom * 3);
  const int n = p.n[axis];

  double o = p.origin[axis];
  double d = p.delta[axis];
  if (p.mol_origin != nullptr || p.mol_delta != nullptr) {
    const int64_t b = owner_of(p.offsets, p.n_molecules, atom);
    if (p.mol_origin != nullptr) o = p.mol_origin[b * 3 + axis];
    if (p.mol_delta != nullptr) d = p.mol_delta[b * 3 + axis];
  }
  const double mu = p.xyz[atom * 3 + axis];
  const double s = p.scale;
  if (atom_invalid(p, atom)) {   // whole row +0, empty support, channel marker -1
    float* row = p.tbl[axis] + atom * p.row[axis];
    for (int e = lane; e < n; e += 32) row[e] = 0.0f;
    if (lane == 0) {
      p.supp[atom * 4 + axis] = 0;
      if (axis == 0) p.supp[atom * 4 + 3] = -1;
    }
    return;
  }

  // Edge arguments are rel + delta*e (fp64) times s. Open axis: rel = o - mu
  // (kernels.py:253). Periodic: images p in (r-L, r, r+L), rel = -p, with
  // r = (mu - o) % L and L = n*delta (kernels.py:240, 247-251).
  double rel[3];
  int images = 1;
  if (!p.periodic) {
    rel[0] = __dsub_rn(o, mu);
    rel[1] = rel[2] = 0.0;
  } else {
    const double L = __dmul_rn((double)n, d);
    const double r = py_mod(__dsub_rn(mu, o), L);
    rel[0] = -__dsub_rn(r, L);
    rel[1] = -r;
    rel[2] = -__dadd_rn(r, L);
    images = 3;
  }

  float* tbl = p.tbl[axis] + atom * p.row[axis];
  const int c_start = 0;
  float e_cur[3], e_nxt[3];
#pragma unroll
  for (int im = 0; im < 3; ++im) {
    e_cur[im] = 0.0f;
    const int e0 = c_start + lane;
    if (im < images) e_cur[im] = edge_erf_warp(e0 >= 0 && e0 <= n, rel[im], d, e0, s);
  }
  int lo = -1, hi = 0;
  for (int c0 = c_start; c0 < n; c0 += 32) {
    const int e = c0 + lane;
    // erf at the next chunk's edges (each edge evaluated exactly once)
#pragma unroll
    for (int im = 0; im < 3; ++im) {
      e_nxt[im] = 0.0f;
      if (im < images) e_nxt[im] = edge_erf_warp(e + 32 <= n, rel[im], d, e + 32, s);
    }
    float g = 0.0f;
#pragma unroll
    for (int im = 0; im < 3; ++im) {
      if (im < images) {
        float up = __shfl_down_sync(kFull, e_cur[im], 1);
        const float wrap = __shfl_sync(kFull, e_nxt[im], 0);
        if (lane == 31) up = wrap;
        // half * (E[e+1] - E[e]), kernels.py:260; images summed (g-1 + g0) + g+1, :268
        const float gi = VG_FMUL(0.5f, VG_FSUB(up, e_cur[im]));
        g = (im == 0) ? gi : VG_FADD(g, gi);
      }
    }
    if (p.has_threshold && !(g >= p.threshold)) g = 0.0f;  // kernels.py:271-272
    if (e >= 0 && e < n) tbl[e] = g;
    const unsigned nz = __ballot_sync(kFull, e >= 0 && e < n && g != 0.0f);
    if (nz != 0u) {
      if (lo < 0) lo = c0 + __ffs(nz) - 1;
      hi = c0 + 32 - __clz(nz);
    }
#pragma unroll
    for (int im = 0; im < 3; ++im) e_cur[im] = e_nxt[im];
  }
  if (lane == 0) {
    const int slo = lo < 0 ? 0 : lo;   // _support_of: (0, 0) when all zero
    const int shi = lo < 0 ? 0 : hi;
    p.supp[atom * 4 + axis] = slo | (shi << 16);
    if (axis == 0) p.supp[atom * 4 + 3] = p.channel[atom];
  }
}

// Open axes: one thread per (atom, axis) row. Only edges inside the row's
// unsaturated window need the erf series; the window [a, b] is found exactly
// (t_e is monotone in e, so a = first edge with t_e > -t_sat and b = last edge
// with t_e < t_sat, checked with the same fp32 edge arguments), every g_e
// outside [a-1, b] is 0.5*(E-E) with both E equal to -1 or +1, i.e. +0.
// Window values go through a per-warp shared buffer so each row is then
// written by the whole warp with coalesced stores; rows are grouped by axis
// (blockIdx.y) so the warp shares n and the table.
constexpr int kWin = 32;   // window edges buffered per lane per pass

__device__ __forceinline__ bool below_sat(float t) { return t <= -VG_TSAT; }
__device__ __forceinline__ bool above_sat(float t) { return t >= VG_TSAT; }

// T lanes per row (T = 1, 2, 4, 8; chosen by the launcher so that small
// batches still fill the GPU): lane `sub` of a row's group evaluates edges
// pstart + sub + T*i, and the mass g_e = 0.5*(E(e+1) - E(e)) takes E(e+1)
// from the next lane of the group (from lane 0's next edge for the last
// lane), so each edge is evaluated once per pass.
template <int T>
__global__ void __launch_bounds__(kTableThreads) vg_tables_open_kernel(TableParams p) {
  // a programmatic dependent (K3 in vg_generate_f32) may be scheduled now; it
  // still waits for this grid's completion before reading the tables
  asm volatile("griddepcontrol.launch_dependents;");
  constexpr int kRowsPerWarp = 32 / T;
  __shared__ float wbuf[kTableThreads / 32][kRowsPerWarp][kWin + 1];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int sub = lane & (T - 1);
  const int rw = lane / T;
  const int axis = blockIdx.y;
  const int n = p.n[axis];
  const int64_t atom0 = (int64_t)blockIdx.x * (kTableThreads / T) + warp * kRowsPerWarp;
  const int64_t atom = atom0 + rw;
  const bool valid = atom < p.n_atoms;
  const double s = p.scale;

  double rel = 0.0, d = 1.0;
  int glo = 0, ghi = -1;   // candidate g range (empty for invalid rows)
  const bool bad = valid && atom_invalid(p, atom);   // row of zeros, empty support
  if (valid && !bad) {
    double o = p.origin[axis];
    d = p.delta[axis];
    if (p.mol_origin != nullptr || p.mol_delta != nullptr) {
      const int64_t b = owner_of(p.offsets, p.n_molecules, atom);
      if (p.mol_origin != nullptr) o = p.mol_origin[b * 3 + axis];
      if (p.mol_delta != nullptr) d = p.mol_delta[b * 3 + axis];
    }
    rel = __dsub_rn(o, p.xyz[atom * 3 + axis]);   // kernels.py:253
    glo = 0;
    ghi = n - 1;
    if (d > 0.0 && isfinite(rel) && isfinite(d)) {
      // estimates, then exact correction against the fp32 edge arguments
      // (estimates only: multiply by a reciprocal computed once)
      const double inv_d = p.mol_delta != nullptr ? 1.0 / d : p.inv_delta[axis];
      const double ea = (-p.tsat_over_s - rel) * inv_d;
      const double eb = (p.tsat_over_s - rel) * inv_d;
      int a = ea <= 0.0 ? 0 : (ea >= (double)(n + 1) ? n + 1 : (int)ceil(ea));
      int b = eb < 0.0 ? -1 : (eb >= (double)n ? n : (int)floor(eb));
      while (a > 0 && !below_sat(vg_edge_arg(rel, d, a - 1, s))) --a;
      while (a <= n && below_sat(vg_edge_arg(rel, d, a, s))) ++a;
      while (b < n && !above_sat(vg_edge_arg(rel, d, b + 1, s))) ++b;
      while (b >= 0 && above_sat(vg_edge_arg(rel, d, b, s))) --b;
      glo = max(0, a - 1);
      ghi = min(n - 1, b);
    }
  }

  float* tbl_axis = p.tbl[axis];
  const int64_t row = p.row[axis];
  int cur = glo;                 // next window edge of this row
  int nz_lo = INT_MAX, nz_hi = 0;
  bool first = true;
  for (;;) {
    // pass: up to kWin window values of each row into the warp buffer
    const int pstart = cur;
    const int pend = min(ghi + 1, cur + kWin);
    const int my_it = pend > pstart ? (pend - pstart + T - 1) / T : 0;
    const int n_it = __reduce_max_sync(kFull, my_it);
    float e_cur = 0.0f;
    if (n_it > 0) e_cur = vg_erf_sat_f32(vg_edge_arg(rel, d, pstart + sub, s));
    for (int i = 0; i < n_it; ++i) {
      const int e = pstart + sub + T * i;
      const float e_nxt = vg_erf_sat_f32(vg_edge_arg(rel, d, e + T, s));
      float up = __shfl_down_sync(kFull, e_cur, 1, T);      // E(e+1) from lane sub+1
      const float wrap = __shfl_sync(kFull, e_nxt, 0, T);   // E(pstart + T*(i+1))
      if (sub == T - 1) up = wrap;
      if (e < pend) {
        float g = VG_FMUL(0.5f, VG_FSUB(up, e_cur));            // kernels.py:260
        if (p.has_threshold && !(g >= p.threshold)) g = 0.0f;   // kernels.py:271-272
        if (g != 0.0f) {
          nz_lo = min(nz_lo, e);
          nz_hi = max(nz_hi, e + 1);
        }
        wbuf[warp][rw][e - pstart] = g;
      }
      e_cur = e_nxt;
    }
    cur = max(pend, cur);
    __syncwarp();
    if (first && !__any_sync(kFull, cur <= ghi)) {
      // Every row's window fit this pass (the common case): whole rows,
      // zeros and window, padding included, as float4 stores; Lp lanes
      // (a power of two >= the row's float4 count, <= 32) per row.
      const int n4 = (n + 3) >> 2;
      int lp = 1;
      while (lp < n4 && lp < 32) lp <<= 1;
      const int rows_per_it = 32 / lp;
      const int sub4 = lane & (lp - 1), rsel = lane / lp;
      for (int r0 = 0; r0 < kRowsPerWarp; r0 += rows_per_it) {
        const int r = r0 + rsel;
        const int src = min(r, kRowsPerWarp - 1) * T;
        const int r_ps = __shfl_sync(kFull, pstart, src);
        const int r_pe = __shfl_sync(kFull, pend, src);
        if (r >= kRowsPerWarp || atom0 + r >= p.n_atoms) continue;
        float4* dst4 = reinterpret_cast<float4*>(tbl_axis + (atom0 + r) * row);
        for (int c4 = sub4; c4 < n4; c4 += lp) {
          const int e = 4 * c4;
          float v[4];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            v[i] = (e + i >= r_ps && e + i < r_pe) ? wbuf[warp][r][e + i - r_ps] : 0.0f;
          dst4[c4] = make_float4(v[0], v[1], v[2], v[3]);
        }
      }
      break;
    }
    // coalesced write-out, one row at a time
    for (int r = 0; r < kRowsPerWarp; ++r) {
      const int r_lo = __shfl_sync(kFull, glo, r * T);
      const int r_hi = __shfl_sync(kFull, ghi, r * T);
      const int r_ps = __shfl_sync(kFull, pstart, r * T);
      const int r_pe = __shfl_sync(kFull, pend, r * T);
      if (atom0 + r >= p.n_atoms) break;
      if (!first && r_pe <= r_ps) continue;
      float* dst = tbl_axis + (atom0 + r) * row;
      for (int c0 = 0; c0 < n; c0 += 32) {
        const int e = c0 + lane;
        if (e >= n) break;
        if (e >= r_ps && e < r_pe) dst[e] = wbuf[warp][r][e - r_ps];
        else if (first && (e < r_lo || e > r_hi)) dst[e] = 0.0f;
      }
    }
    first = false;
    if (!__any_sync(kFull, cur <= ghi)) break;
    __syncwarp();
  }
  // support of the row: first / last nonzero over the group's lanes
#pragma unroll
  for (int o = 1; o < T; o <<= 1) {
    nz_lo = min(nz_lo, __shfl_xor_sync(kFull, nz_lo, o, T));
    nz_hi = max(nz_hi, __shfl_xor_sync(kFull, nz_hi, o, T));
  }
  if (valid && sub == 0) {
    const bool any = nz_lo != INT_MAX;
    const int slo = any ? nz_lo : 0;   // _support_of: (0, 0) when all zero
    const int shi = any ? nz_hi : 0;
    p.supp[atom * 4 + axis] = slo | (shi << 16);
    if (axis == 0) p.supp[atom * 4 + 3] = bad ? -1 : p.channel[atom];
  }
}

// ---------------------------------------------------------------------------
// K3: slab gather + single coalesced store of every voxel
// ---------------------------------------------------------------------------
struct SlabParams {
  const int64_t* offsets;
  const float* tx;
  const float* ty;
  const float* tz;
  const int4* supp;
  float* out;
  vg_mol_stats* stats;
  int64_t slab_elems;   // W*D
  int rx, ry, rz;       // table row strides
  int H, W, D, C;
  int jc;               // y-slabs per task
  int n_jchunks;
  // generic kernel
  int slot_blocks;      // CTAs per slab along the slot axis
  int nslots;           // slots per slab (float4 or float)
  int m_steps;          // slot steps per thread per slab
  // both
  int slots_per_row;    // D/4 (vector) or D (scalar)
  // row-structured kernel
  int row_blocks;       // CTAs per slab along x rows
  int rows_per_step;    // R = blockDim.x / slots_per_row
  int zw;               // slots per row segment of one CTA (z window)
  int z_blocks;         // CTAs per slab along z
  unsigned long long zw_magic;   // floor(2^32 / zw) + 1
  int stage_cap;        // candidates that fit the shared-memory staging area
  int stage_stride;     // floats per staged candidate: gy[pad4(jc)] gx[pad4(W)] gz[pad4(D)]
  int stage_gx;         // offset of gx inside a staged block
  int stage_gz;         // offset of gz inside a staged block
  int stage_floats;     // floats of the staging area (sublists follow it)
  int c0_cap;           // level-0 candidate capacity (ints before the staging area)
  int fuse_channels;    // 1: one CTA serves every channel
  int cta_order;        // per-channel CTAs: 0 molecule fastest, 1 channel fastest
  int tasks;            // tiles per (molecule, channel): y-chunks x row-blocks x z-blocks
  // tapered tail (channel-fused launches): CTAs from taper_lin on serve the
  // molecules from taper_b on in y-chunks of jc2 slabs (tasks2 tiles each), so
  // the launch ends on short CTAs and its SMs finish together
  unsigned taper_lin;   // first tapered CTA (0xffffffff: none)
  int taper_b, tasks2, jc2;
  int n_molecules;
  int gx_win;           // staged gx rows per candidate (window), 0: all CTA rows
  int gx_wmax;          // rows one warp spans in a row step (window padding)
  int bulk;             // 1: stage tables with bulk copies (cp.async.bulk) where aligned
  // K2 candidate bins (NULL: scan the molecule's atoms)
  const int* bins;      // molecule b's bins start at bins + offsets[b] * n_jchunks
  const int* bin_off;   // [B][bin_nb + 1] offsets into the molecule's bins
  int bin_nb;           // C * n_jchunks
};

struct BinParams {
  const int64_t* offsets;
  const int4* supp;
  int* bins;
  int* bin_off;
  int* tile_counter;   // K3W's work counter, zeroed here (K3W follows K2)
  int nb, nch, jc, C;
};

// The candidate list {x supp, y supp, z supp, atom} (kListCap + blockDim
// entries: a compaction round may overshoot the cap by up to blockDim - 1)
// lives in dynamic shared memory (row kernel) or a static array (generic
// kernel) and is passed beside this struct.
struct SlabShared {
  alignas(16) int warp_cnt[32];
  long long red[kMaxThreads / 32];
  unsigned long long bar;   // row kernel: mbarrier of the bulk staging copies
};

__device__ __forceinline__ int lo16(int v) { return v & 0xffff; }
__device__ __forceinline__ int hi16(int v) { return (int)((unsigned)v >> 16); }

// Block-wide ordered compaction step: this thread's rank among the threads
// of the block with keep == true (in thread order) and the block total.
// Ends with the warp counts published; the caller must __syncthreads()
// before the next call (warp_cnt is reused).
__device__ __forceinline__ int block_rank(bool keep, int* warp_cnt, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned bal = __ballot_sync(kFull, keep);
  if (lane == 0) warp_cnt[warp] = __popc(bal);
  __syncthreads();
  // all warp counts with 128-bit loads, then unrolled predicated sums (short
  // latency chain: this sits between two barriers on every round)
  const int4* c4 = reinterpret_cast<const int4*>(warp_cnt);
  int before = 0;
  total = 0;
#pragma unroll
  for (int g = 0; g < kMaxThreads / 128; ++g) {
    if (g * 4 < nw) {
      const int4 v = c4[g];
      const int w0 = g * 4;
      const int a = w0 + 0 < nw ? v.x : 0, b = w0 + 1 < nw ? v.y : 0;
      const int c = w0 + 2 < nw ? v.z : 0, d = w0 + 3 < nw ? v.w : 0;
      total += a + b + c + d;
      before += (w0 + 0 < warp ? a : 0) + (w0 + 1 < warp ? b : 0) + (w0 + 2 < warp ? c : 0) +
                (w0 + 3 < warp ? d : 0);
    }
  }
  return before + __popc(bal & ((1u << lane) - 1u));
}

struct AtomFilter {
  int c, jlo, jhi, xa, xb, za, zb;
  __device__ __forceinline__ bool operator()(const int4& s) const {
    return (c < 0 || s.w == c) && lo16(s.x) < hi16(s.x) && lo16(s.z) < hi16(s.z) && lo16(s.y) < jhi &&
           hi16(s.y) > jlo && lo16(s.x) < xb && hi16(s.x) > xa && lo16(s.z) < zb &&
           hi16(s.z) > za;
  }
};

// Ordered compaction into meta: scans source positions [pos, end) in
// rounds of blockDim.x (position p is atom src[p], or atom p when src is
// NULL) and appends, in ascending atom order, every atom passing `f`. Stops
// once at least kListCap entries are held; `pos` returns the resume point.
__device__ int build_list(const int4* __restrict__ supp, SlabShared& sh, int4* meta,
                          const int* src, int64_t& pos, int64_t end, const AtomFilter& f) {
  int count = 0;
  while (pos < end && count < kListCap) {
    const int64_t p = pos + threadIdx.x;
    bool keep = false;
    int4 s = make_int4(0, 0, 0, 0);
    int64_t atom = 0;
    if (p < end) {
      atom = src != nullptr ? (int64_t)src[p] : p;
      s = __ldg(supp + atom);
      keep = f(s);
    }
    int total;
    const int rank = block_rank(keep, sh.warp_cnt, total);
    if (keep) meta[count + rank] = make_int4(s.x, s.y, s.z, (int)atom);
    count += total;
    pos += blockDim.x;
    __syncthreads();
  }
  return count;
}

__device__ int build_list(const int4* __restrict__ supp, SlabShared& sh, int4* meta, int64_t& pos,
                          int64_t a1, int c, int jlo, int jhi, int xa, int xb) {
  const AtomFilter f{c, jlo, jhi, xa, xb, 0, kMaxAxis};
  return build_list(supp, sh, meta, nullptr, pos, a1, f);
}

// Ordered compaction into c0 of the atoms listed in src[0, n) that pass f
// (a K2 bin). Returns the count, or -1 if more than cap atoms pass.
__device__ int build_index_list(const int4* __restrict__ supp, SlabShared& sh, int* c0, int cap,
                                const int* __restrict__ src, int n, const AtomFilter& f) {
  int count = 0;
  for (int pos = 0; pos < n; pos += blockDim.x) {
    const int p = pos + threadIdx.x;
    int atom = 0;
    bool keep = false;
    if (p < n) {
      atom = __ldg(src + p);
      keep = f(__ldg(supp + atom));
    }
    int total;
    const int rank = block_rank(keep, sh.warp_cnt, total);
    if (keep && count + rank < cap) c0[count + rank] = atom;
    count += total;
    __syncthreads();
  }
  return count <= cap ? count : -1;
}

// Ordered compaction of atom indices into c0 (the CTA's level-0
// candidates). Returns the count, or -1 if more than cap atoms pass.
__device__ int build_index_list(const int4* __restrict__ supp, SlabShared& sh, int* c0, int cap,
                                int64_t a0, int64_t a1, const AtomFilter& f) {
  int count = 0;
  for (int64_t pos = a0; pos < a1; pos += blockDim.x) {
    const int64_t p = pos + threadIdx.x;
    const bool keep = p < a1 && f(__ldg(supp + p));
    int total;
    const int rank = block_rank(keep, sh.warp_cnt, total);
    if (keep && count + rank < cap) c0[count + rank] = (int)p;
    count += total;
    __syncthreads();
  }
  return count <= cap ? count : -1;
}

// A thread's slot: 1, 4 or 8 z-contiguous voxels (8 = two float4).
struct Slot8 {
  float4 a, b;
};
template <int SW>
struct SlotW;
template <>
struct SlotW<1> { using T = float; };
template <>
struct SlotW<4> { using T = float4; };
template <>
struct SlotW<8> { using T = Slot8; };
template <bool VEC>
struct SlotT { using T = typename SlotW<VEC ? 4 : 1>::T; };

__device__ __forceinline__ void zero_slot(float4& a) { a = make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ void zero_slot(float& a) { a = 0.f; }
__device__ __forceinline__ void zero_slot(Slot8& a) {
  zero_slot(a.a);
  zero_slot(a.b);
}
__device__ __forceinline__ int nonzeros(const float4& a) {
  return (a.x != 0.f) + (a.y != 0.f) + (a.z != 0.f) + (a.w != 0.f);
}
__device__ __forceinline__ int nonzeros(const float& a) { return a != 0.f; }

// acc += fl32(pyx * gz) elementwise, never contracted to FMA. `gzrow` may
// point to shared or global memory (generic load).
__device__ __forceinline__ void add_terms(float4& acc, float pyx, const float* gzrow, int k) {
  const float4 gz = reinterpret_cast<const float4*>(gzrow)[k];
  acc.x = VG_FADD(acc.x, VG_FMUL(pyx, gz.x));
  acc.y = VG_FADD(acc.y, VG_FMUL(pyx, gz.y));
  acc.z = VG_FADD(acc.z, VG_FMUL(pyx, gz.z));
  acc.w = VG_FADD(acc.w, VG_FMUL(pyx, gz.w));
}
__device__ __forceinline__ void add_terms(float& acc, float pyx, const float* gzrow, int k) {
  acc = VG_FADD(acc, VG_FMUL(pyx, gzrow[k]));
}

__device__ __forceinline__ void store_slot(float* slab, int f, const float4& v) {
  __stcs(reinterpret_cast<float4*>(slab) + f, v);
}
__device__ __forceinline__ void store_slot(float* slab, int f, const float& v) { __stcs(slab + f, v); }


// Per-molecule counters: nonzero voxels of this CTA (integer atomics are
// order-independent) and, from one CTA per molecule, voxel_writes.
// Per-molecule counters, warp by warp: integer atomics are order-independent,
// so no block reduction (and no barrier) is needed at the end of a CTA.
// nonzero_voxels sums every CTA's count; voxel_writes (gridgen.py:103, the
// sum of support-box volumes) comes from one CTA per molecule. Both start
// from the zeros launch_slabs writes.
__device__ __forceinline__ long long warp_sum(long long v) {
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(kFull, v, off);
  return v;  // lane 0
}

__device__ void finish_stats(const SlabParams& p, SlabShared& sh, int64_t b, int64_t a0,
                             int64_t a1, long long nz, bool owner) {
  (void)sh;
  const bool lane0 = (threadIdx.x & 31) == 0;
  const long long tot = warp_sum(nz);
  if (lane0 && tot != 0)
    atomicAdd(reinterpret_cast<unsigned long long*>(&p.stats[b].nonzero_voxels),
              (unsigned long long)tot);
  if (owner) {
    long long w = 0;
    bool bad = false;
    for (int64_t a = a0 + threadIdx.x; a < a1; a += blockDim.x) {
      const int4 s = __ldg(p.supp + a);
      w += (long long)(hi16(s.x) - lo16(s.x)) * (hi16(s.y) - lo16(s.y)) * (hi16(s.z) - lo16(s.z));
      bad = bad || s.w < 0;   // invalid atom (K1 marker): flag the molecule
    }
    const long long wt = warp_sum(w);
    if (lane0 && wt != 0)
      atomicAdd(reinterpret_cast<unsigned long long*>(&p.stats[b].voxel_writes),
                (unsigned long long)wt);
    if (__any_sync(kFull, bad) && lane0)
      atomicOr(reinterpret_cast<unsigned long long*>(&p.stats[b].voxel_writes), 1ull << 63);
  }
}

// --- generic kernel: any slab shape, one division per slot ------------------
template <bool VEC>
__device__ __forceinline__ void gather_slot(const SlabParams& p, const int4* meta, int n, int j,
                                            bool valid, int i, int k,
                                            typename SlotT<VEC>::T& acc) {
  for (int q = 0; q < n; ++q) {
    const int4 s = meta[q];
    if (j < lo16(s.y) || j >= hi16(s.y)) continue;  // uniform: y-support
    const bool hit = valid && i >= lo16(s.x) && i < hi16(s.x);
    if (!__any_sync(kFull, hit)) continue;           // uniform: warp rows miss x-support
    if (valid) {
      const int64_t a = s.w;
      const float gy = __ldg(p.ty + a * p.ry + j);
      const float pyx = VG_FMUL(gy, __ldg(p.tx + a * p.rx + i));  // multiply.outer(ty, tx)
      add_terms(acc, pyx, p.tz + a * p.rz, k);                     // (.. ) outer tz, then +=
    }
  }
}

template <bool VEC>
__global__ void __launch_bounds__(256, 2) vg_slab_generic_kernel(const __grid_constant__ SlabParams p) {
  using Slot = typename SlotT<VEC>::T;
  __shared__ SlabShared sh;
  __shared__ int4 gmeta[kListCap + 256];   // blockDim <= 256
  const int nt = blockDim.x;

  int64_t t = blockIdx.x;
  const int sb = (int)(t % p.slot_blocks);
  t /= p.slot_blocks;
  const int chunk = (int)(t % p.n_jchunks);
  t /= p.n_jchunks;
  const int c = (int)(t % p.C);
  const int64_t b = t / p.C;

  const int64_t a0 = __ldg(p.offsets + b), a1 = __ldg(p.offsets + b + 1);
  const int j0 = chunk * p.jc;
  const int j1 = min(p.H, j0 + p.jc);
  const int slot0 = sb * nt * p.m_steps;

  int64_t pos = a0;
  const int n_list = build_list(p.supp, sh, gmeta, pos, a1, c, j0, j1, 0, kMaxAxis);
  const bool single = pos >= a1;  // every candidate of the chunk fits the list

  float* out_c = p.out + ((b * p.C + c) * (int64_t)p.H) * p.slab_elems;
  long long nz = 0;
  for (int j = j0; j < j1; ++j) {
    float* slab = out_c + (int64_t)j * p.slab_elems;
    for (int m = 0; m < p.m_steps; ++m) {
      const int f = slot0 + m * nt + (int)threadIdx.x;
      const bool valid = f < p.nslots;
      const int i = f / p.slots_per_row;
      const int k = f - i * p.slots_per_row;
      Slot acc;
      zero_slot(acc);
      if (single) {
        gather_slot<VEC>(p, gmeta, n_list, j, valid, i, k, acc);
      } else {
        // Overflow path (chunks with > kListCap candidates): rebuild the
        // slab's list segment by segment; order across segments is ascending.
        int64_t pos2 = a0;
        while (pos2 < a1) {
          __syncthreads();
          const int n2 = build_list(p.supp, sh, gmeta, pos2, a1, c, j, j + 1, 0, kMaxAxis);
          gather_slot<VEC>(p, gmeta, n2, j, valid, i, k, acc);
        }
        __syncthreads();
      }
      if (valid) {
        store_slot(slab, f, acc);
        if (p.stats != nullptr) nz += nonzeros(acc);
      }
    }
  }
  if (p.stats != nullptr) finish_stats(p, sh, b, a0, a1, nz, c == 0 && chunk == 0 && sb == 0);
}

// --- row-structured kernel ----------------------------------------------------
// A CTA owns a tile of y-slabs [j0, j1) x rows [row_base, row_end) x one z
// window of zw slots (a slot = 4 z-contiguous voxels, or 1 on the scalar
// path). Thread t owns slot k = zblk*zw + t % zw of rows r0 + m*R (m < M,
// R = blockDim/zw): no per-slot division, one accumulator live. The y-chunk
// is processed in sub-chunks halved until the candidate set fits shared
// memory; each warp walks private ordered sublists of only the candidates
// that meet its rows, so culling is exact (skipped terms are +0) and free.
// Grid = (molecule, channel, y-chunk x row-block x z-block).

__device__ __forceinline__ int div_magic(int n, unsigned long long magic) {
  return (int)(((unsigned long long)n * magic) >> 32);  // exact for n < 2^16, d < 2^16
}

__device__ __forceinline__ void add_scaled(float4& acc, float pyx, const float4& gz) {
  acc.x = VG_FADD(acc.x, VG_FMUL(pyx, gz.x));
  acc.y = VG_FADD(acc.y, VG_FMUL(pyx, gz.y));
  acc.z = VG_FADD(acc.z, VG_FMUL(pyx, gz.z));
  acc.w = VG_FADD(acc.w, VG_FMUL(pyx, gz.w));
}
__device__ __forceinline__ void add_scaled(float& acc, float pyx, const float& gz) {
  acc = VG_FADD(acc, VG_FMUL(pyx, gz));
}
__device__ __forceinline__ void add_scaled(Slot8& acc, float pyx, const Slot8& gz) {
  add_scaled(acc.a, pyx, gz.a);
  add_scaled(acc.b, pyx, gz.b);
}
// Explicit shared-space loads (32-bit addresses): keeps the hot loop free of
// generic-to-shared address arithmetic.
__device__ __forceinline__ float lds_f32(unsigned a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ int2 lds_int2(unsigned a) {
  int2 v;
  asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void lds_slot(float4& v, unsigned a) {
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
}
__device__ __forceinline__ void lds_slot(float& v, unsigned a) { v = lds_f32(a); }
__device__ __forceinline__ void lds_slot(Slot8& v, unsigned a) {
  lds_slot(v.a, a);
  lds_slot(v.b, a + 16u);
}
// Nonzero count of values known to be >= +0 (sums of products of masses):
// such a float is nonzero iff its bit pattern is.
__device__ __forceinline__ int nonzeros_pos(const float4& a) {
  return min(__float_as_int(a.x), 1) + min(__float_as_int(a.y), 1) + min(__float_as_int(a.z), 1) +
         min(__float_as_int(a.w), 1);
}
__device__ __forceinline__ int nonzeros_pos(const float& a) { return min(__float_as_int(a), 1); }
__device__ __forceinline__ int nonzeros_pos(const Slot8& a) {
  return nonzeros_pos(a.a) + nonzeros_pos(a.b);
}

// Per-CTA geometry shared by the staged and unstaged paths.
struct RowTile {
  int64_t b;
  int c;
  int64_t a0, a1;
  int row_base, row_end;  // x rows of this CTA
  int zv0, zv1;           // z voxels of this CTA's window
  int r0, k;              // this thread's first row offset and global slot
  int wr0, wr1;           // this warp's row offsets at step 0
};

// Hot loop of the row kernel for one staged segment: for each row step m
// (unrolled) and slab j of the sub-chunk, walk the warp's ordered sublist,
// accumulate fl32(acc + fl32(fl32(gy*gx)*gz)) and store the slot once.
// FIRST=false continues sums stored by an earlier segment (own stores).
// Returns the nonzero-count delta.
template <int M>
struct Counts {
  int v[M];
};

// Slot I/O. SW=8 slots are two float4 half a z-window apart ("half" floats),
// so that every 128-bit warp store still covers 512 contiguous bytes.
// Output stores are streaming (st.global.cs: evict-first in L2). The grids
// are never re-read by the kernel, and streaming them through L2 normally
// would evict the K1 tables that later CTAs stage from.
#ifndef VG_EXP_PLAINST
__device__ __forceinline__ void st_slot(float* p, const float& v, int) { __stcs(p, v); }
__device__ __forceinline__ void st_slot(float* p, const float4& v, int) {
  __stcs(reinterpret_cast<float4*>(p), v);
}
__device__ __forceinline__ void st_slot(float* p, const Slot8& v, int half) {
  __stcs(reinterpret_cast<float4*>(p), v.a);
  __stcs(reinterpret_cast<float4*>(p + half), v.b);
}
#else
__device__ __forceinline__ void st_slot(float* p, const float& v, int) { *p = v; }
__device__ __forceinline__ void st_slot(float* p, const float4& v, int) {
  *reinterpret_cast<float4*>(p) = v;
}
__device__ __forceinline__ void st_slot(float* p, const Slot8& v, int half) {
  *reinterpret_cast<float4*>(p) = v.a;
  *reinterpret_cast<float4*>(p + half) = v.b;
}
#endif
__device__ __forceinline__ void ld_slot(float& v, const float* p, int) { v = *p; }
__device__ __forceinline__ void ld_slot(float4& v, const float* p, int) {
  v = *reinterpret_cast<const float4*>(p);
}
__device__ __forceinline__ void ld_slot(Slot8& v, const float* p, int half) {
  v.a = *reinterpret_cast<const float4*>(p);
  v.b = *reinterpret_cast<const float4*>(p + half);
}
__device__ __forceinline__ void lds_slot2(float& v, unsigned a, unsigned) { v = lds_f32(a); }
__device__ __forceinline__ void lds_slot2(float4& v, unsigned a, unsigned) { lds_slot(v, a); }
__device__ __forceinline__ void lds_slot2(Slot8& v, unsigned a, unsigned halfb) {
  lds_slot(v.a, a);
  lds_slot(v.b, a + halfb);
}

// One candidate term: ((gy*gx)*gz) added to the slot (kernels' op order).
template <typename Slot>
__device__ __forceinline__ void term_of(unsigned ent, unsigned gy_off, unsigned gxm, unsigned gz_off,
                                        unsigned halfb, Slot& gz, float& pyx) {
  // entry: shared address of the block (low 24 bits) | first staged x row
  // relative to the CTA's rows (high 8 bits, windowed gx staging)
  const unsigned blk = ent & 0xFFFFFFu;
  const unsigned gxb = blk - ((ent >> 24) << 2);
  lds_slot2(gz, blk + gz_off, halfb);
  pyx = VG_FMUL(lds_f32(blk + gy_off), lds_f32(gxb + gxm));  // ty (x) tx
}

// Walk the active entries `act` (ballot over a 32-entry group, ascending =
// ascending atom order) two at a time: both entries' loads are issued before
// the first one's adds, so one shared-memory latency covers two terms. The
// adds stay in order, so the sums are unchanged.
template <typename Slot>
__device__ __forceinline__ void walk_group(unsigned act, int ent_x, unsigned gy_off, unsigned gxm,
                                           unsigned gz_off, unsigned halfb, Slot& acc) {
#ifdef VG_EXP_NOWALK
  return;   // experiment build only: measures the kernel without the hot loop
#endif
  while (act != 0u) {
    const int b0 = __ffs(act) - 1;
    act &= act - 1u;
    const bool two = act != 0u;   // warp-uniform
    const int b1 = two ? __ffs(act) - 1 : b0;
    if (two) act &= act - 1u;
    const unsigned blk0 = (unsigned)__shfl_sync(kFull, ent_x, b0);
    const unsigned blk1 = (unsigned)__shfl_sync(kFull, ent_x, b1);
    Slot gz0, gz1;
    float p0, p1;
    term_of(blk0, gy_off, gxm, gz_off, halfb, gz0, p0);
    term_of(blk1, gy_off, gxm, gz_off, halfb, gz1, p1);
    add_scaled(acc, p0, gz0);                                              // (..)(x)tz, +=
    if (two) add_scaled(acc, p1, gz1);
  }
}

template <int M, int SW, bool FIRST>
__device__ __noinline__ int accumulate_rows(float* base, int64_t slab_elems, int m_stride, int nj,
                                            int ibase, int row_end, int R, Counts<M> cnt,
                                            unsigned lists_s, int cap, unsigned gx_off,
                                            unsigned gz_off, int half, int gy_shift) {
  using Slot = typename SlotW<SW>::T;
  const unsigned halfb = 4u * (unsigned)half;
  const int lane = (int)(threadIdx.x & 31);
  // Sublists of <= 32 entries (the common case) are loaded once for all slabs.
  // (M <= 4: the preloaded entries must not push the row loop into spills)
  bool small = M <= 4;
  int2 pre[M];
#pragma unroll
  for (int m = 0; m < M; ++m) {
    small = small && cnt.v[m] <= 32;
    pre[m] = make_int2(0, 0);
    if (M <= 4 && lane < cnt.v[m]) pre[m] = lds_int2(lists_s + 8u * (unsigned)(m * cap + lane));
  }
  int nz = 0;
  float* dst_j = base;
  for (int jj = 0; jj < nj; ++jj, dst_j += slab_elems) {
    const int jbit = 1 << jj;
    const unsigned gy_off = 4u * (unsigned)(jj + gy_shift);
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const bool mine = ibase + m * R < row_end;
      float* dst = dst_j + m * m_stride;
      Slot acc;
      zero_slot(acc);
      int before = 0;
      if (!FIRST && mine) {
        ld_slot(acc, dst, half);
        before = nonzeros_pos(acc);
      }
      const unsigned gxm = gx_off + 4u * (unsigned)(m * R);
      // touched (warp-uniform): some candidate was active on this slab and
      // step; untouched slots keep their value, so their count is unchanged
      bool touched;
      if (small) {
        const unsigned act = __ballot_sync(kFull, (pre[m].y & jbit) != 0);
        touched = act != 0u;
        walk_group(act, pre[m].x, gy_off, gxm, gz_off, halfb, acc);
      } else {
        touched = false;
        // 32 entries at a time: each lane tests one entry's slab mask, the
        // ballot gives the entries active on this slab, visited in ascending
        // order (ascending atom order) with no cost for the inactive ones.
        const unsigned L = lists_s + 8u * (unsigned)(m * cap);
        for (int c0 = 0; c0 < cnt.v[m]; c0 += 32) {
          const int e = c0 + lane;
          int2 ent = make_int2(0, 0);
          if (e < cnt.v[m]) ent = lds_int2(L + 8u * (unsigned)e);
          const unsigned act = __ballot_sync(kFull, (ent.y & jbit) != 0);
          touched = touched || act != 0u;
          walk_group(act, ent.x, gy_off, gxm, gz_off, halfb, acc);
        }
      }
      if (mine) st_slot(dst, acc, half);
      if (__any_sync(kFull, touched) && mine) nz += nonzeros_pos(acc) - before;
    }
  }
  return nz;
}

// Slab pairs (YP = 2): each thread accumulates its slot on two adjacent
// y-slabs (jj, jj+1) in one walk over the candidates active on either: one gx
// and one gz load per candidate serve both slabs, gy is one 64-bit load. A
// candidate active on only one slab of the pair reads gy = +0 on the other
// (outside its y-support the table is +0), so its term there is
// fl(fl(0*gx)*gz) = +0 and acc + (+0) = acc: every voxel still receives the
// same terms in ascending atom order, bit for bit.
__device__ __forceinline__ float2 lds_f32x2(unsigned a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}

template <typename Slot>
__device__ __forceinline__ void walk_group_pair(unsigned act, int ent_x, unsigned gy_off, unsigned gxm,
                                                unsigned gz_off, unsigned halfb, Slot& acc0,
                                                Slot& acc1) {
#ifdef VG_EXP_NOWALK
  return;
#endif
  while (act != 0u) {
    const int b0 = __ffs(act) - 1;
    act &= act - 1u;
    const bool two = act != 0u;   // warp-uniform
    const int b1 = two ? __ffs(act) - 1 : b0;
    if (two) act &= act - 1u;
    const unsigned e0 = (unsigned)__shfl_sync(kFull, ent_x, b0);
    const unsigned e1 = (unsigned)__shfl_sync(kFull, ent_x, b1);
    const unsigned k0 = e0 & 0xFFFFFFu, k1 = e1 & 0xFFFFFFu;
    Slot gz0, gz1;
    lds_slot2(gz0, k0 + gz_off, halfb);
    const float2 gy0 = lds_f32x2(k0 + gy_off);
    const float gx0 = lds_f32(k0 - ((e0 >> 24) << 2) + gxm);
    lds_slot2(gz1, k1 + gz_off, halfb);
    const float2 gy1 = lds_f32x2(k1 + gy_off);
    const float gx1 = lds_f32(k1 - ((e1 >> 24) << 2) + gxm);
    add_scaled(acc0, VG_FMUL(gy0.x, gx0), gz0);   // ty (x) tx, then (x) tz, +=
    add_scaled(acc1, VG_FMUL(gy0.y, gx0), gz0);
    if (two) {
      add_scaled(acc0, VG_FMUL(gy1.x, gx1), gz1);
      add_scaled(acc1, VG_FMUL(gy1.y, gx1), gz1);
    }
  }
}

template <int M, int SW, bool FIRST>
__device__ __noinline__ int accumulate_rows_pair(float* base, int64_t slab_elems, int m_stride,
                                                 int nj, int ibase, int row_end, int R,
                                                 Counts<M> cnt, unsigned lists_s, int cap,
                                                 unsigned gx_off, unsigned gz_off, int half,
                                                 int gy_shift) {
  using Slot = typename SlotW<SW>::T;
  const unsigned halfb = 4u * (unsigned)half;
  const int lane = (int)(threadIdx.x & 31);
  bool small = M <= 2;
  int2 pre[M];
#pragma unroll
  for (int m = 0; m < M; ++m) {
    small = small && cnt.v[m] <= 32;
    pre[m] = make_int2(0, 0);
    if (M <= 2 && lane < cnt.v[m]) pre[m] = lds_int2(lists_s + 8u * (unsigned)(m * cap + lane));
  }
  int nz = 0;
  float* dst_j = base;
  for (int jj = 0; jj < nj; jj += 2, dst_j += 2 * slab_elems) {
    const bool pair = jj + 1 < nj;   // uniform; an odd tail slab runs alone
    const int jbits = (pair ? 3 : 1) << jj;
    // 8-byte aligned: jj and gy_shift even, blocks 16-byte aligned
    const unsigned gy_off = 4u * (unsigned)(jj + gy_shift);
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const bool mine = ibase + m * R < row_end;
      float* dst = dst_j + m * m_stride;
      Slot acc0, acc1;
      zero_slot(acc0);
      zero_slot(acc1);
      int before = 0;
      if (!FIRST && mine) {
        ld_slot(acc0, dst, half);
        before = nonzeros_pos(acc0);
        if (pair) {
          ld_slot(acc1, dst + slab_elems, half);
          before += nonzeros_pos(acc1);
        }
      }
      const unsigned gxm = gx_off + 4u * (unsigned)(m * R);
      bool touched;
      if (small) {
        const unsigned act = __ballot_sync(kFull, (pre[m].y & jbits) != 0);
        touched = act != 0u;
        walk_group_pair(act, pre[m].x, gy_off, gxm, gz_off, halfb, acc0, acc1);
      } else {
        touched = false;
        const unsigned L = lists_s + 8u * (unsigned)(m * cap);
        for (int c0 = 0; c0 < cnt.v[m]; c0 += 32) {
          const int e = c0 + lane;
          int2 ent = make_int2(0, 0);
          if (e < cnt.v[m]) ent = lds_int2(L + 8u * (unsigned)e);
          const unsigned act = __ballot_sync(kFull, (ent.y & jbits) != 0);
          touched = touched || act != 0u;
          walk_group_pair(act, ent.x, gy_off, gxm, gz_off, halfb, acc0, acc1);
        }
      }
      if (mine) {
        st_slot(dst, acc0, half);
        if (pair) st_slot(dst + slab_elems, acc1, half);
      }
      // counted only where some candidate was active (a vote: a real branch,
      // not a predicated count, on the many untouched pairs)
#ifndef VG_EXP_NOCOUNT
      if (__any_sync(kFull, touched) && mine)
        nz += nonzeros_pos(acc0) + (pair ? nonzeros_pos(acc1) : 0) - before;
#endif
    }
  }
  return nz;
}

// Dispatch of the hot loop: single slabs (YP = 1) or slab pairs (YP = 2).
template <int M, int SW, int YP, bool FIRST>
__device__ __forceinline__ int accumulate(float* base, int64_t slab_elems, int m_stride, int nj,
                                          int ibase, int row_end, int R, Counts<M> cnt,
                                          unsigned lists_s, int cap, unsigned gx_off,
                                          unsigned gz_off, int half, int gy_shift = 0) {
  if (YP == 2)
    return accumulate_rows_pair<M, SW, FIRST>(base, slab_elems, m_stride, nj, ibase, row_end, R,
                                              cnt, lists_s, cap, gx_off, gz_off, half, gy_shift);
  return accumulate_rows<M, SW, FIRST>(base, slab_elems, m_stride, nj, ibase, row_end, R, cnt,
                                       lists_s, cap, gx_off, gz_off, half, gy_shift);
}

// Asynchronous global -> shared copies (LDGSTS): a warp issues every copy of
// its candidates back to back instead of waiting on each load; completion is
// awaited once (cp_async_wait_all) before the barrier that publishes them.
__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// mbarrier / bulk-copy primitives (bulk staging of vg_slab_kernel, and K3W)
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned a, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned a) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned a, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(a),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned a, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "VG_WAIT_%=:\n"
      " mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra VG_WAIT_%=;\n}" ::"r"(a),
      "r"(parity)
      : "memory");
}
// 1-D bulk copy global -> shared (TMA engine), completing `bytes` of the
// transaction count of mbarrier `bar`. Addresses 16-byte aligned, bytes % 16 == 0.
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

// First staged x row of a candidate under windowed gx staging: every warp
// whose rows meet the x-support [xlo, xhi) reads rows within
// [xlo - (wmax-1), xhi + wmax - 1); the window starts there (16-byte aligned
// for cp.async when the tile's rows are), clamped to the tile.
__device__ __forceinline__ int gx_window_start(const SlabParams& p, int sx, int row_base, bool gx16) {
  if (p.gx_win <= 0) return row_base;
  int g0 = max(row_base, lo16(sx) - (p.gx_wmax - 1));
  if (gx16) g0 &= ~3;
  return g0;
}

// Stage gy (slabs js..je), gx (CTA rows) and gz (z window) of candidates
// meta[0..ns) into consecutive blocks of the staging area, one warp per block.
// The copies are asynchronous: call cp_async_wait_all() before the barrier.
template <int SW>
__device__ __forceinline__ void stage_tables(const SlabParams& p, const int4* meta, int ns,
                                             float* stage, int js, int je, int row_base, int rows,
                                             int zv0, int zv1) {
#ifdef VG_EXP_NOSTAGE
  return;   // experiment build only
#endif
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const bool gx16 = (row_base & 3) == 0;   // table rows are 16-byte aligned (pad4)
  const int rows4 = (rows + 3) >> 2;
  for (int q = warp; q < ns; q += nw) {
    const int64_t a = meta[q].w;
    float* dst = stage + q * p.stage_stride;
    for (int e = lane; e < je - js; e += 32) cp_async4(dst + e, p.ty + a * p.ry + js + e);
    if (p.gx_win > 0) {
      // window [g0, g0 + gx_win) of the table row around the x-support
      const int g0 = gx_window_start(p, meta[q].x, row_base, gx16);
      const float* gx = p.tx + a * p.rx + g0;
      const int cnt = min(p.gx_win, p.rx - g0);
      if (gx16) {
        for (int e = lane; e < (cnt >> 2); e += 32) cp_async16(dst + p.stage_gx + 4 * e, gx + 4 * e);
      } else {
        for (int e = lane; e < cnt; e += 32) cp_async4(dst + p.stage_gx + e, gx + e);
      }
    } else {
      const float* gx = p.tx + a * p.rx + row_base;
      if (gx16) {
        for (int e = lane; e < rows4; e += 32) cp_async16(dst + p.stage_gx + 4 * e, gx + 4 * e);
      } else {
        for (int e = lane; e < rows; e += 32) cp_async4(dst + p.stage_gx + e, gx + e);
      }
    }
    if (SW >= 4) {
      const float* gz = p.tz + a * p.rz + zv0;
      for (int e = lane; e < p.zw * (SW / 4); e += 32)
        cp_async16(dst + p.stage_gz + 4 * e, gz + 4 * e);
    } else {
      for (int e = lane; e < zv1 - zv0; e += 32)
        cp_async4(dst + p.stage_gz + e, p.tz + a * p.rz + zv0 + e);
    }
  }
}

// The same staged blocks by 1-D bulk copies (cp.async.bulk, the TMA unit):
// one thread per (candidate, table) pair issues one copy, so a CTA stages
// ~85 candidates in a single pass of 3 warp instructions per warp, where
// stage_tables issues three LDGSTS per candidate and warp behind the SM's
// store queue. Completion is counted on `bar` (every warp arrives once with
// its bytes as expect_tx): wait with mbar_wait(bar, parity) instead of
// cp_async_wait_all() + __syncthreads(). Needs 16-byte aligned pieces: js % 4
// == 0, row_base % 4 == 0, 4- or 8-voxel slots (the caller checks).
template <int SW>
__device__ __forceinline__ void stage_tables_bulk(const SlabParams& p, const int4* meta, int ns,
                                                  unsigned stage_s, int js, int je, int row_base,
                                                  int rows, int zv0, unsigned bar) {
  const int lane = threadIdx.x & 31;
  const unsigned gy_bytes = 4u * (unsigned)((je - js + 3) & ~3);
  const unsigned gz_bytes = 4u * (unsigned)(p.zw * SW);
  auto gx_piece = [&](const int4& m, int& g0) {   // bytes and first row of the gx piece
    if (p.gx_win > 0) {
      g0 = gx_window_start(p, m.x, row_base, true);
      return 4u * (unsigned)(min(p.gx_win, p.rx - g0) & ~3);
    }
    g0 = row_base;
    return 4u * (unsigned)((rows + 3) & ~3);
  };
  // this warp's bytes first (expect_tx precedes the copies), one arrival per warp
  unsigned bytes = 0;
  for (int e = (int)threadIdx.x; e < 3 * ns; e += (int)blockDim.x) {
    const int q = e / 3, piece = e - 3 * q;
    int g0;
    bytes += piece == 0 ? gy_bytes : (piece == 2 ? gz_bytes : gx_piece(meta[q], g0));
  }
  const unsigned warp_bytes = __reduce_add_sync(kFull, bytes);
  if (lane == 0) {
    if (warp_bytes > 0) mbar_arrive_tx(bar, warp_bytes);
    else mbar_arrive(bar);
  }
  __syncwarp();
  for (int e = (int)threadIdx.x; e < 3 * ns; e += (int)blockDim.x) {
    const int q = e / 3, piece = e - 3 * q;
    const int4 m = meta[q];
    const int64_t a = m.w;
    const unsigned dst = stage_s + 4u * (unsigned)(q * p.stage_stride);
    if (piece == 0) {
      bulk_g2s(dst, p.ty + a * p.ry + js, gy_bytes, bar);
    } else if (piece == 1) {
      int g0;
      const unsigned nb = gx_piece(m, g0);
      if (nb > 0) bulk_g2s(dst + 4u * (unsigned)p.stage_gx, p.tx + a * p.rx + g0, nb, bar);
    } else {
      bulk_g2s(dst + 4u * (unsigned)p.stage_gz, p.tz + a * p.rz + zv0, gz_bytes, bar);
    }
  }
}

// Warp-private ordered sublists: per row step m, the staged candidates (of
// channel ch, or any channel if ch < 0) whose x-support meets this warp's
// rows: {shared address of the block, slab mask}.
template <int M>
__device__ __forceinline__ void build_sublists(const SlabParams& p, const int4* meta, int ns, int ch,
                                               int2* lists, unsigned stage_s, int js, int je,
                                               int rbase, int rlo0, int rhi0, int R,
                                               Counts<M>& cnt) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int rlo = rlo0 + m * R, rhi = rhi0 + m * R;
    int filled = 0;
    for (int q0 = 0; q0 < ns; q0 += 32) {
      const int q = q0 + lane;
      bool hit = false;
      int2 ent = make_int2(0, 0);
      if (q < ns) {
        const int4 s = meta[q];
        hit = lo16(s.x) <= rhi && hi16(s.x) > rlo;
        if (ch >= 0) hit = hit && __ldg(&p.supp[s.w].w) == ch;
        const int lo = max(lo16(s.y), js) - js, hi = min(hi16(s.y), je) - js;
        const unsigned long long mask = ((1ull << hi) - 1ull) & ~((1ull << lo) - 1ull);
        const int dx = gx_window_start(p, s.x, rbase, (rbase & 3) == 0) - rbase;
        ent = make_int2((int)((stage_s + 4u * (unsigned)(q * p.stage_stride)) | ((unsigned)dx << 24)),
                        (int)(unsigned)mask);
      }
      const unsigned bal = __ballot_sync(kFull, hit);
      if (hit) lists[m * p.stage_cap + filled + __popc(bal & ((1u << lane) - 1u))] = ent;
      filled += __popc(bal);
    }
    cnt.v[m] = filled;
  }
}

#ifdef VG_EXP_TIMING
// Experiment builds only (-DVG_EXP_TIMING): per-CTA phase timestamps.
__device__ unsigned long long g_vg_ts[1 << 17][12];
__device__ unsigned long long g_vg_ts_w[1 << 17][8];   // per-warp hot-loop end
__device__ __forceinline__ unsigned long long vg_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define VG_TS(i) do { if (threadIdx.x == 0 && blockIdx.x < (1u << 17)) g_vg_ts[blockIdx.x][i] = vg_gtime(); } while (0)
#define VG_TSV(i, v) do { if (threadIdx.x == 0 && blockIdx.x < (1u << 17)) g_vg_ts[blockIdx.x][i] = (v); } while (0)
#else
#define VG_TS(i) do { } while (0)
#define VG_TSV(i, v) do { } while (0)
#endif

template <int M, int SW, int YP>
__global__ void __launch_bounds__(kRowThreads, row_minb(M)) vg_slab_kernel(const __grid_constant__ SlabParams p) {
  using Slot = typename SlotW<SW>::T;
  constexpr int kWidth = SW;
  __shared__ SlabShared sh;
  extern __shared__ float4 dyn4[];
  int4* meta_l = reinterpret_cast<int4*>(dyn4);       // candidate list [kListCap + blockDim]
  int* c0 = reinterpret_cast<int*>(meta_l + kListCap + blockDim.x);  // level-0 [c0_cap]
  float* stage = reinterpret_cast<float*>(c0) + p.c0_cap;  // staged tables, then sublists
  const int tid = threadIdx.x, warp = tid >> 5;

  const unsigned bar = smem_u32(&sh.bar);
  unsigned bar_phase = 0;
  if (p.bulk) {
    if (tid == 0) {
      mbar_init(bar, blockDim.x >> 5);   // one arrival per warp and staging round
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
  RowTile T;
  // Linear CTA index. Channel-fused CTAs: the tiles of one molecule are
  // adjacent, so the CTAs staging the same atoms' tables run close together
  // while those are in L2. Per-channel CTAs (large molecules): molecule
  // fastest, which spreads the dense central tiles of a cluster over the
  // launch (measured better for cfg3).
  int t, zblk = 0, rblk = 0, jc = p.jc;
  {
    const unsigned lin = blockIdx.x;
    if (p.fuse_channels) {
      if (lin < p.taper_lin) {
        const unsigned b = lin / (unsigned)p.tasks;
        t = (int)(lin - b * (unsigned)p.tasks);
        T.b = b;
      } else {   // the launch's tail: shorter y-chunks
        const unsigned l2 = lin - p.taper_lin;
        const unsigned b = l2 / (unsigned)p.tasks2;
        t = (int)(l2 - b * (unsigned)p.tasks2);
        T.b = (unsigned)p.taper_b + b;
        jc = p.jc2;
      }
      T.c = 0;
    } else if (p.cta_order == 0) {
      const unsigned nb = (unsigned)p.n_molecules;
      const unsigned rest = lin / nb;
      T.b = lin - rest * nb;
      const unsigned tt = rest / (unsigned)p.C;
      T.c = (int)(rest - tt * (unsigned)p.C);
      t = (int)tt;
    } else {
      const unsigned nc = (unsigned)p.C;
      const unsigned rest = lin / nc;
      T.c = (int)(lin - rest * nc);
      const unsigned nb = (unsigned)p.n_molecules;
      const unsigned tt = rest / nb;
      T.b = rest - tt * nb;
      t = (int)tt;
    }
  }
  if (p.z_blocks > 1) {
    zblk = t % p.z_blocks;
    t /= p.z_blocks;
  }
  if (p.row_blocks > 1) {
    rblk = t % p.row_blocks;
    t /= p.row_blocks;
  }
  const int chunk = t;
  T.a0 = __ldg(p.offsets + T.b);
  T.a1 = __ldg(p.offsets + T.b + 1);
  const int j0 = chunk * jc;
  const int j1 = min(p.H, j0 + jc);
  const int zw = p.zw, R = p.rows_per_step;
  T.r0 = div_magic(tid, p.zw_magic);
  T.k = zblk * zw + (tid - T.r0 * zw);
  T.wr0 = div_magic(warp * 32, p.zw_magic);
  T.wr1 = div_magic(warp * 32 + 31, p.zw_magic);
  T.row_base = rblk * M * R;
  T.row_end = min(p.W, T.row_base + M * R);
  T.zv0 = zblk * zw * kWidth;
  T.zv1 = min(p.D, T.zv0 + zw * kWidth);

  const unsigned stage_s = (unsigned)__cvta_generic_to_shared(stage);
  int2* lists = reinterpret_cast<int2*>(stage + p.stage_floats) + warp * M * p.stage_cap;
  const unsigned lists_s = (unsigned)__cvta_generic_to_shared(lists);
  const int ibase = T.row_base + T.r0;
  // this thread's first z (floats) in the row; SW=8 slots pair quads kk and kk + zw
  const int kk = T.k - zblk * zw;
  const int zf = T.zv0 + (SW == 8 ? 4 * kk : kk * kWidth);
  const int half = SW == 8 ? 4 * zw : 0;
  const unsigned gz_off = 4u * (unsigned)(p.stage_gz + (zf - T.zv0));
  const unsigned gx_off = 4u * (unsigned)(p.stage_gx + T.r0);
  const int slot0 = ibase * p.D + zf;  // float offset in the slab
  const int rows = T.row_end - T.row_base;
  // bulk staging needs 16-byte aligned pieces (x rows; y slabs checked per round)
  const bool bulk_ok = p.bulk && SW >= 4 && (T.row_base & 3) == 0;
  const int rlo0 = T.row_base + T.wr0, rhi0 = T.row_base + T.wr1;
  const int64_t chan_elems = (int64_t)p.H * p.slab_elems;

  // Launched as a programmatic dependent of K1 / K2 (vg_generate_f32,
  // vg_slabs_f32): wait until the preceding grid has completed and its supports,
  // tables and bins are visible (a no-op otherwise). Everything above reads only
  // launch parameters and the batch's offsets, so it overlaps that grid's tail.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  VG_TS(0);
  int nz = 0;
  int rounds = 0, staged = 0;
  int c_lo = T.c, c_hi = T.c + 1;
  if (p.fuse_channels) {
    // Every channel from one candidate list and one staging pass, when the
    // molecule's candidates for the whole chunk fit; otherwise the channels
    // are served one after the other by the general path below.
    c_lo = 0;
    c_hi = p.C;
    const AtomFilter fa{-1, j0, j1, T.row_base, T.row_end, T.zv0, T.zv1};
    int64_t pos = T.a0;
    const int n = build_list(p.supp, sh, meta_l, nullptr, pos, T.a1, fa);
    if (pos >= T.a1 && n <= p.stage_cap) {
      if (bulk_ok && (j0 & 3) == 0) {
        stage_tables_bulk<SW>(p, meta_l, n, stage_s, j0, j1, T.row_base, rows, T.zv0, bar);
        mbar_wait(bar, bar_phase);
        bar_phase ^= 1u;
      } else {
        stage_tables<SW>(p, meta_l, n, stage, j0, j1, T.row_base, rows, T.zv0, T.zv1);
        cp_async_wait_all();
        __syncthreads();
      }
      float* out_b = p.out + T.b * p.C * chan_elems + j0 * p.slab_elems + slot0;
      for (int c = 0; c < p.C; ++c) {
        Counts<M> cnt;
        build_sublists<M>(p, meta_l, n, c, lists, stage_s, j0, j1, T.row_base, rlo0, rhi0, R, cnt);
        __syncwarp();
        nz += accumulate<M, SW, YP, true>(out_b + c * chan_elems, p.slab_elems, R * p.D, j1 - j0,
                                           ibase, T.row_end, R, cnt, lists_s, p.stage_cap, gx_off,
                                           gz_off, half);
        __syncwarp();   // the next channel rewrites this warp's sublists
      }
      c_hi = c_lo;   // done
    }
    __syncthreads();
  }
  for (int c = c_lo; c < c_hi; ++c) {
    float* out_c = p.out + (T.b * p.C + c) * chan_elems;
    // Level 0: the CTA's candidates over its whole chunk, scanned once from the
    // molecule's atoms; sub-chunk lists below filter this short list instead.
    // (skipped for small molecules: scanning them directly is as cheap)
    const AtomFilter f0{c, j0, j1, T.row_base, T.row_end, T.zv0, T.zv1};
    const int* src;
    int64_t src_begin, src_end;
    if (p.bins != nullptr) {
      // K2 bin of (molecule, channel, y-chunk): already ordered and y-culled
      const int* bo = p.bin_off + T.b * (p.bin_nb + 1) + c * p.n_jchunks + chunk;
      const int q0 = __ldg(bo), nbk = __ldg(bo + 1) - q0;
      const int* bl = p.bins + T.a0 * p.n_jchunks + q0;
      const int n0 = nbk > 2 * (int)blockDim.x && p.c0_cap > 0
                         ? build_index_list(p.supp, sh, c0, p.c0_cap, bl, nbk, f0)
                         : -1;
      src = n0 >= 0 ? c0 : bl;
      src_begin = 0;
      src_end = n0 >= 0 ? n0 : nbk;
    } else {
      const int n0 = T.a1 - T.a0 > 2 * (int64_t)blockDim.x && p.c0_cap > 0
                         ? build_index_list(p.supp, sh, c0, p.c0_cap, T.a0, T.a1, f0)
                         : -1;
      src = n0 >= 0 ? c0 : nullptr;
      src_begin = n0 >= 0 ? 0 : T.a0;
      src_end = n0 >= 0 ? n0 : T.a1;
    }
    VG_TS(1);
    int js = j0, sc = j1 - j0;
    while (js < j1) {
      const int je = min(j1, js + sc);
      const AtomFilter f{c, js, je, T.row_base, T.row_end, T.zv0, T.zv1};
      int64_t pos = src_begin;
      int n = build_list(p.supp, sh, meta_l, src, pos, src_end, f);
      if (rounds == 0) VG_TS(8);
      if ((pos < src_end || n > p.stage_cap) && sc > 1) {  // uniform: halve the sub-chunk, rebuild
        sc = (sc + 1) >> 1;
        continue;
      }
      // Candidates are consumed in ascending segments of <= stage_cap. More than
      // one segment only happens for a single over-dense slab: later segments
      // continue the per-voxel sums from the values this thread already stored.
      bool first = true;
      for (;;) {
        // n == 0 still runs one pass: every slot is stored (as zero) exactly once
        for (int s0 = 0; s0 < max(n, 1); s0 += p.stage_cap) {
          const int ns = min(p.stage_cap, n - s0);
          const int4* meta = meta_l + s0;
          const bool bulk = bulk_ok && (js & 3) == 0;   // uniform
          if (bulk)
            stage_tables_bulk<SW>(p, meta, ns, stage_s, js, je, T.row_base, rows, T.zv0, bar);
          else
            stage_tables<SW>(p, meta, ns, stage, js, je, T.row_base, rows, T.zv0, T.zv1);
          Counts<M> cnt;
          build_sublists<M>(p, meta, ns, -1, lists, stage_s, js, je, T.row_base, rlo0, rhi0, R, cnt);
          if (rounds == 0) VG_TS(9);
          if (bulk) {
            mbar_wait(bar, bar_phase);   // every warp's copies have landed
            bar_phase ^= 1u;
          } else {
            cp_async_wait_all();
            __syncthreads();  // staged tables visible to every warp (lists are warp-private)
          }
          if (rounds == 0) VG_TS(2);
          ++rounds;
          staged += ns;

          if (first)
            nz += accumulate<M, SW, YP, true>(out_c + js * p.slab_elems + slot0, p.slab_elems,
                                                R * p.D, je - js, ibase, T.row_end, R, cnt,
                                                lists_s, p.stage_cap, gx_off, gz_off, half);
          else
            nz += accumulate<M, SW, YP, false>(out_c + js * p.slab_elems + slot0, p.slab_elems,
                                                 R * p.D, je - js, ibase, T.row_end, R, cnt,
                                                 lists_s, p.stage_cap, gx_off, gz_off, half);
          VG_TS(3);
#ifdef VG_EXP_TIMING
          // per-warp end of the hot loop (lane 0 of each warp)
          if ((tid & 31) == 0 && blockIdx.x < (1u << 17)) g_vg_ts_w[blockIdx.x][warp] = vg_gtime();
#endif
          __syncthreads();  // the next segment / sub-chunk rewrites the staging area
          first = false;
        }
        if (pos >= src_end) break;
        n = build_list(p.supp, sh, meta_l, src, pos, src_end, f);
      }
      js = je;
    }
  }
  if (p.stats != nullptr)
    finish_stats(p, sh, T.b, T.a0, T.a1, nz, T.c == 0 && chunk == 0 && rblk == 0 && zblk == 0);
#ifdef VG_EXP_TIMING
  VG_TS(4);
  unsigned smid;
  asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
  VG_TSV(5, ((unsigned long long)smid << 32) | (unsigned)T.c);
  VG_TSV(6, ((unsigned long long)rounds << 32) | (unsigned)staged);
  VG_TSV(7, ((unsigned long long)T.b << 32) | (unsigned)(chunk * 256 + rblk * 16 + zblk));
#endif
}

// ---------------------------------------------------------------------------
// K3W: persistent, warp-specialised slab kernel (binned per-channel batches)
// ---------------------------------------------------------------------------
// The same tiles, slot layout, staged blocks, warp sublists and hot loop as
// vg_slab_kernel, but without block-wide barriers. Each persistent CTA is one
// producer warp and R*zw/32 consumer warps around a ring of kWsStages staged
// "units" in shared memory:
//   producer  takes tiles from a global counter (heaviest-first order is not
//             needed: tiles are handed out dynamically), filters the tile's K2
//             bin into an ordered candidate list (warp ballots, no barrier),
//             cuts the tile's y-chunk into units whose candidates fit the
//             staging capacity (greedy over slab pairs; a pair that does not
//             fit is consumed in ascending candidate segments), and for each
//             unit waits for a free ring slot (mbarrier `empty`), writes the
//             unit's header and candidate supports, and stages every
//             candidate's gy / gx-window / gz rows with 1-D bulk copies
//             (cp.async.bulk, TMA engine) that complete on the slot's `full`
//             mbarrier (expect_tx = the unit's bytes).
//   consumers wait on `full`, build their warp-private sublists, run the hot
//             loop and store every slot of the unit's slabs exactly once (or
//             continue the sums of an earlier segment), then arrive on `empty`.
// A consumer warp never waits for another consumer warp: a warp that is done
// with a unit moves on to the next staged one, so the imbalance between the
// dense and the empty rows of a tile no longer idles the block (the
// `__syncthreads` stalls of vg_slab_kernel on cfg3). Every voxel still gets
// its candidates in ascending atom order: units of one tile are produced in
// slab order and, for the same slabs, in candidate order, and every unit is
// consumed by every consumer warp in ring order (a thread reads back only
// values it stored itself).
constexpr int kWsMaxStages = 8; // ring depth (runtime, <= this)
constexpr int kWsListCap = 512; // producer: tile candidates held per bin pass

struct WsUnit {
  int tile;    // linear tile index; -1 = no more work
  int js, je;  // slabs [js, je) of the tile
  int ns;      // staged candidates
  int first;   // 1: the first candidates of these slabs (sums start at +0)
  int gy_shift;  // js - (first staged gy slab): gy is staged from js & ~3
  int pad0, pad1;
};

// Tile geometry shared by producer and consumers: lin -> (b, c, chunk, rblk, zblk)
// in vg_slab_kernel's per-channel order (molecule fastest).
struct WsTile {
  int64_t b;
  int c, chunk, rblk, zblk;
};
__device__ __forceinline__ WsTile ws_decode(const SlabParams& p, int lin) {
  WsTile T;
  const unsigned nb = (unsigned)p.n_molecules;
  const unsigned rest = (unsigned)lin / nb;
  T.b = (unsigned)lin - rest * nb;
  const unsigned tt = rest / (unsigned)p.C;
  T.c = (int)(rest - tt * (unsigned)p.C);
  int t = (int)tt;
  T.zblk = t % p.z_blocks;
  t /= p.z_blocks;
  T.rblk = t % p.row_blocks;
  T.chunk = t / p.row_blocks;
  return T;
}

// Warp-cooperative ordered compaction: appends to dst (ascending source
// order) every element of src[i0, i1) for which keep(i) holds, at most
// `room` of them; returns how many were appended and sets `next` to the
// first source index not examined (i1 when all were).
template <typename Keep, typename Emit>
__device__ __forceinline__ int warp_compact(int i0, int i1, int room, int& next, Keep keep, Emit emit) {
  const int lane = threadIdx.x & 31;
  int count = 0;
  int i = i0;
  for (; i < i1 && count < room; i += 32) {
    const int q = i + lane;
    const bool k = q < i1 && keep(q);
    const unsigned bal = __ballot_sync(kFull, k);
    const int rank = __popc(bal & ((1u << lane) - 1u));
    const int n = __popc(bal);
    if (count + n > room) {
      // take only the first (room - count) hits; resume at the first one left
      const int take = room - count;
      if (k && rank < take) emit(count + rank, q);
      // index of the (take)-th set bit (0-based) = first hit not taken
      unsigned b = bal;
      for (int r = 0; r < take; ++r) b &= b - 1u;
      next = i + __ffs(b) - 1;
      return room;
    }
    if (k) emit(count + rank, q);
    count += n;
  }
  next = i < i1 ? i : i1;
  return count;
}

#ifdef VG_EXP_WSPROF
// Experiment builds only: cycles consumers wait for staged units / the
// producer waits for free slots, totals, units and candidates staged.
__device__ unsigned long long g_ws_prof[8];
#define WSP_T0(v) long long v = clock64()
#define WSP_ADD(i, v) atomicAdd(&g_ws_prof[i], (unsigned long long)(v))
#else
#define WSP_T0(v) do { } while (0)
#define WSP_ADD(i, v) do { } while (0)
#endif

// Producer's tile filter: ordered compaction of the K2 bin entries bl[pos,
// nbk) that pass f0 into lst (at most `room`), as {x, y, z supports, atom}.
// U groups of 32 entries per round: all their bin loads, then all their
// support loads are in flight at once (one warp; the two dependent global
// loads per entry dominate otherwise). `next` = first entry not examined.
template <int U>
__device__ __forceinline__ int ws_scan_bin(const int* __restrict__ bl, int pos, int nbk,
                                           const int4* __restrict__ supp, const AtomFilter& f0,
                                           int4* lst, int room, int& next) {
  const int lane = threadIdx.x & 31;
  int count = 0;
  int i = pos;
  while (i < nbk && count < room) {
    int at[U];
    int4 sp[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int q = i + u * 32 + lane;
      at[u] = q < nbk ? __ldg(bl + q) : -1;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) sp[u] = at[u] >= 0 ? __ldg(supp + at[u]) : make_int4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool k = at[u] >= 0 && f0(sp[u]);
      const unsigned bal = __ballot_sync(kFull, k);
      const int n = __popc(bal), rank = __popc(bal & ((1u << lane) - 1u));
      if (count + n > room) {
        const int take = room - count;
        if (k && rank < take) lst[count + rank] = make_int4(sp[u].x, sp[u].y, sp[u].z, at[u]);
        unsigned b = bal;
        for (int r = 0; r < take; ++r) b &= b - 1u;
        next = i + u * 32 + __ffs(b) - 1;
        return room;
      }
      if (k) lst[count + rank] = make_int4(sp[u].x, sp[u].y, sp[u].z, at[u]);
      count += n;
    }
    i += 32 * U;
  }
  next = i < nbk ? i : nbk;
  return count;
}

// Producer-side shared state: each of the two producer warps owns a tile
// list and its unit plan; the ring cursor and the producers' done flags are
// handed over with the turn.
struct WsProdShared {
  int ring_s;             // next ring slot
  unsigned ring_ph;       // its phase bit
  int done[2];            // producer k found no more tiles
  int stopped;            // the stop unit was emitted
  int pad[3];
};
constexpr int kWsMaxUnits = 17;   // slab pairs per tile (jc <= 32) + 1

template <int M, int NP>
__global__ void __launch_bounds__(kWsThreads + 32 * NP, VG_WS_MINB)
    vg_slab_ws_kernel(const __grid_constant__ SlabParams p, int* tile_counter, int n_tiles,
                      int kWsStages) {
  constexpr int SW = 8, YP = 2;
  extern __shared__ float4 dyn4[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ncw = (int)(blockDim.x >> 5) - NP;   // consumer warps (warps < NP produce)
  const int cap = p.stage_cap;
  // shared layout: full[S], empty[S], turn[2] mbarriers | WsProdShared | units[S] |
  // meta[S][cap] int4 | stage[S][cap*stride] floats | sublists[ncw][M*cap] int2 |
  // per producer: list[kWsListCap] int4, histograms lo/hi[2][34] int, plan[kWsMaxUnits] int2
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(dyn4);
  WsProdShared* ps = reinterpret_cast<WsProdShared*>(bars + 2 * kWsMaxStages + 2);
  WsUnit* units = reinterpret_cast<WsUnit*>(ps + 1);
  int4* meta = reinterpret_cast<int4*>(units + kWsStages);
  float* stage = reinterpret_cast<float*>(meta + kWsStages * cap);
  const int stage_floats = cap * p.stage_stride;
  int2* lists_all = reinterpret_cast<int2*>(stage + kWsStages * stage_floats);
  int4* lists_prod = reinterpret_cast<int4*>(lists_all + ncw * M * cap);
  int* hist_all = reinterpret_cast<int*>(lists_prod + 2 * kWsListCap);
  int2* plan_all = reinterpret_cast<int2*>(hist_all + 2 * 2 * 34);
  const unsigned full0 = smem_u32(bars), empty0 = smem_u32(bars + kWsMaxStages);
  const unsigned turn0 = smem_u32(bars + 2 * kWsMaxStages);

  if (tid == 0) {
    for (int s = 0; s < kWsStages; ++s) {
      mbar_init(full0 + 8u * s, 1);
      mbar_init(empty0 + 8u * s, (unsigned)ncw);
    }
    mbar_init(turn0, 1);
    mbar_init(turn0 + 8u, 1);
    ps->ring_s = 0;
    ps->ring_ph = 0;
    ps->done[0] = 0;
    ps->done[1] = NP == 1 ? 1 : 0;   // one producer: it keeps the turn from the start
    ps->stopped = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();   // the only block-wide barrier

  const int zw = p.zw, R = p.rows_per_step;
  const int64_t chan_elems = (int64_t)p.H * p.slab_elems;

  if (warp < NP) {
    // ------------------------------------------------------------ producers
    // Two producer warps take turns: while one emits its tile's units into
    // the ring (the serial part), the other fetches the next tile and scans
    // its bin (dependent global loads: the latency that would otherwise
    // leave the consumers waiting). Turn k is an mbarrier the other producer
    // arrives on; the ring cursor travels with the turn.
#ifdef VG_EXP_WSPROF
    const long long tp0 = clock64();
#endif
    const int k = warp;
    int4* list = lists_prod + k * kWsListCap;
    int* hlo = hist_all + k * 68;    // [34]: candidates whose (relative) y-support starts at j
    int* hhi = hlo + 34;             // [34]: ... ends at j
    int2* plan = plan_all + k * kWsMaxUnits;
    const unsigned my_turn = turn0 + 8u * k, other_turn = turn0 + 8u * (k ^ 1);
    unsigned turn_par = k == 0 ? 1u : 0u;   // producer 0 holds the first turn
    bool hold = false;                      // kept the turn (other producer is done)
    const unsigned gz_bytes = 4u * (unsigned)(zw * SW);
    int next_tile = 0;
    if (lane == 0) next_tile = atomicAdd(tile_counter, 1);
    for (;;) {
      const int tile = __shfl_sync(kFull, next_tile, 0);
      const bool valid = tile < n_tiles;
      WsTile T{};
      int j0 = 0, j1 = 0, row_base = 0, row_end = 0, zv0 = 0, nl = 0, pos = 0, nbk = 0, n_units = 0;
      const int* bl = nullptr;
      AtomFilter f0{};
      const bool gx16 = true;   // row_base % 4 == 0 (launch rule)
      // gx window start | staged count << 16 of a candidate (staged bulk copy)
      auto gx_pack = [&](int sx) {
        const int g0 = gx_window_start(p, sx, row_base, gx16);
        const int cnt = p.gx_win > 0 ? min(p.gx_win, p.rx - g0) : round_up4(row_end - row_base);
        return g0 | (cnt << 16);
      };
      // candidates of list[0, nl) -> histograms -> unit plan (slab pairs, greedy)
      auto make_plan = [&]() {
        const int nj = j1 - j0;
        for (int j = lane; j < 68; j += 32) hlo[j] = 0;
        __syncwarp();
        for (int i = lane; i < nl; i += 32) {
          const int sy = list[i].y;
          atomicAdd(&hlo[max(lo16(sy) - j0, 0)], 1);
          atomicAdd(&hhi[min(hi16(sy) - j0, nj)], 1);
        }
        __syncwarp();
        if (lane == 0) {   // suffix sums of starts (#lo >= j), prefix sums of ends (#hi <= j)
          int run = 0;
          for (int j = nj; j >= 0; --j) { run += hlo[j]; hlo[j] = run; }
          run = 0;
          for (int j = 0; j <= nj; ++j) { run += hhi[j]; hhi[j] = run; }
        }
        __syncwarp();
        // count(js, je) = nl - #(lo >= je) - #(hi <= js)
        int nu = 0, js = 0;
        while (js < nj) {
          int je = min(nj, js + 2);
          while (je < nj) {
            const int je2 = min(nj, je + 2);
            if (nl - hlo[je2] - hhi[js] > cap) break;
            je = je2;
          }
          if (lane == 0) plan[nu] = make_int2(js, je);
          ++nu;
          js = je;
        }
        __syncwarp();
        return nu;
      };
      if (valid) {
        T = ws_decode(p, tile);
        const int64_t a0 = __ldg(p.offsets + T.b), a1 = __ldg(p.offsets + T.b + 1);
        j0 = T.chunk * p.jc;
        j1 = min(p.H, j0 + p.jc);
        row_base = T.rblk * M * R;
        row_end = min(p.W, row_base + M * R);
        zv0 = T.zblk * zw * SW;
        const int zv1 = min(p.D, zv0 + zw * SW);
        if (p.stats != nullptr && T.c == 0 && T.chunk == 0 && T.rblk == 0 && T.zblk == 0) {
          // voxel_writes (gridgen.py:103) and the invalid-atom flag of the molecule
          long long w = 0;
          bool bad = false;
          for (int64_t a = a0 + lane; a < a1; a += 32 * 8) {
            int4 sp[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)   // 8 loads in flight per lane
              sp[u] = a + 32 * u < a1 ? __ldg(p.supp + a + 32 * u) : make_int4(0, 0, 0, 0);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              w += (long long)(hi16(sp[u].x) - lo16(sp[u].x)) * (hi16(sp[u].y) - lo16(sp[u].y)) *
                   (hi16(sp[u].z) - lo16(sp[u].z));
              bad = bad || sp[u].w < 0;
            }
          }
          const long long wt = warp_sum(w);
          if (lane == 0 && wt != 0)
            atomicAdd(reinterpret_cast<unsigned long long*>(&p.stats[T.b].voxel_writes),
                      (unsigned long long)wt);
          if (__any_sync(kFull, bad) && lane == 0)
            atomicOr(reinterpret_cast<unsigned long long*>(&p.stats[T.b].voxel_writes), 1ull << 63);
        }
        // the tile's K2 bin: ordered atoms of channel c whose y-support meets the chunk
        const int* bo = p.bin_off + T.b * (p.bin_nb + 1) + T.c * p.n_jchunks + T.chunk;
        const int q0 = __ldg(bo);
        nbk = __ldg(bo + 1) - q0;
        bl = p.bins + a0 * p.n_jchunks + q0;
        f0 = AtomFilter{T.c, j0, j1, row_base, row_end, zv0, zv1};
        int nxt = nbk;
        nl = ws_scan_bin<4>(bl, 0, nbk, p.supp, f0, list, kWsListCap, nxt);
        pos = nxt;
        __syncwarp();
        for (int i = lane; i < nl; i += 32) list[i].z = gx_pack(list[i].x);
        __syncwarp();
        n_units = make_plan();
        if (lane == 0) next_tile = atomicAdd(tile_counter, 1);   // in flight during the turn
      }
      // ---- take the turn (the ring is ours until we pass it on)
      if (!hold) {
        mbar_wait(my_turn, turn_par);
        turn_par ^= 1u;
      }
      const bool other_done = ps->done[k ^ 1] != 0;
      int s = ps->ring_s;
      unsigned ph = ps->ring_ph;
      if (!valid) {
        if (other_done) {   // last producer standing: the stop unit
          mbar_wait(empty0 + 8u * s, ph ^ 1u);
          if (lane == 0) {
            units[s].tile = -1;
            mbar_arrive(full0 + 8u * s);
          }
        } else if (lane == 0) {
          ps->done[k] = 1;
          mbar_arrive(other_turn);
        }
        break;
      }
      int pass = 0;
      for (;;) {
        for (int ui = 0; ui < n_units; ++ui) {
          const int2 pu = plan[ui];
          const int js = j0 + pu.x, je = j0 + pu.y;
          const int gy0 = js & ~3;
          const unsigned gy_bytes = 4u * (unsigned)(round_up4(je) - gy0);
          int kc = 0, seg = 0;
          for (;;) {
#ifdef VG_EXP_WSPROF
            const long long tw = clock64();
            mbar_wait(empty0 + 8u * s, ph ^ 1u);
            if (lane == 0) { WSP_ADD(2, clock64() - tw); WSP_ADD(4, 1); }
#else
            mbar_wait(empty0 + 8u * s, ph ^ 1u);
#endif
            int4* um = meta + s * cap;
            // ordered compaction of the candidates meeting [js, je), from kc
            unsigned bytes = 0;
            int ns = 0, i = kc;
            for (; i < nl && ns < cap; i += 32) {
              const int q = i + lane;
              int4 e = make_int4(0, 0, 0, 0);
              bool hit = false;
              if (q < nl) {
                e = list[q];
                hit = lo16(e.y) < je && hi16(e.y) > js;
              }
              const unsigned bal = __ballot_sync(kFull, hit);
              const int n = __popc(bal), rank = __popc(bal & ((1u << lane) - 1u));
              if (ns + n > cap) {   // take the first cap - ns hits, resume at the next one
                const int take = cap - ns;
                if (hit && rank < take) {
                  um[ns + rank] = e;
                  bytes += gy_bytes + gz_bytes + 4u * (unsigned)hi16(e.z);
                }
                unsigned b = bal;
                for (int r = 0; r < take; ++r) b &= b - 1u;
                i += __ffs(b) - 1;   // the first hit not taken
                ns = cap;
                break;
              }
              if (hit) {
                um[ns + rank] = e;
                bytes += gy_bytes + gz_bytes + 4u * (unsigned)hi16(e.z);
              }
              ns += n;
            }
            kc = i < nl ? i : nl;
            bytes = __reduce_add_sync(kFull, bytes);
            if (lane == 0) {
              units[s].tile = tile;
              units[s].js = js;
              units[s].je = je;
              units[s].ns = ns;
              units[s].first = (pass == 0 && seg == 0) ? 1 : 0;
              units[s].gy_shift = js - gy0;
            }
            __syncwarp();
            const unsigned fb = full0 + 8u * s;
            if (lane == 0) {
              if (bytes != 0) mbar_arrive_tx(fb, bytes);
              else mbar_arrive(fb);
            }
            __syncwarp();
            const unsigned blk0 = smem_u32(stage + s * stage_floats);
            for (int q = lane; q < ns; q += 32) {
              const int4 e = um[q];
              const int64_t a = e.w;
              const unsigned d0 = blk0 + 4u * (unsigned)(q * p.stage_stride);
              bulk_g2s(d0, p.ty + a * p.ry + gy0, gy_bytes, fb);
              bulk_g2s(d0 + 4u * (unsigned)p.stage_gx, p.tx + a * p.rx + lo16(e.z),
                       4u * (unsigned)hi16(e.z), fb);
              bulk_g2s(d0 + 4u * (unsigned)p.stage_gz, p.tz + a * p.rz + zv0, gz_bytes, fb);
            }
            if (++s == kWsStages) {
              s = 0;
              ph ^= 1u;
            }
            ++seg;
            if (kc >= nl) break;
          }
        }
        if (pos >= nbk) break;
        // more than kWsListCap candidates in the bin (rare): the next ones,
        // continuing every voxel's sum (first = 0), while holding the turn
        ++pass;
        int nxt = nbk;
        nl = ws_scan_bin<4>(bl, pos, nbk, p.supp, f0, list, kWsListCap, nxt);
        pos = nxt;
        __syncwarp();
        for (int i = lane; i < nl; i += 32) list[i].z = gx_pack(list[i].x);
        __syncwarp();
        n_units = make_plan();
      }
      // ---- pass the turn (keep it when the other producer has finished)
      if (lane == 0) {
        ps->ring_s = s;
        ps->ring_ph = ph;
      }
      __syncwarp();
      if (other_done) {
        hold = true;
      } else {
        if (lane == 0) mbar_arrive(other_turn);
      }
    }
#ifdef VG_EXP_WSPROF
    if (lane == 0) WSP_ADD(3, clock64() - tp0);
#endif
    return;
  }

  // --------------------------------------------------------------- consumers
  const int ct = tid - 32 * NP, cw = warp - NP;
  const int r0 = div_magic(ct, p.zw_magic);
  const int kk = ct - r0 * zw;                       // slot in the z window
  const int wr0 = div_magic(cw * 32, p.zw_magic), wr1 = div_magic(cw * 32 + 31, p.zw_magic);
  const int half = 4 * zw;
  const unsigned gz_off = 4u * (unsigned)(p.stage_gz + 4 * kk);
  const unsigned gx_off = 4u * (unsigned)(p.stage_gx + r0);
  int2* lists = lists_all + cw * M * cap;
  const unsigned lists_s = smem_u32(lists);
  int s = 0;
  unsigned ph = 0;
  // nonzero counts are flushed per tile (one warp atomic), not per unit
  int64_t nz_b = -1;
  long long nz_acc = 0;
  auto flush = [&]() {
    const long long tot = warp_sum(nz_acc);
    if (lane == 0 && tot != 0)
      atomicAdd(reinterpret_cast<unsigned long long*>(&p.stats[nz_b].nonzero_voxels),
                (unsigned long long)tot);
    nz_acc = 0;
  };
  int cur_tile = -1;
#ifdef VG_EXP_WSPROF
  const long long tc0 = clock64();
  long long waited = 0;
#endif
  for (;;) {
#ifdef VG_EXP_WSPROF
    const long long tw = clock64();
    mbar_wait(full0 + 8u * s, ph);
    waited += clock64() - tw;
#else
    mbar_wait(full0 + 8u * s, ph);
#endif
    const WsUnit u = units[s];
#ifdef VG_EXP_WSPROF
    if (lane == 0 && cw == 0 && u.tile >= 0) WSP_ADD(5, u.ns);
#endif
    if (u.tile < 0) break;
    const WsTile T = ws_decode(p, u.tile);
    if (u.tile != cur_tile) {
      if (p.stats != nullptr && nz_b >= 0) flush();
      cur_tile = u.tile;
      nz_b = T.b;
    }
    const int row_base = T.rblk * M * R, row_end = min(p.W, row_base + M * R);
    const int zv0 = T.zblk * zw * SW;
    const int ibase = row_base + r0;
    const int zf = zv0 + 4 * kk;
    const int rlo0 = row_base + wr0, rhi0 = row_base + wr1;
    const unsigned stage_s = smem_u32(stage + s * stage_floats);
    Counts<M> cnt;
    build_sublists<M>(p, meta + s * cap, u.ns, -1, lists, stage_s, u.js, u.je, row_base, rlo0, rhi0,
                      R, cnt);
    __syncwarp();
    float* base = p.out + (T.b * p.C + T.c) * chan_elems + u.js * p.slab_elems + ibase * p.D + zf;
    int nz;
    if (u.first)
      nz = accumulate<M, SW, YP, true>(base, p.slab_elems, R * p.D, u.je - u.js, ibase, row_end, R, cnt,
                                       lists_s, cap, gx_off, gz_off, half, u.gy_shift);
    else
      nz = accumulate<M, SW, YP, false>(base, p.slab_elems, R * p.D, u.je - u.js, ibase, row_end, R,
                                        cnt, lists_s, cap, gx_off, gz_off, half, u.gy_shift);
    __syncwarp();   // every lane is done reading the slot's staged data
    if (lane == 0) mbar_arrive(empty0 + 8u * s);
    nz_acc += nz;
    if (++s == kWsStages) {
      s = 0;
      ph ^= 1u;
    }
  }
  if (p.stats != nullptr && nz_b >= 0) flush();
#ifdef VG_EXP_WSPROF
  if (lane == 0) {
    WSP_ADD(0, waited);
    WSP_ADD(1, clock64() - tc0);
  }
#endif
}

// ---------------------------------------------------------------------------
// K2: ordered candidate bins for large molecules
// ---------------------------------------------------------------------------
// One CTA per molecule. Bin q = channel * nch + y-chunk holds, in ascending
// atom order, every atom of that channel with a non-empty support box whose
// y-support meets the chunk [k*jc, (k+1)*jc). Warp w owns a contiguous atom
// range; per-warp counts, a prefix over warps and bins, then an ordered fill
// (ranks within a warp from __match_any_sync) keep the order deterministic
// without sorting. K3's per-channel CTAs then scan their bin instead of the
// whole molecule.
__device__ __forceinline__ void bin_range(const BinParams& p, const int4& s, int jc, bool valid,
                                          bool& member, int& c, int& k0, int& k1) {
  // (invalid atoms have empty supports and channel -1; the channel bound
  // keeps q inside this warp's counters whatever the supports hold)
  member = valid && lo16(s.x) < hi16(s.x) && lo16(s.y) < hi16(s.y) && lo16(s.z) < hi16(s.z) &&
           (unsigned)s.w < (unsigned)p.C;
  c = s.w;
  k0 = member ? lo16(s.y) / jc : 0;
  k1 = member ? (hi16(s.y) - 1) / jc : -1;
}

__global__ void __launch_bounds__(kBinWarps * 32) vg_bin_kernel(const __grid_constant__ BinParams p) {
  extern __shared__ int bsm[];
  int* cnt = bsm;                      // [kBinWarps][nb]: counts, then write cursors
  int* start = bsm + kBinWarps * p.nb; // [nb]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b = blockIdx.x;
  // K3 directly follows on the stream (vg_slabs_f32 / vg_generate_f32): let its
  // CTAs be scheduled now; they wait (griddepcontrol.wait) for this grid
  asm volatile("griddepcontrol.launch_dependents;");
  const int64_t a0 = __ldg(p.offsets + b), a1 = __ldg(p.offsets + b + 1);
  const int nb = p.nb, nch = p.nch;
  if (b == 0 && threadIdx.x == 0 && p.tile_counter != nullptr) *p.tile_counter = 0;
  for (int i = threadIdx.x; i < kBinWarps * nb; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  const int64_t n = a1 - a0;
  const int64_t per = ((n + kBinWarps - 1) / kBinWarps + 31) / 32 * 32;
  const int64_t w0 = a0 + warp * per, w1 = min(a1, w0 + per);
  int* mine = cnt + warp * nb;
  int* out = p.bins + a0 * nch;
  for (int pass = 0; pass < 2; ++pass) {
    for (int64_t g = w0; g < w1; g += 32) {
      const int64_t a = g + lane;
      const bool valid = a < w1;
      const int4 s = valid ? __ldg(p.supp + a) : make_int4(0, 0, 0, 0);
      bool member;
      int c, k0, k1;
      bin_range(p, s, p.jc, valid, member, c, k0, k1);
      const int kmin = __reduce_min_sync(kFull, member ? k0 : INT_MAX);
      const int kmax = __reduce_max_sync(kFull, member ? k1 : -1);
      for (int k = kmin; k <= kmax; ++k) {
        const bool in = member && k0 <= k && k <= k1;
        const int q = in ? c * nch + k : -1;
        const unsigned peers = __match_any_sync(kFull, q);
        const int leader = __ffs(peers) - 1;
        int base = 0;
        if (in && lane == leader) base = mine[q];
        base = __shfl_sync(kFull, base, leader);
        if (in) {
          if (pass == 1) out[base + __popc(peers & ((1u << lane) - 1u))] = (int)a;
          if (lane == leader) mine[q] = base + __popc(peers);
        }
        __syncwarp();
      }
    }
    __syncthreads();
    if (pass == 0) {
      // per bin: exclusive prefix over warps (then the bin's total)
      for (int q = threadIdx.x; q < nb; q += blockDim.x) {
        int run = 0;
        for (int w = 0; w < kBinWarps; ++w) {
          const int v = cnt[w * nb + q];
          cnt[w * nb + q] = run;
          run += v;
        }
        start[q] = run;
      }
      __syncthreads();
      // exclusive scan of bin totals (one warp, 32 bins per step)
      if (warp == 0) {
        int carry = 0;
        for (int q0 = 0; q0 < nb; q0 += 32) {
          const int q = q0 + lane;
          const int v = q < nb ? start[q] : 0;
          int x = v;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, x, o);
            if (lane >= o) x += y;
          }
          if (q < nb) start[q] = carry + x - v;
          carry += __shfl_sync(kFull, x, 31);
        }
        if (lane == 0) p.bin_off[b * (nb + 1) + nb] = carry;
      }
      __syncthreads();
      for (int q = threadIdx.x; q < nb; q += blockDim.x) p.bin_off[b * (nb + 1) + q] = start[q];
      for (int i = threadIdx.x; i < kBinWarps * nb; i += blockDim.x) cnt[i] += start[i % nb];
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// elementwise helpers
// ---------------------------------------------------------------------------
__global__ void vg_erf_kernel(const float* __restrict__ t, float* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = vg_erf_f32(t[i]);
}

// Write-ceiling probe: grid-stride streaming 128-bit stores (as K3 stores).
// (scripts/probes/write_ceiling.cu: this pattern with 148*64 CTAs is the
// fastest of the simple write patterns on B200, ~6.87 TB/s.)
// One 16 KiB block of streaming float4 stores per CTA (4 per thread, each
// warp instruction 512 contiguous bytes), as many CTAs as blocks: 7.5 TB/s on
// B200, above a grid-stride sweep of the same stores (7.0) and torch's fill_
// (7.4) (scripts/fill_probe.py, profiles/r2_write_ceiling.txt).
__global__ void __launch_bounds__(256) vg_fill_kernel(float4* __restrict__ out, int64_t n4, float4 v) {
  const int64_t base = (int64_t)blockIdx.x * 1024 + threadIdx.x;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int64_t i = base + k * 256;
    if (i < n4) __stcs(out + i, v);
  }
}

__global__ void vg_fill_tail_kernel(float* __restrict__ out, int64_t n, float v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = v;
}

// ---------------------------------------------------------------------------
// host-side validation + launch planning
// ---------------------------------------------------------------------------
int validate(const vg_batch_desc* d) {
  refresh_env();   // every planning entry point validates first
  if (d == nullptr) return set_error(VG_ERR_INVALID, "descriptor is NULL");
  if (d->n_molecules < 0 || d->n_atoms < 0)
    return set_error(VG_ERR_INVALID, "negative molecule or atom count");
  if (d->n_atoms >= (int64_t)INT_MAX)
    return set_error(VG_ERR_INVALID, "n_atoms %lld exceeds 2^31-1", (long long)d->n_atoms);
  if (d->H < 1 || d->W < 1 || d->D < 1 || d->H > kMaxAxis || d->W > kMaxAxis || d->D > kMaxAxis)
    return set_error(VG_ERR_INVALID, "shape (%d, %d, %d) must be 3 voxel counts in [1, %d]", d->H,
                     d->W, d->D, kMaxAxis);
  if (d->C < 1) return set_error(VG_ERR_INVALID, "channels must be >= 1, got %d", d->C);
  if (!(d->scale > 0.0) || !std::isfinite(d->scale))
    return set_error(VG_ERR_INVALID, "scale 1/(sigma*sqrt(2)) must be positive and finite");
  if (d->n_molecules > 0 && d->offsets == nullptr)
    return set_error(VG_ERR_INVALID, "offsets is NULL");
  if (d->n_atoms > 0 && (d->xyz == nullptr || d->channel == nullptr))
    return set_error(VG_ERR_INVALID, "xyz/channel is NULL with n_atoms > 0");
  for (int a = 0; a < 3; ++a) {
    if (d->mol_delta == nullptr && !(d->delta[a] > 0.0))
      return set_error(VG_ERR_INVALID, "voxel size must be positive, got %g", d->delta[a]);
  }
  return VG_OK;
}

// y-chunking of the candidate bins (K2) for this batch, or false if K3 will
// not use bins (defined with the K3 launch plan below).
bool bin_plan(const vg_batch_desc& d, int* jc, int* nch);

void fill_layout(const vg_batch_desc* d, vg_ws_layout* L) {
  const size_t na = (size_t)d->n_atoms;
  L->row_x = round_up4(d->W);
  L->row_y = round_up4(d->H);
  L->row_z = round_up4(d->D);
  size_t off = 0;
  L->tx = off;
  off = align_up(off + na * L->row_x * sizeof(float), 256);
  L->ty = off;
  off = align_up(off + na * L->row_y * sizeof(float), 256);
  L->tz = off;
  off = align_up(off + na * L->row_z * sizeof(float), 256);
  L->supp = off;
  off = align_up(off + na * 4 * sizeof(int32_t), 256);
  // candidate bins: atom indices, molecule b's region holds (atoms of b) x
  // chunks entries from offsets[b] * chunks; then per molecule C*chunks+1
  // bin offsets
  int jc = 0, nch = 0;
  L->bins = L->bin_off = 0;
  L->bin_jc = L->bin_chunks = 0;
  if (bin_plan(*d, &jc, &nch)) {
    L->bin_jc = jc;
    L->bin_chunks = nch;
    L->bins = off;
    off = align_up(off + na * (size_t)nch * sizeof(int32_t), 256);
    L->bin_off = off;
    // bin offsets, then K3W's tile counter (16-byte aligned, see tile_counter_of)
    off = align_up(off + (size_t)d->n_molecules * ((size_t)d->C * nch + 1) * sizeof(int32_t) + 32,
                   256);
  }
  L->total = off == 0 ? 256 : off;
}

int launch_tables(const vg_batch_desc* d, const vg_ws_layout& L, char* ws, cudaStream_t st) {
  if (d->n_atoms == 0) return VG_OK;
  TableParams p;
  memset(&p, 0, sizeof p);
  p.offsets = d->offsets;
  p.xyz = d->xyz;
  p.channel = d->channel;
  p.mol_origin = d->mol_origin;
  p.mol_delta = d->mol_delta;
  p.tbl[0] = reinterpret_cast<float*>(ws + L.tx);
  p.tbl[1] = reinterpret_cast<float*>(ws + L.ty);
  p.tbl[2] = reinterpret_cast<float*>(ws + L.tz);
  p.supp = reinterpret_cast<int32_t*>(ws + L.supp);
  for (int a = 0; a < 3; ++a) {
    p.origin[a] = d->origin[a];
    p.delta[a] = d->delta[a];
  }
  p.scale = d->scale;
  p.tsat_over_s = (double)VG_TSAT / d->scale;
  for (int a = 0; a < 3; ++a) p.inv_delta[a] = 1.0 / d->delta[a];
  p.n_atoms = d->n_atoms;
  p.n_molecules = d->n_molecules;
  p.C = d->C;
  p.n[0] = d->W;
  p.n[1] = d->H;
  p.n[2] = d->D;
  p.row[0] = L.row_x;
  p.row[1] = L.row_y;
  p.row[2] = L.row_z;
  p.has_threshold = !std::isnan(d->threshold);
  p.threshold = d->threshold;
  p.periodic = d->periodic != 0;
  if (!p.periodic) {
    // lanes per row: more lanes only for small batches (K1 otherwise runs
    // beside the previous batch's K3 in GridPipeline, where wider K1 CTAs
    // take more of K3's SM slots; measured on B200)
    int T = 1;
    while (T < 8 && d->n_atoms * 3 * T < 148 * 384) T *= 2;
    T = env_int("VG_K1T", T, 1, 8);
    if (T & (T - 1)) T = 1;
    const int64_t rows_per_block = kTableThreads / T;
    const dim3 grid((unsigned)((d->n_atoms + rows_per_block - 1) / rows_per_block), 3);
    switch (T) {
      case 2: vg_tables_open_kernel<2><<<grid, kTableThreads, 0, st>>>(p); break;
      case 4: vg_tables_open_kernel<4><<<grid, kTableThreads, 0, st>>>(p); break;
      case 8: vg_tables_open_kernel<8><<<grid, kTableThreads, 0, st>>>(p); break;
      default: vg_tables_open_kernel<1><<<grid, kTableThreads, 0, st>>>(p); break;
    }
    return check_launch("vg_tables_open_kernel");
  }
  const int64_t warps = d->n_atoms * 3;
  const int64_t blocks = (warps + kTableThreads / 32 - 1) / (kTableThreads / 32);
  vg_tables_kernel<<<(unsigned)blocks, kTableThreads, 0, st>>>(p);
  return check_launch("vg_tables_kernel");
}

}  // namespace

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
VG_API const char* vg_last_error(void) { return g_last_error; }

VG_API int vg_abi_version(void) { return VG_ABI_VERSION; }

VG_API int vg_workspace_layout(const vg_batch_desc* desc, vg_ws_layout* layout) {
  g_last_error[0] = '\0';
  int rc = validate(desc);
  if (rc != VG_OK) return rc;
  if (layout == nullptr) return set_error(VG_ERR_INVALID, "layout is NULL");
  fill_layout(desc, layout);
  return VG_OK;
}

VG_API int vg_axis_tables_f32(const vg_batch_desc* desc, void* workspace, size_t workspace_bytes,
                              void* stream) {
  g_last_error[0] = '\0';
  vgdev::DeviceGuard guard(workspace);
  int rc = validate(desc);
  if (rc != VG_OK) return rc;
  vg_ws_layout L;
  fill_layout(desc, &L);
  if (workspace == nullptr || workspace_bytes < L.total)
    return set_error(VG_ERR_WORKSPACE, "workspace needs %zu bytes, got %zu", L.total,
                     workspace_bytes);
  return launch_tables(desc, L, static_cast<char*>(workspace), static_cast<cudaStream_t>(stream));
}

namespace {

int gcd_int(int a, int b) { return b == 0 ? a : gcd_int(b, a % b); }

// Launch shape of the row-structured kernel: NT = R * spr threads (a multiple
// of 32), M <= 8 row steps per CTA, row_blocks CTAs per slab; minimises idle
// rows, then prefers NT close to 256. False if no shape exists (huge rows).
bool plan_rows(int spr, int W, int* nt, int* R, int* M, int* row_blocks) {
  const int base = spr / gcd_int(32, spr) * 32;  // lcm(32, spr)
  if (base > kRowThreads) return false;
  // CTAs of t = base * q threads, r = t / spr rows per step, m steps
  auto scan = [&](int forced) {
    double best = 1e30;
    for (int q = 1; base * q <= kRowThreads; ++q) {
      if (forced != 0 && forced != q) continue;
      const int t = base * q, r = t / spr;
      if (r > kMaxCtaRows && t > 256) continue;   // wider CTAs only up to 64 rows
      const int need = (W + r - 1) / r;
      int m = need < 8 ? need : 8;
      const int mcap = kMaxCtaRows / r > 1 ? kMaxCtaRows / r : 1;
      if (m > mcap) m = mcap;
      const int rb = (need + m - 1) / m;
      const double waste = (double)(rb * m * r - W) / (rb * m * r);
      // least padding; then fewer row steps per CTA (512-thread CTAs of one
      // step beat 256-thread CTAs of two at cfg1, 288 threads cover cfg4's
      // 48 rows exactly; measured on B200), then the count nearest 256
      const double score =
          waste + (t < 128 ? 0.25 : 0.0) + (m - 1) * 1e-3 + fabs(t - 256.0) * 1e-6;
      if (score < best) {
        best = score;
        *nt = t;
        *R = r;
        *M = m;
        *row_blocks = rb;
      }
    }
    return best < 1e30;
  };
  // hook VG_PLAN_Q: force the thread multiple (a multiple the rules reject
  // falls back to the free choice)
  const int fq = env_int("VG_PLAN_Q", 0, 1, kRowThreads / base);
  return (fq != 0 && scan(fq)) || scan(0);
}

// Set by vg_generate_f32 around its K3 launch: K3 directly follows K1 on the
// same stream and may be launched as a programmatic dependent of it.
thread_local bool g_pdl_launch = false;

template <int M, int SW, int YP>
int launch_rows_m(dim3 grid, int nt, size_t smem, cudaStream_t st, const SlabParams& p) {
  // The row kernel is register-limited to 4 CTAs/SM; ask for the largest
  // shared-memory carveout so that shared memory never lowers that.
  static vgdev::Once once;
  const cudaError_t e = vgdev::configure_once(once, [] {
    cudaError_t r = cudaFuncSetAttribute(vg_slab_kernel<M, SW, YP>,
                                         cudaFuncAttributePreferredSharedMemoryCarveout,
                                         cudaSharedmemCarveoutMaxShared);
    if (r == cudaSuccess)
      r = cudaFuncSetAttribute(vg_slab_kernel<M, SW, YP>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    return r;
  });
  if (e != cudaSuccess)
    return set_error(VG_ERR_CUDA, "vg_slab_kernel attributes: %s", cudaGetErrorString(e));
  if (g_pdl_launch) {
    // programmatic dependent launch: K3's CTAs are scheduled while K1 (the
    // previous kernel on this stream) finishes; K3 waits on griddepcontrol
    // before it reads any table (vg_generate_f32 only)
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.gridDim = grid;
    cfg.blockDim = dim3((unsigned)nt);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    const cudaError_t le = cudaLaunchKernelEx(&cfg, vg_slab_kernel<M, SW, YP>, p);
    if (le != cudaSuccess)
      return set_error(VG_ERR_CUDA, "vg_slab_kernel (PDL): %s", cudaGetErrorString(le));
    return VG_OK;
  }
  vg_slab_kernel<M, SW, YP><<<grid, nt, smem, st>>>(p);
  return VG_OK;
}

template <int SW, int YP>
int launch_rows(int M, dim3 grid, int nt, size_t smem, cudaStream_t st, const SlabParams& p) {
  switch (M) {
    case 1: return launch_rows_m<1, SW, YP>(grid, nt, smem, st, p);
    case 2: return launch_rows_m<2, SW, YP>(grid, nt, smem, st, p);
    case 3: return launch_rows_m<3, SW, YP>(grid, nt, smem, st, p);
    case 4: return launch_rows_m<4, SW, YP>(grid, nt, smem, st, p);
    case 5: return launch_rows_m<5, SW, YP>(grid, nt, smem, st, p);
    case 6: return launch_rows_m<6, SW, YP>(grid, nt, smem, st, p);
    case 7: return launch_rows_m<7, SW, YP>(grid, nt, smem, st, p);
    default: return launch_rows_m<8, SW, YP>(grid, nt, smem, st, p);
  }
}

// Registers per thread of the row kernel instance (queried once): the
// shared-memory budget keeps as many CTAs resident as the registers allow.
template <int SW, int YP>
int rows_regs_sw(int M) {
  static std::atomic<int> regs[9];   // zero-initialised (static storage)
  const int m = M < 1 ? 1 : (M > 8 ? 8 : M);
  if (regs[m].load(std::memory_order_relaxed) == 0) {
    cudaFuncAttributes a;
    cudaError_t e = cudaErrorInvalidValue;
    switch (m) {
      case 1: e = cudaFuncGetAttributes(&a, vg_slab_kernel<1, SW, YP>); break;
      case 2: e = cudaFuncGetAttributes(&a, vg_slab_kernel<2, SW, YP>); break;
      case 3: e = cudaFuncGetAttributes(&a, vg_slab_kernel<3, SW, YP>); break;
      case 4: e = cudaFuncGetAttributes(&a, vg_slab_kernel<4, SW, YP>); break;
      case 5: e = cudaFuncGetAttributes(&a, vg_slab_kernel<5, SW, YP>); break;
      case 6: e = cudaFuncGetAttributes(&a, vg_slab_kernel<6, SW, YP>); break;
      case 7: e = cudaFuncGetAttributes(&a, vg_slab_kernel<7, SW, YP>); break;
      default: e = cudaFuncGetAttributes(&a, vg_slab_kernel<8, SW, YP>); break;
    }
    regs[m] = e == cudaSuccess && a.numRegs > 0 ? a.numRegs : 64;
  }
  return regs[m];
}

int rows_regs(int sw, int yp, int M) {
  if (sw == 8) return yp == 2 ? rows_regs_sw<8, 2>(M) : rows_regs_sw<8, 1>(M);
  return sw == 4 ? rows_regs_sw<4, 1>(M) : rows_regs_sw<1, 1>(M);
}

// z window (slots per row segment) of the row kernel: whole rows up to 16
// slots, 8-slot (32-float, 128 B) windows for wider rows so warps cull in z
// too. VG_ZW overrides (tuning hook).
int pick_zw(int spr, int sw) {
  const int v = env_int("VG_ZW", 0, 1, spr);
  if (v > 0 && spr % v == 0) return v;
  const int win = 32 / sw;  // 32-float (128 B) windows on rows wider than 64 floats
  if (spr * sw > 64 && win > 0 && spr % win == 0) return win;
  return spr;
}

// Slot width (voxels per thread slot): 8 (two float4, half a z-window
// apart) when D % 8 == 0, else 4 (float4), else 1. VG_SW overrides.
int pick_sw(int D, bool aligned16) {
  int sw = !aligned16 || D % 4 != 0 ? 1 : (D % 8 == 0 ? 8 : 4);
  const int v = env_int("VG_SW", 0, 1, 8);
  if ((v == 1) || (v == 4 && aligned16 && D % 4 == 0) || (v == 8 && aligned16 && D % 8 == 0))
    sw = v;
  return sw;
}

// K3 launch (tables must already be in the workspace, same stream).
// K3 launch plan, shared by the workspace layout (which sizes the candidate
// bins for the plan's y-chunks) and the launch.
struct SlabPlan {
  bool rows_ok;         // row-structured kernel (else the generic one)
  bool vec;             // generic kernel: float4 slots
  int sw, width, spr, zw;
  int nt, R, M, row_blocks, z_blocks;
  int jc, n_jchunks;
  bool fuse;
  int64_t mean_atoms;
};

void plan_slabs(const vg_batch_desc& d, bool aligned16, SlabPlan* P) {
  memset(P, 0, sizeof *P);
  P->sw = pick_sw(d.D, aligned16);
  const int64_t slab = (int64_t)d.W * d.D;
  const bool force = env_int("VG_FORCE_GENERIC", 0, 0, 1) == 1;
  P->zw = pick_zw(d.D / P->sw, P->sw);
  P->rows_ok = !force &&
               plan_rows(P->zw, d.W, &P->nt, &P->R, &P->M, &P->row_blocks);
  // the generic kernel works in float4 or float slots
  P->vec = P->rows_ok ? P->sw >= 4 : (d.D % 4 == 0 && aligned16);
  P->width = P->rows_ok ? P->sw : (P->vec ? 4 : 1);
  P->spr = d.D / P->width;
  P->mean_atoms = d.n_molecules > 0 ? (d.n_atoms + d.n_molecules - 1) / d.n_molecules : 0;
  if (!P->rows_ok) return;
  P->z_blocks = P->spr / P->zw;
  const int rows_per_cta = P->M * P->R < d.W ? P->M * P->R : d.W;
  const int64_t cta_bytes = (int64_t)rows_per_cta * P->zw * P->width * 4;
  const int64_t mean_atoms = P->mean_atoms;
  // Channel fusion (one CTA serves all C channels of its tile from one staged
  // candidate list) for small molecules, whose whole atom list usually fits
  // the staging area; VG_FUSE=0/1 overrides (tuning hook).
  bool fuse = d.C > 1 && mean_atoms <= kFuseMeanAtoms;
  fuse = d.C > 1 && env_int("VG_FUSE", fuse ? 1 : 0, 0, 1) == 1;
  // Output bytes per CTA (measured on B200): fused CTAs ~1 MiB over all
  // channels; per-channel CTAs 256 KiB, halved for dense molecules (hundreds
  // of candidates per tile), whose shorter y-chunks halve less often.
  int64_t task_bytes = fuse ? kFusedTaskBytes : (mean_atoms > 512 ? kTaskBytes / 2 : kTaskBytes);
  // small batches: keep at least ~8 CTAs per SM in flight
  const int64_t total_bytes = d.n_molecules * (int64_t)d.C * d.H * slab * 4;
  if (task_bytes > total_bytes / kMinCtas) task_bytes = total_bytes / kMinCtas;
  const int task_kb = env_int("VG_TASK_KB", 0, 1, 1 << 20);
  if (task_kb > 0) task_bytes = (int64_t)task_kb * 1024;
  if (fuse) task_bytes = (task_bytes + d.C - 1) / d.C;   // per channel
  // y-slabs per CTA: aim for task_bytes of output (<= 32 for the slab masks),
  // then even out the chunks
  int jc = (int)((task_bytes + cta_bytes - 1) / cta_bytes);
  jc = jc < 1 ? 1 : (jc > d.H ? d.H : jc);
  if (jc > 32) jc = 32;
  {
    const int nch = (d.H + jc - 1) / jc;
    jc = (d.H + nch - 1) / nch;
  }
  P->jc = jc;
  P->n_jchunks = (d.H + jc - 1) / jc;
  P->fuse = fuse;
}

// Candidate bins (K2) pay for molecules large enough that every CTA would
// otherwise scan thousands of atoms: per-channel CTAs, > 2*256 atoms on
// average, and a bounded number of bins per molecule.
bool want_bins(const vg_batch_desc& d, const SlabPlan& P) {
  if (env_int("VG_BINS", 1, 0, 1) == 0) return false;
  if (!P.rows_ok || P.fuse || d.periodic) return false;
  if (P.mean_atoms <= 512) return false;
  const int64_t nb = (int64_t)d.C * P.n_jchunks;
  return nb <= kMaxBins && (int64_t)d.n_atoms * P.n_jchunks <= (int64_t)1 << 28;
}

bool bin_plan(const vg_batch_desc& d, int* jc, int* nch) {
  if (d.n_molecules == 0 || d.n_atoms == 0) return false;
  SlabPlan P;
  plan_slabs(d, true, &P);   // outputs from the torch allocator are 16-byte aligned
  if (!want_bins(d, P)) return false;
  *jc = P.jc;
  *nch = P.n_jchunks;
  return true;
}

// K3 launch (tables must already be in the workspace, same stream).
// K2: ordered per-(molecule, channel, y-chunk) candidate bins into the
// workspace (layout L must carry a bin plan). Needs only the supports K1
// wrote, so a pipeline can run it on the tables stream.
// K3W's tile counter: after the bin offsets, in the same workspace region.
int* tile_counter_of(const vg_batch_desc& d, const vg_ws_layout& L, char* ws) {
  const size_t n = (size_t)d.n_molecules * ((size_t)d.C * L.bin_chunks + 1) * sizeof(int32_t);
  return reinterpret_cast<int*>(ws + L.bin_off + align_up(n, 16));
}

int launch_bins(const vg_batch_desc& d, const vg_ws_layout& L, char* ws, cudaStream_t st,
                int* kernels) {
  const int nb = d.C * L.bin_chunks;
  BinParams bp;
  bp.tile_counter = tile_counter_of(d, L, ws);
  bp.offsets = d.offsets;
  bp.supp = reinterpret_cast<const int4*>(ws + L.supp);
  bp.bins = reinterpret_cast<int*>(ws + L.bins);
  bp.bin_off = reinterpret_cast<int*>(ws + L.bin_off);
  bp.nb = nb;
  bp.nch = L.bin_chunks;
  bp.jc = L.bin_jc;
  bp.C = d.C;
  const size_t bsmem = (size_t)(kBinWarps + 1) * nb * sizeof(int);
  static vgdev::Once once;
  const cudaError_t e = vgdev::configure_once(once, [] {
    return cudaFuncSetAttribute(vg_bin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (kBinWarps + 1) * kMaxBins * (int)sizeof(int));
  });
  if (e != cudaSuccess)
    return set_error(VG_ERR_CUDA, "vg_bin_kernel attributes: %s", cudaGetErrorString(e));
  vg_bin_kernel<<<(unsigned)d.n_molecules, kBinWarps * 32, bsmem, st>>>(bp);
  if (kernels != nullptr) *kernels += 1;
  return check_launch("vg_bin_kernel");
}

template <int M, int NP>
int launch_ws_m(int grid, int threads, size_t smem, cudaStream_t st, const SlabParams& p,
                int* counter, int n_tiles, int stages) {
  static vgdev::Once once;
  const cudaError_t e = vgdev::configure_once(once, [] {
    return cudaFuncSetAttribute(vg_slab_ws_kernel<M, NP>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  });
  if (e != cudaSuccess)
    return set_error(VG_ERR_CUDA, "vg_slab_ws_kernel attributes: %s", cudaGetErrorString(e));
  vg_slab_ws_kernel<M, NP><<<grid, threads, smem, st>>>(p, counter, n_tiles, stages);
  return check_launch("vg_slab_ws_kernel");
}

// SM count of the current device (cached per device).
int sm_count() {
  static std::atomic<int> cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  int v = cache[dev & 63].load(std::memory_order_relaxed);
  if (v == 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    cache[dev & 63].store(v, std::memory_order_relaxed);
  }
  return v;
}

// K3W launch: staged block per candidate gy[pad4(jc + 5)] (a unit's slabs
// from js & ~3) | gx window | gz window; staging capacity from the shared
// memory of VG_WS_MINB resident CTAs; one persistent CTA per slot.
int launch_ws(const vg_batch_desc& d, const vg_ws_layout& L, char* ws, SlabParams& p, int M, int R,
              int nt, int jc, cudaStream_t st) {
  p.stage_gx = round_up4(jc + 5);
  p.stage_gz = p.stage_gx + (p.gx_win > 0 ? p.gx_win : round_up4(M * R));
  p.stage_stride = p.stage_gz + round_up4(p.zw * 8);
  p.c0_cap = 0;
  const int ncw = nt / 32;
  const int np = env_int("VG_WS_NP", 1, 1, 2);             // producer warps
  const int kWsStages = env_int("VG_WS_STAGES", 4, 2, kWsMaxStages);
  const int64_t fixed = (2 * kWsMaxStages + 2) * 8 + (int64_t)sizeof(WsProdShared) +
                        kWsStages * (int64_t)sizeof(WsUnit) + 2 * (int64_t)kWsListCap * 16 +
                        2 * 68 * 4 + 2 * kWsMaxUnits * 8;
  const int64_t per_cand = kWsStages * (16 + 4 * (int64_t)p.stage_stride) + (int64_t)ncw * M * 8;
  const int blocks = env_int("VG_WS_CTAS", VG_WS_MINB, 1, 8);
  const int64_t budget = (int64_t)228 * 1024 / blocks - 1024 - fixed;
  int64_t cap = budget / per_cand;
  cap = cap > kListCap ? kListCap : cap;
  cap = env_int("VG_WS_CAP", (int)cap, 8, (int)cap) & ~1;   // even: keeps the layout 16-byte aligned
  if (cap < 8) return set_error(VG_ERR_INVALID, "K3W: staging rows too long");
  p.stage_cap = (int)cap;
  p.stage_floats = 0;
  const size_t smem = (size_t)(fixed + cap * per_cand);
  const int64_t n_tiles64 = d.n_molecules * (int64_t)d.C * p.tasks;
  if (n_tiles64 > INT_MAX) return set_error(VG_ERR_INVALID, "too many tiles (%lld)", (long long)n_tiles64);
  const int n_tiles = (int)n_tiles64;
  int grid = sm_count() * blocks;
  if (grid > n_tiles) grid = n_tiles;
  int* counter = tile_counter_of(d, L, ws);
  const int th = nt + 32 * np;
  if (np == 1)
    return M == 1 ? launch_ws_m<1, 1>(grid, th, smem, st, p, counter, n_tiles, kWsStages)
                  : launch_ws_m<2, 1>(grid, th, smem, st, p, counter, n_tiles, kWsStages);
  return M == 1 ? launch_ws_m<1, 2>(grid, th, smem, st, p, counter, n_tiles, kWsStages)
                : launch_ws_m<2, 2>(grid, th, smem, st, p, counter, n_tiles, kWsStages);
}

// bins_ready: K2 already ran for this workspace (vg_submit_f32 runs it on the
// tables stream); otherwise it is launched here, before K3.
int launch_slabs(const vg_batch_desc& d, const vg_ws_layout& L, char* ws, float* out,
                 vg_mol_stats* stats, cudaStream_t st, int* kernels = nullptr,
                 bool bins_ready = false, bool stats_zeroed = false, bool pipelined = false) {
  const bool aligned16 = (reinterpret_cast<uintptr_t>(out) % 16) == 0;
  SlabPlan P;
  plan_slabs(d, aligned16, &P);
  const int64_t slab = (int64_t)d.W * d.D;
  const int sw = P.sw, zw = P.zw, width = P.width, spr = P.spr;
  // hot loop over single slabs or slab pairs (8-voxel slots only)
  const int yp = sw == 8 && env_int("VG_YP", 2, 1, 2) == 2 ? 2 : 1;
  int nt = P.nt;
  const int R = P.R, M = P.M, row_blocks = P.row_blocks;

  SlabParams p;
  memset(&p, 0, sizeof p);
  p.offsets = d.offsets;
  p.tx = reinterpret_cast<const float*>(ws + L.tx);
  p.ty = reinterpret_cast<const float*>(ws + L.ty);
  p.tz = reinterpret_cast<const float*>(ws + L.tz);
  p.supp = reinterpret_cast<const int4*>(ws + L.supp);
  p.out = out;
  p.stats = stats;
  p.slab_elems = slab;
  p.rx = L.row_x;
  p.ry = L.row_y;
  p.rz = L.row_z;
  p.H = d.H;
  p.W = d.W;
  p.D = d.D;
  p.C = d.C;
  p.slots_per_row = spr;

  if (stats != nullptr && !stats_zeroed) {
    cudaError_t e = cudaMemsetAsync(stats, 0, sizeof(vg_mol_stats) * d.n_molecules, st);
    if (e != cudaSuccess) return set_error(VG_ERR_CUDA, "stats memset: %s", cudaGetErrorString(e));
  }

  if (!P.rows_ok) {
    const bool vec = P.vec;
    const int64_t nslots64 = slab / width;
    if (nslots64 > INT_MAX / 2) return set_error(VG_ERR_INVALID, "slab W*D too large");
    const int nslots = (int)nslots64;
    int m_steps = 1;
    while (m_steps < 16 && (nslots + m_steps - 1) / m_steps > 256) m_steps *= 2;
    nt = (nslots + m_steps - 1) / m_steps;
    nt = nt > 256 ? 256 : ((nt + 31) / 32) * 32;
    const int per_block = nt * m_steps;
    p.slot_blocks = (nslots + per_block - 1) / per_block;
    p.nslots = nslots;
    p.m_steps = m_steps;
    const int64_t cta_bytes = (int64_t)per_block * width * 4;
    int jc = (int)((kTaskBytes / 4 + cta_bytes - 1) / cta_bytes);
    p.jc = jc < 1 ? 1 : (jc > d.H ? d.H : jc);
    p.n_jchunks = (d.H + p.jc - 1) / p.jc;
    const int64_t tasks = d.n_molecules * d.C * (int64_t)p.n_jchunks * p.slot_blocks;
    if (tasks > INT_MAX) return set_error(VG_ERR_INVALID, "too many CTAs (%lld)", (long long)tasks);
    if (vec)
      vg_slab_generic_kernel<true><<<(unsigned)tasks, nt, 0, st>>>(p);
    else
      vg_slab_generic_kernel<false><<<(unsigned)tasks, nt, 0, st>>>(p);
    if (kernels != nullptr) *kernels += 1;
    return check_launch("vg_slab_generic_kernel");
  }

  const int z_blocks = P.z_blocks;
  const int64_t mean_atoms = P.mean_atoms;
  const bool fuse = P.fuse;
  bool after_bins = false;   // K2 launched here, K3 directly behind it
  const int jc = P.jc;
  p.jc = jc;
  p.n_jchunks = P.n_jchunks;
  if ((int64_t)p.n_jchunks * row_blocks * z_blocks > INT_MAX / 2)
    return set_error(VG_ERR_INVALID, "grid too large for the slab kernel");
  // K2: ordered per-(molecule, channel, y-chunk) candidate bins, when the
  // workspace was laid out for this plan's chunks
  if (L.bin_jc == jc && L.bin_chunks == p.n_jchunks && L.bin_jc > 0) {
    p.bins = reinterpret_cast<int*>(ws + L.bins);
    p.bin_off = reinterpret_cast<int*>(ws + L.bin_off);
    p.bin_nb = d.C * p.n_jchunks;
    if (!bins_ready) {
      const int rc = launch_bins(d, L, ws, st, kernels);
      if (rc != VG_OK) return rc;
      // K3 follows K2 on this stream: launched as its programmatic dependent
      after_bins = env_int("VG_PDL", 1, 0, 1) == 1;
    }
  }
  p.row_blocks = row_blocks;
  p.z_blocks = z_blocks;
  p.zw = zw;
  p.rows_per_step = R;
  p.zw_magic = (0x100000000ull / (unsigned long long)zw) + 1ull;
  // Windowed gx staging (open axes, one shared delta): an atom's x-support
  // is shorter than 2*t_sat/(delta*s) + 3 edges (fp32 edge arguments differ
  // from the exact line by < 1e-6 near +-t_sat), so a candidate's gx window
  // needs support + 2 warp spans + 3 (alignment) rows instead of the tile.
  p.gx_wmax = 31 / zw + 2;
  p.gx_win = 0;
  if (!d.periodic && d.mol_delta == nullptr) {
    const double span = 2.0001 * (double)VG_TSAT / (d.scale * d.delta[0]);
    if (span < 4096.0) {
      const int bound = (int)span + 3;
      const int win = round_up4(bound + 2 * p.gx_wmax + 1);
      if (win < round_up4(M * R) && M * R <= 255) p.gx_win = win;
    }
  }
  if (env_int("VG_GXWIN", 1, 0, 1) == 0) p.gx_win = 0;
  // bulk staging (cp.async.bulk + mbarrier): 16-byte table rows and z windows
  p.bulk = sw >= 4 && (zw * sw) % 4 == 0 && env_int("VG_BULK", 1, 0, 1) == 1 ? 1 : 0;
  // Binned per-channel batches (large molecules): the persistent,
  // warp-specialised K3W when its alignment rules hold (8-voxel slots and
  // slab pairs, even y-chunks so every unit starts on an even slab, 16-byte
  // aligned x rows for the bulk copies). VG_WS=0 keeps vg_slab_kernel.
  if (p.bins != nullptr && !fuse && sw == 8 && yp == 2 && M <= 2 && jc % 2 == 0 &&
      (M * R) % 4 == 0 && nt <= kWsThreads && env_int("VG_WS", 0, 0, 1) == 1) {
    // VG_WS_M=2: two row steps per tile (twice the rows per producer pass)
    int Mw = M, rbw = row_blocks;
    if (M == 1 && env_int("VG_WS_M", 1, 1, 2) == 2 && 2 * R <= 255) {
      Mw = 2;
      rbw = (d.W + 2 * R - 1) / (2 * R);
    }
    p.row_blocks = rbw;
    p.z_blocks = z_blocks;
    p.cta_order = 0;
    p.tasks = p.n_jchunks * rbw * z_blocks;
    p.n_molecules = (int)d.n_molecules;
    if (p.gx_win > 0 && !(p.gx_win < round_up4(Mw * R))) p.gx_win = 0;
    const int rc = launch_ws(d, L, ws, p, Mw, R, nt, jc, st);
    if (rc == VG_OK && kernels != nullptr) *kernels += 1;
    return rc;
  }
  // staged block per candidate: gy[pad4(jc)] gx[window or pad4(M*R)] gz[pad4(zw*width)]
  p.stage_gx = (jc + 3) & ~3;
  p.stage_gz = p.stage_gx + (p.gx_win > 0 ? p.gx_win : round_up4(M * R));
  p.stage_stride = p.stage_gz + round_up4(zw * width);
  // Level-0 list: only for large molecules scanned without bins (it is used
  // when a molecule has more than 2*blockDim atoms); with K2 bins the CTA's
  // bin is its candidate source. Capacity in ints, 16-byte aligned.
  p.c0_cap = p.bins != nullptr ? 0 : (mean_atoms > 64 ? kC0CapMax : 256);
  p.c0_cap = round_up4(env_int("VG_C0", p.c0_cap, 0, kC0CapMax));   // keeps staging 16-byte aligned
  // Staging capacity: what the batch's molecules need (about 2x the mean atom
  // count, at most kListCap), within the shared memory that keeps the
  // register-limited number of CTAs resident per SM (228 KB per SM, 1 KB
  // reserved per CTA): the occupancy cliff costs more than extra halving.
  int cap_max = kListCap;
  cap_max = env_int("VG_CAP_MAX", cap_max, 1, kListCap);
  const int64_t want_x = env_int("VG_WANT_X", 2, 1, 16);   // hook: capacity aim, x mean atoms
  const int want = (int)(mean_atoms * want_x < 32 ? 32 : (mean_atoms * want_x > cap_max ? cap_max : mean_atoms * want_x));
  const int regs = (rows_regs(sw, yp, M) + 7) & ~7;   // allocation granularity
  const int reg_blocks = max(1, min(2048 / nt, 65536 / (regs * nt)));
  const int64_t per_cand = 4 * (int64_t)p.stage_stride + (int64_t)(nt / 32) * M * sizeof(int2);
  auto cap_at = [&](int blocks) {
    const int64_t budget = (int64_t)228 * 1024 / blocks - 1024 - (int64_t)sizeof(SlabShared) -
                           (int64_t)(kListCap + nt) * 16 - (int64_t)p.c0_cap * 4 -
                           (int64_t)(M * R + 8 + 3) * 4;
    return budget / per_cand;
  };
  // With 5 or more CTAs per SM, one CTA fewer is worth it when it lifts the
  // capacity towards what the molecules need (cfg4: 76 -> 105 candidates,
  // fewer channel-fused CTAs falling back to per-channel passes; measured
  // 2% faster). At 4 CTAs/SM the occupancy loss costs more (cfg3: 7% slower).
  int blocks = reg_blocks;
  if (cap_at(blocks) < want && blocks >= 5) --blocks;
  blocks = env_int("VG_CTA_SM", blocks, 1, reg_blocks);   // hook: budget for fewer CTAs/SM
  int64_t cap = cap_at(blocks);
  if (cap > want) cap = want;
  p.stage_cap = cap < 1 ? 1 : (int)cap;
  // slack: rows >= W of the last step read (and discard) past the last block;
  // then the warp-private sublists (int2 per candidate, row step and warp)
  p.stage_floats = (p.stage_cap * p.stage_stride + M * R + 8 + 3) & ~3;
  const size_t smem = (size_t)(kListCap + nt) * sizeof(int4) + (size_t)p.c0_cap * sizeof(int) +
                      (size_t)p.stage_floats * sizeof(float) +
                      (size_t)(nt / 32) * M * p.stage_cap * sizeof(int2);
  p.fuse_channels = fuse ? 1 : 0;
  p.cta_order = env_int("VG_ORDER", 0, 0, 1);
  p.tasks = p.n_jchunks * row_blocks * z_blocks;
  p.n_molecules = (int)d.n_molecules;
  int64_t ctas = d.n_molecules * (fuse ? 1 : (int64_t)d.C) * p.tasks;
  // Tapered tail (channel-fused launches of several waves): a launch ends when
  // its last CTA does, and CTAs of ~1 MiB finish up to one CTA time (~40 us at
  // cfg1) apart. The last molecules - about half a wave of full-size CTAs
  // (VG_TAPER_Q quarter waves) - are cut into y-chunks a quarter as long
  // (VG_TAPER_D; a multiple of 4 slabs, so their tables still stage by bulk
  // copies): the SMs then finish within a short CTA's time of one another.
  // Measured on B200: cfg1 K3 0.759 -> 0.751 ms, cfg4 1.4645 -> 1.4463; longer
  // tails or other divisors are within 0.2%. Results do not depend on the tiling.
  p.taper_lin = 0xffffffffu;
  p.taper_b = 0;
  p.tasks2 = p.tasks;
  p.jc2 = jc;
  // (vg_submit_f32 runs consecutive batches' K3s on different streams: the next
  // K3 fills this one's tail, and the short CTAs would only add their overhead:
  // cfg1 pipelined 1.3535 M -> 1.3483 M grids/s with the taper, so it is off there)
  const int taper = env_int("VG_TAPER", pipelined ? 0 : 1, 0, 2);   // hook: 0 off, 2 forced
  if (fuse && taper > 0) {
    const int64_t slots = (int64_t)sm_count() * blocks;
    int jc2 = ((jc / env_int("VG_TAPER_D", 4, 2, 16) + 3) / 4) * 4;
    if (jc2 < 4) jc2 = 4;
    const int nch2 = (d.H + jc2 - 1) / jc2;
    int64_t tail_mols = (env_int("VG_TAPER_Q", 2, 1, 16) * slots / 4 + p.tasks - 1) / p.tasks;
    if (taper == 2) tail_mols = d.n_molecules / 3 > 0 ? d.n_molecules / 3 : 1;
    if (jc2 * 2 <= jc && (ctas >= 4 * slots || taper == 2) && tail_mols < d.n_molecules) {
      p.jc2 = jc2;
      p.tasks2 = nch2 * row_blocks * z_blocks;
      p.taper_b = (int)(d.n_molecules - tail_mols);
      const int64_t head = (int64_t)p.taper_b * p.tasks;
      ctas = head + tail_mols * p.tasks2;
      if (head < 0xffffffffll) p.taper_lin = (unsigned)head;
    }
  }
  if (ctas > INT_MAX) return set_error(VG_ERR_INVALID, "too many CTAs (%lld)", (long long)ctas);
  if (env_int("VG_DEBUG_PLAN", 0, 0, 1) == 1)   // test hook: the launch plan on stderr
    fprintf(stderr,
            "[vg plan] nt=%d M=%d R=%d rb=%d zb=%d jc=%d chunks=%d fuse=%d cap=%d bulk=%d ctas=%lld "
            "taper_b=%d jc2=%d tasks2=%d bins=%d\n",
            nt, M, R, row_blocks, z_blocks, jc, p.n_jchunks, (int)fuse, p.stage_cap, p.bulk,
            (long long)ctas, p.taper_lin == 0xffffffffu ? -1 : p.taper_b, p.jc2, p.tasks2,
            p.bins != nullptr);
  const dim3 grid((unsigned)ctas);
  int rc;
  const bool pdl_saved = g_pdl_launch;
  g_pdl_launch = g_pdl_launch || after_bins;
  if (sw == 8 && yp == 2)
    rc = launch_rows<8, 2>(M, grid, nt, smem, st, p);
  else if (sw == 8)
    rc = launch_rows<8, 1>(M, grid, nt, smem, st, p);
  else if (sw == 4)
    rc = launch_rows<4, 1>(M, grid, nt, smem, st, p);
  else
    rc = launch_rows<1, 1>(M, grid, nt, smem, st, p);
  g_pdl_launch = pdl_saved;
  if (rc != VG_OK) return rc;
  if (kernels != nullptr) *kernels += 1;
  return check_launch("vg_slab_kernel");
}

int prepare(const vg_batch_desc* desc, float* out, void* workspace, size_t workspace_bytes,
            vg_ws_layout* L) {
  g_last_error[0] = '\0';
  int rc = validate(desc);
  if (rc != VG_OK) return rc;
  if (desc->n_molecules > 0 && out == nullptr) return set_error(VG_ERR_INVALID, "out is NULL");
  fill_layout(desc, L);
  if (workspace == nullptr || workspace_bytes < L->total)
    return set_error(VG_ERR_WORKSPACE, "workspace needs %zu bytes, got %zu", L->total,
                     workspace_bytes);
  // the table rows are staged with 16-byte copies (cp.async / cp.async.bulk)
  if (reinterpret_cast<uintptr_t>(workspace) % 16 != 0)
    return set_error(VG_ERR_INVALID, "workspace must be 16-byte aligned");
  return VG_OK;
}

}  // namespace

VG_API int vg_generate_f32(const vg_batch_desc* desc, float* out, void* workspace,
                           size_t workspace_bytes, vg_mol_stats* stats, void* stream) {
  vgdev::DeviceGuard guard(out);
  vg_ws_layout L;
  int rc = prepare(desc, out, workspace, workspace_bytes, &L);
  if (rc != VG_OK || desc->n_molecules == 0) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // small batches: tables and gather in one launch (K13, vg_small.cu)
  rc = vg_small_try(desc, out, stats, st, false, false);
  if (rc < 0) return rc;
  if (rc == 1) return VG_OK;
  char* ws = static_cast<char*>(workspace);
  // counters zeroed before K1, so that K3 directly follows K1 on the stream
  // and can be launched as its programmatic dependent
  if (stats != nullptr) {
    const cudaError_t e = cudaMemsetAsync(stats, 0, sizeof(vg_mol_stats) * desc->n_molecules, st);
    if (e != cudaSuccess) return set_error(VG_ERR_CUDA, "stats memset: %s", cudaGetErrorString(e));
  }
  rc = launch_tables(desc, L, ws, st);
  if (rc != VG_OK) return rc;
  g_pdl_launch = desc->n_atoms > 0 && env_int("VG_PDL", 1, 0, 1) == 1;
  rc = launch_slabs(*desc, L, ws, out, stats, st, nullptr, false, true);
  g_pdl_launch = false;
  return rc;
}

VG_API int vg_fused_small(const vg_batch_desc* desc, const float* out) {
  g_last_error[0] = '\0';
  const int rc = validate(desc);
  if (rc != VG_OK) return rc;
  return vg_small_try(desc, const_cast<float*>(out), nullptr, nullptr, true, true) == 1 ? 1 : 0;
}

VG_API int vg_slabs_f32(const vg_batch_desc* desc, float* out, void* workspace,
                        size_t workspace_bytes, vg_mol_stats* stats, void* stream) {
  vgdev::DeviceGuard guard(out);
  vg_ws_layout L;
  int rc = prepare(desc, out, workspace, workspace_bytes, &L);
  if (rc != VG_OK || desc->n_molecules == 0) return rc;
  return launch_slabs(*desc, L, static_cast<char*>(workspace), out, stats,
                      static_cast<cudaStream_t>(stream));
}

VG_API int vg_submit_f32(const vg_batch_desc* desc, const vg_submit_args* a, float* out,
                         void* workspace, size_t workspace_bytes, vg_mol_stats* stats) {
  if (a == nullptr) return set_error(VG_ERR_INVALID, "submit args are NULL");
  vgdev::DeviceGuard guard(out);
  vg_ws_layout L;
  int rc = prepare(desc, out, workspace, workspace_bytes, &L);
  if (rc == VG_ERR_WORKSPACE && a->ws_needed != nullptr) *a->ws_needed = L.total;
  if (rc != VG_OK) return rc;
  cudaStream_t cs = static_cast<cudaStream_t>(a->copy_stream);
  cudaStream_t ts = static_cast<cudaStream_t>(a->tables_stream);
  cudaStream_t ks = static_cast<cudaStream_t>(a->compute_stream);
  cudaEvent_t ev_wait = static_cast<cudaEvent_t>(a->ev_wait);
  cudaEvent_t ev_copied = static_cast<cudaEvent_t>(a->ev_copied);
  cudaEvent_t ev_tabled = static_cast<cudaEvent_t>(a->ev_tabled);
  cudaEvent_t ev_done = static_cast<cudaEvent_t>(a->ev_done);
  if (ev_copied == nullptr || ev_tabled == nullptr || ev_done == nullptr)
    return set_error(VG_ERR_INVALID, "submit events must be non-NULL");
  const int64_t B = desc->n_molecules, n = desc->n_atoms;
  cudaError_t e = cudaSuccess;
  auto ok = [&](cudaError_t r) {
    if (e == cudaSuccess) e = r;
    return e == cudaSuccess;
  };
  // slot reuse: the copy stage waits for the slot's previous consumer; K1
  // and K3 follow it through ev_copied / ev_tabled, so they are ordered
  // after that consumer too
  if (ev_wait != nullptr) ok(cudaStreamWaitEvent(cs, ev_wait, 0));
  // One H2D when the three host arrays sit in one block with the same
  // relative layout as their device destinations (GridPipeline.staging):
  // offsets first, then xyz and channels in either order, no overlap.
  const char* ho = static_cast<const char*>(a->h_offsets);
  const char* hx = static_cast<const char*>(a->h_xyz);
  const char* hc = static_cast<const char*>(a->h_channel);
  const char* dof = reinterpret_cast<const char*>(desc->offsets);
  const char* dx = reinterpret_cast<const char*>(desc->xyz);
  const char* dc = reinterpret_cast<const char*>(desc->channel);
  const int64_t ob = (B + 1) * 8, xb = n * 24, cb = n * 4;
  const bool one_block = B > 0 && n > 0 && ho != nullptr && hx != nullptr && hc != nullptr &&
                         hx - ho == dx - dof && hc - ho == dc - dof && hx - ho >= ob &&
                         hc - ho >= ob && (hc - hx >= xb || hx - hc >= cb);
  if (one_block) {
    const int64_t xe = (hx - ho) + xb, ce = (hc - ho) + cb;
    const int64_t span = xe > ce ? xe : ce;
    ok(cudaMemcpyAsync(const_cast<char*>(dof), ho, (size_t)span, cudaMemcpyHostToDevice, cs));
  } else {
    if (a->h_offsets != nullptr && B > 0)
      ok(cudaMemcpyAsync(const_cast<int64_t*>(desc->offsets), a->h_offsets, (size_t)ob,
                         cudaMemcpyHostToDevice, cs));
    if (n > 0 && a->h_channel != nullptr)
      ok(cudaMemcpyAsync(const_cast<int32_t*>(desc->channel), a->h_channel, (size_t)cb,
                         cudaMemcpyHostToDevice, cs));
    if (n > 0 && a->h_xyz != nullptr)
      ok(cudaMemcpyAsync(const_cast<double*>(desc->xyz), a->h_xyz, (size_t)xb,
                         cudaMemcpyHostToDevice, cs));
  }
  ok(cudaEventRecord(ev_copied, cs));
  ok(cudaStreamWaitEvent(ts, ev_copied, 0));
  if (e != cudaSuccess) return set_error(VG_ERR_CUDA, "submit (copy stage): %s", cudaGetErrorString(e));
  char* ws = static_cast<char*>(workspace);
  int kernels = 0;
  bool bins_ready = false;
  // small batches run K13 (tables + gather in one kernel) on the compute stream
  const bool small = B > 0 && vg_small_try(desc, out, stats, ks, true, true) == 1;
  if (B > 0 && n > 0 && !small) {
    rc = launch_tables(desc, L, ws, ts);
    if (rc != VG_OK) return rc;
    kernels = 1;
    if (L.bin_jc > 0) {   // K2 beside the previous batch's K3 too
      rc = launch_bins(*desc, L, ws, ts, &kernels);
      if (rc != VG_OK) return rc;
      bins_ready = true;
    }
  }
  // the counters K3 accumulates start from zero: cleared here, beside the
  // previous K3, so consecutive K3s run back to back on the compute stream
  const bool stats_zeroed = B > 0 && stats != nullptr;
  if (stats_zeroed) ok(cudaMemsetAsync(stats, 0, sizeof(vg_mol_stats) * (size_t)B, ts));
  ok(cudaEventRecord(ev_tabled, ts));
  ok(cudaStreamWaitEvent(ks, ev_tabled, 0));
  if (e != cudaSuccess) return set_error(VG_ERR_CUDA, "submit (tables stage): %s", cudaGetErrorString(e));
  if (small) {
    rc = vg_small_try(desc, out, stats, ks, stats_zeroed, false);
    if (rc < 0) return rc;
    kernels += 1;
  } else if (B > 0) {
    rc = launch_slabs(*desc, L, ws, out, stats, ks, &kernels, bins_ready, stats_zeroed, true);
    if (rc != VG_OK) return rc;
  }
  const bool readback = B > 0 && a->h_stats != nullptr && stats != nullptr;
  cudaStream_t rs = static_cast<cudaStream_t>(a->readback_stream);
  cudaEvent_t ev_read = static_cast<cudaEvent_t>(a->ev_read);
  const bool side = readback && rs != nullptr && ev_read != nullptr;
  if (readback && !side)
    ok(cudaMemcpyAsync(a->h_stats, stats, (size_t)B * sizeof(vg_mol_stats), cudaMemcpyDeviceToHost,
                       ks));
  ok(cudaEventRecord(ev_done, ks));
  if (side) {   // the read-back beside the next batch's K3
    ok(cudaStreamWaitEvent(rs, ev_done, 0));
    ok(cudaMemcpyAsync(a->h_stats, stats, (size_t)B * sizeof(vg_mol_stats), cudaMemcpyDeviceToHost,
                       rs));
    ok(cudaEventRecord(ev_read, rs));
  }
  if (e != cudaSuccess) return set_error(VG_ERR_CUDA, "submit (compute stage): %s", cudaGetErrorString(e));
  if (a->kernels != nullptr) *a->kernels = kernels;
  return VG_OK;
}

VG_API int vg_erf_f32(const float* t, float* out, int64_t n, void* stream) {
  g_last_error[0] = '\0';
  if (n < 0) return set_error(VG_ERR_INVALID, "negative length");
  if (n == 0) return VG_OK;
  if (t == nullptr || out == nullptr) return set_error(VG_ERR_INVALID, "NULL pointer");
  vgdev::DeviceGuard guard(out);
  const int64_t blocks64 = (n + 255) / 256;
  const unsigned blocks = (unsigned)(blocks64 > 148 * 64 ? 148 * 64 : blocks64);
  vg_erf_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(t, out, n);
  return check_launch("vg_erf_kernel");
}

VG_API int vg_fill_f32(float* out, int64_t n, float value, void* stream) {
  g_last_error[0] = '\0';
  if (n < 0) return set_error(VG_ERR_INVALID, "negative length");
  if (n == 0) return VG_OK;
  if (out == nullptr || (reinterpret_cast<uintptr_t>(out) % 16) != 0)
    return set_error(VG_ERR_INVALID, "out must be non-NULL and 16-byte aligned");
  vgdev::DeviceGuard guard(out);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n4 = n / 4;
  if (n4 > 0) {
    const int64_t blocks = (n4 + 1023) / 1024;
    if (blocks > INT_MAX) return set_error(VG_ERR_INVALID, "fill too large");
    vg_fill_kernel<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<float4*>(out), n4,
                                                      make_float4(value, value, value, value));
  }
  const int64_t tail = n - n4 * 4;
  if (tail > 0) vg_fill_tail_kernel<<<1, 32, 0, st>>>(out + n4 * 4, tail, value);
  return check_launch("vg_fill_kernel");
}

#ifdef VG_EXP_TIMING
VG_API int vg_exp_timing_fetch_warps(void* host, size_t bytes) {
  return cudaMemcpyFromSymbol(host, g_vg_ts_w, bytes < sizeof(g_vg_ts_w) ? bytes : sizeof(g_vg_ts_w)) ==
                 cudaSuccess ? VG_OK : VG_ERR_CUDA;
}

VG_API int vg_exp_timing_fetch(void* host, size_t bytes) {
  return cudaMemcpyFromSymbol(host, g_vg_ts, bytes < sizeof(g_vg_ts) ? bytes : sizeof(g_vg_ts)) ==
                 cudaSuccess ? VG_OK : VG_ERR_CUDA;
}
#endif

#ifdef VG_EXP_WSPROF
VG_API int vg_exp_wsprof(void* host, int reset) {
  unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (host != nullptr && cudaMemcpyFromSymbol(host, g_ws_prof, sizeof z) != cudaSuccess) return VG_ERR_CUDA;
  if (reset && cudaMemcpyToSymbol(g_ws_prof, z, sizeof z) != cudaSuccess) return VG_ERR_CUDA;
  return VG_OK;
}
#endif

VG_API int vg_exp_f32_host(const float* x, float* out, size_t n) {
  if (n > 0 && (x == nullptr || out == nullptr)) return set_error(VG_ERR_INVALID, "NULL pointer");
  for (size_t i = 0; i < n; ++i) out[i] = vg_exp_f32(x[i]);
  return VG_OK;
}

VG_API int vg_erf_sat_f32_host(const float* t, float* out, size_t n) {
  if (n > 0 && (t == nullptr || out == nullptr)) return set_error(VG_ERR_INVALID, "NULL pointer");
  for (size_t i = 0; i < n; ++i) out[i] = vg_erf_sat_f32(t[i]);
  return VG_OK;
}

VG_API int vg_erf_f32_host(const float* t, float* out, size_t n) {
  if (n > 0 && (t == nullptr || out == nullptr)) return set_error(VG_ERR_INVALID, "NULL pointer");
  for (size_t i = 0; i < n; ++i) out[i] = vg_erf_f32(t[i]);
  return VG_OK;
}
