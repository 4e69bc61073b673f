// vg_small.cu — K13: one launch for a small batch (tables + gather fused).
//
// A small batch (BASELINE configs[0]: 64 molecules of 9-29 atoms, 32^3 x 5
// channels, 42 MB) is latency-bound on the two-kernel path: K1 (per-atom axis
// tables into the workspace) and K3 (gather/store) each take a few launch and
// CTA latencies for microseconds of work, and K3 cannot start before K1 ends.
// K13 does both in one kernel: each CTA owns a y-chunk of one (molecule,
// channel) grid, builds the axis tables of that channel's atoms in shared
// memory (the K1 numerics: fp64 edge arguments, saturated Bürmann erf,
// 0.5*(E(e+1)-E(e)), threshold), then accumulates its voxels over those atoms
// in ascending atom order and writes every voxel once with streaming 128-bit
// stores. Reference: fused_axis_tables kernels.py:217-274 (tables),
// splat_atom gridgen.py:97-109 + generate_grid gridgen.py:130-153
// (accumulation, count_nonzero), GenStats gridgen.py:39-54.
//
// Bits equal the two-kernel path:
//   * every table value is evaluated as K1 does (K1 skips the series outside
//     the unsaturated window, where both E are the same +-1 and the mass is
//     0.5*(E-E) = +0 — the series gives exactly that value too);
//   * per voxel the terms fl(fl(gy*gx)*gz) are added in ascending atom order;
//     K3 and K13 skip atoms whose x/y support misses the voxels of a warp:
//     such terms are +-0, and acc + (+-0) == acc;
//   * atoms the reference rejects (channel outside [0, C), non-finite
//     coordinate) never contribute and flag their molecule (sign bit of
//     voxel_writes), as K1/K3 do.
// Periodic grids keep the two-kernel path (three images per edge).

#include <cuda_runtime.h>

#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/voxgrid_b200.h"
#include "vg_device.cuh"
#include "vg_math.cuh"

extern "C" int vg_internal_set_error(int code, const char* msg);

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kThreads = 256;
// Measured on B200 (profiles/r2_k13_small_batches.txt): one launch beats
// K1 + K3 (K3 launched as K1's programmatic dependent) for a few small grids
// (12.3 vs 15.2 us for one 32^3 x 5 molecule); from ~16 grids the two-kernel
// path is faster (21.3 vs 22.5 us; 25.4 vs 38.9 us at cfg0's 64), its per-CTA
// chain being shorter than K13's.
constexpr int64_t kMaxBytes = 4ll << 20;         // batches up to 4 MiB of output
constexpr int kMaxMeanAtoms = 64;                // small molecules only
constexpr int kSmemBudget = 46 * 1024;           // dynamic smem per CTA (no opt-in)
constexpr int kMaxCap = 64;                      // candidates per pass

struct SmallParams {
  const int64_t* offsets;
  const double* xyz;
  const int32_t* channel;
  const double* mol_origin;
  const double* mol_delta;
  float* out;
  vg_mol_stats* stats;
  double origin[3];
  double delta[3];
  double scale;
  int H, W, D, C;
  int jc, n_jchunks;
  int rx, ry, rz;      // table rows in shared memory (floats, multiples of 4)
  int cap;             // candidates per pass
  float threshold;
  int has_threshold;
};

__device__ __forceinline__ float mass(double rel, double d, int e, double s, const SmallParams& p) {
  // kernels.py:252-262: g_e = fl32(0.5 * (E(t_{e+1}) - E(t_e))), t in fp64 -> fp32
  const float lo = vg_erf_sat_f32(vg_edge_arg(rel, d, e, s));
  const float hi = vg_erf_sat_f32(vg_edge_arg(rel, d, e + 1, s));
  float g = VG_FMUL(0.5f, VG_FSUB(hi, lo));
  if (p.has_threshold && !(g >= p.threshold)) g = 0.0f;  // kernels.py:271-272
  return g;
}

__device__ __forceinline__ bool finite3(const double* x) {
  return isfinite(x[0]) && isfinite(x[1]) && isfinite(x[2]);
}

__device__ __forceinline__ int lo16(int v) { return v & 0xffff; }
__device__ __forceinline__ int hi16(int v) { return (int)((unsigned)v >> 16); }

// First / last+1 nonzero of a shared table row, by one warp, as lo | hi << 16
// ((0, 0) if none: _support_of, kernels.py:147-151).
__device__ __forceinline__ int row_support(const float* row, int n) {
  int lo = -1, hi = 0;
  for (int c0 = 0; c0 < n; c0 += 32) {
    const int e = c0 + (threadIdx.x & 31);
    const unsigned nz = __ballot_sync(kFull, e < n && row[e] != 0.0f);
    if (nz != 0u) {
      if (lo < 0) lo = c0 + __ffs(nz) - 1;
      hi = c0 + 32 - __clz(nz);
    }
  }
  return lo < 0 ? 0 : (lo | (hi << 16));
}

template <int K>
__global__ void __launch_bounds__(kThreads) vg_small_kernel(const __grid_constant__ SmallParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int warp_cnt[kThreads / 32];
  __shared__ long long s_next;
  int* cand = reinterpret_cast<int*>(smem);
  float* tx = reinterpret_cast<float*>(smem + ((p.cap * 4 + 15) & ~15));
  float* ty = tx + p.cap * p.rx;
  float* tz = ty + p.cap * p.ry;
  float* ebuf = tz + p.cap * p.rz;     // E(t_e) at every edge of every candidate row
  int* sxy = reinterpret_cast<int*>(ebuf + p.cap * (p.W + p.H + p.D + 3));   // x, y supports

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned cta = blockIdx.x;
  const int split = (int)(cta % (unsigned)p.n_jchunks);
  cta /= (unsigned)p.n_jchunks;
  const int c = (int)(cta % (unsigned)p.C);
  const int64_t b = cta / (unsigned)p.C;
  const int64_t a0 = __ldg(p.offsets + b), a1 = __ldg(p.offsets + b + 1);
  const int j0 = split * p.jc;
  const int nj = min(p.jc, p.H - j0);
  const int D4 = p.D >> 2;
  const int plane = p.W * D4;            // float4 slots per y row of the grid
  const int nslots = nj * plane;         // this CTA's slots, in groups of K * kThreads
  const double s = p.scale;
  double o[3], dl[3];
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    o[ax] = p.mol_origin != nullptr ? p.mol_origin[b * 3 + ax] : p.origin[ax];
    dl[ax] = p.mol_delta != nullptr ? p.mol_delta[b * 3 + ax] : p.delta[ax];
  }
  float4* dst = reinterpret_cast<float4*>(
      p.out + (((b * p.C + c) * (int64_t)p.H + j0) * p.W) * (int64_t)p.D);
  const int ne = p.W + p.H + p.D + 3;    // edges per candidate (x, y, z)
  long long writes = 0;                  // voxel_writes of this channel's atoms (split 0)
  int nz = 0;
  bool first = true;
  int64_t pos = a0;
  for (;;) {
    // ordered compaction: the next <= cap atoms of channel c with finite
    // coordinates, ascending (input order = accumulation order)
    int count = 0;
    while (pos < a1 && count < p.cap) {
      const int64_t a = pos + tid;
      bool keep = false;
      if (a < a1) keep = __ldg(p.channel + a) == c && finite3(p.xyz + a * 3);
      const unsigned bal = __ballot_sync(kFull, keep);
      if (lane == 0) warp_cnt[warp] = __popc(bal);
      __syncthreads();
      int before = 0, total = 0;
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) {
        const int v = warp_cnt[w];
        before += w < warp ? v : 0;
        total += v;
      }
      const int rank = before + __popc(bal & ((1u << lane) - 1u));
      const int room = p.cap - count;
      if (keep && rank < room) cand[count + rank] = (int)a;
      if (total > room) {
        if (keep && rank == room - 1) s_next = a + 1;
        __syncthreads();
        pos = s_next;
        count = p.cap;
      } else {
        count += total;
        pos += kThreads;
      }
      __syncthreads();
    }
    const bool last = pos >= a1;

    if (count > 0) {
      // E(t_e) once per edge of every candidate row (K1 numerics): fp64 edge
      // arguments (kernels.py:252-254) through the saturated erf
      for (int idx = tid; idx < count * ne; idx += kThreads) {
        const int q = idx / ne;
        int e = idx - q * ne, ax;
        if (e <= p.W) {
          ax = 0;
        } else if (e <= p.W + 1 + p.H) {
          ax = 1;
          e -= p.W + 1;
        } else {
          ax = 2;
          e -= p.W + p.H + 2;
        }
        // (register selects, not a dynamically indexed local array)
        const double oa = ax == 0 ? o[0] : (ax == 1 ? o[1] : o[2]);
        const double da = ax == 0 ? dl[0] : (ax == 1 ? dl[1] : dl[2]);
        const double rel = __dsub_rn(oa, __ldg(p.xyz + (int64_t)cand[q] * 3 + ax));
        ebuf[idx] = vg_erf_sat_f32(vg_edge_arg(rel, da, e, s));
      }
      __syncthreads();
      // masses g_e = fl32(0.5 * (E(e+1) - E(e))) (kernels.py:260), threshold (:271-272)
      for (int idx = tid; idx < count * (ne - 3); idx += kThreads) {
        const int q = idx / (ne - 3);
        int e = idx - q * (ne - 3);
        float* row;
        int eo;   // offset of the row's first edge in ebuf
        if (e < p.W) {
          row = tx + q * p.rx;
          eo = q * ne;
        } else if (e < p.W + p.H) {
          e -= p.W;
          row = ty + q * p.ry;
          eo = q * ne + p.W + 1;
        } else {
          e -= p.W + p.H;
          row = tz + q * p.rz;
          eo = q * ne + p.W + p.H + 2;
        }
        float g = VG_FMUL(0.5f, VG_FSUB(ebuf[eo + e + 1], ebuf[eo + e]));
        if (p.has_threshold && !(g >= p.threshold)) g = 0.0f;
        row[e] = g;
      }
      __syncthreads();
      // supports (first / last+1 nonzero, kernels.py:147-151): x and y for
      // the warp-level culling below, the volume for voxel_writes
      // (gridgen.py:103, from split 0)
      for (int q = warp; q < count; q += kThreads / 32) {
        const int ex = row_support(tx + q * p.rx, p.W);
        const int ey = row_support(ty + q * p.ry, p.H);
        if (lane == 0) {
          sxy[2 * q] = ex;
          sxy[2 * q + 1] = ey;
        }
        if (split == 0 && p.stats != nullptr) {
          const int ez = row_support(tz + q * p.rz, p.D);
          if (lane == 0)
            writes += (long long)(hi16(ex) - lo16(ex)) * (hi16(ey) - lo16(ey)) *
                      (hi16(ez) - lo16(ez));
        }
      }
      __syncthreads();
    }

    // the CTA's voxels, K float4 slots per thread at a time: start from
    // zero (first pass) or from this thread's own earlier stores, add this
    // pass's candidates in ascending atom order, store
    if (first || count > 0 || last) {
      for (int g0 = 0; g0 < nslots; g0 += K * kThreads) {
        int sj[K], si[K], sz[K];
        float4 acc[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int slot = g0 + tid + k * kThreads;
          const int j = slot / plane;
          const int r = slot - j * plane;
          si[k] = r / D4;
          sz[k] = r - si[k] * D4;
          sj[k] = slot < nslots ? j0 + j : -1;
          acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (!first && sj[k] >= 0) acc[k] = dst[slot];
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
          // the warp's rows and x rows for slot k; a candidate whose support
          // misses them adds only +-0 terms there and is skipped (warp-uniform)
          const bool valid = sj[k] >= 0;
          const int jmin = __reduce_min_sync(kFull, valid ? sj[k] : INT_MAX);
          const int jmax = __reduce_max_sync(kFull, valid ? sj[k] : -1);
          const int imin = __reduce_min_sync(kFull, valid ? si[k] : INT_MAX);
          const int imax = __reduce_max_sync(kFull, valid ? si[k] : -1);
          const int yk = valid ? sj[k] : 0, xk = si[k], zk = sz[k];
          for (int c0 = 0; c0 < count; c0 += 32) {
            const int q = c0 + lane;
            bool hit = false;
            if (q < count) {
              const int ex = sxy[2 * q], ey = sxy[2 * q + 1];
              hit = lo16(ey) <= jmax && hi16(ey) > jmin && lo16(ex) <= imax && hi16(ex) > imin;
            }
            unsigned m = __ballot_sync(kFull, hit);
            while (m != 0u) {   // ascending candidates = ascending atom order
              const int qq = c0 + __ffs(m) - 1;
              m &= m - 1u;
              const float pyx = VG_FMUL(ty[qq * p.ry + yk], tx[qq * p.rx + xk]);  // ty (x) tx
              const float4 gz = reinterpret_cast<const float4*>(tz + qq * p.rz)[zk];
              acc[k].x = VG_FADD(acc[k].x, VG_FMUL(pyx, gz.x));   // (..) (x) tz, +=
              acc[k].y = VG_FADD(acc[k].y, VG_FMUL(pyx, gz.y));
              acc[k].z = VG_FADD(acc[k].z, VG_FMUL(pyx, gz.z));
              acc[k].w = VG_FADD(acc[k].w, VG_FMUL(pyx, gz.w));
            }
          }
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
          if (sj[k] >= 0) {
            if (first || count > 0) __stcs(dst + g0 + tid + k * kThreads, acc[k]);
            if (last)
              nz += (acc[k].x != 0.f) + (acc[k].y != 0.f) + (acc[k].z != 0.f) + (acc[k].w != 0.f);
          }
        }
      }
    }
    first = false;
    if (last) break;
    __syncthreads();   // tables are rewritten by the next pass
  }

  if (p.stats == nullptr) return;
  long long tot = nz;
  for (int off = 16; off > 0; off >>= 1) tot += __shfl_down_sync(kFull, tot, off);
  if (lane == 0 && tot != 0)
    atomicAdd(reinterpret_cast<unsigned long long*>(&p.stats[b].nonzero_voxels),
              (unsigned long long)tot);
  if (split == 0) {
    if (lane == 0 && writes != 0)
      atomicAdd(reinterpret_cast<unsigned long long*>(&p.stats[b].voxel_writes),
                (unsigned long long)writes);
    if (c == 0) {
      // atoms the reference rejects flag the molecule (gridgen.py:86-90)
      bool bad = false;
      for (int64_t a = a0 + tid; a < a1; a += kThreads) {
        const int ch = __ldg(p.channel + a);
        bad = bad || (unsigned)ch >= (unsigned)p.C || !finite3(p.xyz + a * 3);
      }
      if (__any_sync(kFull, bad) && lane == 0)
        atomicOr(reinterpret_cast<unsigned long long*>(&p.stats[b].voxel_writes), 1ull << 63);
    }
  }
}

int env_small(const char* name, int dflt) {
  const char* v = getenv(name);
  if (v == nullptr || *v == '\0') return dflt;
  char* end = nullptr;
  const long x = strtol(v, &end, 10);
  return *end == '\0' ? (int)x : dflt;
}

template <int K>
cudaError_t launch_k(unsigned grid, size_t smem, cudaStream_t st, const SmallParams& p) {
  vg_small_kernel<K><<<grid, kThreads, smem, st>>>(p);
  return cudaGetLastError();
}

}  // namespace

// K13 for a validated descriptor (vg_kernels.cu calls this first from
// vg_generate_f32 / vg_submit_f32). Returns 1 when it launched (stats zeroed
// unless `stats_zeroed`, and the kernel queued on `st`), 0 when the batch is
// not a K13 batch (the caller runs K1 + K3), or a negative VG_ERR_* with the
// error set. `dry_run`: only answer whether it would launch (1 / 0).
int vg_small_try(const vg_batch_desc* d, float* out, vg_mol_stats* stats, cudaStream_t st,
                 bool stats_zeroed, bool dry_run) {
  const int mode = env_small("VG_SMALL", -1);   // hook: 0 never, 1 whenever it can run
  if (mode == 0 || d->periodic || d->D % 4 != 0 || d->n_molecules <= 0) return 0;
  if ((reinterpret_cast<uintptr_t>(out) & 15) != 0) return 0;
  const int64_t total = d->n_molecules * (int64_t)d->C * d->H * d->W * d->D * 4;
  const int64_t mean_atoms = (d->n_atoms + d->n_molecules - 1) / d->n_molecules;
  if (mode != 1 && (total > kMaxBytes || mean_atoms > kMaxMeanAtoms)) return 0;
  // float4 slots per thread per group (K) and y-splits per (molecule,
  // channel): enough CTAs for ~4 per SM, each CTA a contiguous run of rows
  const int kk = env_small("VG_SMALL_K", 4);
  const int K = kk <= 1 ? 1 : kk <= 2 ? 2 : kk <= 4 ? 4 : 8;
  const int64_t grids = d->n_molecules * (int64_t)d->C;
  int n_split = (int)((148 * 4 + grids - 1) / grids);
  n_split = env_small("VG_SMALL_SPLIT", n_split);
  n_split = n_split < 1 ? 1 : (n_split > d->H ? d->H : n_split);
  int jc = (d->H + n_split - 1) / n_split;
  const int n_jchunks = (d->H + jc - 1) / jc;
  const int64_t ctas = grids * n_jchunks;
  if (ctas > INT_MAX) return 0;

  SmallParams p;
  memset(&p, 0, sizeof p);
  p.offsets = d->offsets;
  p.xyz = d->xyz;
  p.channel = d->channel;
  p.mol_origin = d->mol_origin;
  p.mol_delta = d->mol_delta;
  p.out = out;
  p.stats = stats;
  for (int a = 0; a < 3; ++a) {
    p.origin[a] = d->origin[a];
    p.delta[a] = d->delta[a];
  }
  p.scale = d->scale;
  p.H = d->H;
  p.W = d->W;
  p.D = d->D;
  p.C = d->C;
  p.jc = jc;
  p.n_jchunks = n_jchunks;
  p.rx = (d->W + 3) & ~3;
  p.ry = (d->H + 3) & ~3;
  p.rz = (d->D + 3) & ~3;
  const int per_cand = 4 * (p.rx + p.ry + p.rz) + 4 * (d->W + d->H + d->D + 3) + 12;
  int cap = (kSmemBudget - 16) / per_cand;
  cap = cap > kMaxCap ? kMaxCap : cap;
  if (cap < 1) return 0;
  p.cap = cap;
  p.has_threshold = !std::isnan(d->threshold);
  p.threshold = d->threshold;
  const size_t smem = (size_t)((cap * 4 + 15) & ~15) +
                      (size_t)cap * 4 * (p.rx + p.ry + p.rz + d->W + d->H + d->D + 3) +
                      (size_t)cap * 8;
  if (dry_run) return 1;

  if (stats != nullptr && !stats_zeroed) {
    const cudaError_t e = cudaMemsetAsync(stats, 0, sizeof(vg_mol_stats) * d->n_molecules, st);
    if (e != cudaSuccess) {
      char msg[256];
      snprintf(msg, sizeof msg, "stats memset: %s", cudaGetErrorString(e));
      return vg_internal_set_error(VG_ERR_CUDA, msg);
    }
  }
  cudaError_t e;
  switch (K) {
    case 1: e = launch_k<1>((unsigned)ctas, smem, st, p); break;
    case 2: e = launch_k<2>((unsigned)ctas, smem, st, p); break;
    case 4: e = launch_k<4>((unsigned)ctas, smem, st, p); break;
    default: e = launch_k<8>((unsigned)ctas, smem, st, p); break;
  }
  if (e != cudaSuccess) {
    char msg[256];
    snprintf(msg, sizeof msg, "vg_small_kernel: %s", cudaGetErrorString(e));
    return vg_internal_set_error(VG_ERR_CUDA, msg);
  }
  return 1;
}
