/* voxgrid_b200.h — C-ABI of the B200 grid-generation hot path.
 *
 * Drop-in boundary for the reference package `voxgrid` (pure Python/numpy,
 * /root/reference/pkg/src/voxgrid). Each entry point names the reference
 * interface it replaces. Plain pointers and sizes only: device pointers are
 * CUDA global-memory addresses, `stream` is a cudaStream_t passed as void*.
 * The library never allocates or frees device memory and keeps no global
 * state besides a thread-local error string; every launch is stream-ordered
 * with no host synchronisation, so calls are reentrant across streams.
 *
 * Return codes: VG_OK (0) or a negative VG_ERR_*; vg_last_error() explains.
 */
#ifndef VOXGRID_B200_H
#define VOXGRID_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VG_OK 0
#define VG_ERR_INVALID -1   /* bad descriptor / argument (ValueError in Python) */
#define VG_ERR_CUDA -2      /* a CUDA launch or runtime call failed             */
#define VG_ERR_WORKSPACE -3 /* workspace pointer NULL or too small              */

#define VG_ABI_VERSION 5

/* One batch of molecules in CSR form plus the grid geometry.
 *
 * Geometry follows GridSpec (reference core.py:92-166): shape (H, W, D) =
 * voxels along (y, x, z); axis_params() gives per world axis x,y,z the triple
 * (n, origin, delta) = (W, ox, A/W), (H, oy, B/H), (D, oz, C/D)
 * (core.py:161-166). Output layout is (B, C, H, W, D) fp32, z contiguous
 * (core.py:3-19); voxel (i, j, k) of channel c is out[b, c, j, i, k].
 */
typedef struct vg_batch_desc {
  int64_t n_molecules;       /* B                                               */
  int64_t n_atoms;           /* total atoms over the batch                      */
  const int64_t* offsets;    /* device [B+1]; molecule b owns atoms [o[b],o[b+1]) */
  const double* xyz;         /* device [n_atoms*3] world positions (x,y,z), fp64 */
  const int32_t* channel;    /* device [n_atoms] channel in [0, C)              */
  const double* mol_origin;  /* device [B*3] per-molecule box origin, or NULL   */
  const double* mol_delta;   /* device [B*3] per-molecule voxel sizes, or NULL  */
  double origin[3];          /* shared box origin (x,y,z) when mol_origin==NULL */
  double delta[3];           /* shared voxel sizes (dx,dy,dz) when mol_delta==NULL */
  double scale;              /* 1/(sigma*sqrt(2)) in fp64, kernels.py:235        */
  float threshold;           /* fl32(threshold), or NaN for None (kernels.py:271) */
  int32_t periodic;          /* 1: wrap every axis, cell edge = n*delta (kernels.py:239-251) */
  int32_t H, W, D, C;        /* grid shape (y, x, z) and channel count          */
} vg_batch_desc;

/* Per-molecule work counters, GenStats (gridgen.py:39-54) minus the
 * host-side fields. voxel_writes = sum over atoms of the support-box volume
 * (gridgen.py:103); nonzero_voxels = count_nonzero of the grid (gridgen.py:151).
 * Invalid atoms — channel outside [0, C) or a non-finite coordinate, which the
 * reference rejects with ValueError (gridgen.py:86-90, 114-119; core.py:190-199)
 * — are never splatted and set the sign bit of their molecule's voxel_writes
 * (voxel_writes < 0 flags the molecule; hosts validate before the launch, the
 * flag reports device-resident inputs). */
typedef struct vg_mol_stats {
  int64_t voxel_writes;
  int64_t nonzero_voxels;
} vg_mol_stats;

/* Byte offsets of the per-atom tables inside the workspace (all 256-aligned;
 * the workspace pointer itself must be 16-byte aligned: VG_ERR_INVALID otherwise).
 * tx: [n_atoms][row_x] fp32 masses along x (W used), ty: [n_atoms][row_y] (H),
 * tz: [n_atoms][row_z] (D); supp: [n_atoms] x int32[4] =
 * {xlo | xhi<<16, ylo | yhi<<16, zlo | zhi<<16, channel} (AxisTable.support,
 * kernels.py:101-119, 147-151). */
typedef struct vg_ws_layout {
  size_t tx, ty, tz, supp, total;
  int32_t row_x, row_y, row_z;
  /* K3 candidate bins (large molecules only; bin_jc == 0 when unused):
   * ordered atom indices per (molecule, channel, y-chunk of bin_jc slabs)
   * at `bins`, per-molecule bin offsets at `bin_off`. Scratch written by
   * vg_generate_f32 / vg_slabs_f32. */
  size_t bins, bin_off;
  int32_t bin_jc, bin_chunks;
} vg_ws_layout;

/* Workspace needed by vg_generate_f32 / vg_axis_tables_f32. */
int vg_workspace_layout(const vg_batch_desc* desc, vg_ws_layout* layout);

/* Replaces generate_batch (gridgen.py:173-221) / generate_grid
 * (gridgen.py:130-153) for float32 grids: writes every voxel of
 * out[B, C, H, W, D] (zeros included; no prior memset needed). Per voxel the
 * atoms of its channel are accumulated in input order in fp32 exactly as
 * splat_atom (gridgen.py:97-109). stats (device [B]) may be NULL. */
int vg_generate_f32(const vg_batch_desc* desc, float* out, void* workspace,
                    size_t workspace_bytes, vg_mol_stats* stats, void* stream);

/* Which kernels vg_generate_f32 / vg_submit_f32 run for this batch into
 * `out`: 1 = the one-launch small-batch kernel (K13: per-CTA axis tables in
 * shared memory + gather; small molecules, output <= 4 MiB, open axes,
 * D % 4 == 0, 16-byte aligned out), 0 = the tables kernel then the slab
 * kernel (K1, K2 for large molecules, K3). Negative VG_ERR_* for an invalid
 * descriptor. No GPU work. */
int vg_fused_small(const vg_batch_desc* desc, const float* out);

/* The second half of vg_generate_f32 alone: writes out[B, C, H, W, D] from
 * tables already computed into `workspace` by vg_axis_tables_f32 for the same
 * descriptor (stream-ordered). Lets a caller time the slab kernel by itself or
 * regenerate grids from cached tables. */
int vg_slabs_f32(const vg_batch_desc* desc, float* out, void* workspace,
                 size_t workspace_bytes, vg_mol_stats* stats, void* stream);

/* One pipelined submission (the loader stage around the path: GridPipeline,
 * paper_2211_08506_b200/loader.py; it replaces the per-batch body of
 * GaussianVoxelizer.transform, estimator.py:134-151, minus the np.stack):
 * copy_stream  waits ev_wait, H2D of the host CSR arrays (when h_* != NULL)
 *              into desc->offsets/channel/xyz, records ev_copied;
 * tables_stream waits ev_copied (hence ev_wait), K1, records ev_tabled;
 * compute_stream waits ev_tabled (hence ev_wait), K2/K3, then the D2H of the
 *              per-grid stats into h_stats (when != NULL), records ev_done;
 *              with a readback_stream, the D2H runs there instead, after ev_done,
 *              followed by ev_read (K3s of consecutive batches stay back to back).
 * Events are caller-created cudaEvent_t (passed as void*); ev_wait may be
 * NULL and may be the same event as ev_done (the wait uses its previous
 * record). Returns at once: no host synchronisation. Host buffers must stay
 * valid (pinned for asynchronous copies) until ev_copied / ev_done. When the
 * three host arrays lie in one block with the same relative offsets as their
 * device destinations (offsets first, xyz and channel not overlapping), the
 * copy stage is a single H2D of that span.
 * VG_ERR_WORKSPACE sets *ws_needed (if non-NULL) to the bytes required. */
typedef struct vg_submit_args {
  const void* h_offsets;   /* host [B+1] int64, or NULL: desc->offsets already filled   */
  const void* h_channel;   /* host [n_atoms] int32, or NULL                              */
  const void* h_xyz;       /* host [n_atoms*3] fp64, or NULL                             */
  void* h_stats;           /* host [B] vg_mol_stats (pinned), or NULL: no read-back      */
  void* copy_stream;
  void* tables_stream;
  void* compute_stream;
  void* ev_wait;
  void* ev_copied;
  void* ev_tabled;
  void* ev_done;
  size_t* ws_needed;
  int32_t* kernels;        /* out (if non-NULL): kernels this call launched (K1, K2, K3) */
  void* readback_stream;   /* NULL: the stats D2H runs on compute_stream before ev_done;
                              else on this stream after ev_done, then ev_read is recorded */
  void* ev_read;
} vg_submit_args;

int vg_submit_f32(const vg_batch_desc* desc, const vg_submit_args* args, float* out,
                  void* workspace, size_t workspace_bytes, vg_mol_stats* stats);

/* Replaces fused_axis_tables (kernels.py:217-274) for every atom of the
 * batch: fills the workspace tables + supports (layout above). Test hook and
 * building block for consumers (reversal) that need the tables. */
int vg_axis_tables_f32(const vg_batch_desc* desc, void* workspace, size_t workspace_bytes,
                       void* stream);

/* Replaces erf_approx(t, float32) (kernels.py:59-70) on a device array. */
int vg_erf_f32(const float* t, float* out, int64_t n, void* stream);

/* Grid reversal (reference reversal.py) building blocks.
 * vg_mse_f64 replaces _mse (reversal.py:256-258) for n_grids candidate grids
 * at once: out[g] = mean over n_voxels of (grids[g] - ref)^2 in fp64, fixed
 * reduction order (deterministic). Workspace: vg_mse_workspace_bytes(). */
size_t vg_mse_workspace_bytes(int64_t n_voxels, int32_t n_grids);
int vg_mse_f64(const float* ref, const float* grids, int64_t n_voxels, int32_t n_grids,
               double* out, void* workspace, size_t workspace_bytes, void* stream);
/* The same for several references: grid g is compared with refs[g / grids_per_ref]
 * (refs: consecutive grids of n_voxels floats) — batched reversal. */
int vg_mse_grouped_f64(const float* refs, const float* grids, int64_t n_voxels, int32_t n_grids,
                       int32_t grids_per_ref, double* out, void* workspace,
                       size_t workspace_bytes, void* stream);

/* Replaces _gradient_from_diff / loss_gradient (reversal.py:271-318): grad
 * [n_atoms*3] (x, y, z per atom, fp64) of mean((regen - ref)^2) w.r.t. the
 * atom coordinates of the molecules described by desc (open boundaries;
 * regen = the grids generated from desc, ref the targets, both
 * (B, C, H, W, D); molecule b's atoms use grid b). */
int vg_loss_gradient_f64(const vg_batch_desc* desc, const float* ref, const float* regen,
                         double* grad, void* stream);

/* Device-resident descent of refine_coords (reversal.py:325-398): the loop
 * state lives in device memory so that an iteration (gradient, candidates,
 * batched regeneration, batched loss, selection) needs no host round trip;
 * the host reads `done` every few iterations. Once `done` is set, both calls
 * leave the state, positions and regen untouched. */
typedef struct vg_descent_state {
  double current;       /* loss at the current positions                        */
  double best;          /* lowest loss seen (its positions are in best_pos)     */
  int64_t iterations;   /* accepted steps                                       */
  int64_t forced;       /* consecutive steps with no candidate <= current       */
  int32_t done;         /* a stop rule fired                                    */
  int32_t diverged;     /* stopped after `patience` forced steps                */
  int32_t sel;          /* last selected candidate (internal)                   */
  int32_t moved;        /* last select call took a step (internal)              */
} vg_descent_state;

/* Loop top: done if iterations >= max_iters or current < tolerance, or if
 * the gradient is all zero; otherwise cands[g] = pos - steps[g] * grad for
 * g < n_steps (fp64, unfused: the reference's positions - (step0*h)*grad).
 * n_coords = 3 * atoms. */
int vg_descent_candidates_f64(vg_descent_state* state, const double* pos, const double* grad,
                              const double* steps, double* cands, int32_t n_coords,
                              int32_t n_steps, int64_t max_iters, double tolerance, void* stream);

/* After the candidates' losses: take the first g with losses[g] <= current
 * (else the last, smallest step), move pos and regen (grids[g], n_voxels
 * floats) to it, count the step, track the best, and stop after `patience`
 * consecutive forced steps. */
int vg_descent_select_f64(vg_descent_state* state, const double* losses, const double* cands,
                          const float* grids, int32_t n_coords, int32_t n_steps,
                          int64_t n_voxels, int32_t patience, double* pos, double* best_pos,
                          float* regen, void* stream);

/* Batched descent: n_molecules independent reversals at once. states[k],
 * coordinates [coord_offsets[k], coord_offsets[k+1]) (device int32, 3 per
 * atom), steps[k*n_steps + g]; molecule k's candidates are at
 * cands[n_steps*coord_offsets[k] + g*(its coordinate count)] (the CSR order
 * of the batched regeneration), losses[k*n_steps + g], grids[k*n_steps + g]
 * and regen[k] (n_voxels floats each). Per molecule the same rules as the
 * single calls, so each result equals its own single reversal. */
int vg_descent_candidates_batch_f64(vg_descent_state* states, const int32_t* coord_offsets,
                                    int32_t n_molecules, const double* pos, const double* grad,
                                    const double* steps, double* cands, int32_t n_steps,
                                    int64_t max_iters, double tolerance, void* stream);
int vg_descent_select_batch_f64(vg_descent_state* states, const int32_t* coord_offsets,
                                int32_t n_molecules, const double* losses, const double* cands,
                                const float* grids, int32_t n_steps, int64_t n_voxels,
                                int32_t patience, double* pos, double* best_pos, float* regen,
                                void* stream);

/* Device fill with 128-bit stores (HBM write-bandwidth probe for the roofline). */
int vg_fill_f32(float* out, int64_t n, float value, void* stream);

/* Host builds of the exact device numerics, for conformance tests only:
 * np.exp on float32 (numpy SIMD algorithm) and the Bürmann erf. */
int vg_exp_f32_host(const float* x, float* out, size_t n);
int vg_erf_f32_host(const float* t, float* out, size_t n);
/* The saturated erf K1 evaluates: +-1 beyond +-VG_TSAT, else the series with
 * the exp range checks dropped (bit-identical to vg_erf_f32_host). */
int vg_erf_sat_f32_host(const float* t, float* out, size_t n);

/* Thread-local description of the last error (empty string if none). */
const char* vg_last_error(void);

/* VG_ABI_VERSION of the loaded library. */
int vg_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* VOXGRID_B200_H */
