/*
 * hpgmxp.h -- C ABI of libhpgmxp.so, the B200 (sm_100a) solve path of HPG-MxP.
 *
 * The reference (mxpbench, pure Python + numpy) has no FFI: its "boundary" is
 * a set of Python call signatures.  Each entry point below
 * replaces one of them; the Python package paper_2507_11512_b200 binds these
 * through ctypes and keeps the reference's names, argument meaning and errors.
 *
 * Conventions
 *   - int return: 0 ok, < 0 error (HPG_E_*); hpg_last_error() has the text.
 *   - prec: HPG_F64 (0) or HPG_F32 (1); vectors are caller-owned DEVICE
 *     pointers of that precision.  "ext" vectors carry the halo tail
 *     (n_ext = n + halo entries), exactly like the reference's halo-tailed
 *     arrays (ref: problem.py:39-40, comm.py:158-172).
 *   - Everything is enqueued on the context's compute stream (hpg_stream());
 *     only functions returning host values synchronise.
 *   - One context per process / GPU, driven from one host thread.
 */
#ifndef HPGMXP_H
#define HPGMXP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HPG_F64 0
#define HPG_F32 1

#define HPG_OK 0
#define HPG_E_ARG -1          /* bad argument                        -> ValueError            */
#define HPG_E_CUDA -2         /* CUDA runtime failure                -> RuntimeError          */
#define HPG_E_NCCL -3         /* NCCL failure                        -> ProtocolError         */
#define HPG_E_COARSEN -4      /* odd local extent while coarsening   -> CoarseningError       */
#define HPG_E_UNSUPPORTED -5  /* e.g. restart length > 63            -> ValueError            */
#define HPG_E_SINGULAR -6     /* zero diagonal reached the smoother  -> SingularDiagonal      */

typedef struct hpg_ctx hpg_ctx;

int hpg_abi_version(void);
const char* hpg_last_error(void);

/* ---- host-only structure (no GPU needed; used by the CPU parity tests) ---- */

/* Rank-level ELL in the reference layout (row-major [n][27], padding col -1).
 * replaces: problem.generate_matrix + coloring.color/permute_system +
 *           comm.build_halo_plan's column rewrite (problem.py:88-142,
 *           coloring.py:36-123, comm.py:180-236).
 * info[0..]: n, n_ext, nnz, ncolors, color_offsets[0..8], halo_size        */
int hpg_host_level(const int local_dims[3], const int rank_coords[3], const int proc_dims[3],
                   double* values, int32_t* col_idx, int32_t* row_nnz, int32_t* diag_pos,
                   int64_t* info, int ninfo);

/* Send list towards the neighbour across face/edge/corner (sx,sy,sz):
 * permuted local rows in the peer's request order (ref: comm.py:209-217).
 * Returns the count (rows may be NULL to query it).                         */
int64_t hpg_host_send_rows(const int local_dims[3], const int rank_coords[3], const int proc_dims[3],
                           int sx, int sy, int sz, int64_t* rows);

/* Byte offset, inside `receiver`'s peer-memory symmetric buffer, of the staging
 * region where `sender`'s halo messages for `level` land (count receives the
 * element count, -1 if the two are not neighbours; sender < 0 returns the
 * buffer size).  Host-only, used by the CPU layout tests. */
int64_t hpg_host_stage_offset(const int local_dims[3], const int proc_dims[3], int levels, int receiver,
                              int level, int sender, int64_t* count);

/* ---- lifecycle ---- */

/* ncclGetUniqueId into out[0..127] (rank 0 calls it, then broadcasts). */
int hpg_nccl_unique_id(void* out, int len);

/* Build the whole hierarchy on device: `levels` levels below local_dims,
 * greedy coloring, permuted ELL (fp64 + fp32 values, shared int32 columns),
 * halo plans, injection maps, V-cycle workspaces.
 * replaces: multigrid.build_hierarchy (multigrid.py:54-84).
 * nccl_uid may be NULL: no NCCL communicator; a multi-rank context then moves
 * every halo and reduction over peer memory (hpg_p2p_open is mandatory) and
 * several ranks may share one GPU.  stream: cudaStream_t to enqueue on
 * (borrowed), or NULL for a context-owned non-blocking stream.              */
int hpg_create(hpg_ctx** out, int device, int rank, int nranks, const int proc_dims[3],
               const int local_dims[3], int levels, int nu1, int nu2, int nu_c,
               const void* nccl_uid, void* stream);
int hpg_destroy(hpg_ctx* ctx);
void* hpg_stream(hpg_ctx* ctx);   /* cudaStream_t of the compute stream */

/* info: n, n_ext, nnz, ncolors, offsets[9], halo_size, ld, nneighbours, device_bytes,
 *       zero_sweep_slots (slots a zero-initial-guess sweep streams, sum over colors
 *       of lower width x rows; 27 n when the lower split is absent) */
int hpg_level_info(hpg_ctx* ctx, int level, int64_t* info, int ninfo);
/* Copy a device level back in the reference layout (host buffers [n][27]). */
int hpg_export_level(hpg_ctx* ctx, int level, double* values, int32_t* col_idx,
                     int32_t* row_nnz, int32_t* diag_pos);
/* Replace level `level`'s (greedy, closed-form) coloring by an explicit one --
 * e.g. JPL (ref: coloring.py:56-70): perm[new row] = natural row, rows sorted by
 * (color, natural); offsets[0..ncolors] the color blocks.  Rebuilds the level's
 * ELL, send lists and the injection maps touching it (general gather kernels
 * then serve restriction / prolongation).  Synchronises. */
int hpg_set_coloring(hpg_ctx* ctx, int level, int ncolors, const int64_t* offsets, const int64_t* perm);
/* Jones-Plassmann-Luby colouring of an lx x ly x lz box on device `device`
 * (ref: coloring.py:56-70, color(A, "jpl", seed)): colors[n] receives each
 * natural row's colour, bit-identical to the reference -- same random stream:
 * state / inc are the low / high 64-bit words of numpy's PCG64 state and
 * increment of default_rng(seed); *rounds the independent-set rounds taken. */
int hpg_jpl_color(int device, int lx, int ly, int lz, const uint64_t* state, const uint64_t* inc, int32_t* colors,
                  int* rounds);
/* Injection map f2c of coarse level `level` (>=1) into its parent (ref: multigrid.py:87-99). */
int hpg_export_f2c(hpg_ctx* ctx, int level, int64_t* f2c);

/* ---- stencil kernels ---- */

/* y = A x with a fresh halo (exchange first).  replaces krylov.spmv (krylov.py:83-107) */
int hpg_spmv(hpg_ctx* ctx, int level, int prec, void* x_ext, void* y);
/* Fill v's halo tail from the neighbours.  replaces comm.exchange (comm.py:239-251) */
int hpg_exchange(hpg_ctx* ctx, int level, int prec, void* v_ext);
/* One forward multicolor GS sweep; z_is_zero zeroes z (tail too) and skips the
 * exchange.  replaces smoother.forward_gs_sweep (smoother.py:78-114)        */
int hpg_gs_sweep(hpg_ctx* ctx, int level, int prec, const void* r, void* z_ext, int z_is_zero);
/* r_c = (r_f - A_f z_f) at the injected rows; z_f's halo must be fresh.
 * `level` is the FINE level.  replaces multigrid.fused_residual_restrict    */
int hpg_restrict(hpg_ctx* ctx, int level, int prec, const void* r_f, const void* z_f_ext, void* r_c);
/* z_f[f2c] += z_c.  `level` is the FINE level.  replaces multigrid.prolong_add */
int hpg_prolong(hpg_ctx* ctx, int level, int prec, void* z_f, const void* z_c);
/* One V-cycle from level 0 with zero initial guess; z_ext (n_ext) receives z.
 * replaces multigrid.MgHierarchy.apply / mg_vcycle (multigrid.py:49-51,140-171) */
int hpg_vcycle(hpg_ctx* ctx, int prec, const void* r, void* z_ext);

/* ---- Krylov ---- */

/* CGS2 of w against Q rows 0..k (Q row-major, row stride ldq elements).
 * host_out receives h1[0..k], h2[0..k] (the two passes) and, when q_next is
 * non-NULL, beta = ||w|| with q_next = w / beta written (ref: krylov.py:110-129,
 * 266-273).  Synchronises.  Reductions are rank-ordered (ref: comm.py:97-108). */
int hpg_cgs2(hpg_ctx* ctx, int prec, void* Q, int64_t ldq, int k, void* w, void* q_next,
             double* host_out);
/* The same step split in two: _begin enqueues everything (no host wait),
 * _end blocks until (h1, h2, beta) of the step in flight are on the host. */
int hpg_cgs2_begin(hpg_ctx* ctx, int prec, void* Q, int64_t ldq, int k, void* w, void* q_next);
int hpg_cgs2_end(hpg_ctx* ctx, double* host_out);
/* out = Q[0:k]^T y  (y given on the host in fp64, narrowed to prec first;
 * ref: krylov.py:288-289) */
int hpg_gemv_combine(hpg_ctx* ctx, int prec, const void* Q, int64_t ldq, int k,
                     const double* y_host, void* out);
/* x += z (x fp64, z of precision prec).  ref: krylov.py:292-293 */
int hpg_axpy_mixed(hpg_ctx* ctx, int prec, double* x, const void* z, int64_t n);
/* fp64 outer residual r = b - A x (x_ext exchanged first) and *rho2 = sum r^2
 * over all ranks.  Synchronises.  ref: krylov.py:215-222 */
int hpg_residual(hpg_ctx* ctx, const double* b, double* x_ext, double* r, double* rho2);
/* q0 = (prec)(r / rho).  ref: krylov.py:250-252 */
int hpg_scale_cast(hpg_ctx* ctx, int prec, const double* r, double rho, void* q0, int64_t n);
/* *out = sum x^2 over all ranks (in prec arithmetic).  Synchronises. */
int hpg_sumsq(hpg_ctx* ctx, int prec, const void* x, int64_t n, double* out);
int hpg_sync(hpg_ctx* ctx);
/* Rank-ordered sum of n doubles on the host side (flags, counters). */
int hpg_allreduce_host(hpg_ctx* ctx, double* vals, int n);
/* Number of kernels this context has launched (for the bench's gpu_launches). */
int64_t hpg_launch_count(hpg_ctx* ctx);
/* Per-motif CUDA-event timers (ref: metrics.py:111-143 Tally).  mode 1 enable,
 * 0 disable, 2 synchronise + ADD seconds per motif into seconds[8]
 * (GS, SpMV, Ortho, Restriction, Prolongation, Vector ops, and two subsets of
 * GS: level-0 full sweeps, level-0 zero-initial-guess sweeps) and reset.     */
int hpg_timers(hpg_ctx* ctx, int mode, double* seconds);
/* Tuning switches (results are identical up to reduction order):
 *   "cgs_fused"  1: CGS2 as one cooperative kernel (single rank, or NVLink peers), 0: per-pass kernels
 *   "cgs_cfg"    force one configuration of that kernel: [CTAs per SM * 1000 +] row groups * 100
 *                + rows per warp * 10 + tiles (e.g. 481, 3441)
 *   "cgs_zigzag" 1: its passes B and D walk each CTA's range backwards (L2 reuse; default 1)
 *   "cgs_solo"   1: single rank, every CTA folds the dot partials itself (one grid barrier
 *                per fold instead of two; bitwise the same values; default 1)
 *   "tail_rows"  levels with at most this many rows run in the persistent V-cycle tail kernel
 *   "tail_cluster" > 0: that tail kernel runs as ONE cluster of this many CTAs (<= 16,
 *                hardware cluster barrier); 0: a cooperative grid (grid-wide barrier)
 *   "pdl"        1: stencil kernels use programmatic dependent launch
 *   "overlap"    1: multi-rank SpMV / GS overlap the halo exchange with interior rows (default 1)
 *   "overlap_rows" only levels with at least this many rows overlap (default 0: all)
 *   "p2p"        1: NVLink peer-memory halo exchange + all-reduce (after hpg_p2p_open)
 *   "graphs"     1: single-rank V-cycles replay a captured CUDA graph per (prec, r, z)
 *   "known_zero" 1: zero-initial-guess sweeps skip the loads of not-yet-updated colors
 *   "gs_minb"    blocks per SM the color-pass kernel is compiled for (2 or 3)
 *   "gs_rev"     1: odd colors' passes walk their block backwards (L2 reuse at the turn)
 *   "spmv_ilv"   fp64 SpMV / residual CTAs interleaved over this many row segments
 *                (the color blocks) so x gathers hit L2 (default 4; bitwise identical)
 *   "spmv_ilv32" the same for the fp32 SpMV (default 8)
 *   "wave"       bit mask (1 fp64, 2 fp32): forward sweeps as one dataflow kernel
 *                (bitwise identical; default 1)
 *   "wave_min_rows" levels with fewer rows keep the per-color passes
 *   "lower"      1: zero-initial-guess sweeps run the strictly-lower kernel (bitwise
 *                identical, but it skips the products against z = 0 that the
 *                reference forms and the flop model counts; default 0)
 *   "stencil"    1: rows whose 27 neighbours are local compute their columns in
 *                closed form instead of loading the index plane (default 1)
 *   "tma"        bit mask (1 fp64, 2 fp32): colour passes of levels with >= "tma_min_rows"
 *                rows stage their 27 value planes with one tensor copy (hpg_tma.cuh)
 *   "tma_cfg32" / "tma_cfg64"  rows per CTA * 100 + CTAs per SM of that pass (12808 / 3220)
 *   "spmv_tma"   bit mask: SpMV, fp64 residual and restriction with staged values;
 *                "spmv_cfg32" / "spmv_cfg64" / "resid_cfg" / "restr_cfg32" / "restr_cfg64"
 *   "face_cols"  bits: face rows off rank interfaces compute their columns (1 SpMV-type,
 *                2 fp64 passes, 4 fp32 passes, 8 passes' x-face slot map, 16 SpMV x-face map)
 *   "brick" / "bpp" / "tma_sweep"  experimental pass kernels (hpg_brick.cuh, the
 *                persistent sweep); measured slower, off
 *   "l2_window"  bytes of persisting L2 set-aside for z during the big passes (0: off)
 * Every option change drops the captured V-cycle graphs (re-captured on next use). */
int hpg_set_option(hpg_ctx* ctx, const char* key, int64_t value);

/* NVLink peer memory (csrc/hpg_p2p.cuh).  Collective setup, nranks > 1:
 *   1. every rank: hpg_p2p_handle -> its symmetric buffer's CUDA IPC handle
 *      (writes sizeof(cudaIpcMemHandle_t) = 64 bytes);
 *   2. all-gather the handles (host control plane);
 *   3. every rank: hpg_p2p_open(all handles, stride) maps the peers, then a
 *      host barrier before the first exchange.
 * Afterwards the halo exchange and the rank-ordered reductions run as P2P
 * kernels over NVLink instead of NCCL (ref: comm.py:97-108, 239-272). */
int hpg_p2p_handle(hpg_ctx* ctx, void* out, int len);
int hpg_p2p_open(hpg_ctx* ctx, const void* handles, int stride);

#ifdef __cplusplus
}
#endif
#endif
