/*
 * slabewald.h — C-ABI of the B200-native doubly periodic spectral Ewald
 * solver (arXiv 2101.07088), libslabewald_cuda.so.
 *
 * The reference has no FFI: its boundary is the Python class API
 *   SlabSolver(system, params, threads=1, refine=1)      slab.py:197
 *   SlabSolver.solve(positions=None, need_energy=True, need_forces=True,
 *                    need_potential=True, subtract_self=False,
 *                    include_correction=True, force_general=False)
 *                                                         slab.py:259-261
 *   near_field_sum(...)                                   slab.py:184-191
 *   build_partition(...)                                  slab.py:51-82
 * Each entry point below replaces the compute behind one of those calls; the
 * Python package paper_2101_07088_b200 (slab.py) binds them with ctypes and
 * keeps the reference's signatures, exceptions and diagnostics keys.
 *
 * Conventions: plain pointers and sizes only.  "host" buffers are caller
 * owned and only read/written during the call; "device" buffers are device
 * pointers on the plan's device.  Positions are [n][3] row-major doubles,
 * fields [n][3].  A plan is not thread safe: one call at a time.  All calls
 * return SE_OK or an error code; se_last_error() gives the message.
 */
#ifndef SLABEWALD_H
#define SLABEWALD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error codes -> Python exception (slab.py maps them) */
#define SE_OK          0
#define SE_ERR_VALUE   1  /* ValueError (bad input, point outside z domain) */
#define SE_ERR_FLOAT   2  /* FloatingPointError (non-finite mismatch, k=0)  */
#define SE_ERR_LINALG  3  /* numpy.linalg.LinAlgError (Schur conditioning)  */
#define SE_ERR_CUDA    4  /* RuntimeError (CUDA / cuFFT failure)            */
#define SE_ERR_MEMORY  5  /* MemoryError (device allocation)                */

/* solve flags (defaults of SlabSolver.solve are ENERGY|FORCES|POTENTIAL|CORRECTION) */
#define SE_NEED_ENERGY     (1u << 0)
#define SE_NEED_FORCES     (1u << 1)
#define SE_NEED_POTENTIAL  (1u << 2)
#define SE_SUBTRACT_SELF   (1u << 3)
#define SE_CORRECTION      (1u << 4)
#define SE_FORCE_GENERAL   (1u << 5)
#define SE_TIMINGS         (1u << 6)   /* fill se_diag.t_ms (adds syncs) */
#define SE_FP32            (1u << 7)   /* fp32 mode: near-field pair kernels in
                                          single precision (pair membership stays
                                          the exact fp64 test); results within
                                          the run's Ewald tolerance */

#define SE_GRAPH           (1u << 9)   /* capture the solve as a CUDA graph
                                          (after one warm solve with the same
                                          buffers, size and flags) and replay
                                          it while those repeat: no per-kernel
                                          launch cost (BD loops, small N) */
#define SE_PAIR_HASH       (1u << 8)   /* record the near-field pair SET of the
                                          charges (se_debug_fetch 6) for
                                          parity tests */

/* Solver parameters: the geometry plus the EwaldParams fields the device
 * path needs (params.py:28-50). */
typedef struct {
    double Lx, Ly, H, eps, eps_b, eps_t;
    double g_w, xi, g_t, H_E, r_nf, r_cut, k_max, z0, z1;
    double xi_is_inf;          /* 1.0 when xi == inf (no near field) */
    int32_t Nx, Ny, Nz, refine;
} se_params;

/* Diagnostics of one solve (slab.py:275,332,384-385 keys + timings). */
typedef struct {
    double ai1, ai2, discrepancy, B_i;
    double A_i, A_b, A_t, psi_i_bottom, psi_i_top, psi_b_bottom, psi_t_top;
    double U_wall;             /* wall-charge energy part of U (0 if sigma=0) */
    int32_t warn_discrepancy;  /* 1 when 1e-3 < discrepancy <= 1e-2 */
    int32_t n_sources;         /* spread sources (charges + images) */
    int64_t n_pairs;           /* near-field pairs evaluated for the charges */
    int64_t n_launches;        /* own kernels launched by this call */
    double t_ms[16];           /* SE_TIMINGS: 0-7 stages (sources, spread,
                                  forward, bvp, inverse, interp, near,
                                  finish); 8-11 kernels (spread, bvp, interp,
                                  near field of the charges: scan + eval);
                                  12 near scan kernel, 13 near eval kernel */
} se_diag;

typedef struct se_plan se_plan;

/* SlabSolver.__init__ (slab.py:197-233).  Host arrays computed by the
 * Python planner exactly as the reference does (bit-identical constants):
 *   z_nodes[Nz]  ascending Chebyshev points   (chebyshev.py:14-19)
 *   cc_w[Nz]     Clenshaw-Curtis weights      (chebyshev.py:22-43)
 *   t_wall0[Nz], t_wallH[Nz]  T_n(z=0), T_n(z=H) (slab.py:214-222)
 *   kx[Nx], ky[Ny]            fft-ordered wavenumbers (chebyshev.py:98-102)
 *   sigma_b, sigma_t          [Nx][Ny] wall charge samples or NULL (zero)
 * device: CUDA ordinal.  Factorises the per-|k| BVPs on the device; an
 * ill-conditioned Schur block returns SE_ERR_LINALG (bvp.py:187-192). */
int se_plan_create(const se_params* params, const double* z_nodes,
                   const double* cc_w, const double* t_wall0,
                   const double* t_wallH, const double* kx, const double* ky,
                   const double* sigma_b, const double* sigma_t, int device,
                   se_plan** out);

void se_plan_destroy(se_plan* plan);

/* Run the plan's work on a caller-provided cudaStream_t (e.g. PyTorch's
 * current stream) instead of its own; NULL selects the legacy stream. */
int se_plan_set_stream(se_plan* plan, void* stream);

/* Bind the charges (system.charges, slab.py:274).  host q[n]. */
int se_set_charges(se_plan* plan, const double* q, int64_t n);

/* SlabSolver.solve with host buffers (positions in, results out):
 * pos[n][3] -> phi_bar[n], E_bar[n][3] (may be NULL without FORCES), U. */
int se_solve(se_plan* plan, const double* pos, int64_t n, uint32_t flags,
             double* phi_bar, double* E_bar, double* U, se_diag* diag);

/* Same with device-resident positions and outputs (no host copies; the
 * stream is synchronised before return). */
int se_solve_device(se_plan* plan, const double* d_pos, int64_t n,
                    uint32_t flags, double* d_phi_bar, double* d_E_bar,
                    double* U, se_diag* diag);

/* Sharded solve (one rank per GPU, charges split by index): the same solve
 * in three phases.  Phase 1 spreads the charges first..first+count-1 (and
 * their images) into the plan's grids and returns the grid buffer
 * (device, rho_len doubles) for the caller to SUM over ranks in place
 * (e.g. an NCCL all-reduce on the plan's stream).  Phase 2 runs the grid
 * pipeline on the summed grids.  Phase 3 interpolates and evaluates the near
 * field (sources: all n_all charges) for this rank's charges, writes
 * d_phi[count], d_E[count][3] (device) and this rank's part of U (the
 * ranks' parts sum to U). */
int se_shard_spread(se_plan* plan, const double* d_pos_all, int64_t n_all,
                    int64_t first, int64_t count, uint32_t flags,
                    double** d_rho, int64_t* rho_len);
int se_shard_fields(se_plan* plan);
int se_shard_charges(se_plan* plan, const double* d_pos_all, double* d_phi,
                     double* d_E, double* U_part, se_diag* diag);

/* Sharded solve with only the own shard's positions and the near field
 * routed by cell (replaces the every-source near field
 * of NearField, slab.py:94-181, on each rank):
 *   se_shard_spread_own   as se_shard_spread, d_pos_own = [count][3] rows of
 *                         charges first..first+count-1 only
 *   se_shard_near         on `stream` (may run concurrently with the grid
 *                         pipeline on the plan's stream): near-field sums of
 *                         the first nt of ns sources (the charges this rank
 *                         owns by cell; the rest are its halo) with all ns
 *                         charges and their mirror images as sources;
 *                         d_out [4][nt] (phi, E); gauge != 0: also the point
 *                         kernel sum at the origin (device scalar d_near0,
 *                         the gauge's near part, to be summed over ranks);
 *                         device int64 d_npairs: the pairs.  d_zsrc_min
 *                         (device scalar, optional): the minimum z over ALL
 *                         ranks' sources incl. mirror layers, so pairs at
 *                         the exact cutoff are decided as the reference's
 *                         single KD tree does (slab.py:120-131).  No host sync.
 *   se_shard_charges_own  interpolation + finalisation of the own shard with
 *                         the caller's near sums in shard order d_near_own
 *                         [4][count] and the summed near0 (device scalar;
 *                         zero surface charge only). */
int se_shard_spread_own(se_plan* plan, const double* d_pos_own, int64_t n_all,
                        int64_t first, int64_t count, uint32_t flags,
                        double** d_rho, int64_t* rho_len);
int se_shard_near(se_plan* plan, void* stream, const double* d_src_pos,
                  const double* d_src_q, int64_t ns, int64_t nt, int gauge,
                  const double* d_zsrc_min, double* d_out, double* d_near0,
                  int64_t* d_npairs);
int se_shard_charges_own(se_plan* plan, const double* d_pos_own,
                         const double* d_near_own, const double* d_near0,
                         double* d_phi, double* d_E, double* U_part,
                         se_diag* diag);

/* Distributed grid pipeline for a sharded solve: after
 * se_dist_setup(plan, rank, nranks, sizes) a rank's solve is
 *   se_shard_spread          -> caller: reduce-scatter  rho_full -> rho_slab
 *   se_dist_forward          -> caller: all-to-all      a2a_send -> a2a_recv
 *   se_dist_modes            -> caller: all-to-all      a2a_send -> a2a_recv
 *                               caller: all-reduce(sum) dsc
 *   se_dist_fields           -> caller: all-gather      fields_slab -> fields
 *   se_shard_charges
 * Rank r owns the z planes [r zc, (r+1) zc) for the xy FFTs and the
 * half-spectrum modes [r mc, (r+1) mc) for the z transforms and BVPs.
 * sizes[0..6] = doubles in rho_full, rho_slab, a2a forward block (all
 * ranks), a2a back block (all ranks), fields_slab, fields, dsc;
 * se_dist_buffers returns the seven device pointers in the same order. */
int se_dist_setup(se_plan* plan, int rank, int nranks, int64_t* sizes);
int se_dist_buffers(se_plan* plan, void** ptrs);
int se_dist_forward(se_plan* plan);
int se_dist_modes(se_plan* plan);
int se_dist_fields(se_plan* plan);

/* Brownian-dynamics steric pair forces (bd.py:246-270): truncated LJ
 * repulsion 4 U0 ((2a/r)^2p - (2a/r)^p) + U0 cut at 2^(1/p) 2a, core capped
 * below r_m, minimum image on the periodic axes (box length > 0; Lz <= 0
 * means open z, the slab case; Lz > 0 the triply periodic box of the g2
 * experiment, validate.py:245).  pos[n][3], out[n][3] host buffers. */
int se_steric_forces(int device, const double* pos, int64_t n, double Lx, double Ly,
                     double Lz, double a, double U0, double r_m, int p, double* out);

/* Device-resident Brownian dynamics (SURVEY 8f next #1 at scale).
 *   se_steric_forces_device: se_steric_forces on device buffers on a
 *     caller's stream; open z (Lz <= 0) uses the cell range [zlo, zhi].
 *   se_bd_first_noise_device: the initial noise W_0 (Philox, subsequence i).
 *   se_bd_step_device: bd_step (bd.py:101-133) on device buffers: forces
 *     q E + f_ext (+ the mirror-wall steric force when wall != 0,
 *     bd.py:273-279), W_{n+1} from Philox4x32-10 (seed, subsequence i,
 *     offset 8 per draw; *draws counts the draws), max_disp cap, z-bound
 *     rejection with a full redraw (*rejections incremented), x/y wrap with
 *     numpy's mod when Lx / Ly > 0.  pos, prev [n][3] updated in place; E
 *     [n][3] (or NULL), q [n] (or NULL), f_ext [n][3] (or NULL).  The noise
 *     stream is NOT numpy's: the host path (bd.py) reproduces the
 *     reference draw for draw, this one is for device-resident runs. */
typedef struct {
    double dt, mu, kT, max_disp, z_lo, z_hi, Lx, Ly, H, a, U0, r_m;
    int32_t p, wall, has_zb, max_retries;
    uint64_t seed;
} se_bd_params;
int se_steric_forces_device(int device, void* stream, const double* d_pos, int64_t n, double Lx,
                            double Ly, double Lz, double zlo, double zhi, double a, double U0,
                            double r_m, int p, double* d_out);
int se_bd_first_noise_device(int device, void* stream, int64_t n, uint64_t seed, double* d_prev);
int se_bd_step_device(int device, void* stream, double* d_pos, double* d_prev, const double* d_E,
                      const double* d_q, const double* d_fext, int64_t n,
                      const se_bd_params* params, uint64_t* draws, int64_t* rejections);

/* Triply periodic twin.  A plan holds the uniform
 * periodic grid nx x ny x nz of the box Lx x Ly x Lz and the permittivity.
 *   se_tp_poisson: solve_triply_periodic (dpsolver.py:221-249); rho, phi
 *     [nx][ny][nz], E [3][nx][ny][nz] (NULL or with_field 0: no field).
 *   se_tp_forces: TriplyPeriodicSolver.forces (bd.py:323-331): spread with
 *     Gaussian width g_t inside radius, FFT Poisson solve, field
 *     interpolation, near_gradient_avg pair forces within r_cut (split g_w,
 *     xi); forces[n][3] = q (far + near).  Host buffers.
 *   se_tp_forces_device: the same on device buffers, on the plan's stream.
 *   se_tp_set_graph: (new) with enable != 0, se_tp_forces_device captures
 *     its kernels as a CUDA graph on the second call with the same buffers
 *     and parameters and replays the graph from then on. */
typedef struct se_tp se_tp;
int se_tp_create(int device, double Lx, double Ly, double Lz, int nx, int ny, int nz,
                 double eps, se_tp** plan);
int se_tp_destroy(se_tp* plan);
int se_tp_set_stream(se_tp* plan, void* stream);
int se_tp_set_graph(se_tp* plan, int enable);
int se_tp_poisson(se_tp* plan, const double* rho, int with_field, double* phi, double* E);
int se_tp_forces(se_tp* plan, const double* pos, const double* q, int64_t n, double g_t,
                 double radius, double g_w, double xi, double r_cut, double* forces);
int se_tp_forces_device(se_tp* plan, const double* d_pos, const double* d_q, int64_t n,
                        double g_t, double radius, double g_w, double xi, double r_cut,
                        double* d_forces);

/* near_field_sum (slab.py:184-191): sources = pos[n] with charges q[n]
 * (plus the mirrored layers of the geometry in params), evaluated at
 * eval_pos[ne].  kind 0 = "avg" (r_cut), 1 = "point" (r_nf).  Host buffers.
 * E may be NULL when need_field == 0.  No plan needed (grid fields of
 * params are ignored). */
int se_near_field(const se_params* params, int device, const double* pos,
                  const double* q, int64_t n, const double* eval_pos,
                  int64_t ne, int kind, int need_field, int subtract_unsplit,
                  double* phi, double* E);

/* build_partition (slab.py:51-82).  Host in/out; index arrays int64, sized
 * by the caller for the worst case (n over/far, 2n images).  Counts out. */
int se_build_partition(const se_params* params, int device, const double* pos,
                       const double* q, int64_t n, int64_t* n_over,
                       int64_t* over, int64_t* n_far, int64_t* far,
                       int64_t* n_img, double* img_pos, double* img_str,
                       int64_t* img_src, int32_t* img_wall);

/* Stage buffers of the last solve, for parity tests (host copy):
 * 0 rho[Nz][2][Nx][Ny] (slot 0 = over, 1 = in), 1 psi coefficients
 * [Nz][2][Nx][Ny/2+1] complex (slot 0 = psi_o, 1 = psi_i) — only when the
 * plan was created with SE_KEEP_STAGES=1 in the environment, 2 field grids
 * [Nz][4][Nx][Ny] (inverse xy FFTs of psi, i kx psi, i ky psi, dpsi/dz
 * before the signs and the k = 0 A_i terms), 3 mismatch fields
 * [4][Nx][Ny/2+1] complex (phi_b, e_b, phi_t, e_t), 4 far-field interpolation
 * sums [4][N], 5 near-field sums [4][N].
 * Returns the byte size when host == NULL. */
int64_t se_debug_fetch(se_plan* plan, int which, void* host, int64_t nbytes);

/* Measured FP64 FMA throughput of the device (TFLOP/s, 2 flops per DFMA):
 * the roofline denominator of the FP64-bound kernels (spread, interpolation,
 * near field), which MEASURED_PEAKS.json does not cover. */
int se_fp64_peak(int device, double* tflops);

const char* se_last_error(void);
const char* se_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SLABEWALD_H */
