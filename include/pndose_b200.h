/* Drop-in C-ABI of the B200 collided-flux DLRA stepper (libpndose_b200.so).
 *
 * The reference (`pndose`, pure Python) has no FFI; its boundary for this hot
 * path is the Python API of pkg/src/pndose/dlra.py, spatial.py, raytracer.py
 * and the energy loop of driver.py. Each entry point below replaces one of
 * those reference interfaces (cited per function); the Python shim
 * paper_2508_04484_b200/{dlra,spatial,raytracer,driver}.py binds them with
 * ctypes and keeps the reference's names, argument meanings and exceptions.
 *
 * Conventions
 *   - every function returns 0 on success or the reference's exit category:
 *     2 ConfigError, 3 PhysicsDataError, 4 NumericalError, 5 OutputIOError
 *     (pkg/src/pndose/errors.py:13-31), 6 for a CUDA runtime failure;
 *     pnd_last_error() copies the message (the shim raises the matching
 *     Python class with it, so message fragments such as "column" or
 *     "rank_max" match the reference's);
 *   - host arrays are C-contiguous float64 (int32 for indices), read or
 *     written only during the call; n = nx*ny*nz cells in the flat order
 *     k*nx*ny + j*nx + i (spatial.py:62-63), m = (N+1)^2 moments;
 *   - all device memory is owned by the handle; calls on one handle are
 *     stream-ordered and not thread-safe.
 */
#ifndef PNDOSE_B200_H
#define PNDOSE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pnd_handle pnd_handle;

/* ---- lifecycle ------------------------------------------------------- */
/* Grid3D + n_moments of an assembled problem (spatial.py:32-78). Raises
 * ConfigError for a 2-cell axis (spatial.py:84-88, "3-point"). */
int pnd_create(pnd_handle** h, int nx, int ny, int nz, double dx, double dy, double dz, int m,
               int device);
int pnd_destroy(pnd_handle* h);
int pnd_last_error(pnd_handle* h, char* buf, size_t len);
int pnd_synchronize(pnd_handle* h);
/* bytes of device memory held by the handle */
int pnd_device_bytes(pnd_handle* h, double* bytes);

/* ---- frozen operators / per-step coefficients (driver.py:523-538) --- */
/* A_d^+- = V_d diag(lambda_d^+-) V_d^T, 3 x m x m each (replaces
 * PNOperators.eig_v/lam_plus/lam_minus as used by dlra.py:155-194). */
int pnd_set_angular(pnd_handle* h, const double* a_plus, const double* a_minus);
/* Material classes: cell_class (n) indexes class_atomic (n_class x 12)
 * atomic densities N_i (ScatteringContext.element_weights, dlra.py:240). */
int pnd_set_materials(pnd_handle* h, const int32_t* cell_class, int n_class,
                      const double* class_atomic);
/* 1/S per cell (StreamingContext.inv_s / ScatteringContext.inv_s). */
int pnd_set_inv_s(pnd_handle* h, const double* inv_s);
/* S(E_mid) per class -> inv_s and the S field on device (Problem.stopping_field,
 * driver.py:331-335, gathered per cell on the GPU). */
int pnd_set_class_stopping(pnd_handle* h, const double* class_s);
/* g_diags (12 x m) and sigma_t (12) of Problem.scattering_tables (driver.py:337-362). */
int pnd_set_scattering(pnd_handle* h, const double* g_diags, const double* sigma_t);
/* Uncollided sources [(psi_u (n), T_M (m))] (ScatteringContext.sources). */
int pnd_set_sources(pnd_handle* h, int n_beams, const double* psi, const double* t_m);
/* Device-resident group table of one beam's uncollided flux (UncollidedFlux.values,
 * n x G row-major) and its T_M; pnd_select_flux then forms at_energy() on the GPU
 * (raytracer.py:440-449): which = 0 -> source slice (E_mid), 1 -> tally slice (E_lo). */
int pnd_set_flux_table(pnd_handle* h, int beam, int n_beams, int n_groups, const double* values,
                       const double* t_m);
int pnd_select_flux(pnd_handle* h, int which, const int32_t* j0, const double* w0,
                    const int32_t* j1, const double* w1);
/* The same group table stored on its ray footprint only (trace_beam deposits
 * into the cells its rays cross, raytracer.py:509-519): cells (nnz, strictly
 * increasing) and their values (nnz x G row-major); at_energy() is 0 in every
 * other cell. A traced pencil beam touches a small fraction of a 256^3 grid,
 * whose dense table would be 17 GB per beam at 128 groups. */
int pnd_set_flux_table_sparse(pnd_handle* h, int beam, int n_beams, int n_groups, int nnz,
                              const int32_t* cells, const double* values, const double* t_m);
/* Per-step coefficient assembly on the device: the
 * tables behind Problem.class_stopping (stopping.py:48-56, 107-120: log E and
 * log S per element, 12 x K), Problem.scattering_tables (driver.py:277-362,
 * angular.py:217-248: moment-table energies (P), Boltzmann moments 12 x P x nd,
 * Fokker-Planck xi1 12 x P; model 0 Boltzmann / 1 Fokker-Planck) and the
 * uncollided group grids ((e_min, e_max) per beam, raytracer.py:440-449), uploaded
 * once. Needs pnd_set_materials and, for the sources, pnd_set_flux_table. */
int pnd_set_coefficient_tables(pnd_handle* h, int k, const double* log_e, const double* log_s,
                               const double* class_density, const double* class_weights, int p,
                               const double* mom_e, int nd, const double* mom_g,
                               const double* mom_xi1, int model, int pn_order,
                               int boltzmann_correction, double fp_correction_scale,
                               int n_beams, const double* flux_range);
/* driver.step_contexts (driver.py:523-538) on the device: S and 1/S per cell, the
 * scattering tables and the uncollided slice at e_mid (+ the tally slice at e_lo
 * when want_lo), with no host->device copy. */
int pnd_coefficients_at(pnd_handle* h, double e_mid, double e_lo, int want_lo);
/* Read back the current coefficients (tests): class S (n_cls), g_diags (12 x m),
 * sigma_t (12), psi and psi_lo (n_beams x n each; null to skip). */
int pnd_get_coefficients(pnd_handle* h, double* class_s, double* g_diags, double* sigma_t,
                         double* psi, double* psi_lo);

/* Per-element Legendre moments of the screened elastic kernel on an energy
 * grid -- MomentTables (driver.py:269-307) via legendre_moments
 * (physics/moliere.py:111-147): the de-peaked Gauss-Legendre quadrature with
 * nn and 2 nn nodes per piece (x1/w1, x2/w2: numpy leggauss nodes) and the
 * doubled-node convergence test (rtol; NumericalError "did not converge").
 * z, a: atomic and mass numbers of the n_el elements; g is n_el x n_e x
 * (max_degree + 1), xi1 n_el x n_e, both per atom [cm^2], the 2 nn results. */
int pnd_moment_tables(pnd_handle* h, int n_e, const double* energies, int n_el,
                      const int32_t* z, const int32_t* a, int nn, const double* x1,
                      const double* w1, const double* x2, const double* w2, int max_degree,
                      double exponent, double rtol, double* g, double* xi1);

/* ---- full-rank oracle on the device (fullrank.py:16-45) --
 * The dense n x m moment matrix (u, row-major on the host) kept on the GPU in
 * 32-column blocks; the streaming step is RK4 on apply_streaming (the K-stage
 * kernel block by block), the scattering step implicit Euler on the
 * self-scattering rates plus the explicit source (same contexts as the
 * low-rank steps). pnd_fullrank_step = streaming + scattering + dose tally
 * (driver.py:607-621). */
int pnd_fullrank_reset(pnd_handle* h);
int pnd_fullrank_set(pnd_handle* h, const double* u);
int pnd_fullrank_get(pnd_handle* h, double* u);
int pnd_fullrank_streaming_step(pnd_handle* h, double dt);
int pnd_fullrank_scattering_step(pnd_handle* h, double dt);
int pnd_fullrank_step(pnd_handle* h, double dt, int tally_steps);

/* ---- low-rank state (LowRankState, dlra.py:46-72) --------------------- */
int pnd_state_set(pnd_handle* h, int ru, int rv, const double* u, const double* s, const double* v);
int pnd_state_shape(pnd_handle* h, int* ru, int* rv);
int pnd_state_get(pnd_handle* h, double* u, double* s, double* v);

/* ---- the hot path ----------------------------------------------------- */
/* streaming_step(state, dt, ctx) (dlra.py:213-225): state -> augmented state. */
int pnd_streaming_step(pnd_handle* h, double dt);
/* scattering_step(state, dt, ctx) (dlra.py:270-322). */
int pnd_scattering_step(pnd_handle* h, double dt);
/* truncate(state, TruncationPolicy(theta, rank_min, rank_max)) (dlra.py:90-115). */
int pnd_truncate(pnd_handle* h, double theta, int rank_min, int rank_max, double* tail,
                 int* rank);
/* one step of the energy loop (driver.py:578-622): streaming, truncate
 * (truncate_after & 1), scattering, truncate (truncate_after & 2), dose
 * trapezoid; tally_steps adds S * sum_b psi_b(E_lo) to the integrand.
 * out[0..7] = tail after streaming, tail after scattering, rank, defect
 * (defect only when want_defect != 0), the (U, V) ranks entering the
 * streaming substep and entering the scattering substep (the driver's
 * augmented-size diagnostics, driver.py:583-601).
 * On small single-device grids (n x rank <= 2^22) with truncation after both
 * substeps the step runs speculatively: the augmentation and truncation
 * ranks are predicted on the host (full increments, last step's ranks), the
 * whole step is launched without a host round trip and the device flags a
 * wrong prediction; the one synchronisation at the end either accepts the
 * step or restores the state and recomputes it on the synchronous path, so
 * the result is the same either way (PND_NO_SPEC=1 disables it). */
int pnd_step(pnd_handle* h, double dt, double theta, int rank_min, int rank_max,
             int truncate_after, int tally_steps, int want_defect, double* out);
/* speculative steps accepted / recomputed so far (two long longs) */
int pnd_spec_stats(pnd_handle* h, long long* hits_misses);
int pnd_dose_reset(pnd_handle* h);
int pnd_dose_accumulate(pnd_handle* h, double dt, int tally_steps);
int pnd_get_dose(pnd_handle* h, double* deposited);
/* Checkpoint / resume at a step boundary (a LowRankState
 * snapshot plus the dose trapezoid's running sum and previous integrand,
 * driver.py:613-621): read and restore the tally (n values each); the
 * factors go through pnd_state_get / pnd_state_set. */
int pnd_dose_state(pnd_handle* h, double* deposited, double* prev);
int pnd_dose_restore(pnd_handle* h, const double* deposited, const double* prev);
/* LowRankState.orthonormality_defect() (dlra.py:67-70) on the device state. */
int pnd_orth_defect(pnd_handle* h, double* defect);

/* ---- unit-parity entry points (host in / host out) -------------------- */
/* apply_streaming(u, inv_s, stencils, ops) (spatial.py:148-167), m <= 64. */
int pnd_apply_streaming(pnd_handle* h, const double* u, double* out);
/* [X^T D_s S^-1 Y] for every stencil s (the L/S-phase factors of
 * dlra.py:183-184, 199-209); out is ns x a x b. */
int pnd_stencil_grams(pnd_handle* h, const double* x, int a, const double* y, int b,
                      double* out);
/* k_rhs(K, F) = -sum_s (D_s S^-1 K) F_s (dlra.py:168-174); f is ns x r x r. */
int pnd_k_rhs(pnd_handle* h, const double* k, int r, const double* f, double* out);
/* The n-side augmentation of streaming_step / scattering_step (the span of
 * orthonormal_columns([K1, U0]), dlra.py:26-43, 220, 304): u (n x a, orthonormal
 * columns) and an increment x (n x b); q (n x b, row-major) receives, in its
 * first *k_out columns, an orthonormal basis of (I - u u^T) x as the device
 * computes it in the step (Gram-based CGS2 + SVQB with the graded-increment
 * second level); rank_bound <= 0 means none. */
int pnd_augment_basis(pnd_handle* h, const double* u, int a, const double* x, int b,
                      int rank_bound, double* q, int* k_out);
/* orthonormal_columns(a) (dlra.py:26-43) via device TSQR; q is rows x min(rows, cols),
 * r is min(rows, cols) x cols. Independent of the handle's grid. */
int pnd_orthonormalize(pnd_handle* h, const double* a, int rows, int cols, double* q, double* r);
/* np.linalg.svd(s, full_matrices=False) of a p x q matrix (dlra.py:99). */
int pnd_svd_small(pnd_handle* h, const double* s, int p, int q, double* pm, double* sig,
                  double* qt);

/* ---- uncollided ray traversal (raytracer.py:353-403) ------------------ */
/* Amanatides-Woo walk of n_rays rays through the handle's grid (origin given),
 * bit-exact with the reference. Pass cells == NULL to get only counts
 * (counts[i] = segments of ray i); otherwise offsets (n_rays + 1, exclusive
 * scan of counts) place ray i's segments at [offsets[i], offsets[i+1]). */
int pnd_traverse(pnd_handle* h, const double* origin3, int n_rays, const double* starts,
                 const double* dirs, int32_t* counts, const int64_t* offsets, int64_t* cells,
                 double* t0, double* t1);

/* ---- uncollided flux: energy march + deposit ---------------------------- */
/* Crank-Nicolson march of a batch of distinct ray signatures (march_ray,
 * raytracer.py:285-350). gmats: n_keys dense (ng*nl)^2 energy operators G
 * (assemble_energy_operators, raytracer.py:169-274; block tridiagonal);
 * steppers = distinct (key, dz) pairs (the reference's LU cache), with the dz
 * each was first built at; per march segment two halves (dz, substeps,
 * stepper). Outputs per segment the group averages after the first half and
 * the below-cutoff residual energy; psi_exit per march (may be NULL).
 * NumericalError "Crank-Nicolson solve failed" / "non-finite flux" as the
 * reference. */
int pnd_march(pnd_handle* h, int nl, int ng, int n_keys, const double* gmats,
              const double* mass, const double* p_lo, double e_min, const double* s_min,
              const double* psi0, int n_steppers, const int32_t* st_key, const double* st_dz,
              int n_marches, const int32_t* seg_off, const int32_t* seg_key,
              const double* half_dz, const int32_t* half_n, const int32_t* half_st,
              double* averages, double* residual, double* psi_exit);
/* track-length deposit of trace_beam (raytracer.py:509-519), rays in
 * enumeration order: values (n x ng row-major) += w * len/V * averages,
 * residual (n) += w * res / V; segments of ray r are [ray_seg_off[r],
 * ray_seg_off[r+1]) and map onto march ray_march[r]'s segments. */
int pnd_deposit(pnd_handle* h, int ng, int n_rays, const int32_t* ray_seg_off,
                const int64_t* cells, const double* lengths, const int32_t* ray_march,
                const int32_t* march_seg_off, const double* weight, double volume,
                int n_march_segs, const double* averages, const double* mres, double* values,
                double* residual);

/* ---- z-slab decomposition (one process per GPU) -------- */
/* NCCL unique id (128 bytes) made on rank 0 and broadcast by the caller */
int pnd_comm_unique_id(char* out128);
/* This handle's grid (nx, ny, nz) is planes [z0, z0 + nz) of a grid with
 * nz_global planes; with world > 1 the stencil halo planes and every Gram sum
 * go over NCCL (comm.cu). Call right after pnd_create. */
int pnd_set_slab(pnd_handle* h, int z0, int nz_global, const char* id128, int rank, int world);

/* ---- measurement and synthetic inputs (bench.py) ------------------------ */
/* phase timer (CUDA events on the handle stream around every phase of the step) */
int pnd_timing(pnd_handle* h, int enable);
int pnd_timing_get(pnd_handle* h, int nphase, double* ms, int* count);
int pnd_event_record(pnd_handle* h, int slot);
int pnd_event_elapsed(pnd_handle* h, int slot_a, int slot_b, double* ms);
/* kernels launched by this process since load */
int pnd_launch_count(pnd_handle* h, long long* count);
/* uncollided group table of a +z pencil beam in a laterally uniform phantom:
 * values[c][g] = lateral[j*nx + i] * depth[k*G + g]; only the two factors are
 * kept on the device and each step's flux slices are formed from them (the
 * dense n x G table is 137 GB per beam at 512^3 x 128 groups) */
int pnd_set_flux_separable(pnd_handle* h, int beam, int n_beams, int n_groups,
                           const double* lateral, const double* depth, const double* t_m);
/* preset rank-r state: orthonormalised pseudo-random U, V; S = diag(logspace(0, -3, r)) */
int pnd_state_random(pnd_handle* h, int r, unsigned long long seed);

#ifdef __cplusplus
}
#endif

#endif /* PNDOSE_B200_H */
