/*
 * libvelreg_b200 -- C ABI of the B200-native (sm_100a) registration hot path.
 *
 * Drop-in boundary for the stationary-velocity Gauss-Newton-Krylov path of the
 * reference package `velreg` (/root/reference/pkg/src/velreg).  The reference
 * has no FFI layer: its operators are Python functions over numpy arrays and
 * its only native code is the numba kernel call
 *     kern(vals, px, py, pz, out, h1, h2, h3)          (interp.py:127)
 * Every entry below replaces one of those Python operators; the Python host
 * package (paper_2209_08189_b200/) keeps the reference's names, argument
 * meaning and exception classes on top of it.
 *
 * Conventions
 *  - All pointers are DEVICE pointers unless stated; the caller owns them.
 *  - dims = {N1, N2, N3}, C order, x3 contiguous (grid.py:3-5); vector fields
 *    are SoA float[3][N1][N2][N3] (grid.py:99).  One field must have < 2^31
 *    voxels.
 *  - Characteristics are displacements in index units: the departure point of
 *    voxel (i,j,k) is (i-d1, j-d2, k-d3).
 *  - Alignment: field pointers need only 4-byte (float) alignment.  The
 *    shared-memory-staged cubic sweeps (cp.async.bulk) are used only when the
 *    source pointers (src / ghost blocks) are 16-byte aligned; otherwise the
 *    direct gather runs (same results).  torch / cudaMalloc allocations are
 *    256-byte aligned.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  All calls are
 *    asynchronous; reductions write f64 results to device memory.
 *  - Return 0 on success, negative VR_ERR_* on invalid arguments / launch
 *    failure.  Non-finite results are reported through an optional device int
 *    flag (set to non-zero), read back where the reference checks
 *    (transport.py:57-59,119-121; optim.py:157-158,179-180).
 */
#ifndef VELREG_B200_H
#define VELREG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VR_ORDER_LINEAR 1
#define VR_ORDER_CUBIC 3

/* spectral operator kinds (diffops.py:108-154) */
#define VR_SPEC_IDENTITY 0  /* FFT round trip (SpectralWorkspace.forward/inverse, diffops.py:51-55) */
#define VR_SPEC_A 1         /* apply_A, symbol |k|^2 (diffops.py:116-118) */
#define VR_SPEC_INVSHIFT 2  /* apply_inv_shifted_A, 1/(beta_v|k|^2+shift) (diffops.py:121-126) */
#define VR_SPEC_K 3         /* apply_K Leray blend (diffops.py:129-146) */
#define VR_SPEC_GAUSS 4     /* Gaussian smoothing exp(-sigma^2|k|^2/2) (north-star extra, no ref) */
#define VR_SPEC_A2 5        /* H2 operator |k|^4 (north-star extra, no ref) */
#define VR_SPEC_INVSHIFT2 6 /* 1/(beta_v|k|^4+shift) (north-star extra, no ref) */

#define VR_RED_SUM 0
#define VR_RED_MINMAX 1

typedef struct vr_spec_plan vr_spec_plan;

/* ---- interpolation (interp.py:112-128 interpolate_values) ------------------
 * out[p] = periodic trilinear (order 1) / tricubic-Lagrange (order 3)
 * interpolant of src at points pts[0..2][p] given in RADIANS (any finite
 * value; wrapped).  pts is float32 (pts_is_f64 = 0) or float64 (1). */
int vr_interp_points(const float* src, const int64_t dims[3], const void* pts, int pts_is_f64, int64_t npts,
                     int order, float* out, void* stream);

/* ---- characteristics (transport.py:66-76 trace_characteristics and
 * transport.py:94-110 TransportOperators.__init__) ----------------------------
 * Forward and backward RK2 traces of velocity v (3 x N, rad / unit time).
 * If div != NULL also the trapezoidal source factors
 *   fac_jac = jac_numer/jac_denom, fac_adj = adj_numer/adj_denom. */
int vr_trace_rk2(const float* v, const int64_t dims[3], double dt, int order, float* disp_fwd, float* disp_bwd,
                 const float* div, float* fac_jac, float* fac_adj, void* stream);

/* displacement -> absolute points wrapped to [0, 2pi) (Characteristics.points) */
int vr_disp_to_points(const float* disp, const int64_t dims[3], double* pts, void* stream);

/* Tuning switch (no reference counterpart) for the semi-Lagrangian sweeps:
 * 1 (default) = shared-memory-staged gathers (stage_tma.cuh; rows of a multiple
 * of 32 voxels), 0 = direct per-point gathers.  Same results (same taps and
 * arithmetic order).  Returns the previous mode. */
int vr_set_gather_mode(int mode);

/* Tuning switch (no reference counterpart) for the power-of-two spectral path:
 * 1 (default) = four-step register FFT kernels where they apply (spectral_4step.cuh),
 * 0 = radix-8 Stockham kernels only.  Returns the previous mode. */
int vr_set_fft_mode(int mode);

/* Tuning switch (no reference counterpart) for VR_SPEC_A: 1 (default) = the
 * separable f64 line engine (spectral_d2.cuh: A = D11 + D22 + D33, each a 1-D
 * f64 transform pair per line, for line lengths 128 / 256), 0 = the 3-D path
 * with an f64 forward half.  Returns the previous mode. */
int vr_set_spec_a_mode(int mode);

/* Tuning switches of the spectral engine (no reference counterpart; results
 * agree to rounding).  key 1: run component-diagonal symbols (A, shifted
 * inverses, Gaussian) on 3-component fields one component at a time (value 1)
 * or all components per pass (0, default; measured faster on B200).  Returns the previous value, or
 * VR_ERR_ARG for an unknown key. */
int vr_set_spectral_tuning(int key, int value);

/* Tuning switch (no reference counterpart) for FD8: 0 (default) = the
 * cp.async tile kernel, 1 = row-tile kernel staging whole x3 rows with
 * cp.async.bulk (N3 in {128, 256}, 16-byte-aligned fields; measured slower).
 * Bit-identical results.  Returns the previous mode. */
int vr_set_fd8_mode(int mode);

/* Number of kernel launches one vr_spec_apply(p, kind, ., ncomp, ...) makes
 * with the current tuning (launch accounting for benchmarks). */
int vr_spec_apply_launches(const vr_spec_plan* p, int kind, int ncomp);

/* Tuning switch (no reference counterpart) for the single-domain RK2 trace:
 * 0 (default) = general flat-index gathers, 1 = lean periodic gathers on a 3-D
 * launch (measured slower: 3.83 vs 2.41 ms at C2 cubic).  Same taps; summation
 * order may differ by an ulp.  Returns the previous mode. */
int vr_set_trace_mode(int mode);

/* ---- semi-Lagrangian sweeps -------------------------------------------------
 * one step dst = interp(src, X) [* factor]:
 *   state    transport.py:130-133 (factor NULL, forward trace)
 *   adjoint  transport.py:154-155 (factor = fac_adj, backward trace)
 *   Jacobian transport.py:194-195 (factor = fac_jac, forward trace) */
int vr_advect(const float* src, const int64_t dims[3], const float* disp, const float* factor, int order,
              float* dst, int* nonfinite_flag, void* stream);

/* incremental state (transport.py:160-185): u0 = dt/2 * s_0, s_j = -vt.grad m^j */
int vr_incstate_init(const float* vt, const float* gradm0, const int64_t dims[3], double dt, float* u0,
                     void* stream);
/* m~_{j+1} = interp(u_j) + dt/2 s_{j+1}; writes u_{j+1} = m~_{j+1} + dt/2 s_{j+1}
 * (last = 0), m~_n itself (last = 1) or -m~_n, the incremental adjoint's final
 * condition (optim.py:206), (last = 2) */
int vr_incstate_step(const float* u, const int64_t dims[3], const float* disp_fwd, const float* vt,
                     const float* gradm_next, double dt, int order, int last, float* out, int* nonfinite_flag,
                     void* stream);

/* trapezoidal body force sum_j w_j lam^j grad m^j (optim.py:162-171);
 * lam_series (n_t+1) x N, gradm_series (n_t+1) x 3 x N */
int vr_body_force(const float* lam_series, const float* gradm_series, int n_t, const int64_t dims[3], double dt,
                  float* out, void* stream);

/* Lean layout (no stored grad-m series): one term j of the same trapezoid,
 * weight w_j = dt/2 at the ends and dt inside, with an f64 accumulator acc
 * (3 x N doubles).  mode 0 = first term (acc = term), 1 = middle (acc +=),
 * 2 = last (acc += term, out = (float)acc).  Calling it for j = 0..n_t in order
 * reproduces vr_body_force bit for bit (optim.py:162-171 accumulates in f64). */
int vr_body_force_term(const float* lam, const float* gradm, const int64_t dims[3], double weight, int mode,
                       double* acc, float* out, void* stream);

/* label transport step (synth.py:121-131): source = labels_in==label_id
 * (if labels_in) else src; destination = float field (dst) or thresholded
 * write of label_id where value >= 0.5 (labels_out). */
int vr_label_step(const float* src, const int* labels_in, int label_id, const int64_t dims[3], const float* disp,
                  int order, float* dst, int* labels_out, void* stream);

/* ---- FD8 (diffops.py:84-105); bit-identical to numpy for float32 input ---- */
int vr_fd8_grad(const float* f, const int64_t dims[3], float* out3, void* stream);
int vr_fd8_div(const float* v3, const int64_t dims[3], float* out, void* stream);

/* ---- spectral (diffops.py:24-55 SpectralWorkspace; :108-154 operators) ---- */
int vr_spec_plan_create(const int64_t dims[3], vr_spec_plan** plan);
int vr_spec_plan_destroy(vr_spec_plan* plan);
int vr_spec_plan_dims(const vr_spec_plan* plan, int64_t dims_out[3]);
/* out = alpha * irfftn(symbol * rfftn(in)) [+ add] for ncomp (1 or 3) components */
int vr_spec_apply(vr_spec_plan* plan, int kind, const float* in, int ncomp, double beta_v, double beta_w,
                  double shift, double sigma, double alpha, const float* add, float* out, void* stream);
/* prolong_spectral (grid.py:181-226): `in` on plan_coarse's grid (ncomp
 * components) -> `out` on plan_fine's grid (each fine dim >= coarse dim). */
int vr_prolong_spectral(vr_spec_plan* plan_coarse, vr_spec_plan* plan_fine, const float* in, int ncomp,
                        float* out, void* stream);
/* h1_energy (diffops.py:149-154) -> *out_dev */
int vr_h1_energy(vr_spec_plan* plan, const float* f, double* out_dev, void* stream);

/* ---- reductions (optim.py:80-85,231-258; grid.py:129-130) -----------------
 * scratch: device f64 buffer of vr_reduce_scratch_doubles() entries. */
int vr_reduce_scratch_doubles(void);
/* out[q] = sum_i a[q][i]*b[q][i], q < k <= 4 (a, b: HOST arrays of device ptrs) */
int vr_dots(int k, const float* const* a, const float* const* b, int64_t n, double* scratch, double* out,
            void* stream);
/* out2 = {sum (a-b)^2, sum (c-b)^2} (c may be NULL) -- relative_residual */
int vr_sqdiff(const float* a, const float* b, const float* c, int64_t n, double* scratch, double* out2,
              void* stream);
/* out4 = {min a, max a, min b, max b} -- _intensity_shift, J extrema */
int vr_minmax(const float* a, const float* b, int64_t n, double* scratch, double* out4, void* stream);
/* out4 = {-max|v|^2, max|v|^2, #non-finite, #non-zero} over a 3 x n field */
int vr_vecstats(const float* v, int64_t n, double* scratch, double* out4, void* stream);

/* ---- vector updates --------------------------------------------------------- */
int vr_axpby(int64_t n, double a, const float* x, double b, const float* y, float* out, void* stream);
int vr_pcg_update(int64_t n, double alpha, const float* p, const float* hp, float* x, float* r, void* stream);
/* PCG step with a device step length: alpha = *rz_dev / *php_dev (f64), then
 * x_out = x + alpha p, r_out = r - alpha hp (f64 arithmetic, f32 storage);
 * outputs may alias inputs. */
int vr_pcg_update2(int64_t n, const double* rz_dev, const double* php_dev, const float* p, const float* hp,
                   const float* x, const float* r, float* x_out, float* r_out, void* stream);
int vr_fill(int64_t n, float value, float* out, void* stream);

/* ---- SYN benchmark template (synth.py:77-101 make_template) -------------------
 * labels / image (either may be NULL) of x1 planes [x_begin, x_begin + x_count)
 * of the global lattice dims: the largest shape index s + 1 whose star shape
 * |u| <= norm |P_l^m(cos(phi(u) + phi_hat_s))| covers the voxel, u = (x - pi)
 * - c_s; or |u| <= fixed_radius when fixed_radius >= 0.  shapes_host: HOST
 * doubles {c1, c2, c3, phi_hat} per shape (the reference's default_rng draws);
 * norm = |Y_l^m| normalisation, dfact_m = (2m-1)!! (host f64, synth.py:51,69). */
int vr_syn_template(const int64_t dims[3], int x_begin, int x_count, const double* shapes_host, int nshapes, int l,
                    int m, double norm, double dfact_m, double fixed_radius, int* labels, float* image,
                    void* stream);

/* (min l0, max l0, min l1, max l1) of one or two int32 label maps (l1 may be
 * NULL), written to out[4] (int32, device).  Validates label ids (grid.py
 * LabelMap, non-negative) and sizes vr_label_counts with one host read. */
int vr_label_range(const int* l0, const int* l1, int64_t n, int* out, void* stream);

/* ---- Dice counts (metrics.py:45-57,72-73) ------------------------------------
 * counts[3*id+{0,1,2}] = |l0==id|, |l1==id|, |l0==id & l1==id|, id <= max_id */
int vr_label_counts(const int* l0, const int* l1, int64_t n, int max_id, unsigned long long* counts,
                    void* stream);

/* ---- x1-slab (multi-GPU) variants ---------------------------------------------
 * A rank owns x1 planes [r*L1, (r+1)*L1) of every field.  A gathered source is
 * passed as its local slab plus two ghost blocks of w planes each: `*_lo` holds
 * the w planes before the slab, `*_hi` the w planes after it (filled by the
 * host's NCCL halo exchange, paper_2209_08189_b200/dist.py; vector sources have
 * ghost blocks of shape (3, w, N2, N3)).  dims are the LOCAL (L1, N2, N3);
 * outputs are local.  w must cover the largest x1 displacement plus the stencil
 * (the host sizes it from an allreduce-max of the velocity). */
/* trace on a slab: v_ext (3, L1+2w, N2, N3) and div_ext (L1+2w, N2, N3) are
 * contiguous ghost-extended copies (built once per velocity iterate) */
int vr_trace_rk2_slab(const float* v_ext, const int64_t dims[3], int64_t n1_global, int w, double dt, int order,
                      float* disp_fwd, float* disp_bwd, const float* div_ext, float* fac_jac, float* fac_adj,
                      void* stream);
/* sweeps on a slab cover output planes [x_begin, x_begin + x_count): planes
 * [w, L1 - w) never touch the ghosts, so the host sweeps them while the ghost
 * exchange is in flight and the 2w boundary planes afterwards */
int vr_advect_slab(const float* src, const float* src_lo, const float* src_hi, const int64_t dims[3], int w,
                   const float* disp, const float* factor, int order, float* dst, int* nonfinite_flag, int x_begin,
                   int x_count, void* stream);
int vr_incstate_step_slab(const float* u, const float* u_lo, const float* u_hi, const int64_t dims[3], int w,
                          const float* disp_fwd, const float* vt, const float* gradm_next, double dt, int order,
                          int last, float* out, int* nonfinite_flag, int x_begin, int x_count, void* stream);
int vr_label_step_slab(const float* src, const float* src_lo, const float* src_hi, int label_id,
                       const int64_t dims[3], int w, const float* disp, int order, float* dst, int* labels_out,
                       void* stream);
/* FD8 on a slab: ghost blocks of exactly 4 planes (component 0 only for the
 * divergence: x1 derivatives are taken of v1 alone) */
int vr_fd8_grad_slab(const float* f, const float* f_lo, const float* f_hi, const int64_t dims[3], int64_t n1_global,
                     float* out3, void* stream);
int vr_fd8_div_slab(const float* v3, const float* v1_lo, const float* v1_hi, const int64_t dims[3],
                    int64_t n1_global, float* out, void* stream);

/* distributed spectral operator = forward (x3, x2 local + pack) -> host
 * all-to-all per component -> X pass on x1 lines -> host all-to-all back ->
 * inverse (unpack + x2, x3).  pl: plan of the local slab (L1, N2, N3); px: plan
 * of the transposed block (N1, N2/P, N3).  Power-of-two sizes only. */
int vr_spec_plan_is_fast(const vr_spec_plan* plan);
int vr_dspec_forward(vr_spec_plan* pl, const float* in, int ncomp, int f64, int nranks, void* sendbuf, void* stream);
int vr_dspec_xpass(vr_spec_plan* px, int kind, int ncomp, int f64, double beta_v, double beta_w, double shift,
                   double sigma, double alpha, int64_t n_global, int j0, int n2_global, int l1, const void* recv,
                   void* xout, void* stream);
int vr_dspec_h1_partial(vr_spec_plan* px, const void* recv, int j0, int n2_global, int l1, double scale,
                        double* out_dev, void* stream);
int vr_dspec_inverse(vr_spec_plan* pl, const void* recv_inv, int ncomp, int nranks, const float* add, float* out,
                     void* stream);

/* Peer variants (multi-GPU over NVLink; dist.py PeerMesh): the transposes are
 * fused into the passes.  vr_dspec_forward_peer stores Y-pass row j straight
 * into rank j / L2's receive buffer dst[j / L2] (block `me`);
 * vr_dspec_xpass_peer stores x1 block p into rank p's inverse receive buffer
 * dst[p]; vr_dspec_inverse_peer reads this rank's blocked inverse receive
 * buffer directly (no unpack pass).  `dst` is a HOST array of nranks device
 * pointers (IPC mappings); nranks a power of two <= 8, N2 = 256 on the slab
 * plan (VR_ERR_UNSUPPORTED otherwise: use the packed NCCL / copy path).  The
 * caller signals completion (vr_peer_signal) after each producing call. */
int vr_dspec_forward_peer(vr_spec_plan* pl, const float* in, int ncomp, int f64, int nranks, int me,
                          void* const* dst, void* stream);
int vr_dspec_xpass_peer(vr_spec_plan* px, int kind, int ncomp, int f64, double beta_v, double beta_w, double shift,
                        double sigma, double alpha, int64_t n_global, int j0, int n2_global, int l1, const void* recv,
                        int nranks, int me, void* const* dst, void* stream);
int vr_dspec_inverse_peer(vr_spec_plan* pl, const void* recv_inv, int ncomp, int nranks, const float* add,
                          float* out, void* stream);

/* A = -Laplacian on x1 slabs through the separable line engine (replaces the
 * 3-D path above for A; reference diffops.py:116-118, optim.py:109-116).
 * pl = slab plan {L1, N2, N3}, px = block plan {N1, N2 / nranks, N3};
 * N3 and N2 in {128, 256}, N1 in {128 .. 2048} (powers of two), N2 / nranks
 * even.  Sequence per operator (one stream; the caller signals / waits the
 * epoch flags between the phases):
 *   vr_dspec_a_rows     acc = D33 in, and every slab row stored into the block
 *                       buffer blk[j / L2] ([c][N1][L2][N3] f32) of its owner
 *   vr_dspec_a_x2       acc += D22 in
 *   vr_dspec_a_x1_peer  D11 of this rank's received block, each x1 line's
 *                       values stored into back[i / L1] ([c][L1][N2][N3] f32)
 *   vr_dspec_a_final    out = alpha (acc + back) (+ add)
 * Bit-identical to vr_spec_apply(VR_SPEC_A) on the whole grid.  blk / back
 * are HOST arrays of nranks device pointers (IPC mappings). */
int vr_dspec_a_ok(const vr_spec_plan* pl, const vr_spec_plan* px, int nranks);
int vr_dspec_a_rows(vr_spec_plan* pl, vr_spec_plan* px, const float* in, int ncomp, int nranks, int me,
                    void* const* blk, void* stream);
int vr_dspec_a_x2(vr_spec_plan* pl, const float* in, int ncomp, void* stream);
int vr_dspec_a_x1_peer(vr_spec_plan* pl, vr_spec_plan* px, const float* blk_local, int ncomp, int nranks, int me,
                       void* const* back, void* stream);
int vr_dspec_a_final(vr_spec_plan* pl, const float* back_local, int ncomp, double alpha, const float* add,
                     float* out, void* stream);
/* vr_dspec_a_x2 and vr_dspec_a_final as one pass, run after the x1 exchange:
 * out = alpha ((acc + D22 in) + back) (+ add), same roundings. */
int vr_dspec_a_x2_final(vr_spec_plan* pl, const float* in, const float* back_local, int ncomp, double alpha,
                        const float* add, float* out, void* stream);

/* ---- peer-memory transport (multi-GPU, one process per GPU; dist.py) ---------
 * Symmetric buffers: vr_peer_malloc allocates (zeroed) device memory and
 * returns its CUDA IPC handle (vr_peer_handle_bytes() bytes, host memory);
 * peers map it with vr_peer_open.  vr_peer_copy = copy-engine D2D copy (dst
 * may be a peer mapping).  vr_peer_signal stores `value` into a (peer) uint64
 * flag after all prior work on `stream` (system-scope release);
 * vr_peer_wait makes `stream` wait until a local flag >= value
 * (cuStreamWaitValue64; VR_ERR_UNSUPPORTED without stream memory ops). */
int vr_peer_malloc(int64_t bytes, void** ptr, void* handle_out);
int vr_peer_free(void* ptr);
int vr_peer_open(const void* handle, void** ptr);
int vr_peer_close(void* ptr);
int vr_peer_handle_bytes(void);
int vr_peer_copy(void* dst, const void* src, int64_t bytes, void* stream);
int vr_peer_signal(unsigned long long* flag, unsigned long long value, void* stream);
/* n <= 8 flags (HOST array of device addresses) in one launch / one batched
 * stream memory operation (cuStreamBatchMemOp; falls back to n waits). */
int vr_peer_signal_many(unsigned long long* const* flags, int n, unsigned long long value, void* stream);
int vr_peer_wait_many(const unsigned long long* const* flags, int n, unsigned long long value, void* stream);
int vr_peer_wait(const unsigned long long* flag, unsigned long long value, void* stream);
/* ghost planes of a float slab src (ncomp, L1, N2, N3): planes [0, w) of every
 * component -> left_hi (ncomp, w, N2, N3), planes [L1-w, L1) -> right_lo;
 * plane = N2*N3 (multiple of 4), 16-byte-aligned (peer-mapped) pointers. */
int vr_peer_halo_put(const float* src, int ncomp, int L1, int64_t plane, int w, float* left_hi, float* right_lo,
                     void* stream);

#ifdef __cplusplus
}
#endif

#endif /* VELREG_B200_H */
