/*
 * ovx.h — C ABI of the B200-native OVFEM / TCOVFEM explicit time step
 * (arxiv 2404.13683, "Low-ordered Orthogonal Voxel Finite Element with INT8
 * Tensor Cores for GPU-based Explicit Elastic Wave Propagation Analysis").
 *
 * The library computes, per time step, the element-by-element stiffness
 * product  f = Σ_e K_e^o u_e  of the orthogonal voxel element (Eq. 5,
 * L66-L69) through the paper's integer form (Eq. 9; Eqs. 10-17,
 * L112-L146) on tcgen05 kind::i8 tensor cores, or through an FP64 CUDA-core
 * reference kernel, fused with the diagonal-mass central-difference update
 * (Eq. 3; update L263-L266 with the sign of Eq. 3).
 *
 * Conventions (all entry points)
 *  - Every function returns ovx_status.  On failure the context keeps a
 *    message readable with ovx_last_error(); the context stays usable unless
 *    the status is OVX_ECUDA (sticky device error).
 *  - ovx_ctx is opaque and not thread-safe: one host thread per context.
 *  - Host pointers are owned by the caller, read/written only during the call
 *    and never retained.  *_device variants take device pointers on the
 *    context's device, valid for the duration of the call.
 *  - Work is enqueued on the context stream (ovx_set_stream) and is
 *    asynchronous unless stated; functions returning host data synchronise.
 *  - Layouts:
 *      node (ix,iy,iz)     -> ix + (nx+1)*(iy + (ny+1)*iz)
 *      element (ex,ey,ez)  -> ex + nx*(ey + ny*ez)
 *      node arrays         3 doubles per node, node-major (x,y,z)
 *      element materials   uint8 per element (material id)
 *      Dirichlet mask      uint8 per node, bit a set = component a fixed to 0
 *      local node order    (---),(+--),(++-),(-+-),(--+),(+-+),(+++),(-++)
 *                          (Fig. 1 is missing from PAPER.md; reading Q1)
 */
#ifndef OVX_H
#define OVX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ovx_ctx ovx_ctx;
typedef int ovx_status;

enum {
    OVX_OK = 0,
    OVX_EINVAL = 2,     /* rejected input: dims <= 0, ds <= 0, unknown material id, NaN/Inf, size mismatch */
    OVX_EUNSTABLE = 3,  /* a non-finite displacement appeared (ovx_check_finite) */
    OVX_ESTATE = 6,     /* call-order violation (e.g. step before setup) */
    OVX_ECUDA = 7,      /* CUDA runtime error (message has the CUDA error string) */
    OVX_ENCCL = 8,      /* NCCL unavailable or an NCCL call failed (multi-GPU contexts) */
    OVX_ENOMEM = 9      /* device allocation failed */
};

enum {
    OVX_INT8 = 0,       /* tcgen05 kind::i8 path: Eqs. 10-17 with byte slices (DESIGN.md variant B) */
    OVX_FP64 = 1,       /* FP64 CUDA-core reference, factored form of Eq. 5 (Walsh-Hadamard of the
                           corner values, ≈180 FP64 ops/element); equal to K_e^o u_e up to rounding */
    OVX_VFEM = 3,       /* NEXT-3: the paper's conventional VFEM element (trilinear hex, exact = 2x2x2
                           Gauss integration, lumped mass), factored FP64 form
                           (Walsh-Hadamard modes) */
    OVX_VFEM_DENSE = 4, /* VFEM, literal dense form f_e = (κds/72)(Vk u_e) + (Gds/216)(Vg u_e) with
                           sequential sums (bit-exact mirror of the oracle's VFEM path) */
    OVX_FP64_DENSE = 2, /* FP64, literal dense form f_e = (κds/256)(K^κ u_e) + (Gds/384)((K̄^G+128I)u_e)
                           with sequential sums: bit-identical to the oracle's FP64 definition */
    OVX_INT8_DIRECT = 5 /* NEXT-4: the paper's DIRECT FP64→INT8 method (Fig. 2 left, Eqs. 11-14, a = 2^7,
                           N = 8 stages): every stage converts the FP64 remainder to an INT8 digit (2N
                           conversions per value instead of one), same integer image and results as the
                           hierarchical paper-digit path (L146); tensor cores as OVX_INT8.  M = 8, undamped. */
};

/* ---- lifetime ------------------------------------------------------------ */
/* Create a context on CUDA device `device` (must be sm_100).  *out is NULL on error. */
ovx_status ovx_create(int device, ovx_ctx **out);
ovx_status ovx_destroy(ovx_ctx *ctx);
/* Last error message of ctx ("" if none).  ctx may be NULL (global message). */
const char *ovx_last_error(const ovx_ctx *ctx);
/* Library version string. */
const char *ovx_version(void);
/* Order all work of ctx on `stream`, a cudaStream_t of the context's device.  NULL is the CUDA
 * default (legacy) stream; OVX_LIBRARY_STREAM gives the context its own non-blocking stream
 * (the state after ovx_create). */
#define OVX_LIBRARY_STREAM ((void *)(intptr_t)-1)
ovx_status ovx_set_stream(ovx_ctx *ctx, void *stream);

/* ---- model (cubes of side ds on a structured grid; L94: κ, G) -- */
/* Global element counts and edge length; nx,ny,nz >= 1, ds > 0.  Resets the model. */
ovx_status ovx_set_grid(ovx_ctx *ctx, int64_t nx, int64_t ny, int64_t nz, double ds);
/* n <= 255 materials; rho, kappa, G > 0 and finite (host arrays of length n). */
ovx_status ovx_set_materials(ovx_ctx *ctx, int n, const double *rho, const double *kappa,
                             const double *G);
/* Per-element material ids (host, nx*ny*nz bytes); every id < n materials. */
ovx_status ovx_set_element_materials(ovx_ctx *ctx, const uint8_t *mat);
/* Per-node Dirichlet mask (host, Nn bytes) or NULL for free surfaces (the default). */
ovx_status ovx_set_dirichlet(ovx_ctx *ctx, const uint8_t *mask);
/* Time step dt > 0 (Eq. 3). */
ovx_status ovx_set_dt(ovx_ctx *ctx, double dt);
/* Rayleigh damping C = alpha·M + beta·K ("Rayleigh damping (100--125 kHz) is
 * used"; coefficients and discretisation unstated — DESIGN.md reading R1): one (alpha, beta) for
 * the model, both finite and >= 0; (0, 0) (the default) is the undamped Eq. 3.  ovx_step then
 * advances u^{it+1} = fma(w, F − K ũ, (2u − u_prev) − RN(alpha·dt)·(u − u_prev)) with the EBE
 * input ũ = u + RN(beta/dt)·(u − u_prev) (backward-difference velocity, explicit).  Allocates a
 * third state buffer (24 B/node).  On z-slab contexts the interface update (ovx_step_iface) applies
 * the same damped recurrence and ovx_step_end rotates the three buffers.
 * ovx_apply_K is unaffected (it computes K u). */
ovx_status ovx_set_damping(ovx_ctx *ctx, double alpha, double beta);
/* Derive K_e^INT8 on the host in exact rational arithmetic,
 * check that all 1152 entries are integers in [-128,127] (L110; else OVX_EINVAL),
 * build per-material constants and the per-node w = dt²/m (Eq. 6, m_n = Σ ρ_e ds³/8).
 * path: OVX_INT8, OVX_FP64, OVX_FP64_DENSE, OVX_VFEM or OVX_VFEM_DENSE.  stages: M, the number of INT8 stages (a = 2^{7M},
 * PAPER.md Eq. 16, Table 3): 8 (FP64-class), or 4 / 6 on the INT8 path (the paper's M = 4 is
 * FP32-class); the FP64 paths require 8. */
ovx_status ovx_setup_elements(ovx_ctx *ctx, int path, int stages);
/* Copy the library's derived K_e^INT8 (24x48 row-major) to host memory. */
ovx_status ovx_get_int8_matrix(ovx_ctx *ctx, int8_t *out);
/* Stability limits of the central-difference scheme (Eq. 3; reading Q19: dt ≤ 2/√λ_max(M⁻¹K)).
 *   dt_elem_bound: 2/sqrt(max_e λ_max(M_e⁻¹ K_e)) over the materials present (host, exact element
 *                  matrices; a safe bound, 20-35 % conservative).  Needs grid and materials.
 *   dt_power_iter: 2/sqrt(λ) with λ the Rayleigh quotient xᵀKx/xᵀMx after 300 power iterations of
 *                  M⁻¹K on the assembled model (the context's own EBE product on the device, fixed
 *                  DOFs removed, deterministic start vector).  λ approaches λ_max
 *                  from below, so this dt is the sharper but not a guaranteed bound.  Needs
 *                  ovx_setup_elements and ovx_set_dt (M = dt²/w); single-GPU contexts only.
 * Either pointer may be NULL (not computed); both NULL is OVX_EINVAL. */
ovx_status ovx_critical_dt(ovx_ctx *ctx, double *dt_elem_bound, double *dt_power_iter);
/* Point sources: component axis[k] of node[k] receives amp[k*n_t + it] at step it (0 after n_t).
 * n <= 16.  (impulse force at an input point.) */
ovx_status ovx_set_sources(ovx_ctx *ctx, int n, const int64_t *node, const int32_t *axis,
                           int64_t n_t, const double *amp);

/* Receivers (Table 1 observation points, L196-L212): at every step it < n_t, the new
 * displacement u^{it+1} of node[k], component c, is recorded at trace index (3k + c)·n_t + it.
 * n <= 32; replaces any previous receiver set and zeroes the traces. */
ovx_status ovx_set_receivers(ovx_ctx *ctx, int n, const int64_t *node, int64_t n_t);
/* Copy the traces (n × 3 × n_t doubles, receiver-major, then component, then step) to host memory. */
ovx_status ovx_get_traces(ovx_ctx *ctx, double *out);

/* ---- state (u^{it}, u^{it-1}, it) is the complete state: also checkpoint/resume -- */
/* Host arrays of 3*Nn doubles (node-major xyz), caller-owned; pinned memory makes the copies DMA.
 * set: both arrays required; the uploaded state is checked on the device and a NaN/Inf anywhere
 * gives OVX_EINVAL (the state is then unset).  get: u and/or u_prev may be NULL (skipped); it may
 * be NULL.  Both synchronise the context stream. */
ovx_status ovx_set_state(ovx_ctx *ctx, const double *u, const double *u_prev, int64_t it);
ovx_status ovx_get_state(ovx_ctx *ctx, double *u, double *u_prev, int64_t *it);
ovx_status ovx_set_state_device(ovx_ctx *ctx, const double *u, const double *u_prev, int64_t it);
ovx_status ovx_get_state_device(ovx_ctx *ctx, double *u, double *u_prev, int64_t *it);

/* ---- time stepping ------------------------------------------------------- */
/* Advance n steps: u^{it+1} = fma(w, F^{it} − K u^{it}, 2u^{it} − u^{it−1}), Dirichlet
 * components forced to 0.  One fused kernel launch per step, asynchronous. */
ovx_status ovx_step(ovx_ctx *ctx, int64_t n);
/* Wait for all work on the context stream. */
ovx_status ovx_sync(ovx_ctx *ctx);
/* OVX_EUNSTABLE if u^{it} holds a NaN/Inf (synchronises). */
ovx_status ovx_check_finite(ovx_ctx *ctx);

/* ---- z-slab decomposition (multi-GPU) ---------------------
 * Rank r owns element layers [ez0, ez1) of the global grid and node planes ez0..ez1 (both
 * interface planes are stored on both neighbours).  Its context is set up with the local grid
 * (nz = ez1 - ez0).  The rank ABOVE owns (updates) each interface plane, so the result is
 * bit-identical to one GPU: the node force is f_n = T_n + B_n (reading U2: T_n, B_n =
 * pairwise sums of the 4 corner contributions of the element layer below / above the plane);
 * the rank below sends T (a_send), the owner adds its own B, updates the plane and sends it back
 * down.
 * flags: bit 0 = local plane 0 is an interface owned here (needs mat_below, the nx*ny material
 * ids of the element layer below, for its nodal mass); bit 1 = the top local plane is owned
 * by the rank above.  Call after ovx_set_element_materials, before stepping. */
ovx_status ovx_set_slab(ovx_ctx *ctx, int flags, const uint8_t *mat_below);
/* Device buffers of 3*(nx+1)*(ny+1) doubles each, owned by the caller (e.g. torch tensors used
 * by the NCCL transport): a_send (T of the top plane, written by ovx_step_begin),
 * a_recv (T from below, read by ovx_step_iface), u_send (updated plane 0, written by
 * ovx_step_iface), u_recv (updated top plane from above, read by ovx_step_end). */
ovx_status ovx_set_iface_buffers(ovx_ctx *ctx, double *a_send, double *a_recv, double *u_send, double *u_recv);
/* One slab time step in three stream-ordered parts; the caller exchanges a_send -> a_recv
 * (upwards) between begin and iface, and u_send -> u_recv (downwards) between iface and end. */
ovx_status ovx_step_begin(ovx_ctx *ctx);
ovx_status ovx_step_iface(ovx_ctx *ctx);
ovx_status ovx_step_end(ovx_ctx *ctx);
/* Overlapped form (exchange overlapped with interior compute): ovx_step_begin is
 * ovx_step_begin_part(0) (the first and last z-chunk of the slab — the CTAs that produce a_send and
 * the plane-0 partial) followed by ovx_step_begin_part(1) (the interior chunks), both on the context
 * stream.  Once part 0 has completed (an event recorded after it), the caller may exchange and call
 * ovx_step_iface_stream on another stream while part 1 runs: the interior chunks neither read nor
 * write plane 0, the top plane or the interface buffers.  ovx_step_end must be ordered after both
 * (the context stream waits for the other stream).  stream: a cudaStream_t, NULL = default stream,
 * OVX_LIBRARY_STREAM = the context stream.  Results are identical to the serial form. */
ovx_status ovx_step_begin_part(ovx_ctx *ctx, int part);
ovx_status ovx_step_iface_stream(ovx_ctx *ctx, void *stream);

/* ---- parity hooks -------------------------------------------------------- */
/* f = K u for one EBE product (same kernel as ovx_step, update disabled).
 * Host arrays of 3*Nn doubles.  Does not change the state. */
ovx_status ovx_apply_K(ovx_ctx *ctx, const double *u, double *f);
ovx_status ovx_apply_K_device(ovx_ctx *ctx, const double *u, double *f);
/* Bit-level integer-path record for elements [e0, e0+ne) of the product with the host
 * field u (3*Nn doubles), from the production kernel (INT8 path only):
 *   s[ne]            Eq. 10 scale s_e = max|ū_e|
 *   v[ne*48]         INT64 image trunc(2^56 ū_e/s_e)   (Eq. 12, a = 2^56)
 *   d[ne*8*48]       byte slices of v + 2^56, stage-major (variant B of Eq. 16)
 *   C[ne*8*24]       per-stage tensor-core products K_e^INT8 · d_j (INT32, Eq. 17)
 *   y_hi,y_lo[ne*24] y = K_e^INT8 v as a 128-bit integer (y_hi*2^64 + (uint64)y_lo)
 *   fe[ne*24]        element force f_e (Eq. 9)
 * Any output pointer may be NULL. */
ovx_status ovx_debug_element_ints(ovx_ctx *ctx, const double *u, int64_t e0, int64_t ne,
                                  double *s, int64_t *v, uint8_t *d, int32_t *C,
                                  int64_t *y_hi, int64_t *y_lo, double *fe);
/* Per-node w = dt²/m_n (host, Nn doubles). */
ovx_status ovx_get_node_w(ovx_ctx *ctx, double *w);

/* ---- instrumentation ----------------------------------------------------- */
/* Device time of the step kernels launched since the last reset, from CUDA events on
 * the context stream (synchronises); resets the counters if reset != 0. */
ovx_status ovx_get_timers(ovx_ctx *ctx, double *ms_step, int64_t *launches, int reset);
/* Number of CTAs / threads / dynamic smem bytes of the step kernel for the current model. */
ovx_status ovx_get_launch_config(ovx_ctx *ctx, int64_t *ctas, int *threads, int *smem_bytes);
/* Per-phase device time since the last reset (synchronises):
 *   ms_ebe    single GPU: the fused step kernels (EBE product, scatter and update are one kernel);
 *             distributed: from each step's start to the end of its edge z-chunks;
 *   ms_halo   distributed: from the edge z-chunks to the end of the interface exchanges and the
 *             interface update (hidden under the interior chunks when it is shorter); 0 on one GPU;
 *   ms_update 0: the update is fused into the EBE kernels (there is no separate update kernel). */
ovx_status ovx_get_phase_timers(ovx_ctx *ctx, double *ms_ebe, double *ms_halo, double *ms_update, int reset);

/* ---- multi-GPU: z-slabs (PAPER.md L288 names the multi-GPU extension as future work) --
 * The element layers are split into contiguous z-slabs balanced to ±1 layer; rank r stores node
 * planes ez0..ez1 (inclusive) and the rank ABOVE owns (updates) each interface plane.  A
 * distributed context runs the whole step in the library: per step the edge z-chunks on a
 * high-priority stream, the interior chunks concurrently on the context stream, the interface
 * partial force exchanged with NCCL point-to-point (NVLink), the owner's interface update, the
 * updated plane sent back — results identical bit for bit to one GPU.
 * On a distributed context:
 *   ovx_set_grid            takes the GLOBAL element counts; the rank's slab is derived from it;
 *   ovx_set_element_materials  the rank's layers [ez0, ez1), preceded by layer ez0-1 when rank > 0
 *                           (nx*ny*(ez1-ez0) entries, + nx*ny in front for rank > 0);
 *   ovx_set_dirichlet, ovx_set_state / ovx_get_state: the rank's node planes ez0..ez1;
 *   ovx_set_sources / ovx_set_receivers: GLOBAL node ids; a rank keeps the sources of the planes
 *                           it owns, and records only the receivers of its owned planes (the other
 *                           traces stay 0: sum the traces over the ranks);
 *   ovx_step                the distributed schedule (NCCL contexts; loopback groups use
 *                           ovx_step_group). */
/* Element layers [*ez0, *ez1) of rank `rank` among `world` for nz global layers. */
ovx_status ovx_get_partition(int64_t nz, int world, int rank, int64_t *ez0, int64_t *ez1);
/* A new NCCL unique id (128 bytes) on the rank that creates the communicator; the caller
 * broadcasts it to the other ranks (e.g. through torch.distributed).  OVX_ENCCL if libnccl.so.2
 * cannot be loaded. */
ovx_status ovx_nccl_unique_id(uint8_t out[128]);
/* A context for rank `rank` of `world` on `device`, with a library-owned NCCL communicator
 * (ncclCommInitRank: a collective call — every rank must call it).  world = 1 is a plain context. */
ovx_status ovx_create_dist(int device, int rank, int world, const uint8_t id[128], ovx_ctx **out);
/* `world` contexts (out[0..world-1], ranks in order, devices[r] each) that exchange interface
 * data by device-to-device copies inside this process: the distributed schedule without NCCL
 * (tests; several ranks may share one device, which NCCL refuses).  Step them with ovx_step_group;
 * destroy each with ovx_destroy. */
ovx_status ovx_create_group(int world, const int *devices, ovx_ctx **out);
/* n steps of all ranks of a loopback group, phase by phase in lock step (the same kernels, streams
 * and events as a distributed ovx_step, with copies in place of the NCCL calls). */
ovx_status ovx_step_group(ovx_ctx **ranks, int world, int64_t n);

#ifdef __cplusplus
}
#endif
#endif /* OVX_H */
