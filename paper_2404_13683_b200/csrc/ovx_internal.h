// ovx_internal.h — declarations shared by the C-ABI layer (capi.cu) and the kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ovx {

constexpr int kMaxMat = 256;   // constant-table size; id 255 is the reserved zero material
constexpr int kZeroMat = kMaxMat - 1;
constexpr int kMaxSrc = 16;
constexpr int kMaxRec = 32;

// Per-material constants, computed on the host in the operation order the
// oracle's definition fixes (DESIGN.md §Integer path):
//   cG = (2G)/(3κ)   c1 = κ ds/256   c2 = (256G)/(3κ)     (Eq. 9)
//   ck = κ ds/256    cg = G ds/384                           (FP64 path: κ ds A_κ + G ds A_G)
//   L0..C2: factored FP64 path, (ds/16)(3/4)^k λ and μ, λ = κ − 2G/3, μ = G
struct MatConst {
    double cG, c1, c2, ck, cg, rho_vol8;
    double L0, M0, M0x2, L1, M1, M1x3, C2;
    double vl[3], vm[3];   // factored VFEM: (ds/16)·3^{-|T|}·λ and ·μ for |T| = 0, 1, 2
};

enum Mode { MODE_STEP = 0, MODE_APPLY = 1, MODE_DEBUG = 2 };

struct StepParams {
    int64_t nx, ny, nz;
    const MatConst *mc;   // the context's material table (device, kMaxMat entries; kZeroMat = zeros)
    int kset;             // dense matrices of step_v1: 0 OVFEM (K^κ, K̄^G + 128 I), 1 VFEM (Vk, Vg)
    const double *u;      // u^{it} (3 per node)
    double *uo;           // MODE_STEP: in u^{it-1}, out u^{it+1}
    const double *w;      // dt²/m per node
    const uint8_t *mat;   // material id per element
    const uint8_t *dmask; // Dirichlet mask per node (may be null)
    double *fout;         // MODE_APPLY / MODE_DEBUG: f = K u
    int nsrc;
    int64_t src_dof[kMaxSrc];
    double src_val[kMaxSrc];
    // receivers (Table 1 observation points): u^{it+1} of node rec_node[k] is stored at
    // traces[(3k + c)·rec_nt + it] when it < rec_nt
    int nrec;
    int64_t rec_node[kMaxRec];
    double *traces;
    int64_t it, rec_nt;
    // z-slab decomposition (multi-GPU): bit 0 = local plane 0 is an interface
    // owned by this rank (its lower-layer partial arrives from below), bit 1 = the top local
    // plane is an interface owned by the rank above (send its partial, do not update it)
    // Rayleigh damping (reading R1, MODE_STEP only): the EBE input is ũ = u + cb·(u − u_prev) and
    // u^{it+1} = fma(w, F − K ũ, (2u − u_prev) − ca·(u − u_prev)), written to un (a third buffer:
    // halo nodes read u_prev, so the update cannot be in place)
    int damped;
    double ca, cb;         // RN(alpha·dt), RN(beta/dt)
    double *un;
    int stages;            // INT8 path: M (4, 6 or 8)
    int direct;            // INT8 path: the direct N-stage conversion (OVX_INT8_DIRECT, NEXT-4)
    int nmat;              // materials in mc[0, nmat) (ids < 255; 255 = zero material)
    int slab_flags;
    double *iface_top_A;   // [NX1*NY1][3]   partial force of the top plane (bit 1)
    double *iface_bot_b;   // [NX1*NY1][3] the layer-0 bottom-face sum B of plane 0 (bit 0)
    // tiling
    int tiles_x, tiles_y, zchunk;
    int tz0;               // first z-chunk of this launch (z-slab overlap: edge chunks, then the interior)
    // MODE_DEBUG outputs for elements [dbg_e0, dbg_e0 + dbg_ne)
    int64_t dbg_e0, dbg_ne;
    double *dbg_s;
    int64_t *dbg_v;
    uint8_t *dbg_d;
    int32_t *dbg_C;
    int64_t *dbg_yhi, *dbg_ylo;
    double *dbg_fe;
};

struct LaunchInfo {
    int64_t ctas;
    int threads;
    int smem;
};

// kernels.cu
// The element matrices, which are the same for every context: K_e^INT8 (and the INT8 kernels' B-operand
// images built from it) and the dense integer matrices of both elements (kk, kg: 2 × 576, OVFEM then
// VFEM).  Uploaded once per device, synchronously; per-context data (materials) never goes to
// __constant__ memory, so contexts on one device are independent.
cudaError_t upload_device_constants(const int8_t *k8, const double *kk2, const double *kg2);
LaunchInfo step_launch_info(int path, int64_t nx, int64_t ny, int64_t nz);
// part: -1 all z-chunks; 0 the first and the last chunk (the ones holding interface planes);
// 1 the others.  Launching part 0 then part 1 computes the same step as part -1.
cudaError_t launch_step(int path, int mode, StepParams p, cudaStream_t st, int part = -1, int *nlaunch = nullptr);
cudaError_t launch_node_w(int64_t nx, int64_t ny, int64_t nz, const uint8_t *mat, const uint8_t *mat_below,
                          const MatConst *mc, double dt, double *w, cudaStream_t st);
cudaError_t launch_iface_update(const StepParams &p, const double *a_recv, double *u_send, cudaStream_t st);
cudaError_t launch_finite_check(const double *u, int64_t n, int *flag, cudaStream_t st);
cudaError_t launch_power_iter(int64_t nn, const double *x, const double *y, const double *w, const uint8_t *dmask,
                              double dt2, double *z, double *acc, double *xnext, cudaStream_t st);

// element_setup.cpp
int derive_element_matrices(int8_t *k8, double *Ak, double *Ag);
int derive_vfem_matrices(double *Vk, double *Vg);
double sym_lambda_max(const double *A);

}  // namespace ovx
