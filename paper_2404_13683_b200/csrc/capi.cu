// capi.cu — the C ABI declared in include/ovx.h (host-side L1/L4 logic).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <array>
#include <dlfcn.h>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ovx.h"
#include "ovx_internal.h"

using namespace ovx;

struct EventPair {
    cudaEvent_t a, b;
};

struct ovx_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::string err;
    int64_t nx = 0, ny = 0, nz = 0;
    double ds = 0;
    int nmat = 0;
    std::vector<double> rho, kappa, G;
    bool have_grid = false, have_emat = false, setup = false, have_state = false;
    double dt = 0;
    int path = OVX_INT8, stages = 8;
    uint8_t *d_mat = nullptr, *d_mask = nullptr;
    int *d_flag = nullptr;   // finiteness flag (allocated once: no cudaMalloc / cudaFree per state upload)
    double *d_u = nullptr, *d_up = nullptr, *d_w = nullptr;
    double alpha = 0, beta = 0;       // Rayleigh damping (reading R1)
    int direct = 0;                   // OVX_INT8_DIRECT: the direct N-stage conversion (NEXT-4)
    double *d_un = nullptr;           // third state buffer of damped steps
    int8_t k8[1152];
    double Ak[576], Ag[576], Kk[576], Kg[576];
    std::vector<MatConst> mc;         // host copy of the material table (kMaxMat entries)
    MatConst *d_mc = nullptr;         // the context's own device copy (kernels read it via StepParams)
    int kset = 0;                     // dense matrix set: 0 OVFEM, 1 VFEM
    int nsrc = 0;
    std::vector<int64_t> src_node;
    std::vector<int32_t> src_axis;
    int64_t n_t = 0;
    std::vector<double> amp;
    int64_t it = 0;
    int nrec = 0;
    std::vector<int64_t> rec_node;
    int64_t rec_nt = 0;
    double *d_traces = nullptr;
    std::vector<EventPair> ev_used, ev_free;
    int64_t launches = 0;
    // z-slab (multi-GPU) state
    int slab_flags = 0;
    uint8_t *d_mat_below = nullptr;
    double *d_bot_b = nullptr;
    double *a_send = nullptr, *a_recv = nullptr, *u_send = nullptr, *u_recv = nullptr;
    // library-driven z-slab rank (ovx_create_dist: NCCL; ovx_create_group: in-process loopback)
    int rank = 0, world = 1;              // world > 1: a distributed context
    void *nccl = nullptr;                 // ncclComm_t (NCCL ranks)
    struct LoopGroup *group = nullptr;    // loopback group (all ranks in this process)
    int64_t nz_global = 0, ez0 = 0, ez1 = 0;
    double *d_iface = nullptr;            // library-owned a_send | a_recv | u_send | u_recv
    cudaStream_t s_hi = nullptr;          // high-priority stream: edge chunks, exchange, interface update
    std::vector<cudaEvent_t> ev_pool;     // per-step phase events
    std::vector<std::array<cudaEvent_t, 4>> ph_used;   // (start, kernels done, halo done, end) per step
    double ph_ebe_ms = 0.0, ph_halo_ms = 0.0;           // folded-in totals of recycled phase events
    int64_t nn2() const { return (nx + 1) * (ny + 1); }
    int64_t nn() const { return (nx + 1) * (ny + 1) * (nz + 1); }
    int64_t ne() const { return nx * ny * nz; }
};

namespace {

std::string g_err;
ovx_status dist_step(ovx_ctx *ctx, int64_t n);
void dist_release(ovx_ctx *ctx);
std::mutex g_const_mu;
bool g_const_done[64] = {false};

ovx_status fail(ovx_ctx *c, ovx_status s, const std::string &m) {
    if (c) c->err = m;
    else g_err = m;
    return s;
}
ovx_status cuda_fail(ovx_ctx *c, cudaError_t e, const char *where) {
    return fail(c, OVX_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define CK(call)                                                        \
    do {                                                                \
        cudaError_t e_ = (call);                                        \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call);        \
    } while (0)

void dfree(void *p) {
    if (p) cudaFree(p);
}

// The element matrices (the same for every context) on the context's device, uploaded once per device.
ovx_status ensure_device_constants(ovx_ctx *ctx) {
    const int dev = ctx->device;
    if (dev < 0 || dev >= 64) return fail(ctx, OVX_EINVAL, "device index out of range");
    std::lock_guard<std::mutex> lk(g_const_mu);
    if (g_const_done[dev]) return OVX_OK;
    int8_t k8[1152];
    double Ak[576], Ag[576], kk2[2 * 576], kg2[2 * 576];
    if (derive_element_matrices(k8, Ak, Ag) != 0) return fail(ctx, OVX_EINVAL, "K_e^INT8 derivation failed");
    for (int r = 0; r < 24; ++r)
        for (int c = 0; c < 24; ++c) {
            kk2[r * 24 + c] = (double)k8[r * 48 + c];
            kg2[r * 24 + c] = (double)k8[r * 48 + 24 + c] + (r == c ? 128.0 : 0.0);
        }
    if (derive_vfem_matrices(kk2 + 576, kg2 + 576) != 0) return fail(ctx, OVX_EINVAL, "VFEM derivation failed");
    CK(upload_device_constants(k8, kk2, kg2));
    g_const_done[dev] = true;
    return OVX_OK;
}

ovx_status refresh_w(ovx_ctx *ctx) {
    if (!ctx->setup || !(ctx->dt > 0)) return OVX_OK;
    CK(launch_node_w(ctx->nx, ctx->ny, ctx->nz, ctx->d_mat, (ctx->slab_flags & 1) ? ctx->d_mat_below : nullptr,
                     ctx->d_mc, ctx->dt, ctx->d_w, ctx->stream));
    return OVX_OK;
}

bool finite_all(const double *a, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
        if (!std::isfinite(a[i])) return false;
    return true;
}

void fill_receivers(ovx_ctx *ctx, StepParams &p) {
    p.nrec = ctx->nrec;
    for (int k = 0; k < ctx->nrec; ++k) p.rec_node[k] = ctx->rec_node[k];
    p.traces = ctx->d_traces;
    p.it = ctx->it;
    p.rec_nt = ctx->d_traces ? ctx->rec_nt : 0;
}

StepParams base_params(ovx_ctx *ctx) {
    StepParams p;
    std::memset(&p, 0, sizeof(p));
    p.nx = ctx->nx;
    p.ny = ctx->ny;
    p.nz = ctx->nz;
    p.mc = ctx->d_mc;
    p.kset = ctx->kset;
    p.w = ctx->d_w;
    p.mat = ctx->d_mat;
    p.dmask = ctx->d_mask;
    p.stages = ctx->stages;
    p.direct = ctx->direct;
    p.nmat = ctx->nmat;
    return p;
}

ovx_status need_ready(ovx_ctx *ctx) {
    if (!ctx) return fail(nullptr, OVX_EINVAL, "null context");
    if (!ctx->have_grid || !ctx->have_emat || !ctx->setup)
        return fail(ctx, OVX_ESTATE, "grid, element materials and ovx_setup_elements are required first");
    return OVX_OK;
}

}  // namespace

extern "C" {

const char *ovx_version(void) { return "ovx 0.1 (sm_100a; tcgen05 kind::i8 + FP64 EBE)"; }

const char *ovx_last_error(const ovx_ctx *ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

ovx_status ovx_create(int device, ovx_ctx **out) {
    if (!out) return fail(nullptr, OVX_EINVAL, "out is null");
    *out = nullptr;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) return fail(nullptr, OVX_ECUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    if (device < 0 || device >= n) return fail(nullptr, OVX_EINVAL, "device index out of range");
    cudaDeviceProp prop;
    e = cudaGetDeviceProperties(&prop, device);
    if (e != cudaSuccess) return fail(nullptr, OVX_ECUDA, cudaGetErrorString(e));
    if (prop.major != 10) return fail(nullptr, OVX_EINVAL, "ovx kernels are built for sm_100a (B200) only");
    if ((e = cudaSetDevice(device)) != cudaSuccess) return fail(nullptr, OVX_ECUDA, cudaGetErrorString(e));
    ovx_ctx *ctx = new ovx_ctx();
    ctx->device = device;
    e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete ctx;
        return fail(nullptr, OVX_ECUDA, cudaGetErrorString(e));
    }
    ctx->own_stream = true;
    *out = ctx;
    return OVX_OK;
}

ovx_status ovx_destroy(ovx_ctx *ctx) {
    if (!ctx) return OVX_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    dfree(ctx->d_mat);
    dfree(ctx->d_mask);
    dfree(ctx->d_u);
    dfree(ctx->d_up);
    dfree(ctx->d_un);
    dfree(ctx->d_w);
    dfree(ctx->d_mat_below);
    dfree(ctx->d_bot_b);
    dfree(ctx->d_traces);
    dfree(ctx->d_mc);
    dfree(ctx->d_flag);
    dfree(ctx->d_iface);
    dist_release(ctx);
    for (auto &p : ctx->ev_used) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
    for (auto &p : ctx->ev_free) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    return OVX_OK;
}

ovx_status ovx_set_stream(ovx_ctx *ctx, void *stream) {
    if (!ctx) return fail(nullptr, OVX_EINVAL, "null context");
    cudaSetDevice(ctx->device);
    if (ctx->own_stream) {
        cudaStreamSynchronize(ctx->stream);
        cudaStreamDestroy(ctx->stream);
        ctx->own_stream = false;
    }
    if (stream != OVX_LIBRARY_STREAM) {
        ctx->stream = (cudaStream_t)stream;   // NULL: the legacy default stream
    } else {
        CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        ctx->own_stream = true;
    }
    return OVX_OK;
}

ovx_status ovx_set_grid(ovx_ctx *ctx, int64_t nx, int64_t ny, int64_t nz, double ds) {
    if (!ctx) return fail(nullptr, OVX_EINVAL, "null context");
    if (nx <= 0 || ny <= 0 || nz <= 0 || !(ds > 0) || !std::isfinite(ds))
        return fail(ctx, OVX_EINVAL, "grid dims must be >= 1 and ds > 0");
    if (nx > (1 << 24) || ny > (1 << 24) || nz > (1 << 24)) return fail(ctx, OVX_EINVAL, "grid too large");
    int64_t ez0 = 0, ez1 = nz;
    if (ctx->world > 1) {   // a z-slab rank: nz is the global element-layer count
        if (nz < ctx->world) return fail(ctx, OVX_EINVAL, "fewer element layers than ranks");
        ovx_get_partition(nz, ctx->world, ctx->rank, &ez0, &ez1);
    }
    const int64_t nz_global = nz;
    nz = ez1 - ez0;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    dfree(ctx->d_mat);
    dfree(ctx->d_mask);
    dfree(ctx->d_u);
    dfree(ctx->d_up);
    dfree(ctx->d_un);
    dfree(ctx->d_w);
    ctx->d_mat = nullptr;
    ctx->d_mask = nullptr;
    ctx->d_u = ctx->d_up = ctx->d_w = ctx->d_un = nullptr;
    ctx->alpha = ctx->beta = 0.0;
    dfree(ctx->d_mat_below);
    dfree(ctx->d_bot_b);
    ctx->d_mat_below = nullptr;
    ctx->d_bot_b = nullptr;
    ctx->slab_flags = 0;
    ctx->a_send = ctx->a_recv = ctx->u_send = ctx->u_recv = nullptr;
    ctx->nx = nx;
    ctx->ny = ny;
    ctx->nz = nz;
    ctx->ds = ds;
    ctx->have_grid = ctx->have_emat = ctx->setup = ctx->have_state = false;
    ctx->it = 0;
    // a new grid is a new model: sources and receivers of the previous one do not carry over
    ctx->nsrc = 0;
    ctx->src_node.clear();
    ctx->src_axis.clear();
    ctx->n_t = 0;
    ctx->amp.clear();
    ctx->nrec = 0;
    ctx->rec_node.clear();
    ctx->rec_nt = 0;
    dfree(ctx->d_traces);
    ctx->d_traces = nullptr;
    const int64_t nn = ctx->nn(), ne = ctx->ne();
    if (cudaMalloc(&ctx->d_mat, ne) != cudaSuccess || cudaMalloc(&ctx->d_u, 24 * nn) != cudaSuccess ||
        cudaMalloc(&ctx->d_up, 24 * nn) != cudaSuccess || cudaMalloc(&ctx->d_w, 8 * nn) != cudaSuccess) {
        cudaGetLastError();
        return fail(ctx, OVX_ENOMEM, "device allocation failed for the grid");
    }
    CK(cudaMemsetAsync(ctx->d_u, 0, 24 * nn, ctx->stream));
    CK(cudaMemsetAsync(ctx->d_up, 0, 24 * nn, ctx->stream));
    ctx->nz_global = nz_global;
    ctx->ez0 = ez0;
    ctx->ez1 = ez1;
    if (ctx->world > 1) {   // library-owned interface buffers and the slab flags of this rank
        const int64_t n2 = 3 * ctx->nn2();
        ctx->slab_flags = (ctx->rank > 0 ? 1 : 0) | (ctx->rank < ctx->world - 1 ? 2 : 0);
        dfree(ctx->d_iface);
        ctx->d_iface = nullptr;
        if (cudaMalloc(&ctx->d_iface, 4 * 8 * n2) != cudaSuccess ||
            ((ctx->slab_flags & 1) && (cudaMalloc(&ctx->d_mat_below, ctx->nx * ctx->ny) != cudaSuccess ||
                                       cudaMalloc(&ctx->d_bot_b, 8 * n2) != cudaSuccess))) {
            cudaGetLastError();
            return fail(ctx, OVX_ENOMEM, "device allocation failed for the interface buffers");
        }
        CK(cudaMemsetAsync(ctx->d_iface, 0, 4 * 8 * n2, ctx->stream));
        ctx->a_send = ctx->d_iface;
        ctx->a_recv = ctx->d_iface + n2;
        ctx->u_send = ctx->d_iface + 2 * n2;
        ctx->u_recv = ctx->d_iface + 3 * n2;
    }
    ctx->have_grid = true;
    return OVX_OK;
}

ovx_status ovx_set_materials(ovx_ctx *ctx, int n, const double *rho, const double *kappa, const double *G) {
    if (!ctx) return fail(nullptr, OVX_EINVAL, "null context");
    if (n < 1 || n > kMaxMat - 1 || !rho || !kappa || !G) return fail(ctx, OVX_EINVAL, "need 1..255 materials");
    for (int i = 0; i < n; ++i)
        if (!(rho[i] > 0) || !(kappa[i] > 0) || !(G[i] > 0) || !std::isfinite(rho[i]) || !std::isfinite(kappa[i]) ||
            !std::isfinite(G[i]))
            return fail(ctx, OVX_EINVAL, "material constants must be finite and > 0");
    ctx->nmat = n;
    ctx->rho.assign(rho, rho + n);
    ctx->kappa.assign(kappa, kappa + n);
    ctx->G.assign(G, G + n);
    ctx->setup = false;
    return OVX_OK;
}

ovx_status ovx_set_element_materials(ovx_ctx *ctx, const uint8_t *mat) {
    if (!ctx) return fail(nullptr, OVX_EINVAL, "null context");
    if (!ctx->have_grid || ctx->nmat == 0) return fail(ctx, OVX_ESTATE, "set grid and materials first");
    if (!mat) return fail(ctx, OVX_EINVAL, "mat is null");
    // a distributed rank with a lower neighbour passes the element layer below its slab first
    const int64_t halo = (ctx->world > 1 && (ctx->slab_flags & 1)) ? ctx->nx * ctx->ny : 0;
    const int64_t ne = ctx->ne();
    for (int64_t e = 0; e < ne + halo; ++e)
        if (mat[e] >= ctx->nmat) return fail(ctx, OVX_EINVAL, "unknown material id at element " + std::to_string(e));
    cudaSetDevice(ctx->device);
    if (halo) CK(cudaMemcpyAsync(ctx->d_mat_below, mat, halo, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->d_mat, mat + halo, ne, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->have_emat = true;
    if (ctx->setup) return refresh_w(ctx);
    return OVX_OK;
}

ovx_status ovx_set_dirichlet(ovx_ctx *ctx, const uint8_t *mask) {
    if (!ctx) return fail(nullptr, OVX_EINVAL, "null context");
    if (!ctx->have_grid) return fail(ctx, OVX_ESTATE, "set grid first");
    cudaSetDevice(ctx->device);
    if (!mask) {
        dfree(ctx->d_mask);
        ctx->d_mask = nullptr;
        return OVX_OK;
    }
    const int64_t nn = ctx->nn();
    for (int64_t i = 0; i < nn; ++i)
        if (mask[i] > 7) return fail(ctx, OVX_EINVAL, "Dirichlet mask values must be in 0..7");
    if (!ctx->d_mask && cudaMalloc(&ctx->d_mask, nn) != cudaSuccess) {
        cudaGetLastError();
        return fail(ctx, OVX_ENOMEM, "mask allocation failed");
    }
    CK(cudaMemcpyAsync(ctx->d_mask, mask, nn, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return OVX_OK;
}

ovx_status ovx_set_dt(ovx_ctx *ctx, double dt) {
    if (!ctx) return fail(nullptr, OVX_EINVAL, "null context");
    if (!(dt > 0) || !std::isfinite(dt)) return fail(ctx, OVX_EINVAL, "dt must be finite and > 0");
    ctx->dt = dt;
    cudaSetDevice(ctx->device);
    return refresh_w(ctx);
}

ovx_status ovx_setup_elements(ovx_ctx *ctx, int path, int stages) {
    if (!ctx) return fail(nullptr, OVX_EINVAL, "null context");
    if (!ctx->have_grid || !ctx->have_emat) return fail(ctx, OVX_ESTATE, "set grid and element materials first");
    if (path != OVX_INT8 && path != OVX_FP64 && path != OVX_FP64_DENSE && path != OVX_VFEM && path != OVX_VFEM_DENSE &&
        path != OVX_INT8_DIRECT)
        return fail(ctx, OVX_EINVAL, "path must be OVX_INT8, OVX_INT8_DIRECT, OVX_FP64, OVX_FP64_DENSE, OVX_VFEM or OVX_VFEM_DENSE");
    if (path == OVX_INT8_DIRECT && stages != 8) return fail(ctx, OVX_EINVAL, "the direct path is built for M = 8");
    ctx->direct = path == OVX_INT8_DIRECT ? 1 : 0;
    if (path == OVX_INT8_DIRECT) path = OVX_INT8;   // the INT8 kernels, direct conversion
    if (stages != 8 && !(path == OVX_INT8 && (stages == 4 || stages == 6)))
        return fail(ctx, OVX_EINVAL, "stages: M = 8 (all paths), or M = 4 / 6 on the INT8 path");
    if (derive_element_matrices(ctx->k8, ctx->Ak, ctx->Ag) != 0)
        return fail(ctx, OVX_EINVAL, "K_e^INT8 derivation produced a non-INT8 entry (PAPER.md L110 violated)");
    double dk = 256.0, dg = 384.0;        // K_e = κ ds Kk/dk + G ds Kg/dg for the dense kernel
    if (path == OVX_VFEM || path == OVX_VFEM_DENSE) {
        if (derive_vfem_matrices(ctx->Kk, ctx->Kg) != 0)
            return fail(ctx, OVX_EINVAL, "VFEM matrices are not integral at denominators 72 / 216");
        dk = 72.0;
        dg = 216.0;
        for (int i = 0; i < 576; ++i) {   // element spectrum (critical dt) from the VFEM matrices
            ctx->Ak[i] = ctx->Kk[i] / dk;
            ctx->Ag[i] = ctx->Kg[i] / dg;
        }
    } else {
        for (int r = 0; r < 24; ++r)
            for (int c = 0; c < 24; ++c) {
                ctx->Kk[r * 24 + c] = (double)ctx->k8[r * 48 + c];
                ctx->Kg[r * 24 + c] = (double)ctx->k8[r * 48 + 24 + c] + (r == c ? 128.0 : 0.0);
            }
    }
    ctx->mc.assign(kMaxMat, MatConst{});   // entries >= nmat (and the zero material 255) are all zero
    ctx->kset = (path == OVX_VFEM || path == OVX_VFEM_DENSE) ? 1 : 0;
    const double ds = ctx->ds;
    const double vol8 = ds * ds * ds / 8.0;
    for (int m = 0; m < ctx->nmat; ++m) {
        const double k = ctx->kappa[m], g = ctx->G[m];
        MatConst &c = ctx->mc[m];
        c.cG = (2.0 * g) / (3.0 * k);
        c.c1 = k * ds / 256.0;
        c.c2 = (256.0 * g) / (3.0 * k);
        c.ck = k * ds / dk;               // the oracle's κ ds / 256 (OVFEM) or κ ds / 72 (VFEM)
        c.cg = g * ds / dg;
        c.rho_vol8 = ctx->rho[m] * vol8;
        const double lam = k - 2.0 * g / 3.0, s0 = ds / 16.0, s1 = s0 * 0.75, s2 = s1 * 0.75;
        c.L0 = s0 * lam;
        c.M0 = s0 * g;
        c.M0x2 = 2.0 * c.M0;
        c.L1 = s1 * lam;
        c.M1 = s1 * g;
        c.M1x3 = 3.0 * c.M1;
        c.C2 = s2 * lam + 4.0 * (s2 * g);
        for (int q = 0; q < 3; ++q) {    // factored VFEM weights w_T = (ds/16) 3^{-|T|}
            const double wq = (ds / 16.0) / (q == 0 ? 1.0 : q == 1 ? 3.0 : 9.0);
            c.vl[q] = wq * lam;
            c.vm[q] = wq * g;
        }
    }
    ctx->path = path;
    ctx->stages = stages;
    cudaSetDevice(ctx->device);
    ovx_status s = ensure_device_constants(ctx);
    if (s) return s;
    if (!ctx->d_mc && cudaMalloc(&ctx->d_mc, sizeof(MatConst) * kMaxMat) != cudaSuccess) {
        cudaGetLastError();
        return fail(ctx, OVX_ENOMEM, "material table allocation failed");
    }
    // stream-ordered before every kernel of this context; no other context reads this table
    CK(cudaMemcpyAsync(ctx->d_mc, ctx->mc.data(), sizeof(MatConst) * kMaxMat, cudaMemcpyHostToDevice, ctx->stream));
    ctx->setup = true;
    return refresh_w(ctx);
}

ovx_status ovx_get_int8_matrix(ovx_ctx *ctx, int8_t *out) {  // ctx may be NULL (host-only)
    if (!out) return fail(ctx, OVX_EINVAL, "null argument");
    int8_t k8[1152];
    if (derive_element_matrices(k8, nullptr, nullptr) != 0) return fail(ctx, OVX_EINVAL, "non-INT8 entry");
    std::memcpy(out, k8, 1152);
    return OVX_OK;
}

ovx_status ovx_critical_dt(ovx_ctx *ctx, double *dt_elem_bound, double *dt_power_iter) {
    if (!ctx || (!dt_elem_bound && !dt_power_iter)) return fail(ctx, OVX_EINVAL, "null argument");
    if (!ctx->have_grid || ctx->nmat == 0) return fail(ctx, OVX_ESTATE, "set grid and materials first");
    if (dt_elem_bound) {
        double Ak[576], Ag[576], K[576];
        if (derive_element_matrices(nullptr, Ak, Ag) != 0) return fail(ctx, OVX_EINVAL, "derivation failed");
        double lmax = 0.0;
        for (int m = 0; m < ctx->nmat; ++m) {
            for (int i = 0; i < 576; ++i) K[i] = ctx->kappa[m] * ctx->ds * Ak[i] + ctx->G[m] * ctx->ds * Ag[i];
            const double lam = sym_lambda_max(K) / (ctx->rho[m] * ctx->ds * ctx->ds * ctx->ds / 8.0);
            if (lam > lmax) lmax = lam;
        }
        *dt_elem_bound = 2.0 / std::sqrt(lmax);
    }
    if (dt_power_iter) {   // λ_max(M⁻¹K) of the assembled model by power iteration with the EBE product
        ovx_status s = need_ready(ctx);
        if (s) return s;
        if (!(ctx->dt > 0)) return fail(ctx, OVX_ESTATE, "the power iteration needs dt (for M = dt²/w)");
        if (ctx->world > 1 || ctx->slab_flags) return fail(ctx, OVX_EINVAL, "power iteration: single-GPU contexts only");
        cudaSetDevice(ctx->device);
        const int64_t nn = ctx->nn(), n3 = 3 * nn;
        double *blk = nullptr;
        if (cudaMalloc(&blk, 8 * (3 * n3 + 4)) != cudaSuccess) {
            cudaGetLastError();
            return fail(ctx, OVX_ENOMEM, "power-iteration scratch allocation failed");
        }
        double *x = blk, *y = blk + n3, *z = blk + 2 * n3, *acc = blk + 3 * n3;
        std::vector<double> hx(n3);
        uint64_t st = 0x9E3779B97F4A7C15ull;   // deterministic start vector (splitmix64 in [-1, 1))
        for (int64_t i = 0; i < n3; ++i) {
            uint64_t q = (st += 0x9E3779B97F4A7C15ull);
            q = (q ^ (q >> 30)) * 0xBF58476D1CE4E5B9ull;
            q = (q ^ (q >> 27)) * 0x94D049BB133111EBull;
            q ^= q >> 31;
            hx[i] = (double)(q >> 11) * 0x1p-52 - 1.0;
        }
        double lam = 0.0, h[3] = {0, 0, 0};
        cudaError_t e = cudaMemcpyAsync(x, hx.data(), 8 * n3, cudaMemcpyHostToDevice, ctx->stream);
        const double dt2 = ctx->dt * ctx->dt;
        for (int k = 0; k < 300 && e == cudaSuccess; ++k) {
            StepParams p = base_params(ctx);
            p.u = x;
            p.fout = y;
            if ((e = cudaMemsetAsync(acc, 0, 24, ctx->stream))) break;
            if ((e = launch_step(ctx->path, MODE_APPLY, p, ctx->stream))) break;
            if ((e = launch_power_iter(nn, x, y, ctx->d_w, ctx->d_mask, dt2, z, acc, x, ctx->stream))) break;
            if ((e = cudaMemcpyAsync(h, acc, 24, cudaMemcpyDeviceToHost, ctx->stream))) break;
            if ((e = cudaStreamSynchronize(ctx->stream))) break;
            lam = h[0] / h[1];   // Rayleigh quotient xᵀKx / xᵀMx (from below)
        }
        cudaFree(blk);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "power iteration");
        if (!(lam > 0)) return fail(ctx, OVX_EUNSTABLE, "power iteration did not produce a positive eigenvalue");
        *dt_power_iter = 2.0 / std::sqrt(lam);
    }
    return OVX_OK;
}

ovx_status ovx_set_sources(ovx_ctx *ctx, int n, const int64_t *node, const int32_t *axis, int64_t n_t,
                           const double *amp) {
    if (!ctx) return fail(nullptr, OVX_EINVAL, "null context");
    if (!ctx->have_grid) return fail(ctx, OVX_ESTATE, "set grid first");
    if (n < 0 || n > kMaxSrc || n_t < 0) return fail(ctx, OVX_EINVAL, "0..16 sources");
    if (n > 0 && (!node || !axis || (n_t > 0 && !amp))) return fail(ctx, OVX_EINVAL, "null source arrays");
    const int64_t nn_all = ctx->world > 1 ? ctx->nn2() * (ctx->nz_global + 1) : ctx->nn();
    for (int k = 0; k < n; ++k)
        if (node[k] < 0 || node[k] >= nn_all || axis[k] < 0 || axis[k] > 2)
            return fail(ctx, OVX_EINVAL, "source node/axis out of range");
    if (n > 0 && n_t > 0 && !finite_all(amp, (int64_t)n * n_t)) return fail(ctx, OVX_EINVAL, "non-finite amplitude");
    ctx->src_node.clear();
    ctx->src_axis.clear();
    ctx->amp.clear();
    for (int k = 0; k < n; ++k) {   // distributed: global node ids; keep the sources of owned planes
        int64_t nd = node[k];
        if (ctx->world > 1) {
            const int64_t pz = nd / ctx->nn2(), p1 = (ctx->slab_flags & 2) ? ctx->ez1 : ctx->ez1 + 1;
            if (pz < ctx->ez0 || pz >= p1) continue;
            nd -= ctx->ez0 * ctx->nn2();
        }
        ctx->src_node.push_back(nd);
        ctx->src_axis.push_back(axis[k]);
        ctx->amp.insert(ctx->amp.end(), amp + (size_t)k * (size_t)n_t, amp + (size_t)(k + 1) * (size_t)n_t);
    }
    ctx->nsrc = (int)ctx->src_node.size();
    ctx->n_t = n_t;
    return OVX_OK;
}

static ovx_status set_state_impl(ovx_ctx *ctx, const double *u, const double *up, int64_t it, cudaMemcpyKind kind) {
    if (!ctx) return fail(nullptr, OVX_EINVAL, "null context");
    if (!ctx->have_grid) return fail(ctx, OVX_ESTATE, "set grid first");
    if (!u || !up) return fail(ctx, OVX_EINVAL, "null state arrays");
    if (it < 0) return fail(ctx, OVX_EINVAL, "the step index it must be >= 0");
    const int64_t n3 = 3 * ctx->nn();
    cudaSetDevice(ctx->device);
    CK(cudaMemcpyAsync(ctx->d_u, u, 8 * n3, kind, ctx->stream));
    CK(cudaMemcpyAsync(ctx->d_up, up, 8 * n3, kind, ctx->stream));
    if (kind == cudaMemcpyHostToDevice) {   // finiteness checked on the device (the host scan was serial)
        int h = 0;
        if (!ctx->d_flag) CK(cudaMalloc(&ctx->d_flag, sizeof(int)));
        CK(cudaMemsetAsync(ctx->d_flag, 0, sizeof(int), ctx->stream));
        CK(launch_finite_check(ctx->d_u, n3, ctx->d_flag, ctx->stream));
        CK(launch_finite_check(ctx->d_up, n3, ctx->d_flag, ctx->stream));
        CK(cudaMemcpyAsync(&h, ctx->d_flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        if (h) {
            ctx->have_state = false;
            return fail(ctx, OVX_EINVAL, "non-finite state");
        }
    }
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->it = it;
    ctx->have_state = true;
    return OVX_OK;
}
static ovx_status get_state_impl(ovx_ctx *ctx, double *u, double *up, int64_t *it, cudaMemcpyKind kind) {
    if (!ctx) return fail(nullptr, OVX_EINVAL, "null context");
    if (!ctx->have_grid) return fail(ctx, OVX_ESTATE, "set grid first");
    const int64_t n3 = 3 * ctx->nn();
    cudaSetDevice(ctx->device);
    if (u) CK(cudaMemcpyAsync(u, ctx->d_u, 8 * n3, kind, ctx->stream));
    if (up) CK(cudaMemcpyAsync(up, ctx->d_up, 8 * n3, kind, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (it) *it = ctx->it;
    return OVX_OK;
}

ovx_status ovx_set_state(ovx_ctx *ctx, const double *u, const double *u_prev, int64_t it) {
    return set_state_impl(ctx, u, u_prev, it, cudaMemcpyHostToDevice);
}
ovx_status ovx_get_state(ovx_ctx *ctx, double *u, double *u_prev, int64_t *it) {
    return get_state_impl(ctx, u, u_prev, it, cudaMemcpyDeviceToHost);
}
ovx_status ovx_set_state_device(ovx_ctx *ctx, const double *u, const double *u_prev, int64_t it) {
    return set_state_impl(ctx, u, u_prev, it, cudaMemcpyDeviceToDevice);
}
ovx_status ovx_get_state_device(ovx_ctx *ctx, double *u, double *u_prev, int64_t *it) {
    return get_state_impl(ctx, u, u_prev, it, cudaMemcpyDeviceToDevice);
}

ovx_status ovx_step(ovx_ctx *ctx, int64_t n) {
    ovx_status s = need_ready(ctx);
    if (s) return s;
    if (!(ctx->dt > 0)) return fail(ctx, OVX_ESTATE, "set dt first");
    if (n < 0) return fail(ctx, OVX_EINVAL, "n must be >= 0");
    if (ctx->direct && (ctx->alpha != 0.0 || ctx->beta != 0.0))
        return fail(ctx, OVX_EINVAL, "the direct N-stage path (OVX_INT8_DIRECT) is undamped only");
    if (ctx->world > 1) {
        if (ctx->group) return fail(ctx, OVX_ESTATE, "loopback-group ranks step together with ovx_step_group");
        return dist_step(ctx, n);
    }
    if (ctx->slab_flags) return fail(ctx, OVX_ESTATE, "slab contexts step with ovx_step_begin/iface/end");
    if (n == 0) return OVX_OK;
    cudaSetDevice(ctx->device);
    EventPair ev;
    if (!ctx->ev_free.empty()) {
        ev = ctx->ev_free.back();
        ctx->ev_free.pop_back();
    } else {
        CK(cudaEventCreate(&ev.a));
        CK(cudaEventCreate(&ev.b));
    }
    CK(cudaEventRecord(ev.a, ctx->stream));
    StepParams p = base_params(ctx);
    const bool damped = ctx->alpha != 0.0 || ctx->beta != 0.0;
    if (damped) {
        p.damped = 1;
        p.ca = ctx->alpha * ctx->dt;   // RN(alpha·dt), RN(beta/dt): the oracle's roundings
        p.cb = ctx->beta / ctx->dt;
    }
    for (int64_t k = 0; k < n; ++k) {
        p.u = ctx->d_u;
        p.uo = ctx->d_up;
        p.un = damped ? ctx->d_un : nullptr;
        p.nsrc = ctx->nsrc;
        for (int q = 0; q < ctx->nsrc; ++q) {
            p.src_dof[q] = 3 * ctx->src_node[q] + ctx->src_axis[q];
            p.src_val[q] = (ctx->it >= 0 && ctx->it < ctx->n_t) ? ctx->amp[(size_t)q * ctx->n_t + ctx->it] : 0.0;
        }
        fill_receivers(ctx, p);
        CK(launch_step(ctx->path, MODE_STEP, p, ctx->stream));
        if (damped) {            // (u_prev, u, u_next) <- (u, u_next, u_prev)
            double *old_up = ctx->d_up;
            ctx->d_up = ctx->d_u;
            ctx->d_u = ctx->d_un;
            ctx->d_un = old_up;
        } else {
            std::swap(ctx->d_u, ctx->d_up);
        }
        ctx->it += 1;
        ctx->launches += 1;
    }
    CK(cudaEventRecord(ev.b, ctx->stream));
    ctx->ev_used.push_back(ev);
    return OVX_OK;
}

ovx_status ovx_set_damping(ovx_ctx *ctx, double alpha, double beta) {
    if (!ctx) return fail(nullptr, OVX_EINVAL, "null context");
    if (!ctx->have_grid) return fail(ctx, OVX_ESTATE, "set the grid first");
    if (!(alpha >= 0) || !(beta >= 0) || !std::isfinite(alpha) || !std::isfinite(beta))
        return fail(ctx, OVX_EINVAL, "Rayleigh coefficients must be finite and >= 0");
    cudaSetDevice(ctx->device);
    if ((alpha != 0.0 || beta != 0.0) && !ctx->d_un) {
        if (cudaMalloc(&ctx->d_un, 24 * ctx->nn()) != cudaSuccess) {
            cudaGetLastError();
            return fail(ctx, OVX_ENOMEM, "device allocation failed for the third state buffer");
        }
    }
    ctx->alpha = alpha;
    ctx->beta = beta;
    return OVX_OK;
}

ovx_status ovx_set_slab(ovx_ctx *ctx, int flags, const uint8_t *mat_below) {
    if (!ctx) return fail(nullptr, OVX_EINVAL, "null context");
    if (!ctx->have_grid || ctx->nmat == 0) return fail(ctx, OVX_ESTATE, "set grid and materials first");
    if (flags < 0 || flags > 3) return fail(ctx, OVX_EINVAL, "slab flags must be in 0..3");
    if ((flags & 1) && !mat_below) return fail(ctx, OVX_EINVAL, "a lower neighbour needs the halo materials");
    cudaSetDevice(ctx->device);
    const int64_t ne2 = ctx->nx * ctx->ny;
    if (flags & 1) {
        for (int64_t e = 0; e < ne2; ++e)
            if (mat_below[e] >= ctx->nmat) return fail(ctx, OVX_EINVAL, "unknown material id in the halo layer");
        if (!ctx->d_mat_below && cudaMalloc(&ctx->d_mat_below, ne2) != cudaSuccess) {
            cudaGetLastError();
            return fail(ctx, OVX_ENOMEM, "halo allocation failed");
        }
        if (!ctx->d_bot_b && cudaMalloc(&ctx->d_bot_b, 8 * 3 * ctx->nn2()) != cudaSuccess) {
            cudaGetLastError();
            return fail(ctx, OVX_ENOMEM, "interface allocation failed");
        }
        CK(cudaMemcpyAsync(ctx->d_mat_below, mat_below, ne2, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    ctx->slab_flags = flags;
    return refresh_w(ctx);
}

ovx_status ovx_set_iface_buffers(ovx_ctx *ctx, double *a_send, double *a_recv, double *u_send, double *u_recv) {
    if (!ctx) return fail(nullptr, OVX_EINVAL, "null context");
    if (((ctx->slab_flags & 2) && !a_send) || ((ctx->slab_flags & 1) && (!a_recv || !u_send)) ||
        ((ctx->slab_flags & 2) && !u_recv))
        return fail(ctx, OVX_EINVAL, "missing interface buffer for the slab flags");
    ctx->a_send = a_send;
    ctx->a_recv = a_recv;
    ctx->u_send = u_send;
    ctx->u_recv = u_recv;
    return OVX_OK;
}

static StepParams step_params(ovx_ctx *ctx) {
    StepParams p = base_params(ctx);
    p.u = ctx->d_u;
    p.uo = ctx->d_up;
    p.nsrc = ctx->nsrc;
    for (int q = 0; q < ctx->nsrc; ++q) {
        p.src_dof[q] = 3 * ctx->src_node[q] + ctx->src_axis[q];
        p.src_val[q] = (ctx->it >= 0 && ctx->it < ctx->n_t) ? ctx->amp[(size_t)q * ctx->n_t + ctx->it] : 0.0;
    }
    p.slab_flags = ctx->slab_flags;
    p.iface_top_A = ctx->a_send;
    p.iface_bot_b = ctx->d_bot_b;
    if (ctx->alpha != 0.0 || ctx->beta != 0.0) {   // Rayleigh damping (reading R1), as in ovx_step
        p.damped = 1;
        p.ca = ctx->alpha * ctx->dt;
        p.cb = ctx->beta / ctx->dt;
        p.un = ctx->d_un;
    }
    fill_receivers(ctx, p);
    return p;
}

static ovx_status step_begin_impl(ovx_ctx *ctx, int part) {
    ovx_status s = need_ready(ctx);
    if (s) return s;
    if (!(ctx->dt > 0)) return fail(ctx, OVX_ESTATE, "set dt first");
    if (((ctx->slab_flags & 2) && !ctx->a_send) || ((ctx->slab_flags & 1) && !ctx->d_bot_b))
        return fail(ctx, OVX_ESTATE, "interface buffers not set");
    cudaSetDevice(ctx->device);
    int nl = 0;
    CK(launch_step(ctx->path, MODE_STEP, step_params(ctx), ctx->stream, part, &nl));
    ctx->launches += nl;
    return OVX_OK;
}

ovx_status ovx_step_begin(ovx_ctx *ctx) { return step_begin_impl(ctx, -1); }

ovx_status ovx_step_begin_part(ovx_ctx *ctx, int part) {
    if (part != 0 && part != 1) return fail(ctx, OVX_EINVAL, "part must be 0 (edge chunks) or 1 (interior)");
    return step_begin_impl(ctx, part);
}

static ovx_status step_iface_impl(ovx_ctx *ctx, cudaStream_t st) {
    ovx_status s = need_ready(ctx);
    if (s) return s;
    if (!(ctx->slab_flags & 1)) return OVX_OK;
    cudaSetDevice(ctx->device);
    CK(launch_iface_update(step_params(ctx), ctx->a_recv, ctx->u_send, st));
    ctx->launches += 1;
    return OVX_OK;
}

ovx_status ovx_step_iface(ovx_ctx *ctx) { return step_iface_impl(ctx, ctx ? ctx->stream : nullptr); }

ovx_status ovx_step_iface_stream(ovx_ctx *ctx, void *stream) {
    if (!ctx) return fail(nullptr, OVX_EINVAL, "null context");
    return step_iface_impl(ctx, stream == OVX_LIBRARY_STREAM ? ctx->stream : (cudaStream_t)stream);
}

ovx_status ovx_step_end(ovx_ctx *ctx) {
    ovx_status s = need_ready(ctx);
    if (s) return s;
    cudaSetDevice(ctx->device);
    const bool damped = ctx->alpha != 0.0 || ctx->beta != 0.0;
    double *next = damped ? ctx->d_un : ctx->d_up;   // the buffer holding u^{it+1}
    if (ctx->slab_flags & 2)   // the owner above sent the updated top plane
        CK(cudaMemcpyAsync(next + 3 * ctx->nn2() * ctx->nz, ctx->u_recv, 24 * ctx->nn2(),
                           cudaMemcpyDeviceToDevice, ctx->stream));
    if (damped) {              // (u_prev, u, u_next) <- (u, u_next, u_prev)
        double *old_up = ctx->d_up;
        ctx->d_up = ctx->d_u;
        ctx->d_u = ctx->d_un;
        ctx->d_un = old_up;
    } else {
        std::swap(ctx->d_u, ctx->d_up);
    }
    ctx->it += 1;
    return OVX_OK;
}

ovx_status ovx_set_receivers(ovx_ctx *ctx, int n, const int64_t *node, int64_t n_t) {
    if (!ctx) return fail(nullptr, OVX_EINVAL, "null context");
    if (!ctx->have_grid) return fail(ctx, OVX_ESTATE, "set grid first");
    if (n < 0 || n > kMaxRec || n_t < 0 || (n > 0 && !node)) return fail(ctx, OVX_EINVAL, "0..32 receivers");
    const int64_t nn_all = ctx->world > 1 ? ctx->nn2() * (ctx->nz_global + 1) : ctx->nn();
    for (int k = 0; k < n; ++k)
        if (node[k] < 0 || node[k] >= nn_all) return fail(ctx, OVX_EINVAL, "receiver node out of range");
    cudaSetDevice(ctx->device);
    dfree(ctx->d_traces);
    ctx->d_traces = nullptr;
    ctx->nrec = n;
    ctx->rec_node.assign(node, node + n);
    if (ctx->world > 1)   // distributed: global ids; receivers of other ranks' planes record nothing (-1)
        for (int k = 0; k < n; ++k) {
            const int64_t pz = node[k] / ctx->nn2(), p1 = (ctx->slab_flags & 2) ? ctx->ez1 : ctx->ez1 + 1;
            ctx->rec_node[k] = (pz >= ctx->ez0 && pz < p1) ? node[k] - ctx->ez0 * ctx->nn2() : -1;
        }
    ctx->rec_nt = n_t;
    if (n > 0 && n_t > 0) {
        if (cudaMalloc(&ctx->d_traces, 8 * 3 * (size_t)n * (size_t)n_t) != cudaSuccess) {
            cudaGetLastError();
            return fail(ctx, OVX_ENOMEM, "trace allocation failed");
        }
        CK(cudaMemsetAsync(ctx->d_traces, 0, 8 * 3 * (size_t)n * (size_t)n_t, ctx->stream));
    }
    return OVX_OK;
}

ovx_status ovx_get_traces(ovx_ctx *ctx, double *out) {
    if (!ctx || !out) return fail(ctx, OVX_EINVAL, "null argument");
    cudaSetDevice(ctx->device);
    if (ctx->d_traces) {
        CK(cudaMemcpyAsync(out, ctx->d_traces, 8 * 3 * (size_t)ctx->nrec * (size_t)ctx->rec_nt,
                           cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    return OVX_OK;
}

ovx_status ovx_sync(ovx_ctx *ctx) {
    if (!ctx) return fail(nullptr, OVX_EINVAL, "null context");
    cudaSetDevice(ctx->device);
    CK(cudaStreamSynchronize(ctx->stream));
    return OVX_OK;
}

ovx_status ovx_check_finite(ovx_ctx *ctx) {
    if (!ctx) return fail(nullptr, OVX_EINVAL, "null context");
    if (!ctx->have_grid) return fail(ctx, OVX_ESTATE, "set grid first");
    cudaSetDevice(ctx->device);
    int h = 0;
    if (!ctx->d_flag) CK(cudaMalloc(&ctx->d_flag, sizeof(int)));
    CK(cudaMemsetAsync(ctx->d_flag, 0, sizeof(int), ctx->stream));
    CK(launch_finite_check(ctx->d_u, 3 * ctx->nn(), ctx->d_flag, ctx->stream));
    CK(cudaMemcpyAsync(&h, ctx->d_flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (h) return fail(ctx, OVX_EUNSTABLE, "non-finite displacement at step " + std::to_string(ctx->it));
    return OVX_OK;
}

static ovx_status apply_impl(ovx_ctx *ctx, const double *u_dev, double *f_dev) {
    StepParams p = base_params(ctx);
    p.u = u_dev;
    p.fout = f_dev;
    CK(launch_step(ctx->path, MODE_APPLY, p, ctx->stream));
    return OVX_OK;
}

ovx_status ovx_apply_K_device(ovx_ctx *ctx, const double *u, double *f) {
    ovx_status s = need_ready(ctx);
    if (s) return s;
    if (!u || !f) return fail(ctx, OVX_EINVAL, "null array");
    cudaSetDevice(ctx->device);
    return apply_impl(ctx, u, f);
}

ovx_status ovx_apply_K(ovx_ctx *ctx, const double *u, double *f) {
    ovx_status s = need_ready(ctx);
    if (s) return s;
    if (!u || !f) return fail(ctx, OVX_EINVAL, "null array");
    const int64_t n3 = 3 * ctx->nn();
    if (!finite_all(u, n3)) return fail(ctx, OVX_EINVAL, "non-finite u");
    cudaSetDevice(ctx->device);
    double *du = nullptr, *df = nullptr;
    if (cudaMalloc(&du, 8 * n3) != cudaSuccess || cudaMalloc(&df, 8 * n3) != cudaSuccess) {
        cudaGetLastError();
        dfree(du);
        return fail(ctx, OVX_ENOMEM, "scratch allocation failed");
    }
    cudaMemcpyAsync(du, u, 8 * n3, cudaMemcpyHostToDevice, ctx->stream);
    s = apply_impl(ctx, du, df);
    if (!s) {
        cudaError_t e = cudaMemcpyAsync(f, df, 8 * n3, cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) s = cuda_fail(ctx, e, "apply_K readback");
    }
    cudaFree(du);
    cudaFree(df);
    return s;
}

ovx_status ovx_debug_element_ints(ovx_ctx *ctx, const double *u, int64_t e0, int64_t ne, double *s_out,
                                  int64_t *v, uint8_t *d, int32_t *C, int64_t *y_hi, int64_t *y_lo, double *fe) {
    ovx_status s = need_ready(ctx);
    if (s) return s;
    if (!u || e0 < 0 || ne < 0 || e0 + ne > ctx->ne()) return fail(ctx, OVX_EINVAL, "bad element range");
    if (ctx->path != OVX_INT8 && (s_out || v || d || C || y_hi || y_lo))
        return fail(ctx, OVX_EINVAL, "integer records exist only on the INT8 path");
    if (ne == 0) return OVX_OK;
    const int64_t n3 = 3 * ctx->nn();
    cudaSetDevice(ctx->device);
    // one device block for everything
    const size_t bs = 8 * ne, bv = 8 * ne * 48, bd = ne * 384, bC = 4 * ne * 192, by = 8 * ne * 24, bf = 8 * ne * 24;
    const size_t bu = 8 * n3, total = bu * 2 + bs + bv + bd + bC + 2 * by + bf + 16 * 256;
    uint8_t *blk = nullptr;
    if (cudaMalloc(&blk, total) != cudaSuccess) {
        cudaGetLastError();
        return fail(ctx, OVX_ENOMEM, "debug scratch allocation failed");
    }
    size_t o = 0;
    auto take = [&](size_t b) { uint8_t *q = blk + o; o += (b + 255) / 256 * 256; return q; };
    double *du = (double *)take(bu), *df = (double *)take(bu);
    StepParams p = base_params(ctx);
    p.u = du;
    p.fout = df;
    p.dbg_e0 = e0;
    p.dbg_ne = ne;
    p.dbg_s = (double *)take(bs);
    p.dbg_v = (int64_t *)take(bv);
    p.dbg_d = take(bd);
    p.dbg_C = (int32_t *)take(bC);
    p.dbg_yhi = (int64_t *)take(by);
    p.dbg_ylo = (int64_t *)take(by);
    p.dbg_fe = (double *)take(bf);
    cudaError_t e = cudaMemcpyAsync(du, u, bu, cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) e = launch_step(ctx->path, MODE_DEBUG, p, ctx->stream);
    if (e == cudaSuccess && s_out) e = cudaMemcpyAsync(s_out, p.dbg_s, bs, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess && v) e = cudaMemcpyAsync(v, p.dbg_v, bv, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess && d) e = cudaMemcpyAsync(d, p.dbg_d, bd, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess && C) e = cudaMemcpyAsync(C, p.dbg_C, bC, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess && y_hi) e = cudaMemcpyAsync(y_hi, p.dbg_yhi, by, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess && y_lo) e = cudaMemcpyAsync(y_lo, p.dbg_ylo, by, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess && fe) e = cudaMemcpyAsync(fe, p.dbg_fe, bf, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    cudaFree(blk);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "debug_element_ints");
    return OVX_OK;
}

ovx_status ovx_get_node_w(ovx_ctx *ctx, double *w) {
    ovx_status s = need_ready(ctx);
    if (s) return s;
    if (!w) return fail(ctx, OVX_EINVAL, "null array");
    if (!(ctx->dt > 0)) return fail(ctx, OVX_ESTATE, "set dt first");
    cudaSetDevice(ctx->device);
    CK(cudaMemcpyAsync(w, ctx->d_w, 8 * ctx->nn(), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return OVX_OK;
}

ovx_status ovx_get_timers(ovx_ctx *ctx, double *ms_step, int64_t *launches, int reset) {
    if (!ctx) return fail(nullptr, OVX_EINVAL, "null context");
    cudaSetDevice(ctx->device);
    CK(cudaStreamSynchronize(ctx->stream));
    double tot = 0.0;
    for (auto &p : ctx->ev_used) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, p.a, p.b));
        tot += ms;
    }
    if (ms_step) *ms_step = tot;
    if (launches) *launches = ctx->launches;
    if (reset) {
        for (auto &p : ctx->ev_used) ctx->ev_free.push_back(p);
        ctx->ev_used.clear();
        ctx->launches = 0;
    }
    return OVX_OK;
}

ovx_status ovx_get_launch_config(ovx_ctx *ctx, int64_t *ctas, int *threads, int *smem_bytes) {
    if (!ctx) return fail(nullptr, OVX_EINVAL, "null context");
    if (!ctx->have_grid) return fail(ctx, OVX_ESTATE, "set grid first");
    LaunchInfo li = step_launch_info(ctx->path, ctx->nx, ctx->ny, ctx->nz);
    if (ctas) *ctas = li.ctas;
    if (threads) *threads = li.threads;
    if (smem_bytes) *smem_bytes = li.smem;
    return OVX_OK;
}

}  // extern "C"

// ============================================================================================
// z-slab decomposition driven by the library (SURVEY §8(b) "distributed create", §8(e); PAPER.md
// L288 names the multi-GPU extension as future work).  Per step (the overlapped schedule):
//   s_hi (high priority) waits for the previous step; the edge z-chunks (first and last: they
//   produce the top interface's partial force T and plane 0's bottom-face sum B) on s_hi, the
//   interior chunks concurrently on the context stream; on s_hi: T → rank above (NCCL P2P),
//   interface update of plane 0 by its owner (the rank above: f = T + B, reading U2), the updated
//   plane → rank below; the context stream waits for s_hi and installs the received top plane.
// NCCL is loaded at run time (dlopen of libnccl.so.2; the one torch already loaded if any).
// ============================================================================================
namespace {

namespace nccl {
struct UniqueId {
    char internal[128];
};
typedef void *Comm;
typedef int Result;
constexpr int kFloat64 = 8;   // ncclFloat64
struct Api {
    Result (*GetUniqueId)(UniqueId *) = nullptr;
    Result (*CommInitRank)(Comm *, int, UniqueId, int) = nullptr;
    Result (*CommDestroy)(Comm) = nullptr;
    Result (*Send)(const void *, size_t, int, int, Comm, cudaStream_t) = nullptr;
    Result (*Recv)(void *, size_t, int, int, Comm, cudaStream_t) = nullptr;
    Result (*GroupStart)() = nullptr;
    Result (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(Result) = nullptr;
    std::string err;
    bool ok() const { return GetUniqueId && CommInitRank && Send && Recv && GroupStart && GroupEnd; }
};
const Api &api() {
    static Api a = [] {
        Api x;
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // already in the process (torch)
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            x.err = std::string("cannot load libnccl.so.2: ") + dlerror();
            return x;
        }
        x.GetUniqueId = (Result(*)(UniqueId *))dlsym(h, "ncclGetUniqueId");
        x.CommInitRank = (Result(*)(Comm *, int, UniqueId, int))dlsym(h, "ncclCommInitRank");
        x.CommDestroy = (Result(*)(Comm))dlsym(h, "ncclCommDestroy");
        x.Send = (Result(*)(const void *, size_t, int, int, Comm, cudaStream_t))dlsym(h, "ncclSend");
        x.Recv = (Result(*)(void *, size_t, int, int, Comm, cudaStream_t))dlsym(h, "ncclRecv");
        x.GroupStart = (Result(*)())dlsym(h, "ncclGroupStart");
        x.GroupEnd = (Result(*)())dlsym(h, "ncclGroupEnd");
        x.GetErrorString = (const char *(*)(Result))dlsym(h, "ncclGetErrorString");
        if (!x.ok()) x.err = "libnccl.so.2 lacks a needed symbol";
        return x;
    }();
    return a;
}
}  // namespace nccl

#define NK(call)                                                                                        \
    do {                                                                                                \
        nccl::Result r_ = (call);                                                                       \
        if (r_ != 0)                                                                                    \
            return fail(ctx, OVX_ENCCL, std::string(#call) + ": " +                                    \
                                            (nccl::api().GetErrorString ? nccl::api().GetErrorString(r_) : "?")); \
    } while (0)

}  // namespace

// All ranks of a decomposition in this process on one or more devices (tests: the schedule above
// with device-to-device copies in place of NCCL, stepped in lock step by ovx_step_group).
struct LoopGroup {
    std::vector<ovx_ctx *> ranks;
};

namespace {

cudaEvent_t ev_take(ovx_ctx *ctx) {
    if (!ctx->ev_pool.empty()) {
        cudaEvent_t e = ctx->ev_pool.back();
        ctx->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

ovx_status dist_prepare(ovx_ctx *ctx) {
    ovx_status s = need_ready(ctx);
    if (s) return s;
    if (!(ctx->dt > 0)) return fail(ctx, OVX_ESTATE, "set dt first");
    cudaSetDevice(ctx->device);
    if (!ctx->s_hi) {
        int lo = 0, hi = 0;
        CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CK(cudaStreamCreateWithPriority(&ctx->s_hi, cudaStreamNonBlocking, hi));
    }
    return OVX_OK;
}

// phase 1: s_hi after the previous step; edge chunks on s_hi, interior on the context stream
ovx_status dist_phase_compute(ovx_ctx *ctx, std::array<cudaEvent_t, 4> &ev) {
    for (auto &e : ev) e = ev_take(ctx);
    CK(cudaEventRecord(ev[0], ctx->stream));
    CK(cudaStreamWaitEvent(ctx->s_hi, ev[0], 0));
    const StepParams p = step_params(ctx);
    int n0 = 0, n1 = 0;
    CK(launch_step(ctx->path, MODE_STEP, p, ctx->s_hi, 0, &n0));
    CK(launch_step(ctx->path, MODE_STEP, p, ctx->stream, 1, &n1));
    CK(cudaEventRecord(ev[1], ctx->s_hi));
    ctx->launches += n0 + n1;
    return OVX_OK;
}
// interface update of plane 0 (owner = this rank, when it has a lower neighbour)
ovx_status dist_phase_iface(ovx_ctx *ctx) {
    if (!(ctx->slab_flags & 1)) return OVX_OK;
    CK(launch_iface_update(step_params(ctx), ctx->a_recv, ctx->u_send, ctx->s_hi));
    ctx->launches += 1;
    return OVX_OK;
}
// the context stream waits for s_hi; installs the top plane; swap
// accumulate the recorded phase times into the running totals and recycle the events
ovx_status fold_phase_events(ovx_ctx *ctx) {
    CK(cudaStreamSynchronize(ctx->stream));
    for (auto &ev : ctx->ph_used) {
        float t01 = 0.f, t12 = 0.f;
        CK(cudaEventElapsedTime(&t01, ev[0], ev[1]));   // step start -> edge chunks done
        CK(cudaEventElapsedTime(&t12, ev[1], ev[2]));   // edge chunks done -> exchanges + interface done
        ctx->ph_ebe_ms += t01;
        ctx->ph_halo_ms += t12;
        for (auto e : ev) ctx->ev_pool.push_back(e);
    }
    ctx->ph_used.clear();
    return OVX_OK;
}

ovx_status dist_phase_end(ovx_ctx *ctx, std::array<cudaEvent_t, 4> &ev) {
    CK(cudaEventRecord(ev[2], ctx->s_hi));
    CK(cudaStreamWaitEvent(ctx->stream, ev[2], 0));
    ovx_status s = ovx_step_end(ctx);
    if (s) return s;
    CK(cudaEventRecord(ev[3], ctx->stream));
    ctx->ph_used.push_back(ev);
    if (ctx->ph_used.size() >= 4096) return fold_phase_events(ctx);   // bounded event use on long runs
    return OVX_OK;
}

ovx_status dist_step(ovx_ctx *ctx, int64_t n) {
    ovx_status s = dist_prepare(ctx);
    if (s) return s;
    const nccl::Api &A = nccl::api();
    if (!ctx->nccl || !A.ok()) return fail(ctx, OVX_ENCCL, "no NCCL communicator (" + A.err + ")");
    const size_t cnt = (size_t)(3 * ctx->nn2());
    nccl::Comm comm = (nccl::Comm)ctx->nccl;
    const bool up = ctx->rank < ctx->world - 1, down = ctx->rank > 0;
    for (int64_t k = 0; k < n; ++k) {
        std::array<cudaEvent_t, 4> ev;
        if ((s = dist_phase_compute(ctx, ev))) return s;
        NK(A.GroupStart());   // T: the top interface's partial force to the owner above
        if (up) NK(A.Send(ctx->a_send, cnt, nccl::kFloat64, ctx->rank + 1, comm, ctx->s_hi));
        if (down) NK(A.Recv(ctx->a_recv, cnt, nccl::kFloat64, ctx->rank - 1, comm, ctx->s_hi));
        NK(A.GroupEnd());
        if ((s = dist_phase_iface(ctx))) return s;
        NK(A.GroupStart());   // the updated interface plane back to the rank below
        if (down) NK(A.Send(ctx->u_send, cnt, nccl::kFloat64, ctx->rank - 1, comm, ctx->s_hi));
        if (up) NK(A.Recv(ctx->u_recv, cnt, nccl::kFloat64, ctx->rank + 1, comm, ctx->s_hi));
        NK(A.GroupEnd());
        if ((s = dist_phase_end(ctx, ev))) return s;
    }
    return OVX_OK;
}

void dist_release(ovx_ctx *ctx) {
    for (auto &ev : ctx->ph_used)
        for (auto e : ev) ctx->ev_pool.push_back(e);
    ctx->ph_used.clear();
    for (auto e : ctx->ev_pool) cudaEventDestroy(e);
    ctx->ev_pool.clear();
    if (ctx->s_hi) cudaStreamDestroy(ctx->s_hi);
    ctx->s_hi = nullptr;
    if (ctx->nccl && nccl::api().CommDestroy) nccl::api().CommDestroy((nccl::Comm)ctx->nccl);
    ctx->nccl = nullptr;
    if (ctx->group) {
        auto &v = ctx->group->ranks;
        for (auto &r : v)
            if (r == ctx) r = nullptr;
        bool empty = true;
        for (auto r : v) empty &= (r == nullptr);
        if (empty) delete ctx->group;
        ctx->group = nullptr;
    }
}

}  // namespace

extern "C" {

ovx_status ovx_get_partition(int64_t nz, int world, int rank, int64_t *ez0, int64_t *ez1) {
    if (!ez0 || !ez1 || nz < 1 || world < 1 || rank < 0 || rank >= world)
        return fail(nullptr, OVX_EINVAL, "partition: need nz >= 1, 0 <= rank < world");
    const int64_t base = nz / world, rem = nz % world;
    *ez0 = rank * base + std::min<int64_t>(rank, rem);
    *ez1 = *ez0 + base + (rank < rem ? 1 : 0);
    return OVX_OK;
}

ovx_status ovx_nccl_unique_id(uint8_t out[128]) {
    if (!out) return fail(nullptr, OVX_EINVAL, "null argument");
    const nccl::Api &A = nccl::api();
    if (!A.ok()) return fail(nullptr, OVX_ENCCL, A.err);
    nccl::UniqueId id;
    ovx_ctx *ctx = nullptr;
    NK(A.GetUniqueId(&id));
    std::memcpy(out, id.internal, 128);
    return OVX_OK;
}

ovx_status ovx_create_dist(int device, int rank, int world, const uint8_t id[128], ovx_ctx **out) {
    if (!out || !id || world < 1 || rank < 0 || rank >= world) return fail(nullptr, OVX_EINVAL, "bad rank / world / id");
    ovx_status s = ovx_create(device, out);
    if (s) return s;
    ovx_ctx *ctx = *out;
    ctx->rank = rank;
    ctx->world = world;
    const nccl::Api &A = nccl::api();   // world = 1: a communicator of one (checks the NCCL setup)
    if (!A.ok()) {
        ovx_destroy(ctx);
        *out = nullptr;
        return fail(nullptr, OVX_ENCCL, A.err);
    }
    nccl::UniqueId uid;
    std::memcpy(uid.internal, id, 128);
    nccl::Comm comm = nullptr;
    cudaSetDevice(device);
    const nccl::Result r = A.CommInitRank(&comm, world, uid, rank);   // collective over the ranks
    if (r != 0) {
        ovx_destroy(ctx);
        *out = nullptr;
        return fail(nullptr, OVX_ENCCL, std::string("ncclCommInitRank: ") + (A.GetErrorString ? A.GetErrorString(r) : "?"));
    }
    ctx->nccl = comm;
    return OVX_OK;
}

ovx_status ovx_create_group(int world, const int *devices, ovx_ctx **out) {
    if (!out || !devices || world < 1) return fail(nullptr, OVX_EINVAL, "bad group arguments");
    LoopGroup *g = new LoopGroup();
    for (int r = 0; r < world; ++r) {
        ovx_ctx *c = nullptr;
        ovx_status s = ovx_create(devices[r], &c);
        if (s) {
            for (int q = 0; q < r; ++q) ovx_destroy(out[q]);   // the last destroy frees the group
            if (r == 0) delete g;
            return s;
        }
        c->rank = r;
        c->world = world;
        c->group = world > 1 ? g : nullptr;
        g->ranks.push_back(c);
        out[r] = c;
    }
    if (world == 1) delete g;
    return OVX_OK;
}

ovx_status ovx_step_group(ovx_ctx **ranks, int world, int64_t n) {
    if (!ranks || world < 1) return fail(nullptr, OVX_EINVAL, "bad group arguments");
    if (world == 1) return ovx_step(ranks[0], n);
    for (int r = 0; r < world; ++r) {
        ovx_ctx *ctx = ranks[r];
        if (!ctx || ctx->group == nullptr || ctx->group != ranks[0]->group || ctx->rank != r || ctx->world != world)
            return fail(ctx, OVX_EINVAL, "not the ranks of one loopback group, in rank order");
        ovx_status s = dist_prepare(ctx);
        if (s) return s;
    }
    std::vector<std::array<cudaEvent_t, 4>> ev(world);
    for (int64_t k = 0; k < n; ++k) {
        for (int r = 0; r < world; ++r) {
            ovx_ctx *ctx = ranks[r];
            cudaSetDevice(ctx->device);
            ovx_status s = dist_phase_compute(ctx, ev[r]);
            if (s) return s;
        }
        // T: a_send(r) -> a_recv(r+1), on the receiver's s_hi after the sender's edge chunks
        for (int r = 0; r + 1 < world; ++r) {
            ovx_ctx *ctx = ranks[r + 1];
            cudaSetDevice(ctx->device);
            CK(cudaStreamWaitEvent(ctx->s_hi, ev[r][1], 0));
            CK(cudaMemcpyPeerAsync(ctx->a_recv, ctx->device, ranks[r]->a_send, ranks[r]->device,
                                   8 * 3 * ctx->nn2(), ctx->s_hi));
        }
        for (int r = 0; r < world; ++r) {
            ovx_ctx *ctx = ranks[r];
            cudaSetDevice(ctx->device);
            ovx_status s = dist_phase_iface(ctx);
            if (s) return s;
            CK(cudaEventRecord(ev[r][2], ctx->s_hi));   // (re-recorded by the end phase)
        }
        // the updated plane: u_send(r) -> u_recv(r-1), on the receiver's s_hi after the owner's update
        for (int r = 1; r < world; ++r) {
            ovx_ctx *ctx = ranks[r - 1];
            cudaSetDevice(ctx->device);
            CK(cudaStreamWaitEvent(ctx->s_hi, ev[r][2], 0));
            CK(cudaMemcpyPeerAsync(ctx->u_recv, ctx->device, ranks[r]->u_send, ranks[r]->device,
                                   8 * 3 * ctx->nn2(), ctx->s_hi));
        }
        // the senders' next edge chunks must not overwrite a_send / u_send before the copies: every
        // s_hi waits for its neighbours' s_hi at the end of the step (through the context streams)
        for (int r = 0; r < world; ++r) {
            ovx_ctx *ctx = ranks[r];
            cudaSetDevice(ctx->device);
            ovx_status s = dist_phase_end(ctx, ev[r]);
            if (s) return s;
        }
        for (int r = 0; r < world; ++r) {
            ovx_ctx *ctx = ranks[r];
            cudaSetDevice(ctx->device);
            if (r > 0) CK(cudaStreamWaitEvent(ctx->stream, ev[r - 1][2], 0));
            if (r + 1 < world) CK(cudaStreamWaitEvent(ctx->stream, ev[r + 1][2], 0));
        }
    }
    return OVX_OK;
}

ovx_status ovx_get_phase_timers(ovx_ctx *ctx, double *ms_ebe, double *ms_halo, double *ms_update, int reset) {
    if (!ctx) return fail(nullptr, OVX_EINVAL, "null context");
    cudaSetDevice(ctx->device);
    CK(cudaStreamSynchronize(ctx->stream));
    double a = 0.0, b = 0.0;
    if (ctx->world > 1) {
        ovx_status s = fold_phase_events(ctx);
        if (s) return s;
        a = ctx->ph_ebe_ms;
        b = ctx->ph_halo_ms;
    } else {
        for (auto &p : ctx->ev_used) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, p.a, p.b));
            a += ms;
        }
    }
    if (ms_ebe) *ms_ebe = a;
    if (ms_halo) *ms_halo = b;
    if (ms_update) *ms_update = 0.0;   // the update is fused into the EBE kernels
    if (reset) {
        ctx->ph_ebe_ms = ctx->ph_halo_ms = 0.0;
        for (auto &p : ctx->ev_used) ctx->ev_free.push_back(p);
        ctx->ev_used.clear();
    }
    return OVX_OK;
}

}  // extern "C"
