// capi.cu — the C ABI declared in include/ovx.h (host-side L1/L4 logic).
#include <cmath>
#include <cstdio>
#include <cstring>
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
    double *d_un = nullptr;           // third state buffer of damped steps
    int8_t k8[1152];
    double Ak[576], Ag[576], Kk[576], Kg[576];
    std::vector<MatConst> mc;
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
    int64_t nn2() const { return (nx + 1) * (ny + 1); }
    int64_t nn() const { return (nx + 1) * (ny + 1) * (nz + 1); }
    int64_t ne() const { return nx * ny * nz; }
};

namespace {

std::string g_err;
const ovx_ctx *g_const_owner[64] = {nullptr};

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

ovx_status ensure_constants(ovx_ctx *ctx) {
    if (ctx->device >= 0 && ctx->device < 64 && g_const_owner[ctx->device] == ctx) return OVX_OK;
    CK(upload_constants(ctx->mc.data(), ctx->nmat, ctx->k8, ctx->Kk, ctx->Kg, ctx->stream));
    if (ctx->device >= 0 && ctx->device < 64) g_const_owner[ctx->device] = ctx;
    return OVX_OK;
}

ovx_status refresh_w(ovx_ctx *ctx) {
    if (!ctx->setup || !(ctx->dt > 0)) return OVX_OK;
    ovx_status s = ensure_constants(ctx);
    if (s) return s;
    CK(launch_node_w(ctx->nx, ctx->ny, ctx->nz, ctx->d_mat, (ctx->slab_flags & 1) ? ctx->d_mat_below : nullptr,
                     ctx->dt, ctx->d_w, ctx->stream));
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
    p.w = ctx->d_w;
    p.mat = ctx->d_mat;
    p.dmask = ctx->d_mask;
    p.stages = ctx->stages;
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
    for (auto &p : ctx->ev_used) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
    for (auto &p : ctx->ev_free) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    if (ctx->device >= 0 && ctx->device < 64 && g_const_owner[ctx->device] == ctx) g_const_owner[ctx->device] = nullptr;
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
    const int64_t nn = ctx->nn(), ne = ctx->ne();
    if (cudaMalloc(&ctx->d_mat, ne) != cudaSuccess || cudaMalloc(&ctx->d_u, 24 * nn) != cudaSuccess ||
        cudaMalloc(&ctx->d_up, 24 * nn) != cudaSuccess || cudaMalloc(&ctx->d_w, 8 * nn) != cudaSuccess) {
        cudaGetLastError();
        return fail(ctx, OVX_ENOMEM, "device allocation failed for the grid");
    }
    CK(cudaMemsetAsync(ctx->d_u, 0, 24 * nn, ctx->stream));
    CK(cudaMemsetAsync(ctx->d_up, 0, 24 * nn, ctx->stream));
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
    const int64_t ne = ctx->ne();
    for (int64_t e = 0; e < ne; ++e)
        if (mat[e] >= ctx->nmat) return fail(ctx, OVX_EINVAL, "unknown material id at element " + std::to_string(e));
    cudaSetDevice(ctx->device);
    CK(cudaMemcpyAsync(ctx->d_mat, mat, ne, cudaMemcpyHostToDevice, ctx->stream));
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
    if (path != OVX_INT8 && path != OVX_FP64 && path != OVX_FP64_DENSE && path != OVX_VFEM && path != OVX_VFEM_DENSE)
        return fail(ctx, OVX_EINVAL, "path must be OVX_INT8, OVX_FP64, OVX_FP64_DENSE, OVX_VFEM or OVX_VFEM_DENSE");
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
    ctx->mc.resize(ctx->nmat);
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
    ctx->setup = true;
    cudaSetDevice(ctx->device);
    if (ctx->device >= 0 && ctx->device < 64 && g_const_owner[ctx->device] == ctx) g_const_owner[ctx->device] = nullptr;
    ovx_status s = ensure_constants(ctx);
    if (s) return s;
    return refresh_w(ctx);
}

ovx_status ovx_get_int8_matrix(ovx_ctx *ctx, int8_t *out) {  // ctx may be NULL (host-only)
    if (!out) return fail(ctx, OVX_EINVAL, "null argument");
    int8_t k8[1152];
    if (derive_element_matrices(k8, nullptr, nullptr) != 0) return fail(ctx, OVX_EINVAL, "non-INT8 entry");
    std::memcpy(out, k8, 1152);
    return OVX_OK;
}

ovx_status ovx_critical_dt(ovx_ctx *ctx, double *dt_elem_bound) {
    if (!ctx || !dt_elem_bound) return fail(ctx, OVX_EINVAL, "null argument");
    if (!ctx->have_grid || ctx->nmat == 0) return fail(ctx, OVX_ESTATE, "set grid and materials first");
    double Ak[576], Ag[576], K[576];
    if (derive_element_matrices(nullptr, Ak, Ag) != 0) return fail(ctx, OVX_EINVAL, "derivation failed");
    double lmax = 0.0;
    for (int m = 0; m < ctx->nmat; ++m) {
        for (int i = 0; i < 576; ++i) K[i] = ctx->kappa[m] * ctx->ds * Ak[i] + ctx->G[m] * ctx->ds * Ag[i];
        const double lam = sym_lambda_max(K) / (ctx->rho[m] * ctx->ds * ctx->ds * ctx->ds / 8.0);
        if (lam > lmax) lmax = lam;
    }
    *dt_elem_bound = 2.0 / std::sqrt(lmax);
    return OVX_OK;
}

ovx_status ovx_set_sources(ovx_ctx *ctx, int n, const int64_t *node, const int32_t *axis, int64_t n_t,
                           const double *amp) {
    if (!ctx) return fail(nullptr, OVX_EINVAL, "null context");
    if (!ctx->have_grid) return fail(ctx, OVX_ESTATE, "set grid first");
    if (n < 0 || n > kMaxSrc || n_t < 0) return fail(ctx, OVX_EINVAL, "0..16 sources");
    if (n > 0 && (!node || !axis || (n_t > 0 && !amp))) return fail(ctx, OVX_EINVAL, "null source arrays");
    for (int k = 0; k < n; ++k)
        if (node[k] < 0 || node[k] >= ctx->nn() || axis[k] < 0 || axis[k] > 2)
            return fail(ctx, OVX_EINVAL, "source node/axis out of range");
    if (n > 0 && n_t > 0 && !finite_all(amp, (int64_t)n * n_t)) return fail(ctx, OVX_EINVAL, "non-finite amplitude");
    ctx->nsrc = n;
    ctx->src_node.assign(node, node + n);
    ctx->src_axis.assign(axis, axis + n);
    ctx->n_t = n_t;
    ctx->amp.assign(amp, amp + (size_t)n * (size_t)n_t);
    return OVX_OK;
}

static ovx_status set_state_impl(ovx_ctx *ctx, const double *u, const double *up, int64_t it, cudaMemcpyKind kind) {
    if (!ctx) return fail(nullptr, OVX_EINVAL, "null context");
    if (!ctx->have_grid) return fail(ctx, OVX_ESTATE, "set grid first");
    if (!u || !up) return fail(ctx, OVX_EINVAL, "null state arrays");
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
    if (ctx->slab_flags) return fail(ctx, OVX_ESTATE, "slab contexts step with ovx_step_begin/iface/end");
    if (n == 0) return OVX_OK;
    cudaSetDevice(ctx->device);
    s = ensure_constants(ctx);
    if (s) return s;
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
            p.src_val[q] = (ctx->it < ctx->n_t) ? ctx->amp[(size_t)q * ctx->n_t + ctx->it] : 0.0;
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
        p.src_val[q] = (ctx->it < ctx->n_t) ? ctx->amp[(size_t)q * ctx->n_t + ctx->it] : 0.0;
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
    s = ensure_constants(ctx);
    if (s) return s;
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
    for (int k = 0; k < n; ++k)
        if (node[k] < 0 || node[k] >= ctx->nn()) return fail(ctx, OVX_EINVAL, "receiver node out of range");
    cudaSetDevice(ctx->device);
    dfree(ctx->d_traces);
    ctx->d_traces = nullptr;
    ctx->nrec = n;
    ctx->rec_node.assign(node, node + n);
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
    ovx_status s = ensure_constants(ctx);
    if (s) return s;
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
    s = ensure_constants(ctx);
    if (s) return s;
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
