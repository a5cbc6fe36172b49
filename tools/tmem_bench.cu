// tmem_bench.cu — per-SM TMEM load / store throughput on sm_100a (tcgen05.ld / tcgen05.st,
// 32x32b shapes), as seen by W warps of one CTA per SM.  Prints JSON lines.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/tmem_bench tools/tmem_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int OP, int X>
__global__ void __launch_bounds__(512, 1) kern(int nwarps, unsigned *out, long long *cyc) {
    __shared__ uint32_t tm;
    const int w = threadIdx.x >> 5;
    if (w == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tm)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = tm + ((uint32_t)((w & 3) * 32) << 16) + (uint32_t)((w >> 2) * 64);
    uint32_t acc = 0;
    long long t0 = clock64();
    if (w < nwarps) {
        for (int it = 0; it < ITERS; ++it) {
            const uint32_t a = base + (uint32_t)((it & 1) * 32);
            if (OP == 0) {
                if (X == 8) {
                    uint32_t r[8];
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                                   "=r"(r[7])
                                 : "r"(a));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    for (int i = 0; i < 8; ++i) acc += r[i];
                } else {
                    uint32_t r[32];
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                        : "r"(a));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    for (int i = 0; i < 32; ++i) acc += r[i];
                }
            } else {
                asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(acc), "r"(acc + 1),
                             "r"(acc + 2), "r"(acc + 3)
                             : "memory");
                asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a + 4), "r"(acc),
                             "r"(acc + 1), "r"(acc + 2), "r"(acc + 3)
                             : "memory");
                if ((it & 3) == 3) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                acc += it;
            }
        }
    }
    long long t1 = clock64();
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * 512 + threadIdx.x] = acc;
}

template <int OP, int X>
void run(const char *name, int nw, unsigned *out, long long *cyc) {
    kern<OP, X><<<148, 512>>>(nw, out, cyc);
    kern<OP, X><<<148, 512>>>(nw, out, cyc);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < 148; ++i) mean += h[i];
    mean /= 148;
    const double bytes = (double)nw * 32 * 4 * (OP == 0 ? X : 8) * ITERS;   // per SM
    printf("{\"op\": \"%s\", \"warps\": %d, \"cycles\": %.0f, \"bytes_per_clk_per_sm\": %.2f}\n", name, nw, mean,
           bytes / mean);
}

int main() {
    unsigned *out;
    long long *cyc;
    cudaMalloc(&out, 148 * 512 * 4);
    cudaMalloc(&cyc, 148 * 8);
    for (int nw : {1, 4, 8, 16}) {
        run<0, 8>("ld.32x32b.x8", nw, out, cyc);
        run<0, 32>("ld.32x32b.x32", nw, out, cyc);
        run<1, 4>("st.32x32b.x4(x2)", nw, out, cyc);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
    return 0;
}
