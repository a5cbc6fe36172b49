// microbench.cu — per-SM throughput of the instructions the INT8 element path issues on CUDA
// cores (F2I.S64.F64, I2F.F64.S64, PRMT, DMUL/DFMA, IMAD.WIDE, IADD) on sm_100a.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

#define BODY8(STMT) STMT(0) STMT(1) STMT(2) STMT(3) STMT(4) STMT(5) STMT(6) STMT(7)

template <int OP>
__global__ void kern(const double *in, unsigned long long *out, long long *cyc) {
    double d[8];
    long long l[8];
    uint32_t u[8];
    for (int i = 0; i < 8; ++i) {
        d[i] = in[(threadIdx.x + i) & 63];
        l[i] = (long long)threadIdx.x * 7919 + i;
        u[i] = threadIdx.x * 2654435761u + i;
    }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
        if (OP == 0) {  // F2I.S64.F64.TRUNC
#define S(i) asm volatile("cvt.rzi.s64.f64 %0, %1;\n\tcvt.rn.f64.s64 %1, %0;" : "=l"(l[i]), "+d"(d[i]));
            BODY8(S)
#undef S
        } else if (OP == 1) {  // I2F.F64.S64
#define S(i) asm volatile("cvt.rn.f64.s64 %0, %1;\n\tadd.s64 %1, %1, 1;" : "=d"(d[i]), "+l"(l[i]));
            BODY8(S)
#undef S
        } else if (OP == 2) {  // PRMT
#define S(i) asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(u[i]) : "r"(u[(i + 1) & 7]));
            BODY8(S)
#undef S
        } else if (OP == 3) {  // DFMA
#define S(i) asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[i]) : "d"(d[(i + 3) & 7]));
            BODY8(S)
#undef S
        } else if (OP == 4) {  // IMAD.WIDE
#define S(i) asm volatile("mad.wide.s32 %0, %1, %2, %0;" : "+l"(l[i]) : "r"(u[i]), "r"(u[(i + 1) & 7]));
            BODY8(S)
#undef S
        } else if (OP == 5) {  // IADD (32-bit)
#define S(i) asm volatile("add.s32 %0, %0, %1;" : "+r"(u[i]) : "r"(u[(i + 5) & 7]));
            BODY8(S)
#undef S
        } else if (OP == 6) {  // I2F.F64.S32
#define S(i) asm volatile("cvt.rn.f64.s32 %0, %1;\n\tcvt.rzi.s32.f64 %1, %0;" : "=d"(d[i]), "+r"(u[i]));
            BODY8(S)
#undef S
        } else if (OP == 7) {  // FP64 max (fmax)
#define S(i) asm volatile("max.f64 %0, %0, %1;" : "+d"(d[i]) : "d"(d[(i + 3) & 7]));
            BODY8(S)
#undef S
        }
    }
    long long t1 = clock64();
    unsigned long long acc = 0;
    for (int i = 0; i < 8; ++i) acc ^= (unsigned long long)l[i] ^ u[i] ^ __double_as_longlong(d[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char *name, const double *in, unsigned long long *out, long long *cyc, int sms) {
    const int threads = 1024;
    kern<OP><<<sms, threads>>>(in, out, cyc);
    cudaDeviceSynchronize();
    kern<OP><<<sms, threads>>>(in, out, cyc);
    cudaDeviceSynchronize();
    long long h[1024];
    cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < sms; ++i) mean += h[i];
    mean /= sms;
    double ops = (double)threads * ITERS * 8;
    printf("{\"op\": \"%s\", \"per_sm_per_clk\": %.2f}\n", name, ops / mean);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *in;
    unsigned long long *out;
    long long *cyc;
    cudaMalloc(&in, 64 * 8);
    double h[64];
    for (int i = 0; i < 64; ++i) h[i] = 0.37 * (i + 1) * (i % 2 ? -1 : 1);
    cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
    cudaMalloc(&out, sizeof(unsigned long long) * sms * 1024);
    cudaMalloc(&cyc, sizeof(long long) * sms);
    run<0>("F2I.S64.F64+I2F.F64.S64 pair", in, out, cyc, sms);
    run<1>("I2F.F64.S64+IADD64", in, out, cyc, sms);
    run<2>("PRMT", in, out, cyc, sms);
    run<3>("DFMA", in, out, cyc, sms);
    run<4>("IMAD.WIDE", in, out, cyc, sms);
    run<5>("IADD", in, out, cyc, sms);
    run<6>("I2F.F64.S32+F2I.S32.F64 pair", in, out, cyc, sms);
    run<7>("DMNMX(max.f64)", in, out, cyc, sms);
    printf("{\"sms\": %d}\n", sms);
    return 0;
}
