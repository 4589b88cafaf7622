// Throughput of the FP64 / 64-bit conversion instructions the model
// evaluation uses (per SM per clock), measured with 8 independent chains.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CH 8
template <int OP>
__global__ void k(uint64_t *out, int iters, uint64_t seed) {
    uint64_t u[CH];
    double d[CH];
    for (int c = 0; c < CH; ++c) { u[c] = seed + threadIdx.x * 77 + c; d[c] = (double)(u[c] & 0xffff) + 0.25; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            if (OP == 0) d[c] = __ull2double_rn(u[c] + (uint64_t)i);          // I2F.F64.U64
            if (OP == 1) u[c] = (uint64_t)(long long)d[c] + (uint64_t)i, d[c] += 1.0;  // F2I.S64.F64 (+DADD)
            if (OP == 2) d[c] = rint(d[c] * 1.0000001);                          // FRND + DMUL
            if (OP == 3) d[c] = __dadd_rn(__dmul_rn(d[c], 1.0000001), 0.5);      // DMUL + DADD
            if (OP == 4) d[c] = __ll2double_rn((long long)u[c] + i);              // I2F.F64.S64
            if (OP == 5) u[c] = (u[c] * 0x9E3779B97F4A7C15ULL) ^ (u[c] >> 29);     // 64-bit int mul/xor/shift
            if (OP == 6) d[c] = (double)(float)d[c];                             // F2F
            if (OP == 7) u[c] = (uint64_t)__double2ll_rn(d[c]) + i, d[c] += 1.0;  // F2I rn
        }
    }
    uint64_t acc = 0;
    for (int c = 0; c < CH; ++c) acc ^= u[c] ^ (uint64_t)__double_as_longlong(d[c]);
    if (acc == 42) out[0] = acc;
}

template <int OP>
void run(const char *name, int sms, int clk_khz) {
    uint64_t *o;
    cudaMalloc(&o, 8);
    int iters = 4096, nt = 256, nb = sms * 8;
    k<OP><<<nb, nt>>>(o, 16, 1);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<OP><<<nb, nt>>>(o, iters, 1);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double ops = (double)nb * nt * iters * CH;
    double per_clk_sm = ops / (ms * 1e-3) / sms / (clk_khz * 1e3);
    printf("%-28s %8.3f ms  %7.2f thread-ops/clk/SM\n", name, ms, per_clk_sm);
    cudaFree(o);
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%s SMs=%d clk=%d kHz\n", p.name, p.multiProcessorCount, clk);
    run<0>("I2F.F64.U64", p.multiProcessorCount, clk);
    run<4>("I2F.F64.S64", p.multiProcessorCount, clk);
    run<1>("F2I.S64.F64.TRUNC+DADD", p.multiProcessorCount, clk);
    run<7>("F2I.S64.F64.RN+DADD", p.multiProcessorCount, clk);
    run<2>("FRND.F64+DMUL", p.multiProcessorCount, clk);
    run<3>("DMUL+DADD", p.multiProcessorCount, clk);
    run<5>("IMAD.WIDE64 mix", p.multiProcessorCount, clk);
    run<6>("F2F f64->f32->f64", p.multiProcessorCount, clk);
    return 0;
}
