// Shared-memory histogram strategies for 2048 bins, uniform vs skewed
// (25% of keys in bin 0): MATCH.ANY aggregation vs plain ATOMS vs
// ballot-filtered hot bin.  Keys per clock per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t h32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

template <int MODE, bool SKEW>
__global__ void __launch_bounds__(1024) k(uint32_t *out, int iters) {
    __shared__ uint32_t h[4 * 2048];
    for (int j = threadIdx.x; j < 4 * 2048; j += blockDim.x) h[j] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t s = blockIdx.x * 1024 + threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        uint32_t r = h32(s + i * 7919u);
        int b = (SKEW && (r & 3) == 0) ? 0 : (int)((r >> 2) & 2047);
        uint32_t *hh = h + (MODE >= 2 ? (warp & 3) * 2048 : 0);
        if (MODE == 0 || MODE == 2) {
            unsigned peers = __match_any_sync(0xffffffffu, b);
            if (lane == __ffs(peers) - 1) atomicAdd(hh + b, __popc(peers));
        } else if (MODE == 1 || MODE == 3) {
            atomicAdd(hh + b, 1u);
        } else {  // hot bin 0 by ballot, rest plain
            unsigned hot = __ballot_sync(0xffffffffu, b == 0);
            if (b != 0) atomicAdd(hh + b, 1u);
            else if (lane == __ffs(hot) - 1) atomicAdd(hh, __popc(hot));
        }
    }
    __syncthreads();
    uint32_t acc = 0;
    for (int j = threadIdx.x; j < 4 * 2048; j += blockDim.x) acc += h[j];
    if (acc == 12345) out[0] = acc;
}

template <int MODE, bool SKEW>
void run(const char *name, int sms, int clk) {
    uint32_t *o;
    cudaMalloc(&o, 4);
    int iters = 2048;
    k<MODE, SKEW><<<sms, 1024>>>(o, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<MODE, SKEW><<<sms, 1024>>>(o, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double keys = (double)sms * 1024 * iters;
    printf("%-34s %s %7.3f ms %6.2f keys/clk/SM\n", name, SKEW ? "skew" : "unif", ms, keys / (ms * 1e-3) / sms / (clk * 1e3));
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    run<0, false>("match+atoms 1 copy", p.multiProcessorCount, clk);
    run<0, true>("match+atoms 1 copy", p.multiProcessorCount, clk);
    run<1, false>("atoms 1 copy", p.multiProcessorCount, clk);
    run<1, true>("atoms 1 copy", p.multiProcessorCount, clk);
    run<2, true>("match+atoms 4 copies", p.multiProcessorCount, clk);
    run<3, false>("atoms 4 copies", p.multiProcessorCount, clk);
    run<3, true>("atoms 4 copies", p.multiProcessorCount, clk);
    run<4, true>("ballot-hot + atoms 4 copies", p.multiProcessorCount, clk);
    return 0;
}
