// Micro-benchmark: dependent latency (cycles) of DFMA/DMUL/DADD/FFMA/FADD on one warp.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/dfp_latency.cu -o /tmp/dfp && gpurun -- /tmp/dfp
#include <cstdio>
__global__ void k(double* out, long long* cyc, double x0, float xf0) {
    double x = x0; float y = xf0; long long t0, t1;
#define BD(slot, expr) t0 = clock64(); for (int i = 0; i < 256; ++i) { x = expr; } t1 = clock64(); cyc[slot] = (t1 - t0); out[slot] = x; x = x0;
#define BF(slot, expr) t0 = clock64(); for (int i = 0; i < 256; ++i) { y = expr; } t1 = clock64(); cyc[slot] = (t1 - t0); out[slot] = y; y = xf0;
    BD(0, __fma_rn(x, 1.0000001, 1e-9))
    BD(1, x * 1.0000001)
    BD(2, x + 1e-9)
    BF(3, __fmaf_rn(y, 1.0000001f, 1e-9f))
    BF(4, y + 1e-9f)
    out[10] = x; out[11] = y;
}
int main() {
    double* d; long long* c; cudaMalloc(&d, 16*8); cudaMalloc(&c, 16 * 8);
    k<<<1, 32>>>(d, c, 0.7, 0.7f); k<<<1, 32>>>(d, c, 0.7, 0.7f); cudaDeviceSynchronize();
    long long h[16]; cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
    const char* names[] = {"DFMA", "DMUL", "DADD", "FFMA", "FADD"};
    for (int i = 0; i < 5; ++i) printf("%-6s %.2f cycles/op (dependent)\n", names[i], h[i] / 256.0);
    return 0;
}
