// Micro-benchmark: latency of the branch-free update helpers (atan2_bf, fast_sqrt, fast_rcp,
// ) against libm atan2 / IEEE division.  nvcc -I include -I paper_1907_00463_b200/csrc ...
#include <cstdio>
#include "correlator.cuh"
using namespace l1rxg;
__global__ void k(double* out, long long* cyc, double y0, double x0) {
    double y = y0, x = x0; long long t0, t1;
    t0 = clock64(); for (int i = 0; i < 256; ++i) { y = atan2_bf(y, x) + 0.5; } t1 = clock64(); cyc[0] = (t1 - t0) / 256; out[0] = y; y = y0;
    t0 = clock64(); for (int i = 0; i < 256; ++i) { y = fast_sqrt(y + 2.0); } t1 = clock64(); cyc[1] = (t1 - t0) / 256; out[1] = y; y = y0;
    t0 = clock64(); for (int i = 0; i < 256; ++i) { y = fast_rcp(y + 2.0); } t1 = clock64(); cyc[2] = (t1 - t0) / 256; out[2] = y; y = y0;
    cyc[3] = 0;
    t0 = clock64(); for (int i = 0; i < 256; ++i) { y = atan2(y, x) + 0.5; } t1 = clock64(); cyc[4] = (t1 - t0) / 256; out[4] = y; y = y0;
    t0 = clock64(); for (int i = 0; i < 256; ++i) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y)); y = r + 1.0; } t1 = clock64(); cyc[5] = (t1 - t0) / 256; out[5] = y; y = y0;
    t0 = clock64(); for (int i = 0; i < 256; ++i) { y = y / 16.368e6 + 3.0; } t1 = clock64(); cyc[6] = (t1 - t0) / 256; out[6] = y; y = y0;
}
int main() {
    double* d; long long* c; cudaMalloc(&d, 64); cudaMalloc(&c, 64);
    k<<<1, 32>>>(d, c, 0.3, 1.7); k<<<1, 32>>>(d, c, 0.3, 1.7); cudaDeviceSynchronize();
    long long h[8]; cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
    const char* n[] = {"atan2_bf+DADD", "fast_sqrt+DADD", "fast_rcp+DADD", "(removed)", "atan2 (libm)+DADD", "rcp.approx+DADD", "IEEE div+DADD"};
    for (int i = 0; i < 7; ++i) printf("%-22s %lld\n", n[i], h[i]);
}
