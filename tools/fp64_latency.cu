// Micro-benchmark: single-thread latency (cycles) of the fp64 operations on
// the loop-update critical path (one warp, lane 0, dependent chains).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double x0) {
    double x = x0, acc = 0;
    long long t0, t1;
#define BENCH(slot, expr)                                   \
    t0 = clock64();                                         \
    for (int i = 0; i < 64; ++i) { x = expr; }              \
    t1 = clock64(); cyc[slot] = (t1 - t0) / 64; acc += x; x = x0;
    BENCH(0, fma(x, 1.0000001, 1e-9))
    BENCH(1, x * 1.0000001 + 0.5 / (x + 3.0))
    BENCH(2, sqrt(x + 2.0))
    BENCH(3, atan(x * 0.5) + 0.1)
    BENCH(4, atan2(x, 1.5) + 0.2)
    BENCH(5, log10(x + 3.0))
    BENCH(6, fmod(x * 3000.0 + 7.0, 1023.0) * 1e-3)
    BENCH(7, (double)__frcp_rn((float)x) + x)
    BENCH(8, (double)__double2int_ru(x * 7.7) * 0.1)
    BENCH(9, 1.0 / x)
    float xf = (float)x0, accf = 0; float s, c;
    t0 = clock64();
    for (int i = 0; i < 64; ++i) { sincosf(xf, &s, &c); xf = s + 0.5f; }
    t1 = clock64(); cyc[10] = (t1 - t0) / 64; accf += xf;
    t0 = clock64();
    for (int i = 0; i < 64; ++i) { __sincosf(xf, &s, &c); xf = s + 0.5f; }
    t1 = clock64(); cyc[11] = (t1 - t0) / 64; accf += xf;
    out[0] = acc + accf;
}
int main() {
    double* d; long long* c; cudaMalloc(&d, 8); cudaMalloc(&c, 16 * 8);
    k<<<1, 32>>>(d, c, 0.7); k<<<1, 32>>>(d, c, 0.7);
    long long h[16]; cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
    const char* names[] = {"dfma", "fma+div", "sqrt", "atan", "atan2", "log10", "fmod", "frcp", "f2i+i2f", "rcp(div)", "sincosf", "__sincosf"};
    for (int i = 0; i < 12; ++i) printf("%-10s %lld cycles\n", names[i], h[i]);
    return 0;
}
