// Micro-benchmark: latency of fp64<->int conversions, FRND, LDS chains and SHFL on one warp.
#include <cstdio>
__global__ void k(double* out, long long* cyc, double x0, int i0, const short* sp) {
    double x = x0; int iv = i0; long long t0, t1;
    t0 = clock64(); for (int i = 0; i < 256; ++i) { x = (double)(iv + (int)x); } t1 = clock64(); cyc[0] = t1 - t0; out[0] = x; x = x0;
    t0 = clock64(); for (int i = 0; i < 256; ++i) { x = (double)__double2int_ru(x * 1.5) ; } t1 = clock64(); cyc[1] = t1 - t0; out[1] = x; x = x0;
    t0 = clock64(); for (int i = 0; i < 256; ++i) { x = rint(x * 1.5) + 0.25; } t1 = clock64(); cyc[2] = t1 - t0; out[2] = x; x = x0;
    t0 = clock64(); for (int i = 0; i < 256; ++i) { x = x * 1.0000001 + 0.1; } t1 = clock64(); cyc[3] = t1 - t0; out[3] = x; x = x0;
    // LDS latency chain
    __shared__ int sm[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sm[i] = (i + 1) & 255;
    __syncthreads();
    int p = 0;
    t0 = clock64(); for (int i = 0; i < 256; ++i) { p = sm[p]; } t1 = clock64(); cyc[4] = t1 - t0; out[4] = p;
    float f = (float)x0;
    t0 = clock64(); for (int i = 0; i < 256; ++i) { f = __shfl_sync(0xffffffffu, f, 1) + 1.0f; } t1 = clock64(); cyc[5] = t1 - t0; out[5] = f;
}
int main() {
    double* d; long long* c; short* sp; cudaMalloc(&d, 16*8); cudaMalloc(&c, 16 * 8); cudaMalloc(&sp, 64);
    k<<<1, 32>>>(d, c, 0.7, 3, sp); k<<<1, 32>>>(d, c, 0.7, 3, sp); cudaDeviceSynchronize();
    long long h[16]; cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
    const char* names[] = {"I2F.F64(+F2I)", "F2I.CEIL+I2F+DMUL", "FRND+DMUL+DADD", "DFMA", "LDS chain", "SHFL+FADD"};
    for (int i = 0; i < 6; ++i) printf("%-20s %.1f cycles/iter\n", names[i], h[i] / 256.0);
    return 0;
}
