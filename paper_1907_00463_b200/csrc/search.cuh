// search.cuh -- K4: correlator-bank search grid (BASELINE config 5), sm_100a.
//
// Semantics: acquire_pcs's plane (acquisition.hpp:189-222): for PRN p,
// Doppler bin f and 1-ms segment s, the carrier is wiped with
// e^{-j 2 pi f n / fs} anchored at the global sample index n
// (wipe_carrier, :170-182), circularly correlated with the zero-order-hold
// code, and |.| is accumulated over segments; FFTW's inverse is
// unnormalised (fft.hpp:17-19), so a cell is N * |sum_n wiped[n] code[(n-d) mod N]|.
//
// Evaluated directly at the half-chip delays d = k * spc (spc = samples per
// half chip, an integer at the config rates, e.g. 8 at 16.368 MHz) through an
// exact identity: the ZOH code is constant over each chip, so with
//   F0[c] = sum of the wiped samples of chip c,
//   F1[c] = the same shifted by half a chip,
// corr[d = 2j*spc]     = sum_c F0[c] chip[(c - j) mod 1023]
// corr[d = (2j+1)*spc] = sum_c F1[c] chip[(c - j) mod 1023]
// i.e. two 1023-point circular correlations per (PRN, bin, segment) instead of
// N x 2046 multiply-adds.  K4a folds (per bin and segment, shared by all PRNs);
// K4b is a register-tiled circulant +-1 correlation on the FP32 pipes.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace l1rxg {

constexpr int GRID_CHIPS = 1023;

// K4a: one CTA per (bin, segment).  x: baseband [n_seg][N]; F out:
// [bin][seg][2][1023] float2.  spc = samples per half chip.
__global__ void __launch_bounds__(256) grid_fold_kernel(const float2* __restrict__ x, int N, int spc,
                                                        const double* __restrict__ bins, double fs,
                                                        int n_seg, float2* F) {
    extern __shared__ float2 hsum[];  // [2 * 1023] half-chip sums
    const int bin = blockIdx.x / n_seg, seg = blockIdx.x % n_seg;
    const double w = -2.0 * 3.14159265358979323846 * bins[bin] / fs;  // wipe_carrier :172
    const int nh = 2 * GRID_CHIPS;
    const float2* xs = x + (int64_t)seg * N;
    for (int h = threadIdx.x; h < nh; h += blockDim.x) {
        // anchor at the half chip's first sample (global index), fp64 reduced
        const int64_t n0 = (int64_t)seg * N + (int64_t)h * spc;
        const double th = w * (double)n0;
        const double r = fma(-rint(th * (1.0 / (2.0 * 3.14159265358979323846))),
                             2.0 * 3.14159265358979323846, th);
        float sa, ca;
        sincosf((float)r, &sa, &ca);
        float ws, wc;
        sincosf((float)w, &ws, &wc);
        float cr = ca, ci = sa, accr = 0.f, acci = 0.f;
        for (int k = 0; k < spc; ++k) {  // x * e^{j(th + w k)}
            const float2 v = xs[h * spc + k];
            accr = fmaf(v.x, cr, fmaf(-v.y, ci, accr));
            acci = fmaf(v.x, ci, fmaf(v.y, cr, acci));
            const float nr = cr * wc - ci * ws;
            ci = cr * ws + ci * wc;
            cr = nr;
        }
        hsum[h] = make_float2(accr, acci);
    }
    __syncthreads();
    float2* Fo = F + ((int64_t)bin * n_seg + seg) * 2 * GRID_CHIPS;
    for (int c = threadIdx.x; c < GRID_CHIPS; c += blockDim.x) {
        const float2 a = hsum[2 * c], b = hsum[2 * c + 1], d = hsum[(2 * c + 2) % nh];
        Fo[c] = make_float2(a.x + b.x, a.y + b.y);                      // F0
        Fo[GRID_CHIPS + c] = make_float2(b.x + d.x, b.y + d.y);         // F1
    }
}

// K4b: one CTA per (PRN, bin, parity); the n_seg vectors of that (bin,
// parity) sit in shared memory; thread t owns shifts j = t + 256 q (q < 4),
// vectors in groups of VG; cells accumulate N * |corr| over segments.
constexpr int GRID_TPB = 256;
constexpr int GRID_SH = 4;   // shifts per thread (4 * 256 >= 1023)
constexpr int GRID_VG = 5;   // vectors per register group

__global__ void __launch_bounds__(GRID_TPB) grid_corr_kernel(const float2* __restrict__ F,
                                                             const int8_t* __restrict__ codes,
                                                             const int32_t* __restrict__ prns,
                                                             int n_bins, int n_seg, float scale,
                                                             float* plane /*[prn][bin][2046]*/) {
    extern __shared__ __align__(16) unsigned char sm[];
    float* cd = reinterpret_cast<float*>(sm);                 // chips doubled [2 * 1024]
    float2* fv = reinterpret_cast<float2*>(sm + 2 * 1024 * 4);  // [n_seg][1023]
    const int par = blockIdx.x & 1;
    const int bin = (blockIdx.x >> 1) % n_bins;
    const int pi = (blockIdx.x >> 1) / n_bins;
    const int8_t* code = codes + prns[pi] * GRID_CHIPS;
    // cd[u] = chip[(u - 1023) mod 1023] for u in [0, 2046): chip[(c - j) mod 1023] = cd[c - j + 1023]
    for (int u = threadIdx.x; u < 2 * GRID_CHIPS; u += blockDim.x)
        cd[u] = (float)code[u % GRID_CHIPS];
    for (int s = 0; s < n_seg; ++s)
        for (int c = threadIdx.x; c < GRID_CHIPS; c += blockDim.x)
            fv[s * GRID_CHIPS + c] =
                F[(((int64_t)bin * n_seg + s) * 2 + par) * GRID_CHIPS + c];
    __syncthreads();
    float mag[GRID_SH];
#pragma unroll
    for (int q = 0; q < GRID_SH; ++q)
        mag[q] = 0.f;
    const int j0 = threadIdx.x;
    for (int s0 = 0; s0 < n_seg; s0 += GRID_VG) {
        float ar[GRID_SH][GRID_VG], ai[GRID_SH][GRID_VG];
#pragma unroll
        for (int q = 0; q < GRID_SH; ++q)
#pragma unroll
            for (int v = 0; v < GRID_VG; ++v)
                ar[q][v] = ai[q][v] = 0.f;
        const int nv = min(GRID_VG, n_seg - s0);
#pragma unroll 2
        for (int c = 0; c < GRID_CHIPS; ++c) {
            float ch[GRID_SH];
#pragma unroll
            for (int q = 0; q < GRID_SH; ++q) {
                const int j = j0 + q * GRID_TPB;
                ch[q] = j < GRID_CHIPS ? cd[c - j + GRID_CHIPS] : 0.f;
            }
#pragma unroll
            for (int v = 0; v < GRID_VG; ++v) {
                const float2 f = v < nv ? fv[(s0 + v) * GRID_CHIPS + c] : make_float2(0.f, 0.f);
#pragma unroll
                for (int q = 0; q < GRID_SH; ++q) {
                    ar[q][v] = fmaf(ch[q], f.x, ar[q][v]);
                    ai[q][v] = fmaf(ch[q], f.y, ai[q][v]);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < GRID_SH; ++q)
#pragma unroll
            for (int v = 0; v < GRID_VG; ++v)
                if (v < nv)
                    mag[q] += scale * sqrtf(fmaf(ar[q][v], ar[q][v], ai[q][v] * ai[q][v]));
    }
    float* row = plane + ((int64_t)pi * n_bins + bin) * (2 * GRID_CHIPS);
#pragma unroll
    for (int q = 0; q < GRID_SH; ++q) {
        const int j = j0 + q * GRID_TPB;
        if (j < GRID_CHIPS)
            row[2 * j + par] = mag[q];
    }
}

// ---- K4b on the tensor cores ------------------------------------------
// The 2 x n_bins x n_seg circular correlations of a PRN are ONE matrix
// product: with M_p[k][j] = chip_p[(k - j) mod 1023] (a circulant, +-1),
// corr[v][j] = sum_k F[v][k] M_p[k][j] for every fold vector v (re and im
// separately).  The fp32 folds are split into three bf16 terms
// F = F1 + F2 + F3 (24 significant bits, as fp32), and +-1 is exact in bf16,
// so one bf16 GEMM with K = 3 x 1024 ([F1 F2 F3] against [M; M; M]) and fp32
// accumulation reproduces the fp32 correlation on the 5th-gen tensor cores.
constexpr int GRID_K = 1024;      // 1023 chips padded with a zero row/column
constexpr int GRID_KS = 3 * GRID_K;

// A[r][GRID_KS], r = vector * 2 + (0: re, 1: im); vector = (bin*n_seg+seg)*2+par
__global__ void grid_split_kernel(const float2* __restrict__ F, int n_vec, __nv_bfloat16* A) {
    const int v = blockIdx.x;
    for (int c = threadIdx.x; c < GRID_K; c += blockDim.x) {
        const float2 f = c < GRID_CHIPS ? F[(int64_t)v * GRID_CHIPS + c] : make_float2(0.f, 0.f);
#pragma unroll
        for (int ri = 0; ri < 2; ++ri) {
            const float x = ri ? f.y : f.x;
            const __nv_bfloat16 h1 = __float2bfloat16_rn(x);
            const float r1 = x - __bfloat162float(h1);
            const __nv_bfloat16 h2 = __float2bfloat16_rn(r1);
            const __nv_bfloat16 h3 = __float2bfloat16_rn(r1 - __bfloat162float(h2));
            __nv_bfloat16* row = A + ((int64_t)v * 2 + ri) * GRID_KS;
            row[c] = h1;
            row[GRID_K + c] = h2;
            row[2 * GRID_K + c] = h3;
        }
    }
}

// Mt_p (column-major GRID_K x GRID_KS for cuBLAS): Mt[j + GRID_K * k'] =
// chip_p[(k - j) mod 1023] with k = k' mod GRID_K, zero on the padding.
__global__ void grid_circ_kernel(const int8_t* __restrict__ codes, const int32_t* __restrict__ prns,
                                 __nv_bfloat16* Mt) {
    const int pi = blockIdx.y;
    const int kp = blockIdx.x;  // column k'
    const int k = kp % GRID_K;
    const int8_t* code = codes + prns[pi] * GRID_CHIPS;
    __nv_bfloat16* col = Mt + ((int64_t)pi * GRID_KS + kp) * GRID_K;
    for (int j = threadIdx.x; j < GRID_K; j += blockDim.x) {
        float v = 0.f;
        if (k < GRID_CHIPS && j < GRID_CHIPS) {
            int m = k - j;
            if (m < 0)
                m += GRID_CHIPS;
            v = (float)code[m];
        }
        col[j] = __float2bfloat16_rn(v);
    }
}

// plane[p][bin][2j + par] = scale * sum_seg |C_p[re row][j] + i C_p[im row][j]|
// (four delays per thread: 16-byte loads; the product rows of a (bin, par)
// are read once, HBM-bound)
__global__ void grid_mag_kernel(const float* __restrict__ C, int n_rows, int n_bins, int n_seg,
                                float scale, float* plane) {
    const int pi = blockIdx.y;
    const int bp = blockIdx.x;  // bin * 2 + par
    const int bin = bp >> 1, par = bp & 1;
    const float* Cp = C + (int64_t)pi * n_rows * GRID_K;
    float* row = plane + ((int64_t)pi * n_bins + bin) * (2 * GRID_CHIPS);
    const int j4 = threadIdx.x;  // delays 4*j4 .. 4*j4+3 (GRID_K = 4 * 256)
    float4 m = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
    for (int seg = 0; seg < n_seg; ++seg) {
        const int64_t v = ((int64_t)bin * n_seg + seg) * 2 + par;
        const float4 re = __ldcs(reinterpret_cast<const float4*>(Cp + (v * 2) * GRID_K) + j4);
        const float4 im = __ldcs(reinterpret_cast<const float4*>(Cp + (v * 2 + 1) * GRID_K) + j4);
        m.x += scale * sqrtf(fmaf(re.x, re.x, im.x * im.x));
        m.y += scale * sqrtf(fmaf(re.y, re.y, im.y * im.y));
        m.z += scale * sqrtf(fmaf(re.z, re.z, im.z * im.z));
        m.w += scale * sqrtf(fmaf(re.w, re.w, im.w * im.w));
    }
    const float mv[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int j = 4 * j4 + q;
        if (j < GRID_CHIPS)
            row[2 * j + par] = mv[q];
    }
}

// plane [prn][bin][2046] fp32 -> [prn][bin][n_delays] fp32 or fp64
__global__ void grid_plane_out_kernel(const float* __restrict__ plane, int n_delays, int64_t cells, void* out,
                                      int f32) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cells)
        return;
    const int64_t r = i / n_delays, k = i - r * n_delays;
    const float v = plane[r * (2 * GRID_CHIPS) + k];
    if (f32)
        static_cast<float*>(out)[i] = v;
    else
        static_cast<double*>(out)[i] = (double)v;
}

}  // namespace l1rxg
