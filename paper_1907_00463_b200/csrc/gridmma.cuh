// gridmma.cuh -- K4c: the config-5 correlator bank as ONE hand-written
// tcgen05 int8 GEMM per launch with the |.| + noncoherent sum fused into the
// epilogue (sm_100a).
//
// Semantics (acquisition.hpp:189-222, see search.cuh): for PRN p, Doppler
// bin b, parity par (even / odd half-chip delays) and 1-ms segment s,
//   corr[j] = sum_k F[b,s,par][k] * chip_p[(k - j) mod 1023]   (j, k < 1023)
// and plane[p][b][2j + par] = N * sum_s |corr_s[j]| (FFTW's unnormalised
// inverse, fft.hpp:17-19).
//
// Exact integer formulation.  Each fold row (b, s, par, re|im) is quantised
// to 24-bit integers X = round(F / sc), sc = max|F| / (2^23 - 2^16) per row,
// and split into three signed base-256 digits X = 65536 d2 + 256 d1 + d0
// (d_i in [-128, 127]).  The chips are +-1, so every digit correlation
// sum_k d[k] chip[(k - j) mod 1023] is exact in int32 -- one kind::i8 MMA
// with int32 accumulation -- and the epilogue recombines
// corr = sc (65536 c2 + 256 c1 + c0) in fp32 (quantisation 6e-8 of the
// row's largest fold, far inside the 1e-5 parity bar).
//
// GEMM: D[j][r] = sum_k A[j][k] B[r][k], both operands K-major int8:
//   A = the circulant tile of PRN p for 128 delays j (M = 128 TMEM lanes),
//       GENERATED IN SHARED MEMORY from the 1023-chip code (128 KB, all of
//       K = 1024, kept across every fold group of the same (p, delay tile));
//   B = the digit rows of one fold group g = (bin, par): n_seg segments x
//       (re, im) x 3 digits, in chunks of 5 segments per 32 rows
//       (N = 32 ceil(n_seg / 5); 128 for config 5's 20 segments), streamed by
//       TMA (cp.async.bulk.tensor.2d, 128B swizzle) through a 4-stage
//       mbarrier ring, 128 K-bytes per stage;
//   D = int32 in TMEM, double-buffered (2 x N columns) so the epilogue of
//       group g overlaps the MMAs of group g + 1.
// Epilogue (4 warps, thread = delay lane): tcgen05.ld 32 columns (5
// segments) at a time, recombine digits, sqrt(re^2 + im^2), sum over
// segments, one float per (p, b, delay) to the plane -- the products never
// leave the SM.
//
// Warp roles (256 threads): warp 0 = TMA producer, warp 1 = MMA issuer (one
// elected lane), warps 4-7 = epilogue; every warp regenerates A at a (p,
// delay tile) boundary (the pipeline drains there: 1-3 times per CTA).
// Persistent grid: CTA c owns the units [c U / grid, (c + 1) U / grid) of
// the U = n_prns x 8 x n_groups (p, tile, group) units, ordered group-fastest.
#pragma once

#include <cuda.h>
#include <stdint.h>

#include "correlator.cuh"  // smem_u32, mbar_* helpers

namespace l1rxg {

constexpr int GM_M = 128;                  // delays per tile (TMEM lanes)
constexpr int GM_TILES = 8;                // 8 x 128 = 1024 >= 1023 delays
constexpr int GM_KB = 128;                 // K bytes per pipeline stage (one 128-B swizzle row)
constexpr int GM_NKB = 8;                  // K = 1024 (1023 chips + a zero)
constexpr int GM_A_BYTES = GM_M * 1024;    // the circulant tile, all of K
constexpr int GM_THREADS = 384;  // warp 0 TMA, warp 1 MMA, warps 4-11 epilogue (two per TMEM lane quarter)
constexpr int GM_SEG_PER_CHUNK = 5;        // 5 segments x (re, im) x 3 digits = 30 of 32 columns

__host__ __device__ constexpr int gm_rows(int n_seg) { return 32 * ((n_seg + GM_SEG_PER_CHUNK - 1) / GM_SEG_PER_CHUNK); }
__host__ __device__ constexpr int gm_row(int seg, int ri, int d) {
    return (seg / GM_SEG_PER_CHUNK) * 32 + (seg % GM_SEG_PER_CHUNK) * 6 + ri * 3 + d;
}

struct __align__(64) GridMmaArgs {
    CUtensorMap bmap;        // digits [n_groups * n_rows][1024] int8, box {128 B, n_rows}, 128B swizzle
    const int8_t* codes;     // [33][1023]
    const int32_t* prns;     // [n_prns]
    const float* scales;     // [n_groups][n_seg]: the quantisation step of each fold vector
    float* plane;            // [n_prns][n_bins][2046]
    int n_prns, n_groups, n_seg, n_rows;
    float out_scale;         // N: FFTW's unnormalised inverse
    int a_smem;              // 1: the circulant tile in shared memory (SS MMA); 0: in TMEM (TS MMA)
    int ks;                  // K blocks of 128 B per B stage (1, 2, 4 or 8)
    int epi;                 // 0: skip the epilogue arithmetic (timing experiments only)
};

// ---- tcgen05 / TMA primitives (PTX ISA 8.7, sm_100a) ---------------------
__device__ __forceinline__ void gm_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void gm_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// shared-memory matrix descriptor: K-major, 128-byte swizzle, 8-row atoms
// of 1024 B (SBO), version 1 (sm_100)
__device__ __forceinline__ uint64_t gm_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);          // start address
    d |= (uint64_t)1 << 16;                          // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;                // SBO
    d |= (uint64_t)1 << 46;                          // version
    d |= (uint64_t)2 << 61;                          // SWIZZLE_128B
    return d;
}

// instruction descriptor kind::i8: D int32, A/B signed int8, both K-major
__device__ __forceinline__ uint32_t gm_idesc(int n) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(GM_M >> 4) << 24);
}

__device__ __forceinline__ void gm_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void gm_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void gm_tma_2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

// mbarrier wait with a bound (~seconds): a broken pipeline traps (a launch
// error the host reports) instead of hanging the GPU
__device__ __forceinline__ void gm_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0;
    for (uint32_t spin = 0; !ok; ++spin) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (spin > (1u << 22))
            __trap();
    }
}

__device__ __forceinline__ void gm_mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// 32 consecutive TMEM columns of this warp's 32 lanes: thread i gets lane i
#define GM_LD32(taddr, v)                                                                                      \
    asm volatile(                                                                                              \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19," \
        "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                             \
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),      \
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), \
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),           \
          "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),           \
          "=r"(v[30]), "=r"(v[31])                                                                             \
        : "r"(taddr))

// ---- K4c-a: fold rows -> int8 digit rows + per-row quantisation steps ----
// one CTA per (group g = bin * 2 + par, segment); F: [bin][seg][par][1023]
__global__ void __launch_bounds__(256) grid_digits_kernel(const float2* __restrict__ F, int n_seg, int n_rows,
                                                          int8_t* __restrict__ Bq, float* __restrict__ scales) {
    const int g = blockIdx.x / n_seg, seg = blockIdx.x % n_seg;
    const int bin = g >> 1, par = g & 1;
    const float2* f = F + ((int64_t)(bin * n_seg + seg) * 2 + par) * GRID_CHIPS;
    __shared__ float red[2][8];
    float mr = 0.f, mi = 0.f;
    for (int k = threadIdx.x; k < GRID_CHIPS; k += blockDim.x) {
        const float2 v = f[k];
        mr = fmaxf(mr, fabsf(v.x));
        mi = fmaxf(mi, fabsf(v.y));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mr = fmaxf(mr, __shfl_xor_sync(0xffffffffu, mr, o));
        mi = fmaxf(mi, __shfl_xor_sync(0xffffffffu, mi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = mr;
        red[1][threadIdx.x >> 5] = mi;
    }
    __syncthreads();
    mr = mi = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        mr = fmaxf(mr, red[0][w]);
        mi = fmaxf(mi, red[1][w]);
    }
    // quantisation step (one per fold vector, re and im alike): its largest
    // |component| maps to QMAX = 2^23 - 2^16, so the top balanced digit stays
    // in [-127, 127]
    constexpr float QMAX = 8323072.f;
    const float stv = fmaxf(mr, mi) / QMAX;
    const float inv[2] = {stv > 0.f ? 1.f / stv : 0.f, stv > 0.f ? 1.f / stv : 0.f};
    if (threadIdx.x == 0)
        scales[(int64_t)g * n_seg + seg] = stv;
    int8_t* rows = Bq + (int64_t)g * n_rows * 1024;
    for (int k = threadIdx.x; k < 1024; k += blockDim.x) {
        const float2 v = k < GRID_CHIPS ? f[k] : make_float2(0.f, 0.f);
#pragma unroll
        for (int ri = 0; ri < 2; ++ri) {
            int x = __float2int_rn((ri ? v.y : v.x) * inv[ri]);
            x = max(-8323072, min(8323072, x));
            const int d0 = (int)(int8_t)(x & 0xff);  // balanced base-256 digits
            const int x1 = (x - d0) >> 8;
            const int d1 = (int)(int8_t)(x1 & 0xff);
            const int d2 = (x1 - d1) >> 8;
            rows[(int64_t)gm_row(seg, ri, 0) * 1024 + k] = (int8_t)d0;
            rows[(int64_t)gm_row(seg, ri, 1) * 1024 + k] = (int8_t)d1;
            rows[(int64_t)gm_row(seg, ri, 2) * 1024 + k] = (int8_t)d2;
        }
    }
}

// ---- K4c-b: the GEMM + fused epilogue -------------------------------------
// TMEM map (512 columns x 128 lanes of 32 bit):
//   [0, 256)                A: the circulant tile, lane j = delay j0 + j, column
//                           c = chips 4c .. 4c + 3 (one byte each, K-major);
//   [256, 256 + NR)         accumulator 0;  [256 + NR, 256 + 2 NR) accumulator 1
//                           (one buffer when 2 NR > 256, i.e. > 20 segments).
// A[j][k] = chip[(k - j0 - j) mod 1023] (0 for a delay >= 1023; the k = 1023
// column meets the zero digit column of B).  cext[i] = chip[i mod 1023] for
// i < GM_CEXT: lane j's 128 chips from k0 start at i = k0 - J + 1023 and never
// wrap, so each 4-chip word is one funnel shift of two aligned words.
constexpr int GM_CEXT = 2 * GRID_CHIPS + 160;
constexpr int GM_A_COLS = 256;

// 32 consecutive TMEM columns of this warp's 32 lanes from registers
#define GM_ST32(taddr, v)                                                                                      \
    asm volatile(                                                                                              \
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17," \
        "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),                          \
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),     \
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),         \
        "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),        \
        "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])                     \
        : "memory")

// A from TMEM (the ".kind::i8 [d], [a], b_desc" form)
__device__ __forceinline__ void gm_mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// A in shared memory instead (the "SS" form, runtime knob a_smem): the
// K-major 128B-swizzled layout the descriptor names -- K block kb at
// kb * 16 KB, row j at (j / 8) * 1024 + (j % 8) * 128, 16-byte chunk c at
// ((c ^ (j % 8)) * 16).
__device__ __forceinline__ void gm_build_a_smem(unsigned char* A, const unsigned char* cext, int j0, int tid,
                                                int nthr) {
    const uint32_t* cw = reinterpret_cast<const uint32_t*>(cext);
    for (int q = tid; q < GM_A_BYTES / 16; q += nthr) {
        const int kb = q >> 10, j = (q >> 3) & 127, c = q & 7;
        const int J = j0 + j;
        const int i = kb * 128 + c * 16 - J + GRID_CHIPS;
        const int w0 = i >> 2, sh = (i & 3) * 8;
        uint32_t x[5];
#pragma unroll
        for (int t = 0; t < 5; ++t)
            x[t] = cw[w0 + t];
        uint4 o = make_uint4(__funnelshift_r(x[0], x[1], sh), __funnelshift_r(x[1], x[2], sh),
                             __funnelshift_r(x[2], x[3], sh), __funnelshift_r(x[3], x[4], sh));
        if (J >= GRID_CHIPS)
            o = make_uint4(0u, 0u, 0u, 0u);
        *reinterpret_cast<uint4*>(A + kb * 16384 + (j >> 3) * 1024 + (j & 7) * 128 + ((c ^ (j & 7)) << 4)) = o;
    }
}

// B ring: stages of ks K-blocks (each one 128B-swizzled box of n_rows x 128 B)
__host__ __device__ inline int gm_stages(int n_rows, int ks, int a_smem) {
    const int budget = (200 - (a_smem ? 128 : 0)) * 1024;
    const int s = budget / (n_rows * GM_KB * ks);
    return s > 12 ? 12 : s;
}
__host__ __device__ inline size_t gm_smem_bytes_rt(int n_rows, int ks, int a_smem) {
    return 1024 + (a_smem ? (size_t)GM_A_BYTES : 0) + (size_t)gm_stages(n_rows, ks, a_smem) * n_rows * GM_KB * ks +
           2304 + 256 + 2 * GM_M * sizeof(float);
}

template <bool A_SMEM, int KS>
__global__ void __launch_bounds__(GM_THREADS, 1) grid_mma_kernel(const __grid_constant__ GridMmaArgs ga) {
    extern __shared__ unsigned char gm_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(gm_raw) + 1023) & ~uintptr_t(1023));
    const int NR = ga.n_rows;
    constexpr bool a_smem = A_SMEM;
    const int NS = gm_stages(NR, KS, A_SMEM);
    const int box_bytes = NR * GM_KB;
    const int stage_bytes = box_bytes * KS;
    unsigned char* A = sm;                               // a_smem: the circulant tile
    unsigned char* Bst = sm + (a_smem ? GM_A_BYTES : 0);
    unsigned char* cext = Bst + NS * stage_bytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(cext + ((GM_CEXT + 63) & ~63));
    uint64_t* full = bars;                       // [NS] TMA landed
    uint64_t* empty = bars + 12;                 // [NS] MMAs done with the stage
    uint64_t* tfull = bars + 24;                 // [2] accumulator ready
    uint64_t* tempty = bars + 26;                // [2] accumulator drained (8 epilogue warps)
    uint64_t* adone = bars + 28;                 // MMAs of a (p, tile) run complete (A reusable)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 29);
    float* pairsum = reinterpret_cast<float*>(bars + 32);  // [2][128]: the epilogue pairs' partial sums

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n_units = ga.n_prns * GM_TILES * ga.n_groups;
    const int u_begin = (int)((int64_t)blockIdx.x * n_units / gridDim.x);
    const int u_end = (int)((int64_t)(blockIdx.x + 1) * n_units / gridDim.x);
    const int acc0 = a_smem ? 0 : GM_A_COLS;     // accumulators after A (TMEM mode)
    const int nacc = acc0 + 2 * NR <= 512 ? 2 : 1;
    const int nkst = GM_NKB / KS;                // stages per unit

    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 8);
        }
        mbar_init(adone, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {  // all 512 TMEM columns (one CTA per SM)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    gm_fence_before();
    __syncthreads();
    gm_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tacc = tmem + (uint32_t)acc0;
    const uint32_t idesc = gm_idesc(NR);

    int stage = 0, phase = 0;  // B ring (TMA producer and MMA issuer)
    int abuf = 0, aphase = 0;  // accumulator ring (MMA issuer and epilogue)
    int runs = 0;

    for (int u0 = u_begin; u0 < u_end;) {
        // ---- a run: consecutive units of one (PRN, delay tile)
        const int pt = u0 / ga.n_groups;
        const int u1 = min(u_end, (pt + 1) * ga.n_groups);
        const int pi = pt / GM_TILES, mt = pt % GM_TILES;
        if (runs > 0)  // the previous run's MMAs still read A
            gm_wait(adone, (uint32_t)((runs - 1) & 1));
        const int8_t* code = ga.codes + ga.prns[pi] * GRID_CHIPS;
        for (int m = tid; m < GM_CEXT; m += GM_THREADS)
            cext[m] = (unsigned char)code[m % GRID_CHIPS];
        __syncthreads();
        if (a_smem) {
            gm_build_a_smem(A, cext, mt * GM_M, tid, GM_THREADS);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor-core reads
        } else if (warp >= 4 && warp < 8) {  // A into TMEM: lane j = delay, 8 stores of 32 columns (128 chips)
            const int q = warp - 4, j = q * 32 + lane;
            const int J = mt * GM_M + j;
            const uint32_t* cw = reinterpret_cast<const uint32_t*>(cext);
            for (int c0 = 0; c0 < GM_A_COLS; c0 += 32) {
                uint32_t v[32];
                const int i = 4 * c0 - J + GRID_CHIPS;  // chips 4 c0 .. of row J start at cext[i]
                const int w0 = i >> 2, sh = (i & 3) * 8;
                uint32_t lo = cw[w0];
#pragma unroll
                for (int t = 0; t < 32; ++t) {
                    const uint32_t hi = cw[w0 + t + 1];
                    v[t] = J < GRID_CHIPS ? __funnelshift_r(lo, hi, sh) : 0u;
                    lo = hi;
                }
                GM_ST32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c0, v);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        gm_fence_before();
        __syncthreads();
        gm_fence_after();

        if (warp == 0) {
            // ---- TMA producer: the digit rows of each group, KS x 128 K-bytes per stage
            if (lane == 0)
                for (int u = u0; u < u1; ++u) {
                    const int g = u - pt * ga.n_groups;
                    for (int ks = 0; ks < nkst; ++ks) {
                        gm_wait(&empty[stage], (uint32_t)(phase ^ 1));
                        mbar_expect_tx(&full[stage], (uint32_t)stage_bytes);
                        for (int j = 0; j < KS; ++j)
                            gm_tma_2d(smem_u32(Bst + stage * stage_bytes + j * box_bytes), &ga.bmap,
                                      (ks * KS + j) * GM_KB, g * NR, &full[stage]);
                        if (++stage == NS) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
            __syncwarp();
        } else if (warp == 1) {
            // ---- MMA issuer: lane 0 alone walks the run (descriptors advanced
            // by adding (byte offset >> 4) to the start-address field)
            if (lane == 0) {
                const uint64_t adesc0 = gm_desc(smem_u32(A));
                const uint64_t bdesc0 = gm_desc(smem_u32(Bst));
                for (int u = u0; u < u1; ++u) {
                    gm_wait(&tempty[abuf], (uint32_t)(aphase ^ 1));
                    gm_fence_after();
                    const uint32_t dacc = tacc + (uint32_t)(abuf * NR);
                    for (int ks = 0; ks < nkst; ++ks) {
                        gm_wait(&full[stage], (uint32_t)phase);
                        gm_fence_after();
                        const uint64_t bst = bdesc0 + (uint64_t)((stage * stage_bytes) >> 4);
#pragma unroll
                        for (int j = 0; j < KS; ++j) {
#pragma unroll
                            for (int kk = 0; kk < GM_KB / 32; ++kk) {
                                const int kb = ks * KS + j;
                                const uint64_t bd = bst + (uint64_t)((j * box_bytes + kk * 32) >> 4);
                                const uint32_t acc = (ks | j | kk) != 0;
                                if (A_SMEM)
                                    gm_mma(dacc, adesc0 + (uint64_t)((kb * 16384 + kk * 32) >> 4), bd, idesc, acc);
                                else
                                    gm_mma_ts(dacc, tmem + (uint32_t)(kb * 32 + kk * 8), bd, idesc, acc);
                            }
                        }
                        gm_commit(&empty[stage]);  // the stage is free once these MMAs finish
                        if (++stage == NS) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                    gm_commit(&tfull[abuf]);
                    if (++abuf == nacc) {
                        abuf = 0;
                        aphase ^= 1;
                    }
                }
                gm_commit(adone);  // every MMA of this run done -> A may be rebuilt
            }
            __syncwarp();
        } else if (warp >= 4) {
            // ---- epilogue: two warps per TMEM lane quarter (thread = delay
            // lane), each over half of the group's 32-column chunks; the pair
            // adds its partial sums through shared memory
            const int q = warp & 3, h = (warp - 4) >> 2;
            const int J = mt * GM_M + q * 32 + lane;
            const int n_bins = ga.n_groups >> 1;
            const int nch = (ga.n_seg + GM_SEG_PER_CHUNK - 1) / GM_SEG_PER_CHUNK;
            for (int u = u0; u < u1; ++u) {
                const int g = u - pt * ga.n_groups;
                gm_wait(&tfull[abuf], (uint32_t)aphase);
                gm_fence_after();
                const float* sc = ga.scales + (int64_t)g * ga.n_seg;
                float acc = 0.f;
                for (int ch = h; ga.epi && ch < nch; ch += 2) {
                    uint32_t v[32];
                    GM_LD32(tacc + ((uint32_t)(q * 32) << 16) + (uint32_t)(abuf * NR + ch * 32), v);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int sl = 0; sl < GM_SEG_PER_CHUNK; ++sl) {
                        const int seg = ch * GM_SEG_PER_CHUNK + sl;
                        if (seg < ga.n_seg) {
                            // 65536 c2 + (256 c1 + c0): the low part exact in int32
                            const int* c = reinterpret_cast<const int*>(v) + sl * 6;
                            const float re = fmaf(65536.f, (float)c[2], (float)(256 * c[1] + c[0]));
                            const float im = fmaf(65536.f, (float)c[5], (float)(256 * c[4] + c[3]));
                            acc = fmaf(__ldg(sc + seg), sqrtf(fmaf(re, re, im * im)), acc);
                        }
                    }
                }
                gm_fence_before();
                __syncwarp();
                if (lane == 0)
                    gm_mbar_arrive(&tempty[abuf]);
                float* slot = pairsum + (u & 1) * GM_M + q * 32 + lane;
                if (h == 1)
                    *slot = acc;
                asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
                if (h == 0 && J < GRID_CHIPS)
                    ga.plane[((int64_t)pi * n_bins + (g >> 1)) * (2 * GRID_CHIPS) + 2 * J + (g & 1)] =
                        ga.out_scale * (acc + *slot);
                if (++abuf == nacc) {
                    abuf = 0;
                    aphase ^= 1;
                }
            }
        }
        // keep every thread's ring counters in step (each role's lane advanced only its own)
        if (warp >= 2 || lane != 0)
            for (int u = u0; u < u1; ++u)
                for (int ks = 0; ks < nkst; ++ks)
                    if (++stage == NS) {
                        stage = 0;
                        phase ^= 1;
                    }
        if (warp < 4 && !(warp == 1 && lane == 0))
            for (int u = u0; u < u1; ++u)
                if (++abuf == nacc) {
                    abuf = 0;
                    aphase ^= 1;
                }
        ++runs;
        u0 = u1;
        __syncthreads();
    }
    gm_fence_before();
    __syncthreads();
    gm_fence_after();
    if (warp == 2)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

}  // namespace l1rxg
