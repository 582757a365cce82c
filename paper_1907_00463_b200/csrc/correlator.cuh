// correlator.cuh -- K2 correlator + K3 loop update, sm_100a device code.
//
// Hot path (reference: /root/reference/proj/include/l1rx/tracking.hpp):
//   K2 correlate  tracking.hpp:226-282  carrier wipe + K-tap code replica MAC
//   K3 loop       tracking.hpp:520-618 (+ :459-515) DLL/PLL/FLL + metrics
//
// Correlator algorithm ("boundary-prefix").  The replica of
// tap k is a +/-1 staircase whose steps sit where the reference's fp64 chip
// index trunc(fl(fma(i, cps, base) + d_k)) changes.  For the wiped samples
// y_i the tap sum over a run [i0, i1] of consecutive samples is
//     sum_i chip_k(i) y_i = chip_k(i1) * P(i1+1) - sum_b (chip_after - chip_before) * P(b)
// with P(b) the run-local exclusive prefix sum and b the steps inside the
// run.  Phase A (per thread: a run of RUN samples) wipes the carrier,
// stores the prefix sums in place in shared memory and adds each tap's
// chip(end) * total term.  Phase B (flattened over the code's chip
// TRANSITIONS, about 512 per code period, so every thread does the same
// amount of work) locates each step exactly -- fp64 estimate, then the
// reference expression evaluated at the candidate sample and its
// neighbour (it is monotone in the sample index) -- and subtracts
// delta * P(b).  Every chip decision is therefore the reference's, bit for
// bit, while the per-sample cost no longer grows with the number of taps.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "l1rxg.h"

namespace l1rxg {

#ifndef L1RXG_RUN
#define L1RXG_RUN 31
#endif
constexpr int RUN = L1RXG_RUN;  // samples per thread run; odd -> LDS.64 conflict-free
constexpr int MAX_NT = 640; // correlator CTA size cap (<= 102 registers)
constexpr double PI_D = 3.14159265358979323846;  // constants.hpp:20
constexpr double TWO_PI_D = 2.0 * PI_D;
constexpr double F_L1_HZ = 1.57542e9;      // constants.hpp:5
constexpr double CHIP_RATE_HZ = 1.023e6;   // constants.hpp:6
constexpr int CHIP_EXT = 4096;             // chip index domain of one epoch
// transition table domain: the largest chip index of an epoch is below
// 2046 + 1.1 * 1023 + 1 = 3172 (code phase + 1023, code rate < 1.1 x chip
// rate, |tap| <= 1 chip), i.e. below 3 * L + 104 <= 1736 transitions for
// every GPS C/A code (L <= 544 per period)
constexpr int TRANS_EXT = 2048;

// ---------------------------------------------------------------------
// per-epoch NCO constants (tracking.hpp:234-239)
struct EpochConsts {
    double w;        // 2*pi*fD/fs   rad/sample
    double cps;      // code_freq/fs chips/sample
    double inv_cps;  // boundary estimate only (verified exactly)
    double base;     // code_phase + 1023
    double phi;      // carrier phase at epoch start
    int n, nh;
};

__device__ __forceinline__ void make_consts(EpochConsts& c, double code_phase,
                                            double code_freq, double doppler,
                                            double phase, double fs, int n) {
    c.w = 2.0 * PI_D * doppler / fs;  // (2*pi*fD)/fs as the reference orders it
    c.cps = code_freq / fs;
    c.inv_cps = __drcp_rn(c.cps);  // correctly rounded (tap_boundary's fast path)
    c.base = code_phase + 1023.0;
    c.phi = phase;
    c.n = n;
    c.nh = n / 2;
}

// The reference's replica phase of tap d at sample i (tracking.hpp:251-254
// as compiled: ph = fma(i, cps, base), then ph + d rounded).
__device__ __forceinline__ double tap_value(double i, double cps, double base, double d) {
    return __dadd_rn(__fma_rn(i, cps, base), d);
}
__device__ __forceinline__ int tap_index(int i, double cps, double base, double d) {
    return __double2int_rz(tap_value((double)i, cps, base, d));
}
// First b in [lo, hi] with tap_value(b) >= m, given that one exists
// (tap_index(hi) >= m).  The estimate ceil((m - d - base)/cps) is within one
// sample of the answer (its error, < 1e-2 samples, and the reference's
// rounding, < 1e-11 samples, are far below one sample), so checking the
// estimate and its left neighbour with the reference expression pins the
// exact boundary: tap_value is monotone in the sample index.
//
// Fast path: with inv_cps within 2 ulp of 1/cps, |e - x*| < 4e-11 samples for
// the exact crossing x* = (m - d - base)/cps, and the reference's own
// rounding moves its crossing by < 5e-11 samples; so when e is farther than
// 1e-9 from an integer the boundary is ceil(e) with certainty.  Only near
// ties (exact ties occur at commensurate rates) take the exact check.
__device__ __forceinline__ int tap_boundary(int m, double d, const EpochConsts& c, int lo, int hi) {
    const double mm = (double)m;
    const double e = ((mm - d) - c.base) * c.inv_cps;
    int b = max(lo, min(hi, __double2int_ru(e)));
    if (fabs(e - rint(e)) > 1e-9)
        return b;
    const bool dn = (b > lo) && (tap_value((double)(b - 1), c.cps, c.base, d) >= mm);
    const bool up = !dn && (b < hi) && (tap_value((double)b, c.cps, c.base, d) < mm);
    return b - (int)dn + (int)up;
}

// Sample kinds of a tracker ring: SK_F32 (float2: decoded/filtered real IF),
// SK_I16 (raw cint16, 4 B) and SK_I8 (raw cint8, 2 B); raw samples are
// converted while they are wiped (the /32768 or /128 scale is a power of two,
// folded exactly into the rotator table).
constexpr int SK_F32 = 0, SK_I16 = 1, SK_I8 = 2;
constexpr int SK_R8 = 3;  // raw real int8 IF at fs/4 (overlapped kernel with FIR warps, ovlcorr.cuh)
template <int SK>
struct Samp;
template <>
struct Samp<SK_F32> {
    typedef unsigned long long raw_t;
    static constexpr int esz = 8;
};
template <>
struct Samp<SK_I16> {
    typedef uint32_t raw_t;
    static constexpr int esz = 4;
};
template <>
struct Samp<SK_I8> {
    typedef uint16_t raw_t;
    static constexpr int esz = 2;
};

// A complex sample as one 64-bit value (one LDS.64 / STS.64).
typedef unsigned long long f2x;
__device__ __forceinline__ f2x pk2(float a, float b) {
    f2x r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float2 upk2(f2x v) {
    float2 r;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
__device__ __forceinline__ float2 cvt_sample(f2x v) { return upk2(v); }
// Raw complex ints -> exact floats without the (quarter-rate) I2F: flipping
// the sign bit biases each component to an unsigned value u = v + 2^(b-1);
// 0x4B400000 | u is the float 1.5 * 2^23 + u, so one FADD removes the
// bias exactly (|v| < 2^22).  Little endian: the real part is the low half.
__device__ __forceinline__ float2 cvt_sample(uint32_t w) {  // cint16
    const uint32_t u = w ^ 0x80008000u;
    const float re = __uint_as_float(__byte_perm(u, 0x4B400000u, 0x7610));
    const float im = __uint_as_float(__byte_perm(u, 0x4B400000u, 0x7632));
    return make_float2(re - 12615680.0f, im - 12615680.0f);  // 1.5 * 2^23 + 2^15
}
__device__ __forceinline__ float2 cvt_sample(uint16_t h) {  // cint8
    const uint32_t u = (uint32_t)h ^ 0x8080u;
    const float re = __uint_as_float(__byte_perm(u, 0x4B400000u, 0x7640));
    const float im = __uint_as_float(__byte_perm(u, 0x4B400000u, 0x7641));
    return make_float2(re - 12583040.0f, im - 12583040.0f);  // 1.5 * 2^23 + 2^7
}

// ---------------------------------------------------------------------
// Per-PRN chip tables (built once per CTA).
//   chip[m]   = chips[m mod 1023] (+/-1)                (m < CHIP_EXT)
//   tm[g]     = chip index of the g-th chip transition  (g < TRANS_EXT)
//   td[g]     = chips[tm] - chips[tm - 1] in {-2, +2}
//   cum[r]    = number of transitions at indices <= r within one period
// A transition at index m means chips[m mod 1023] != chips[(m-1) mod 1023].
// F(m) = (m / 1023) * L + cum[m mod 1023] counts the transitions in [0, m].
struct CodeTables {
    int8_t chip[CHIP_EXT];
    int16_t tm[TRANS_EXT];
    int8_t td[TRANS_EXT];
    int16_t cum[1024];
    int L;
};

__device__ __forceinline__ int trans_count(const CodeTables& ct, int m) {
    const int p = m / 1023;
    return p * ct.L + ct.cum[m - p * 1023];
}

// Builds the tables for one PRN; all threads participate (ends with a barrier).
__device__ void build_code_tables(CodeTables& ct, const int8_t* codes, int prn) {
    const int8_t* c = codes + prn * 1023;
    for (int k = threadIdx.x; k < CHIP_EXT; k += blockDim.x)
        ct.chip[k] = c[k % 1023];
    if (threadIdx.x < 32) {  // one warp: ballot-scan of the transitions
        const int lane = threadIdx.x;
        int running = 0;
        for (int base = 0; base < 1023; base += 32) {
            const int r = base + lane;
            const bool t = r < 1023 && c[r] != c[(r + 1022) % 1023];
            const unsigned mask = __ballot_sync(0xffffffffu, t);
            const int before = __popc(mask & ((1u << lane) - 1u));
            if (r < 1023) {
                if (t)
                    ct.tm[running + before] = (int16_t)r;
                ct.cum[r] = (int16_t)(running + before + (t ? 1 : 0));
            }
            running += __popc(mask);
        }
        if (lane == 0)
            ct.L = running;
    }
    __syncthreads();
    const int L = ct.L;
    // extend tm/td over TRANS_EXT (entries >= L derive from the first period)
    for (int g = threadIdx.x; g < TRANS_EXT; g += blockDim.x) {
        const int p = g / L, q = g - p * L;
        const int r = ct.tm[q];  // q < L: first-period entries are final
        const int m = p * 1023 + r;
        const int8_t dlt = (int8_t)(c[r] - c[(r + 1022) % 1023]);
        if (g >= L)
            ct.tm[g] = (int16_t)(m < 32767 ? m : 32767);
        ct.td[g] = dlt;
    }
    __syncthreads();
}

// ---------------------------------------------------------------------
// Phase A: one thread's run of samples [i0, i0+cnt) at run[0..RUN).
// Overwrites run[j] with the exclusive prefix of the wiped (but not yet
// anchored) samples, stores the run's carrier anchor e^{-j theta(i0)}, and
// accumulates chip_k(last) * anchor * total into acc[2k..2k+1] for every
// tap, plus the first-half prompt into acc[2T..2T+1].
// raw: the run's samples (any sample kind); run: where its exclusive prefix
// sums go (the same memory for float2 rings: in place).
template <int T, bool FULL, typename R>
__device__ __forceinline__ void phase_a(const EpochConsts& c, const R* raw, float2* run,
                                        const float2* __restrict__ rot,
                                        const int8_t* __restrict__ chip,
                                        const double* __restrict__ d, int kp, int i0, int cnt,
                                        float* acc, float2* anchor_slot) {
    // theta(i0) exactly as the reference computes it (fma(w, i, phi)),
    // reduced to [-pi, pi] in fp64; the fp32 phasor's ~4e-7 error is common
    // to the run's samples
    const double th = __fma_rn(c.w, (double)i0, c.phi);
    const double r = fma(-rint(th * (1.0 / TWO_PI_D)), TWO_PI_D, th);
    float sa, ca;
    __sincosf((float)r, &sa, &ca);
    *anchor_slot = make_float2(ca, sa);

    // P += x_j * conj(rot_j), rot[j] = (c, s): (xr c + xi s, xi c - xr s),
    // the reference's wipe-off form (tracking.hpp:248-249), as four FFMAs
    // straight into the prefix.  Samples and rotators are loaded PF ahead.
    // (A packed FFMA2 form needs a negated pair per sample plus
    // register-pair moves and measured slower.)
    constexpr int PF = 4;
    f2x* runp = reinterpret_cast<f2x*>(run);
    R xw[PF];
    float2 qw[PF];
#pragma unroll
    for (int j = 0; j < PF; ++j) {
        xw[j] = (FULL || j < cnt) ? raw[j] : R(0);
        qw[j] = rot[j];
    }
    f2x P = 0ull;
#pragma unroll
    for (int j = 0; j < RUN; ++j) {
        const float2 x = cvt_sample(xw[j % PF]);
        const float2 q = qw[j % PF];
        if (j + PF < RUN) {
            xw[j % PF] = (FULL || j + PF < cnt) ? raw[j + PF] : R(0);
            qw[j % PF] = rot[j + PF];
        }
        runp[j] = P;
        const float2 Pf = upk2(P);
        P = pk2(fmaf(x.y, q.y, fmaf(x.x, q.x, Pf.x)), fmaf(-x.x, q.y, fmaf(x.y, q.x, Pf.y)));
    }
    const float2 Pt = upk2(P);
    const float pr = Pt.x, pi = Pt.y;
    const int i_last = i0 + (FULL ? RUN : cnt) - 1;
    const double dl = (double)i_last;
    const float zr = fmaf(pr, ca, pi * sa);  // anchored run total
    const float zi = fmaf(pi, ca, -(pr * sa));
    float chip_p = 0.f;
#pragma unroll
    for (int k = 0; k < T; ++k) {
        const float ch = (float)chip[__double2int_rz(tap_value(dl, c.cps, c.base, d[k]))];
        acc[2 * k] = fmaf(ch, zr, acc[2 * k]);
        acc[2 * k + 1] = fmaf(ch, zi, acc[2 * k + 1]);
        if (k == kp)
            chip_p = ch;
    }
    // first-half prompt (tracking.hpp:265-271)
    if (i_last < c.nh) {
        acc[2 * T] = fmaf(chip_p, zr, acc[2 * T]);
        acc[2 * T + 1] = fmaf(chip_p, zi, acc[2 * T + 1]);
    } else if (i0 < c.nh) {  // the run straddling n/2: chip(nh-1) * P(nh)
        const float ch = (float)chip[tap_index(c.nh - 1, c.cps, c.base, d[kp])];
        const float2 pn = run[c.nh - i0];
        acc[2 * T] = fmaf(ch, fmaf(pn.x, ca, pn.y * sa), acc[2 * T]);
        acc[2 * T + 1] = fmaf(ch, fmaf(pn.y, ca, -(pn.x * sa)), acc[2 * T + 1]);
    }
}

template <int T, typename R>
__device__ __forceinline__ void phase_a_dispatch(const EpochConsts& c, const R* raw, float2* run,
                                                 const float2* rot, const int8_t* chip,
                                                 const double* d, int kp, int i0, int cnt,
                                                 float* acc, float2* anchor_slot) {
    if (cnt == RUN)
        phase_a<T, true>(c, raw, run, rot, chip, d, kp, i0, cnt, acc, anchor_slot);
    else
        phase_a<T, false>(c, raw, run, rot, chip, d, kp, i0, cnt, acc, anchor_slot);
}

// Phase B: every chip transition of every tap whose step falls in the
// sub-tile [u0, u0+len): acc_k -= delta * anchor(run(b)) * P(b).
// tile_d[i - u0] holds P(i) (phase A's in-place prefixes).
constexpr int MAXSUB = 24;  // sub-tiles per epoch (n <= 24 * nwork * 31)


// Phase B thread roles: threads are dealt to taps in fixed groups of
// gsz = nthreads / T (thread t -> tap t / gsz, rank t % gsz; leftover
// threads idle), so a thread's tap offset and its accumulators stay in
// registers; a group walks its tap's transitions with stride gsz.
struct PhaseB {
    int kt, jt, gsz;  // tap, rank in the tap's group, group size
    int g0, cnt;      // this unit: first global transition index of the tap, count
    int n1;           // exact steps found before the unit's samples arrived (<= 2)
    int b1[2];        //   their sample positions
    float d1[2];      //   and chip deltas
    double dk;        // tap offset
    bool prompt;      // kt is the prompt tap (first-half prompt too)
    float re, im, hre, him;  // this thread's tap sum and first-half prompt
};

template <int T>
__device__ __forceinline__ void phase_b_init(PhaseB& pb, const double* d, int kp, int tid,
                                             int nthreads) {
    pb.gsz = max(1, nthreads / T);
    pb.kt = tid / pb.gsz;
    pb.jt = tid - pb.kt * pb.gsz;
    pb.dk = pb.kt < T ? d[pb.kt] : 0.0;
    pb.prompt = pb.kt == kp;
    pb.re = pb.im = pb.hre = pb.him = 0.f;
}

// One transition at step b of delta dlt: acc -= dlt * anchor(run(b)) * P(b).
__device__ __forceinline__ void phase_b_one(PhaseB& pb, const float2* tile_d, const float2* anchors,
                                            int u0, int nh, int b, float dlt) {
    const int off = b - u0;
    const float2 p = tile_d[off];
    const float2 an = anchors[off / RUN];
    const float ar = fmaf(p.x, an.x, p.y * an.y);
    const float ai = fmaf(p.y, an.x, -(p.x * an.y));
    pb.re = fmaf(-dlt, ar, pb.re);
    pb.im = fmaf(-dlt, ai, pb.im);
    if (pb.prompt && b < nh) {
        pb.hre = fmaf(-dlt, ar, pb.hre);
        pb.him = fmaf(-dlt, ai, pb.him);
    }
}

// Latency shape (one unit per epoch, its copy long done): the tap's
// transition range, computed right before phase A so it interleaves with it,
// and the whole walk after phase A (two steps at a time).
template <int T>
__device__ __forceinline__ void phase_b_range(PhaseB& pb, const EpochConsts& c, const CodeTables& ct,
                                              int u0, int len) {
    pb.n1 = -1;  // no steps precomputed: phase_b walks from the first
    if (pb.kt >= T) {
        pb.g0 = pb.cnt = 0;
        return;
    }
    const int mlo = tap_index(u0 > 0 ? u0 - 1 : 0, c.cps, c.base, pb.dk);
    const int mhi = tap_index(u0 + len - 1, c.cps, c.base, pb.dk);
    pb.g0 = trans_count(ct, mlo);
    pb.cnt = trans_count(ct, mhi) - pb.g0;
}

// Phase B, part 1 -- before the unit's samples are needed (it depends only
// on the epoch constants, so it runs while the bulk copy lands): the range
// of this thread's tap's transitions whose step falls in the unit
// [u0, u0+len), and the exact steps of the first two of them (the two fp64
// searches overlap).  Part 2 (after phase A) is then only the prefix reads
// and FMAs, so the tile is released sooner.
template <int T>
__device__ __forceinline__ void phase_b_pre(PhaseB& pb, const EpochConsts& c, const CodeTables& ct,
                                            int u0, int len) {
    pb.n1 = 0;
    if (pb.kt >= T) {
        pb.g0 = pb.cnt = 0;
        return;
    }
    const int hi = u0 + len - 1;
    const int mlo = tap_index(u0 > 0 ? u0 - 1 : 0, c.cps, c.base, pb.dk);
    const int mhi = tap_index(hi, c.cps, c.base, pb.dk);
    pb.g0 = trans_count(ct, mlo);
    pb.cnt = trans_count(ct, mhi) - pb.g0;
    const int j1 = pb.jt, j2 = pb.jt + pb.gsz;
    pb.n1 = j1 < pb.cnt ? (j2 < pb.cnt ? 2 : 1) : 0;
    const int ga = pb.g0 + (pb.n1 > 0 ? j1 : 0), gb = pb.g0 + (pb.n1 > 1 ? j2 : 0);
    const int ma = ct.tm[ga], mb = ct.tm[gb];
    pb.d1[0] = (float)ct.td[ga];
    pb.d1[1] = (float)ct.td[gb];
    pb.b1[0] = pb.n1 > 0 ? tap_boundary(ma, pb.dk, c, u0, hi) : u0;
    pb.b1[1] = pb.n1 > 1 ? tap_boundary(mb, pb.dk, c, u0, hi) : u0;
}

// Phase B, part 2: the steps found in part 1, then (low sample rates only)
// the rest of the tap's transitions, two at a time.
template <int T, bool PRE = true>
__device__ __forceinline__ void phase_b(PhaseB& pb, const EpochConsts& c, const float2* tile_d,
                                        const float2* anchors, const CodeTables& ct, int u0,
                                        int len) {
    if (pb.kt >= T)
        return;
    if constexpr (PRE) {
        if (pb.n1 > 0)
            phase_b_one(pb, tile_d, anchors, u0, c.nh, pb.b1[0], pb.d1[0]);
        if (pb.n1 > 1)
            phase_b_one(pb, tile_d, anchors, u0, c.nh, pb.b1[1], pb.d1[1]);
    }
    const int hi = u0 + len - 1;
    const int g0 = pb.g0, cnt = pb.cnt;
    for (int j = PRE ? pb.jt + 2 * pb.gsz : pb.jt; j < cnt; j += 2 * pb.gsz) {
        const int j2 = j + pb.gsz;
        const bool two = j2 < cnt;
        const int ga = g0 + j, gb = g0 + (two ? j2 : j);
        const int ma = ct.tm[ga], mb = ct.tm[gb];
        const float da = (float)ct.td[ga], db = (float)ct.td[gb];
        const int ba = tap_boundary(ma, pb.dk, c, u0, hi);
        const int bb = tap_boundary(mb, pb.dk, c, u0, hi);
        phase_b_one(pb, tile_d, anchors, u0, c.nh, ba, da);
        if (two)
            phase_b_one(pb, tile_d, anchors, u0, c.nh, bb, db);
    }
}

// Folds a thread's phase-B sums into its V = 2T+2 partials (once per epoch).
template <int T>
__device__ __forceinline__ void phase_b_fold(PhaseB& pb, float* acc) {
#pragma unroll
    for (int k = 0; k < T; ++k)
        if (k == pb.kt) {
            acc[2 * k] += pb.re;
            acc[2 * k + 1] += pb.im;
        }
    acc[2 * T] += pb.hre;
    acc[2 * T + 1] += pb.him;
    pb.re = pb.im = pb.hre = pb.him = 0.f;
}

// Per-epoch rotator table rot[j] = scale * (cos wj, sin wj), j < RUN
// (accurate sincosf; scale = the raw samples' power-of-two decode factor, so
// the products equal decode-then-wipe exactly); 8 bytes so phase A's
// broadcast read is one shared wavefront.
__device__ __forceinline__ void fill_rot(float2* rot, double w, int tid, float scale = 1.f) {
    if (tid < RUN) {
        float s, co;
        sincosf((float)(w * (double)tid), &s, &co);
        rot[tid] = make_float2(co * scale, s * scale);
    }
}

// Named barrier over the first `count` threads (a multiple of 32).
__device__ __forceinline__ void named_bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// ---- TMA (cp.async.bulk) + mbarrier helpers ---------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1-D bulk copy global -> shared on the TMA engine, completion on bar.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// ---- thread-block cluster helpers (distributed shared memory) ----------
__device__ __forceinline__ uint32_t cluster_map(const void* local, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(local)), "r"(rank));
    return r;
}
// Asynchronous remote store that completes `8` transaction bytes on the
// remote CTA's mbarrier (no fence / separate arrive needed).
__device__ __forceinline__ void st_async_f64(uint32_t remote_addr, double x, uint32_t remote_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(
                     remote_addr),
                 "d"(x), "r"(remote_bar)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAITC_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}

// ---------------------------------------------------------------------
// K3: loop update (tracking.hpp:542-601 + :459-515).
struct LoopCfg {
    l1rxg_tracking_cfg cfg;
    int kernel;
    double fs;
    // host-precomputed, same operation order as the reference
    double dt;                  // n / fs                     (:542)
    double pll_k1, pll_k2;      // ((wn*wn)*dt)*0.5, (2*zeta)*wn  (:71-84)
    double dll_k1, dll_k2;
    double fll_k;               // ((4*B_fll)*2)*pi            (:88-92)
    double alpha;               // 1 / cn0_window_ms           (:466)
    double inv_fll_c, inv_fll_f;  // 1 / (2 pi (dt/2)), 1 / (2 pi dt) (:113-138)
};

// ---- branch-free fp64 helpers for the per-epoch critical path ----------
// (SIMT lanes evaluate different pieces of the update with the same
// instruction stream; without branches the pieces interleave.)
// Reciprocal to ~1 ulp: hardware seed + two Newton steps.
__device__ __forceinline__ double fast_rcp(double b) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
    r = __fma_rn(r, __fma_rn(-b, r, 1.0), r);
    return __fma_rn(r, __fma_rn(-b, r, 1.0), r);
}
// a / b to ~1 ulp (loop-filter internals, 1e-5 bar)
__device__ __forceinline__ double fast_div(double a, double b) {
    const double r = fast_rcp(b);
    const double q = a * r;
    return __fma_rn(__fma_rn(-b, q, a), r, q);
}
// sqrt to ~1 ulp, x >= 0
__device__ __forceinline__ double fast_sqrt(double x) {
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    r = r * __fma_rn(-0.5 * x * r, r, 1.5);
    r = r * __fma_rn(-0.5 * x * r, r, 1.5);
    const double s = x * r;
    const double t = __fma_rn(0.5 * r, __fma_rn(-s, s, x), s);
    return x > 0.0 ? t : 0.0;
}
// atan2(y, x), branch-free, relative error < 1e-13 (minimax polynomial of
// atan(t)/t in t^2 on |t| <= tan(pi/8) after octant reduction, evaluated by
// Estrin's scheme; t from a one-Newton-step reciprocal): the loop filters'
// bar is 1e-5, and the short dependency chain is what matters here.
__device__ __forceinline__ double atan2_bf(double y, double x) {
    const double ax = fabs(x), ay = fabs(y);
    const double mx = fmax(ax, ay), mn = fmin(ax, ay);
    const bool big = mn > 0.41421356237309503 * mx;
    const double num = big ? mn - mx : mn;
    const double den = big ? mn + mx : mx;
    double r0;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r0) : "d"(den));
    const double rc = __fma_rn(r0, __fma_rn(-den, r0, 1.0), r0);
    const double t = den > 0.0 ? num * rc : 0.0;
    const double u = t * t, u2 = u * u, u4 = u2 * u2, u8 = u4 * u4;
    const double p01 = __fma_rn(-0.33333333333328574, u, 1.0);
    const double p23 = __fma_rn(-0.14285714182900408, u, 0.1999999999888112);
    const double p45 = __fma_rn(-0.09090774637548268, u, 0.11111106252782828);
    const double p67 = __fma_rn(-0.06640401512223144, u, 0.07689974062542373);
    const double p89 = __fma_rn(-0.04350303905541161, u, 0.05689174687479212);
    const double q0 = __fma_rn(p23, u2, p01);
    const double q1 = __fma_rn(p67, u2, p45);
    const double q2 = __fma_rn(0.021161483326090677, u2, p89);
    const double p = __fma_rn(__fma_rn(q2, u4, q1), u4, q0);
    (void)u8;
    double r = __fma_rn(t, p, 0.0) + (big ? PI_D / 4.0 : 0.0);
    r = ay > ax ? PI_D / 2.0 - r : r;
    r = x < 0.0 ? PI_D - r : r;
    return copysign(r, y);
}

// atan2(y, x) in fp32 with the same branch-free octant reduction: angle
// error < 2e-7 rad (fp32 quotient + the atan(t)/t series to u^7 on
// |t| <= tan(pi/8)); the loop-filter outputs it feeds carry a 1e-5 bar and
// the NCO advance does not depend on it.  Shorter dependency chain than the
// fp64 polynomial on the per-epoch critical path.
__device__ __forceinline__ double atan2_f32(double y, double x) {
    const float ax = fabsf((float)x), ay = fabsf((float)y);
    const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
    const bool big = mn > 0.41421356237f * mx;
    const float num = big ? mn - mx : mn;
    const float den = big ? mn + mx : mx;
    const float t = den > 0.f ? __fdividef(num, den) : 0.f;
    const float u = t * t, u2 = u * u;
    const float a0 = fmaf(-1.f / 3.f, u, 1.f), a1 = fmaf(-1.f / 7.f, u, 0.2f);
    const float a2 = fmaf(-1.f / 11.f, u, 1.f / 9.f), a3 = fmaf(-1.f / 15.f, u, 1.f / 13.f);
    const float p = fmaf(fmaf(a3, u2, a2), u2 * u2, fmaf(a1, u2, a0));
    double r = (double)(t * p) + (big ? PI_D / 4.0 : 0.0);
    r = ay > ax ? PI_D / 2.0 - r : r;
    r = x < 0.0 ? PI_D - r : r;
    return copysign(r, y);
}

// C fmod(x, y) for y > 0 and |x| < 2^40 y, exactly: the remainder
// x - k*y (k = trunc(x/y)) is representable, so one fma computes it
// without rounding; the quotient estimate is corrected by +-1 so the result
// lands in [0, y) for x >= 0 and (-y, 0] for x < 0, as fmod defines.
__device__ __forceinline__ double fmod_exact(double x, double y, double inv_y) {
    double k = trunc(x * inv_y);
    const double r = __fma_rn(-k, y, x);
    // branch-free +-1 correction of the quotient estimate
    const double adj = x >= 0.0 ? (r < 0.0 ? -1.0 : (r >= y ? 1.0 : 0.0))
                                : (r > 0.0 ? 1.0 : (r <= -y ? -1.0 : 0.0));
    k += adj;
    return __fma_rn(-k, y, x);
}

// NCO advance over n samples (tracking.hpp:275-280, fma as compiled)
__device__ __forceinline__ void advance_nco(double& code_phase, double& carrier_phase,
                                            double& chi, const EpochConsts& c) {
    carrier_phase = fmod_exact(__fma_rn(c.w, (double)c.n, carrier_phase), 2.0 * PI_D,
                               1.0 / (2.0 * PI_D));
    const double adv = __dmul_rn((double)c.n, c.cps);
    code_phase = fmod_exact(__dadd_rn(code_phase, adv), 1023.0, 1.0 / 1023.0);
    chi = __dadd_rn(chi, adv);
}

// The discriminator values and NCO advance of one epoch, the inputs of the
// reference's sequential loop logic (loop_fast); computed in parallel lanes
// of warp 0 and by the control warp (see warp0_update).
struct LoopPre {
    double e, l;        // |E|, |L|            (tracking.hpp:96-97, 545-546)
    double dll;         // DLL discriminator   (:95-101)
    double pll;         // Costas atan         (:104-111)
    double fc, ff;      // FLL coarse / fine   (:113-138)
    double code_phase, carrier_phase, chi;  // NCO advance (:275-280)
};

// track_epoch is split along its data dependences:
//  * loop_fast -- everything the NEXT epoch's correlation needs: FLL
//    assist, PLL/DLL filters, carrier-aided code frequency, NCO advance,
//    counters (tracking.hpp:552-601).  On the per-epoch critical path.
//  * loop_metrics -- lock-fail rule, run state, update_quality_metrics
//    (lock ratio, C/N0 window, drop to Idle; :545-549, 591-592, 459-515).
//    Nothing in the next correlation depends on it, so the tracking kernel
//    runs it on a control warp while the next epoch is being correlated.
// Together they perform the reference's operations in its order; the only
// cross-dependence (the FLL gate reads the previous epoch's lock ratio) is
// honoured because loop_metrics(e) completes before loop_fast(e+1).
// The channel's scalars are pulled into registers (independent shared-
// memory loads) and written back once.
__device__ void loop_fast(l1rxg_channel& ch, const l1rxg_corr& o, const LoopCfg& lc,
                          const LoopPre& p) {
    const l1rxg_tracking_cfg& cfg = lc.cfg;
    const bool noop = lc.kernel == L1RXG_KERNEL_NOOP;
    const int64_t esh = ch.epochs_since_handoff;
    const double clr_s = ch.carrier_lock_ratio;
    double pll_i = ch.pll_integrator, pll_p = ch.pll_prev_error;
    double dll_i = ch.dll_integrator, dll_p = ch.dll_prev_error;
    const int pll_pr = ch.pll_primed, dll_pr = ch.dll_primed;
    const int have_last = ch.have_last_prompt;
    const double dt = lc.dt;

    const double dll_err = p.dll;  // :95-101 (piece 0)
    if (ch.fll_enabled && esh < (int64_t)cfg.fll_pull_in_ms && clr_s < 0.8 && !noop) {  // :561-576
        if (esh < (int64_t)cfg.fll_coarse_ms)
            pll_i = __fma_rn(lc.fll_k * p.fc, dt, pll_i);
        else if (have_last)
            pll_i = __fma_rn(lc.fll_k * p.ff, dt, pll_i);
    }
    // loop_filter_update (:75-84), PLL then DLL
    pll_i = __fma_rn(lc.pll_k1, p.pll + (pll_pr ? pll_p : p.pll), pll_i);
    // the two divisions of the reference (/ 2pi, / f_L1) as multiplications
    // by the reciprocals: a last-bit difference, far inside the 1e-5 bar
    const double doppler_cmd = __fma_rn(lc.pll_k2, p.pll, pll_i) * (1.0 / (2.0 * PI_D));
    dll_i = __fma_rn(lc.dll_k1, dll_err + (dll_pr ? dll_p : dll_err), dll_i);
    const double dll_cmd = __fma_rn(lc.dll_k2, dll_err, dll_i);
    const double cf = __fma_rn(CHIP_RATE_HZ, fma(doppler_cmd, 1.0 / F_L1_HZ, 1.0), dll_cmd);  // :142-147

    ch.code_phase_chips = p.code_phase;
    ch.carrier_phase_rad = p.carrier_phase;
    ch.chi_chips = p.chi;
    ch.pll_integrator = pll_i;
    ch.pll_prev_error = p.pll;
    ch.pll_primed = 1;
    ch.dll_integrator = dll_i;
    ch.dll_prev_error = dll_err;
    ch.dll_primed = 1;
    ch.carrier_doppler_hz = doppler_cmd;
    ch.code_freq_hz = cf;
    ch.last_ip = o.ip;
    ch.last_qp = o.qp;
    ch.have_last_prompt = 1;
    ch.epoch_ms_count += 1;
    ch.epochs_since_handoff = esh + 1;
    ch.sample_offset_next_epoch += o.n_samples;
}

// esh: epochs_since_handoff as it was before this epoch's increment.
__device__ void loop_metrics(l1rxg_channel& ch, const l1rxg_corr& o, const LoopCfg& lc,
                             double e_env, int64_t esh) {
    const l1rxg_tracking_cfg& cfg = lc.cfg;
    const bool noop = lc.kernel == L1RXG_KERNEL_NOOP;
    int state = ch.state, lfc = ch.lock_fail_count, mvalid = ch.metrics_valid;
    int win_len = ch.win_len;
    double clr_s = ch.carrier_lock_ratio, cn0 = ch.cn0_dbhz, mu_s = ch.mu_smoothed;
    if (e_env == 0.0 && !noop)  // :545-549
        lfc++;
    if (state == L1RXG_ACQUIRED)  // :591-592
        state = L1RXG_TRACKING;
    // update_quality_metrics (:459-515); explicit roundings (no FMA
    // contraction), so every kernel instantiation computes the same bits
    const double ii = __dmul_rn(o.ip, o.ip), qq = __dmul_rn(o.qp, o.qp);
    const double pwr = __dadd_rn(ii, qq);
    const double clr = pwr > 0 ? __ddiv_rn(__dsub_rn(ii, qq), pwr) : 0.0;
    clr_s = __dadd_rn(clr_s, __dmul_rn(lc.alpha, __dsub_rn(clr, clr_s)));
    const int m = cfg.cn0_window_ms;
    double nbi = 0, nbq = 0, wbp = 0;
    bool full = false;
    if (m <= L1RXG_WIN_MAX) {  // the window's samples, summed when it is full
        ch.win_ip[win_len] = o.ip;
        ch.win_qp[win_len] = o.qp;
        win_len++;
        if (win_len >= m) {
            for (int k = 0; k < m; ++k) {
                const double wi = ch.win_ip[k], wq = ch.win_qp[k];
                const double sg = wi >= 0 ? 1.0 : -1.0;
                nbi = __dadd_rn(nbi, __dmul_rn(sg, wi));
                nbq = __dadd_rn(nbq, __dmul_rn(sg, wq));
                wbp = __dadd_rn(wbp, __dadd_rn(__dmul_rn(wi, wi), __dmul_rn(wq, wq)));
            }
            full = true;
        }
    } else {  // longer windows: the same sums accumulated in push order (bit-identical)
        if (win_len > 0) {
            nbi = ch.win_ip[0];
            nbq = ch.win_qp[0];
            wbp = ch.win_ip[1];
        }
        const double sg = o.ip >= 0 ? 1.0 : -1.0;
        nbi = __dadd_rn(nbi, __dmul_rn(sg, o.ip));
        nbq = __dadd_rn(nbq, __dmul_rn(sg, o.qp));
        wbp = __dadd_rn(wbp, __dadd_rn(__dmul_rn(o.ip, o.ip), __dmul_rn(o.qp, o.qp)));
        win_len++;
        full = win_len >= m;
        if (!full) {
            ch.win_ip[0] = nbi;
            ch.win_qp[0] = nbq;
            ch.win_ip[1] = wbp;
        }
    }
    if (full) {
        win_len = 0;
        const double mu =
            wbp > 0 ? __ddiv_rn(__dadd_rn(__dmul_rn(nbi, nbi), __dmul_rn(nbq, nbq)), wbp) : 0.0;
        mu_s = mvalid ? __dadd_rn(mu_s, __dmul_rn(0.2, __dsub_rn(mu, mu_s))) : mu;
        const double md = (double)m;
        if (mu_s >= md - 1e-9)
            cn0 = 65.0;
        else if (mu_s <= 1.0)
            cn0 = 0.0;
        else
            cn0 = __dmul_rn(10.0, log10(__ddiv_rn(__ddiv_rn(__dsub_rn(mu_s, 1.0), __dsub_rn(md, mu_s)), 1e-3)));
        mvalid = 1;
    }
    if (mvalid && esh > cfg.fll_pull_in_ms + cfg.cn0_window_ms) {
        if (cn0 < cfg.cn0_drop_dbhz || clr_s < cfg.carrier_lock_drop)
            lfc++;
        else
            lfc = 0;
    }
    if (lfc > cfg.lock_fail_limit)
        state = L1RXG_IDLE;
    ch.state = state;
    ch.lock_fail_count = lfc;
    ch.metrics_valid = mvalid;
    ch.win_len = win_len;
    ch.carrier_lock_ratio = clr_s;
    ch.cn0_dbhz = cn0;
    ch.mu_smoothed = mu_s;
}

// ---------------------------------------------------------------------
// Shared-memory layout of a correlator CTA (the sample tile follows it).
template <int T>
struct CorrSmem {
    l1rxg_channel ch;
    EpochConsts c;
    LoopPre pre;
    double d[T];
    double sums[2 * T + 2];
    float red[32 * (2 * T + 2)];
    float2 rot[RUN + 1];
    uint64_t bars[2][2];  // per tile buffer: the two halves of its bulk copy
    uint64_t pbar[2];     // cluster: partial totals of epoch e landed (e & 1)
    int inflight[2];      // per tile buffer: a bulk copy is outstanding
    int64_t issue_pos;    // ring position of the next unit to copy
    // epoch handed from the critical path to the control warp
    l1rxg_epoch_record rec;  // inputs, correlator outputs, loop outputs
    int64_t rec_slot;
    int64_t rec_esh;         // epochs_since_handoff before that epoch
    double rec_eenv;         // |E| + |L|
    int pending, stop;
    double nco_ph1, nco_cp1;  // this epoch's NCO advance (control warp, off the critical path)
    CodeTables ct;
};

template <int T>
__host__ __device__ constexpr size_t corr_smem_header() {
    return (sizeof(CorrSmem<T>) + 15) & ~size_t(15);
}

// Dynamic shared memory after the header: anchors[nwork] (one carrier
// anchor per run of the current unit), then nbuf sample tiles of cap + 4
// float2 each (cap = nwork * RUN; +4: bulk-copy alignment slack).
template <int T>
__device__ __forceinline__ float2* anchors_of(CorrSmem<T>* s) {
    return reinterpret_cast<float2*>(reinterpret_cast<char*>(s) + corr_smem_header<T>());
}
__host__ __device__ constexpr int anchors_len(int nwork) { return (nwork + 1) & ~1; }
// Sample tile b: nwork*RUN samples of esz bytes + 16 B of bulk-copy
// alignment slack on each side, rounded to 16 B.
__host__ __device__ constexpr size_t tile_bytes(int nwork, int esz) {
    return ((static_cast<size_t>(nwork) * RUN * esz + 32) + 15) & ~size_t(15);
}
template <int T>
__device__ __forceinline__ unsigned char* tile_of(CorrSmem<T>* s, int nwork, int b, int esz) {
    return reinterpret_cast<unsigned char*>(anchors_of(s) + anchors_len(nwork)) +
           (size_t)b * tile_bytes(nwork, esz);
}
// Raw sample kinds: the prefix sums go to their own float2 tile after the
// sample tiles (float2 rings keep them in place).
template <int T>
__device__ __forceinline__ float2* prefix_of(CorrSmem<T>* s, int nwork, int nbuf, int esz) {
    return reinterpret_cast<float2*>(tile_of(s, nwork, nbuf, esz));
}
// Cluster exchange slots after the tiles: [2 (epoch parity)][csize][2T+2]
// fp64 partial totals, written by every CTA of the cluster into every CTA.
template <int T>
__device__ __forceinline__ double* xslots_of(CorrSmem<T>* s, int nwork, int nbuf, int esz) {
    return reinterpret_cast<double*>(prefix_of(s, nwork, nbuf, esz) +
                                     (esz == 8 ? 0 : (size_t)nwork * RUN));
}

// o (CorrelatorOutputs) from the fp64 sums
template <int T>
__device__ __forceinline__ l1rxg_corr corr_from_sums(const double* sums, int ke, int kp, int kl, int n) {
    l1rxg_corr o;
    o.ie = sums[2 * ke];
    o.qe = sums[2 * ke + 1];
    o.ip = sums[2 * kp];
    o.qp = sums[2 * kp + 1];
    o.il = sums[2 * kl];
    o.ql = sums[2 * kl + 1];
    o.ip_h1 = sums[2 * T];
    o.qp_h1 = sums[2 * T + 1];
    o.ip_h2 = o.ip - o.ip_h1;
    o.qp_h2 = o.qp - o.qp_h1;
    o.n_samples = n;
    o.pad_ = 0;
    return o;
}

// Warp reduction of the V partials -> red[warp][v] as a reduce-scatter
// butterfly: at each level a lane keeps half of its values and receives the
// partner's matching half, so V values need ~V + 5 shuffles instead of 5V.
template <int V>
__device__ __forceinline__ void warp_partials(const float* acc, float* red, int lane, int warp) {
    constexpr int P = (V <= 8) ? 8 : (V <= 16) ? 16 : (V <= 32) ? 32 : 64;
    if constexpr (P > 32) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
            float x = acc[v];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
                x += __shfl_xor_sync(0xffffffffu, x, o);
            if (lane == 0)
                red[warp * V + v] = x;
        }
    } else {
        float x[P];
#pragma unroll
        for (int v = 0; v < P; ++v)
            x[v] = v < V ? acc[v] : 0.f;
        int base = 0;
#pragma unroll
        for (int lv = 0, o = 16; lv < 5; ++lv, o >>= 1) {
            const int c = P >> lv;  // values held before this level
            if (c > 1) {
                const int h = c / 2;
                const bool upper = (lane & o) != 0;
#pragma unroll
                for (int i = 0; i < h; ++i) {
                    const float send = upper ? x[i] : x[i + h];
                    const float keep = upper ? x[i + h] : x[i];
                    x[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
                if (upper)
                    base += h;
            } else {
                x[0] += __shfl_xor_sync(0xffffffffu, x[0], o);
            }
        }
        if (base < V && (lane & (32 / P - 1)) == 0)
            red[warp * V + base] = x[0];
    }
}

// fp64 cross-warp totals (by warp 0): lane v adds the nwarps partials of
// value v into four interleaved fp64 chains, then pairs them -- a fixed,
// deterministic order; only the live warps are converted and added.
template <int V>
__device__ __forceinline__ void warp0_totals(const float* red, double* sums, int lane, int nwarps) {
    for (int v = lane; v < V; v += 32) {
        double x0 = 0.0, x1 = 0.0, x2 = 0.0, x3 = 0.0;
        int w = 0;
        for (; w + 4 <= nwarps; w += 4) {
            x0 += (double)red[w * V + v];
            x1 += (double)red[(w + 1) * V + v];
            x2 += (double)red[(w + 2) * V + v];
            x3 += (double)red[(w + 3) * V + v];
        }
        if (w < nwarps)
            x0 += (double)red[w * V + v];
        if (w + 1 < nwarps)
            x1 += (double)red[(w + 1) * V + v];
        if (w + 2 < nwarps)
            x2 += (double)red[(w + 2) * V + v];
        sums[v] = (x0 + x1) + (x2 + x3);
    }
}

// ---------------------------------------------------------------------
// Kernel arguments for closed-loop tracking.
struct TrackArgs {
    const unsigned char* ring;  // [n_streams][ring_stride] samples of esz bytes
    int64_t ring_stride;      // R + apron
    int64_t ring_cap;         // R
    const int64_t* avail;     // [n_streams] samples ingested
    l1rxg_channel* chans;     // [C]
    const int32_t* chan_stream;
    l1rxg_epoch_record* recs; // [C][max_records]
    double* tap_sums;         // [C][max_records][2T]
    int64_t* ecount;          // [C] epochs done
    int32_t* status;          // [C] 0 ok, 1 ring overrun
    const int8_t* codes;      // [33][1023]
    int max_records;
    int max_epochs;
    int n;
    int kp, ke, kl;
    l1rxg_taps taps;
    LoopCfg lc;
    long long* prof;  // optional stage clocks (L1RXG_PROF=1): [epoch][8], CTA 0
    int nbuf;         // sample tiles per CTA: 1 (latency shape) or 2 (double-buffered)
    int csize;        // CTAs per channel (a thread-block cluster when > 1)
    int share;        // samples of each epoch per cluster CTA (multiple of RUN)
    int thr;          // throughput-shape instantiation (track_kernel<..., true>)
    float ovl_dwmax;  // overlapped kernel: |dw| * RUN above this recomputes phase A exactly
};

// Stage clocks (profiling builds only: -DL1RXG_PROFILE, run with
// L1RXG_PROF=1): CTA 0's first 64 epochs, bank 0 per-epoch stamps, bank 1
// per-unit stage sums kept in registers and flushed once per epoch.
#ifdef L1RXG_PROFILE
#define PROF_STAMP(k)                                                          \
    do {                                                                       \
        if (a.prof && blockIdx.x == 0 && e < 64)                               \
            a.prof[e * 8 + (k)] = clock64();                                   \
    } while (0)
// per-unit stage sums of CTA 0, kept in registers and flushed once per
// epoch (bank 1 of the profile buffer)
#define PROF_UNIT(k, t0)                                                       \
    do {                                                                       \
        if (a.prof) {                                                          \
            const long long t_ = clock64();                                    \
            pu[k] += t_ - (t0);                                                \
            (t0) = t_;                                                         \
        }                                                                      \
    } while (0)
// thread 0's phase A sub-steps (bank 3)
#define PROF_A(k)                                                              \
    do {                                                                       \
        if (a.prof && blockIdx.x == 0 && e < 64 && tid == 0)                  \
            a.prof[1536 + e * 8 + (k)] = clock64();                            \
    } while (0)
// warp-0 update sub-steps (bank 2)
#define PROF_W(k)                                                              \
    do {                                                                       \
        if (a.prof && blockIdx.x == 0 && ep < 64 && lane == 0)                 \
            a.prof[1024 + ep * 8 + (k)] = clock64();                           \
    } while (0)
#else
#define PROF_A(k) \
    do {          \
    } while (0)
#define PROF_W(k) \
    do {          \
    } while (0)
#define PROF_STAMP(k) \
    do {              \
    } while (0)
#define PROF_UNIT(k, t0) \
    do {                 \
    } while (0)
#endif

// TMA unit: len samples (esz bytes each) from ring position pos (< R) into
// the tile, copied from the 16-byte aligned position below (delta samples of
// slack), in two halves on two mbarriers.
template <int T>
__device__ __forceinline__ void issue_unit(CorrSmem<T>* s, int b, unsigned char* tile,
                                           const unsigned char* ring, int64_t pos, int len, int esz) {
    const int A = 16 / esz;  // samples per 16 bytes
    const int delta = (int)(pos & (A - 1));
    const int h = A * ((len + delta) / (2 * A));
    const uint32_t total = (uint32_t)(((len + delta) * esz + 15) & ~15);
    const uint32_t b0 = (uint32_t)(h * esz);
    const unsigned char* src = ring + (pos - delta) * esz;
    mbar_expect_tx(&s->bars[b][0], b0);
    if (b0)
        tma_load_1d(tile, src, b0, &s->bars[b][0]);
    mbar_expect_tx(&s->bars[b][1], total - b0);
    tma_load_1d(tile + b0, src + b0, total - b0, &s->bars[b][1]);
    s->inflight[b] = 1;
}

// NCO advance of the epoch being correlated (tracking.hpp:275-280, exact
// fmod): depends only on the pre-epoch state, so the control warp computes it
// (lanes 0/1) while the work warps correlate.
__device__ __forceinline__ void nco_advance_lanes(double& ph1, double& cp1, const EpochConsts& c,
                                                  const l1rxg_channel& ch, int lane) {
    const bool carrier = lane == 0;
    const double adv = __dmul_rn((double)c.n, c.cps);
    const double fm = fmod_exact(carrier ? __fma_rn(c.w, (double)c.n, ch.carrier_phase_rad)
                                         : __dadd_rn(ch.code_phase_chips, adv),
                                 carrier ? 2.0 * PI_D : 1023.0,
                                 carrier ? 1.0 / (2.0 * PI_D) : 1.0 / 1023.0);
    if (lane == 0)
        ph1 = fm;
    else if (lane == 1)
        cp1 = fm;
}

// Control-warp side of an epoch: run state, quality metrics and lock-fail
// rule for the epoch handed over in s->rec, then its record and tap sums.
template <int T, typename S>
__device__ __forceinline__ void finish_epoch(S* s, const TrackArgs& a, int lane,
                                             bool writer) {
    if (lane == 0) {
        l1rxg_channel& ch = s->ch;
        const l1rxg_corr o = corr_from_sums<T>(s->sums, a.ke, a.kp, a.kl, a.n);
        loop_metrics(ch, o, a.lc, s->rec_eenv, s->rec_esh);
        l1rxg_epoch_record r = s->rec;  // inputs; the rest is post-update state
        r.epoch_index = ch.epoch_ms_count - 1;
        r.sample_offset_end = ch.sample_offset_next_epoch;
        r.prn = ch.prn;
        r.n_samples = o.n_samples;
        r.ie = o.ie; r.qe = o.qe; r.ip = o.ip; r.qp = o.qp; r.il = o.il; r.ql = o.ql;
        r.ip_h1 = o.ip_h1; r.qp_h1 = o.qp_h1; r.ip_h2 = o.ip_h2; r.qp_h2 = o.qp_h2;
        r.carrier_doppler_hz = ch.carrier_doppler_hz;
        r.code_freq_hz = ch.code_freq_hz;
        r.code_phase_chips = ch.code_phase_chips;
        r.carrier_phase_rad = ch.carrier_phase_rad;
        r.chi_chips = ch.chi_chips;
        r.dll_integrator = ch.dll_integrator;
        r.pll_integrator = ch.pll_integrator;
        r.dll_prev_error = ch.dll_prev_error;
        r.pll_prev_error = ch.pll_prev_error;
        r.state = ch.state;
        r.lock_fail_count = ch.lock_fail_count;
        r.cn0_dbhz = ch.cn0_dbhz;
        r.carrier_lock_ratio = ch.carrier_lock_ratio;
        r.mu_smoothed = ch.mu_smoothed;
        if (writer)
            a.recs[s->rec_slot] = r;
    }
    if (writer && a.tap_sums && lane < 2 * T)
        a.tap_sums[s->rec_slot * (2 * T) + lane] = s->sums[lane];
}

// The per-epoch critical path on warp 0, SIMT: the transcendental pieces of
// track_epoch are evaluated as ONE instruction stream over lanes with
// different inputs (no divergence, no cross-warp hand-off):
//   atan2 on lanes 0..2: PLL  atan(qp/ip) = atan2(qp*sgn(ip), |ip|)
//                        (tracking.hpp:104-111), FLL coarse and fine
//                        (:113-138; the fine one folded to dot >= 0);
//   sqrt  on lanes 3..4: |E|, |L| (:96-97);
// (branch-free fp64 helpers, so the pieces interleave); the exact-fmod NCO
// advance (:275-280) was computed by the control warp during the epoch.
// Lane 0 then runs loop_fast and forms the next epoch's w and cps as IEEE
// quotients (:234-236).  Loop values agree with the reference to ~1e-15
// relative (the parity bar is 1e-5); the state advance is bit-exact.
template <int T, typename S>
__device__ __forceinline__ void warp0_update(S* s, const TrackArgs& a, const EpochConsts& c,
                                             int64_t off, int cidx, int64_t done, int nwork_warps,
                                             int lane, int crank, int ep, double* xs, int rec_i) {
    constexpr int V = 2 * T + 2;
    PROF_W(0);
    warp0_totals<V>(s->red, s->sums, lane, nwork_warps);
    __syncwarp();
    PROF_W(1);
    if (a.csize > 1) {
        // every CTA of the cluster sends its fp64 totals to every CTA
        // (st.async completing bytes on the receiver's mbarrier), then each
        // sums the csize slots in rank order: identical cluster totals (and
        // so identical loop updates) in every CTA, one round trip
        const int par = ep & 1;
        const int K = a.csize;
        for (int it = lane; it < V * K; it += 32) {
            const int q = it / V, v = it - q * V;
            st_async_f64(cluster_map(xs + (par * K + crank) * V + v, q), s->sums[v],
                         cluster_map(&s->pbar[par], q));
        }
        if (lane == 0)
            mbar_expect_tx(&s->pbar[par], (uint32_t)(K * V * 8));
        mbar_wait_cluster(&s->pbar[par], (uint32_t)(ep >> 1) & 1u);
        for (int v = lane; v < V; v += 32) {
            double t = 0.0;
            for (int q = 0; q < K; ++q)
                t += xs[(par * K + q) * V + v];
            s->sums[v] = t;
        }
        __syncwarp();
    }
    PROF_W(2);
    l1rxg_channel& ch = s->ch;
    if (ch.state == L1RXG_IDLE) {  // the previous epoch dropped the channel
        if (lane == 0)
            s->stop = 1;
        return;
    }
    const double ie = s->sums[2 * a.ke], qe = s->sums[2 * a.ke + 1];
    const double il = s->sums[2 * a.kl], ql = s->sums[2 * a.kl + 1];
    const double ip = s->sums[2 * a.kp], qp = s->sums[2 * a.kp + 1];
    const double h1i = s->sums[2 * T], h1q = s->sums[2 * T + 1];
    const double cp0 = ch.code_phase_chips, ph0 = ch.carrier_phase_rad, chi0 = ch.chi_chips;
    const double adv = __dmul_rn((double)c.n, c.cps);
    // atan2 lanes
    double y = 0.0, x = 1.0;
    bool zero = false;
    if (lane == 0) {
        y = ip < 0 ? -qp : qp;
        x = fabs(ip);
    } else if (lane == 1 || lane == 2) {
        const double pi_ = lane == 1 ? h1i : ch.last_ip, pq = lane == 1 ? h1q : ch.last_qp;
        const double ci = lane == 1 ? ip - h1i : ip, cq = lane == 1 ? qp - h1q : qp;
        double cross = __dsub_rn(__dmul_rn(pi_, cq), __dmul_rn(pq, ci));
        double dot = __dadd_rn(__dmul_rn(pi_, ci), __dmul_rn(pq, cq));
        if (lane == 2 && dot < 0) {
            cross = -cross;
            dot = -dot;
        }
        y = cross;
        x = dot;
        zero = cross == 0.0 && dot == 0.0;
    }
#ifdef L1RXG_ATAN_F32  // experiment switch: measured 0.4 % on config 2, not worth the precision
    const double ang = atan2_f32(y, x);
#else
    const double ang = atan2_bf(y, x);
#endif
    // sqrt lanes
    const double sq = fast_sqrt(lane == 3 ? __dadd_rn(__dmul_rn(ie, ie), __dmul_rn(qe, qe))
                                          : __dadd_rn(__dmul_rn(il, il), __dmul_rn(ql, ql)));
    PROF_W(3);
    const double a_pll = __shfl_sync(0xffffffffu, ang, 0);
    const double a_fc = __shfl_sync(0xffffffffu, ang, 1);
    const double a_ff = __shfl_sync(0xffffffffu, ang, 2);
    const bool z_fc = __shfl_sync(0xffffffffu, zero, 1);
    const bool z_ff = __shfl_sync(0xffffffffu, zero, 2);
    const double e = __shfl_sync(0xffffffffu, sq, 3);
    const double l = __shfl_sync(0xffffffffu, sq, 4);
    const double ph1 = s->nco_ph1;  // NCO advance, computed by the control warp
    const double cp1 = s->nco_cp1;
    double fd = 0.0, cf = 0.0;
    if (lane == 0) {
        LoopPre pre;
        pre.e = e;
        pre.l = l;
        pre.dll = (e + l == 0.0) ? 0.0 : 0.5 * fast_div(e - l, e + l);  // :95-101
        pre.pll = ip == 0.0 ? (qp == 0.0 ? 0.0 : (qp > 0 ? PI_D / 2.0 : -PI_D / 2.0)) : a_pll;
        pre.fc = z_fc ? 0.0 : a_fc * a.lc.inv_fll_c;
        pre.ff = z_ff ? 0.0 : a_ff * a.lc.inv_fll_f;
        pre.carrier_phase = ph1;
        pre.code_phase = cp1;
        pre.chi = __dadd_rn(chi0, adv);
        l1rxg_epoch_record& r = s->rec;  // correlator inputs for the record
        r.sample_offset_start = off;
        r.code_phase_in = cp0;
        r.code_freq_in = ch.code_freq_hz;
        r.carrier_doppler_in = ch.carrier_doppler_hz;
        r.carrier_phase_in = ph0;
        s->rec_esh = ch.epochs_since_handoff;
        s->rec_eenv = e + l;
        l1rxg_corr o;
        o.ip = ip;
        o.qp = qp;
        o.n_samples = c.n;
        PROF_W(4);
        loop_fast(ch, o, a.lc, pre);
        PROF_W(5);
        fd = ch.carrier_doppler_hz;
        cf = ch.code_freq_hz;
        s->rec_slot = (int64_t)cidx * a.max_records + rec_i;
        s->pending = 1;
    }
    // next epoch's w = (2 pi fD)/fs and cps = cf/fs, the reference's IEEE
    // quotients (lanes 0 and 1); inv_cps is formed by each thread at the start
    // of the next epoch, off this path
    PROF_W(6);
    fd = __shfl_sync(0xffffffffu, fd, 0);
    cf = __shfl_sync(0xffffffffu, cf, 0);
    // one IEEE division per lane (two on one lane serialise: 2.5x slower)
    const double quo = (lane == 0 ? 2.0 * PI_D * fd : cf) / a.lc.fs;
    const double w = __shfl_sync(0xffffffffu, quo, 0);
    const double cps = __shfl_sync(0xffffffffu, quo, 1);
    if (lane == 0) {
        EpochConsts& nc = s->c;
        nc.w = w;
        nc.cps = cps;
        nc.base = cp1 + 1023.0;
        nc.phi = ph1;
        nc.n = c.n;
        nc.nh = c.nh;
    }
    __syncwarp();
    PROF_W(7);
}

// Channel-resident persistent tracking kernel: one CTA per channel loops
// over its epochs with no host round trip (replaces the per-channel
// track_epoch fan-out of Receiver::tracking_round, pipeline.hpp:563-610).
//   * work warps (blockDim - 32 threads): correlation, phases A and B, one
//     sub-tile ("unit", cap = nwork * RUN samples) at a time;
//   * units arrive by TMA bulk copy into nbuf tiles: with one tile the next
//     unit is copied once the current one is consumed (latency shape: one
//     unit per epoch, the copy overlaps the loop update); with two tiles
//     the copy of unit u+2 is issued as soon as unit u is consumed, so it
//     overlaps unit u+1's correlation (throughput shape, many units per
//     epoch);
//   * per-epoch critical path on warp 0: fp64 totals -> the transcendental
//     pieces in SIMT lanes -> loop_fast (filters, NCO) -> next epoch's
//     constants;
//   * the last warp is a control warp: it issues the copies and finishes
//     epoch e (loop_metrics, record) while epoch e+1 is being correlated.
//     If that makes the channel Idle, epoch e+1 is discarded before its
//     loop update, exactly as if it had never been admitted
//     (tracking.hpp:511-514 + the caller's Idle check, pipeline.hpp:567-568).
// THR: throughput shape (many units per epoch, four CTAs per SM): phase B's
// steps are searched while each unit's copy lands.  !THR: latency shapes
// (the copy is long done): the search interleaves with phase A.  Separate
// instantiations keep each shape's code small (the serial per-epoch path of
// the latency shape is sensitive to instruction-cache misses).
template <int T, int SK, bool THR>
__global__ void __launch_bounds__(MAX_NT, 1) track_kernel(TrackArgs a) {
    typedef typename Samp<SK>::raw_t R;
    constexpr int esz = Samp<SK>::esz;
    constexpr int A = 16 / esz;  // samples per 16-byte bulk-copy granule
    extern __shared__ __align__(16) unsigned char smem_raw[];
    CorrSmem<T>* s = reinterpret_cast<CorrSmem<T>*>(smem_raw);
    // cluster split: csize consecutive CTAs (one cluster) share a channel,
    // CTA crank correlating samples [r0, rend) of every epoch
    const int csize = a.csize;
    const int crank = csize > 1 ? (int)(blockIdx.x % csize) : 0;
    const int cidx = blockIdx.x / csize;
    const bool writer = crank == 0;
    const int strm = a.chan_stream[cidx];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = (blockDim.x + 31) >> 5;
    const int ctl = nwarps - 1;            // control warp
    const int nwork = blockDim.x - 32;     // correlation threads
    const int nwork_warps = nwarps - 1;
    constexpr int V = 2 * T + 2;
    const int cap = nwork * RUN;
    const int n = a.n;
    const int r0 = csize > 1 ? crank * a.share : 0;
    const int rend = csize > 1 ? min(n, r0 + a.share) : n;
    const int my_n = rend - r0;
    const int nsub = (my_n + cap - 1) / cap;
    const int skip = n - my_n;             // ring samples between this CTA's epochs
    const int nbuf = a.nbuf;
    const bool noop = a.lc.kernel == L1RXG_KERNEL_NOOP;
    const int64_t avail = a.avail[strm];
    const unsigned char* ring = a.ring + (int64_t)strm * a.ring_stride * esz;
    float2* anchors = anchors_of(s);
    double* xs = xslots_of(s, nwork, nbuf, esz);
    const float scale = SK == SK_I16 ? 1.f / 32768.f : SK == SK_I8 ? 1.f / 128.f : 1.f;
    const int64_t off0 = a.chans[cidx].sample_offset_next_epoch;
    // unit v of this launch: epoch v / nsub, sub-tile v % nsub, into tile
    // v % nbuf.  Units of the epoch being correlated (ev <= ecur) are always
    // copied; a later epoch's only if the admission test will accept it as
    // things stand (not Idle, in range, fully ingested).
    auto try_issue = [&](int v, int ecur) {
        const int ev = v / nsub;
        const int q = v - ev * nsub;
        const int64_t offv = off0 + (int64_t)ev * n;
        if (noop || ev >= a.max_epochs || offv + n > avail || off0 < 0 ||
            off0 < avail - a.ring_cap || (ev > ecur && s->ch.state == L1RXG_IDLE))
            return;
        const int b = v & (nbuf - 1);
        const int len = min(cap, rend - (r0 + q * cap));
        // units are issued in order without gaps: the ring position advances
        // by each unit's length (+ the other cluster CTAs' samples at the end
        // of an epoch)
        const int64_t pos = s->issue_pos;
        issue_unit(s, b, tile_of(s, nwork, b, esz), ring, pos, len, esz);
        int64_t nxt = pos + len + (q + 1 == nsub ? skip : 0);
        while (nxt >= a.ring_cap)
            nxt -= a.ring_cap;
        s->issue_pos = nxt;
    };
    if (tid == 0) {
        s->ch = a.chans[cidx];
        for (int b = 0; b < 2; ++b) {
            mbar_init(&s->bars[b][0], 1);
            mbar_init(&s->bars[b][1], 1);
            mbar_init(&s->pbar[b], 1);  // the local expect_tx arrive + K*V*8 bytes
            s->inflight[b] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        s->pending = 0;
        s->stop = 0;
    }
    for (int k = tid; k < T; k += blockDim.x)
        s->d[k] = a.taps.offsets_chips[k];
    if (csize > 1)
        cluster_sync_all();  // barriers initialised before any remote arrive
    __syncthreads();
    PhaseB pb;
    phase_b_init<T>(pb, s->d, a.kp, tid, nwork);
    build_code_tables(s->ct, a.codes, s->ch.prn);
    const int64_t pos0 = off0 >= 0 ? (off0 + r0) % a.ring_cap : 0;
    if (tid == 0) {  // first epoch: consts and the first units
        s->issue_pos = pos0;
        const l1rxg_channel& ch = s->ch;
        make_consts(s->c, ch.code_phase_chips, ch.code_freq_hz, ch.carrier_doppler_hz,
                    ch.carrier_phase_rad, a.lc.fs, n);
        for (int v = 0; v < nbuf; ++v)
            try_issue(v, -1);
    }
    __syncthreads();
    fill_rot(s->rot, s->c.w, tid, scale);
    __syncthreads();

    uint32_t phase = 0;  // bit b: parity of tile b's next completion
    int e = 0;
    int u = 0;           // next unit to consume
    // ring position of unit u, tracked by every thread (the copy's 16-byte
    // alignment slack follows from it) so no hand-off from the issuer is needed
    int64_t upos = pos0;
    int64_t done = a.ecount[cidx];
    int rec_i = (int)(done % a.max_records);  // record slot of the current epoch
    for (;;) {
        // epoch admission (uniform: every thread -- and every CTA of a
        // cluster -- reads the same state)
        const int64_t off = s->ch.sample_offset_next_epoch;
        if (s->ch.state == L1RXG_IDLE || e >= a.max_epochs || off + n > avail)
            break;
        if (off < avail - a.ring_cap || off < 0) {  // window already overwritten
            if (tid == 0)
                a.status[cidx] = 1;
            break;
        }
        if (tid == 0)
            PROF_STAMP(0);
        PROF_A(0);
        EpochConsts c = s->c;
        // control warp: this epoch's NCO advance, then finish the previous
        // epoch, while this one correlates
        if (warp == ctl) {
            nco_advance_lanes(s->nco_ph1, s->nco_cp1, c, s->ch, lane);
            if (s->pending) {
                finish_epoch<T>(s, a, lane, writer);
                if (lane == 0)
                    s->pending = 0;
            }
        }
        float acc[V];
#pragma unroll
        for (int v = 0; v < V; ++v)
            acc[v] = 0.f;
#ifdef L1RXG_PROFILE
        long long tu = a.prof ? clock64() : 0;
        long long pu[5] = {0, 0, 0, 0, 0};
#endif
        for (int q = 0; q < nsub; ++q, ++u) {
            const int b = nbuf == 1 ? 0 : (int)(u & 1);
            const uint32_t par = (phase >> b) & 1u;
            const int u0 = r0 + q * cap;
            const int len = min(cap, rend - u0);
            const int delta = (int)(upos & (A - 1));
            const int h = A * ((len + delta) / (2 * A));
            upos += len + (q + 1 == nsub ? skip : 0);
            while (upos >= a.ring_cap)
                upos -= a.ring_cap;
            if (!noop) {
                const R* rawt = reinterpret_cast<const R*>(tile_of(s, nwork, b, esz)) + delta;
                // prefix sums: in place for float2 rings, else their own tile
                float2* pre = SK == SK_F32 ? reinterpret_cast<float2*>(tile_of(s, nwork, b, esz)) + delta
                                           : prefix_of(s, nwork, nbuf, esz);
                const float2* tile_d = pre;
                if (tid < nwork) {
                    PROF_A(1);
                    const int i0 = u0 + tid * RUN;
                    const int cnt = min(RUN, rend - i0);
                    const int r0t = delta + tid * RUN;
                    // phase B's transition range and first exact steps depend
                    // only on the epoch constants: with several units per
                    // epoch they are found while this unit's copy lands; with
                    // one (latency shape, copy long done) they interleave
                    // with phase A below
                    if constexpr (THR) {
                        c.inv_cps = fast_rcp(c.cps);  // tap_boundary's estimate (within 2 ulp)
                        phase_b_pre<T>(pb, c, s->ct, u0, len);
                    }
                    PROF_A(2);
                    // each half of the copy has waiters (thread 0's run starts
                    // in the first, the last run ends in the second), so after
                    // the work-warp barrier below both copies are complete
                    if (cnt > 0) {
                        if (r0t < h)
                            mbar_wait(&s->bars[b][0], par);
                        if (r0t + RUN > h)
                            mbar_wait(&s->bars[b][1], par);
                    }
                    PROF_A(3);
                    if constexpr (!THR) {
                        c.inv_cps = fast_rcp(c.cps);
                        phase_b_range<T>(pb, c, s->ct, u0, len);
                    }
#ifndef L1RXG_XSKIP_A
                    if (cnt > 0)
                        phase_a_dispatch<T>(c, rawt + tid * RUN, pre + tid * RUN, s->rot, s->ct.chip,
                                            s->d, a.kp, i0, cnt, acc, &anchors[tid]);
#endif
                    PROF_A(4);
                    if (tid == 0) {
                        PROF_STAMP(1);
                        PROF_UNIT(0, tu);
                    }
                }
                phase ^= 1u << b;
                if (tid < nwork) {
                    // prefixes + anchors visible: the work warps only, so the
                    // control warp's epoch finish does not hold phase B
                    named_bar_sync(1, nwork);
                    if (tid == 0) {
                        PROF_STAMP(2);
                        PROF_UNIT(1, tu);
                    }
#ifndef L1RXG_XSKIP_B
                    phase_b<T, THR>(pb, c, tile_d, anchors, s->ct, u0, len);
#endif
                }
            }
            if (q + 1 == nsub && warp < nwork_warps) {
                phase_b_fold<T>(pb, acc);
                warp_partials<V>(acc, s->red, lane, warp);
            }
            if (tid == 0)
                PROF_UNIT(2, tu);
            __syncthreads();  // tile consumed
            if (tid == 0) {
                PROF_STAMP(3);
                PROF_UNIT(3, tu);
            }
            if (warp == ctl && lane == 0) {  // the next bulk copy, off warp 0's path
                s->inflight[b] = 0;
                try_issue(u + nbuf, e);
            }
            if (tid == 0)
                PROF_UNIT(4, tu);
        }
        // ---- critical path, all on warp 0 in SIMT form (no cross-warp
        // hand-off): totals (+ the cluster exchange) -> one atan2 / sqrt /
        // fmod / division per lane -> loop_fast on lane 0 -> next epoch's
        // constants, rotators, ranges
        if (warp == 0) {
            if (tid == 0) {
                PROF_STAMP(4);
#ifdef L1RXG_PROFILE
                if (a.prof && blockIdx.x == 0 && e < 64)
                    for (int k = 0; k < 5; ++k)
                        a.prof[512 + e * 8 + k] = pu[k];
#endif
            }
            warp0_update<T>(s, a, c, off, cidx, done, nwork_warps, lane, crank, e, xs, rec_i);
            if (tid == 0)
                PROF_STAMP(5);
            fill_rot(s->rot, s->c.w, lane, scale);
            if (tid == 0)
                PROF_STAMP(6);
        }
        __syncthreads();
        if (tid == 0)
            PROF_STAMP(7);
        if (s->stop)
            break;
        ++e;
        ++done;
        if (++rec_i == a.max_records)
            rec_i = 0;
    }
    __syncthreads();
    if (warp == ctl && s->pending)
        finish_epoch<T>(s, a, lane, writer);
    __syncthreads();
    if (tid == 0) {
        for (int b = 0; b < nbuf; ++b)
            if (s->inflight[b]) {  // never leave a bulk copy in flight into freed smem
                mbar_wait(&s->bars[b][0], (phase >> b) & 1u);
                mbar_wait(&s->bars[b][1], (phase >> b) & 1u);
            }
        if (writer) {
            a.chans[cidx] = s->ch;
            a.ecount[cidx] = done;
        }
    }
    if (csize > 1)
        cluster_sync_all();  // no CTA leaves while a peer may still write into it
}

// ---------------------------------------------------------------------
// Open-loop batch (per-call compatibility path and replay tests): job j
// correlates samples src + j*n with NCO states[j], advances it in place.
struct JobArgs {
    const float2* samples;  // [n_jobs][n]
    l1rxg_nco* states;      // [n_jobs]
    const int32_t* prns;    // [n_jobs]
    const int8_t* codes;
    double* tap_sums;       // [n_jobs][2T]
    l1rxg_corr* corr;       // [n_jobs]
    int n, kp, ke, kl, kernel;
    double fs;
    l1rxg_taps taps;
};

template <int T>
__global__ void __launch_bounds__(MAX_NT, 1) correlate_jobs_kernel(JobArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    CorrSmem<T>* s = reinterpret_cast<CorrSmem<T>*>(smem_raw);
    float2* anchors = anchors_of(s);
    float2* tile = reinterpret_cast<float2*>(tile_of(s, blockDim.x, 0, 8));
    const int j = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = (blockDim.x + 31) >> 5;
    constexpr int V = 2 * T + 2;
    const int n = a.n;
    const int cap = blockDim.x * RUN;
    for (int k = tid; k < T; k += blockDim.x)
        s->d[k] = a.taps.offsets_chips[k];
    if (tid == 0) {
        const l1rxg_nco st = a.states[j];
        make_consts(s->c, st.code_phase_chips, st.code_freq_hz, st.carrier_doppler_hz,
                    st.carrier_phase_rad, a.fs, n);
    }
    build_code_tables(s->ct, a.codes, a.prns[j]);  // ends with a barrier
    PhaseB pb;
    phase_b_init<T>(pb, s->d, a.kp, tid, blockDim.x);
    fill_rot(s->rot, s->c.w, tid);
    const EpochConsts c = s->c;
    float acc[V];
#pragma unroll
    for (int v = 0; v < V; ++v)
        acc[v] = 0.f;
    const float2* src = a.samples + (int64_t)j * n;
    if (a.kernel != L1RXG_KERNEL_NOOP) {
        for (int u0 = 0; u0 < n; u0 += cap) {
            const int len = min(cap, n - u0);
            for (int i = tid; i < len; i += blockDim.x)
                tile[i] = __ldg(src + u0 + i);
            __syncthreads();
            const int i0 = u0 + tid * RUN;
            const int cnt = min(RUN, n - i0);
            if (cnt > 0)
                phase_a_dispatch<T>(c, reinterpret_cast<const f2x*>(tile + tid * RUN), tile + tid * RUN,
                                    s->rot, s->ct.chip, s->d, a.kp, i0, cnt, acc, &anchors[tid]);
            __syncthreads();
            phase_b_pre<T>(pb, c, s->ct, u0, len);
            phase_b<T>(pb, c, tile, anchors, s->ct, u0, len);
            __syncthreads();
        }
    }
    phase_b_fold<T>(pb, acc);
    warp_partials<V>(acc, s->red, lane, warp);
    __syncthreads();
    if (warp == 0)
        warp0_totals<V>(s->red, s->sums, lane, nwarps);
    __syncthreads();
    if (tid < 2 * T)
        a.tap_sums[(int64_t)j * 2 * T + tid] = s->sums[tid];
    if (tid == 0) {
        l1rxg_nco st = a.states[j];
        advance_nco(st.code_phase_chips, st.carrier_phase_rad, st.chi_chips, c);
        a.states[j] = st;
        a.corr[j] = corr_from_sums<T>(s->sums, a.ke, a.kp, a.kl, n);
    }
}

}  // namespace l1rxg
