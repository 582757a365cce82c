// segcorr.cuh -- the segment correlator: throughput-shape tracking kernel
// over raw complex-int16 rings (sm_100a).
//
// Same contract as track_kernel (correlator.cuh; reference
// tracking.hpp:226-282 correlate + :520-618 track_epoch), a different
// schedule for the many-channel case (BASELINE config 4):
//
//   * the ring keeps the recording's raw cint16 samples (4 B, no decode
//     pass: the K1 ingest is fused into the correlator) in rows of 32
//     samples (128 B), and each work warp pulls its own 32-row units by TMA
//     TENSOR copies with the 128-byte swizzle, double-buffered per warp (no
//     CTA barrier per unit);
//   * lane l owns row l of a unit: a ring-aligned run of 32 consecutive
//     samples, read as eight conflict-free LDS.128 (the swizzle puts the 8
//     lanes of a quarter-warp on 8 different bank groups);
//   * carrier wipe as in track_kernel (per-epoch rotator table e^{-jwj} +
//     a per-run fp64-anchored phasor) with four FFMAs per sample into the
//     run's running sum P, but NO prefix tile: a tap's replica changes at
//     most once inside a run when a chip spans > 32 samples, and the steps
//     of all taps inside one half-run share one position when the taps'
//     residues are > 15 samples apart (config 4: 64 samples per chip,
//     0.25-chip grid), so P is captured in REGISTERS at the static midpoint
//     and at one dynamic position per half, and tap k's run sum is
//         chip_end * P(32) + (chip_start - chip_end) * P(q_k);
//   * every step position q_k is the reference's exact fp64 chip decision
//     (tap_boundary: estimate + exact check), and whatever does not fit the
//     register captures (ties between taps of one residue, more than one
//     step per run at low sample rates, the run holding the n/2 split of
//     the half-epoch prompt) takes an exact per-sample slow path over the
//     same shared-memory row -- correct for every geometry, fast for the
//     one it is chosen for.
//
//   * per epoch: the step table (every transition of every tap located and
//     entered by all threads), the runs, the warps' partial sums, the loop
//     update on warp 0 (warp0_update / loop_fast, shared with track_kernel);
//     the last warp finishes the previous epoch (loop_metrics, record) before
//     its runs -- all warps correlate (the QD variant below locates each
//     run's crossings itself and has no step table);
//   * persistent CTAs (five or six per SM) take work items of 16 epochs of
//     one channel; a chunk waits for its channel's previous chunk, so a
//     launch has no wave-quantisation tail; the channels of one recording
//     are drawn together by CTAs of one warp-slot class (gang tickets,
//     SegArgs) so that they share the recording's samples through L2.
// DESIGN.md section 3 has the measurements behind each choice.
#pragma once

#include <cuda.h>  // CUtensorMap (the map itself is encoded on the host)

#include <type_traits>

#include "correlator.cuh"

namespace l1rxg {

// Defaults (measured, config 4): four correlating warps per CTA and five
// CTAs per SM (44 KB of shared memory each: the unit buffers first at the
// 1024-B aligned dynamic base, no transition-count table) beat five warps x
// four CTAs by 2 %; the QD variant (36 KB, 80 registers) runs six per SM;
// two or three warps per CTA are no gain (profiles/r3g_seg_qd6_fullsize.txt).
#ifndef L1RXG_SEG_NW
#define L1RXG_SEG_NW 4
#endif
#ifndef L1RXG_SEG_PAD
#define L1RXG_SEG_NOPAD
#define L1RXG_SEG_NOCUM
#endif
constexpr int SEG_NW = L1RXG_SEG_NW;         // warps per CTA, all correlate
constexpr int SEG_NT = 32 * SEG_NW;
constexpr int SEG_NBUF = 2;                  // TMA buffers per work warp
#ifndef L1RXG_SEG_FILL_UNR
#define L1RXG_SEG_FILL_UNR 2
#endif
constexpr int SEG_FILL_UNR = L1RXG_SEG_FILL_UNR;  // step-table transitions located per fill iteration
constexpr int SEG_UNIT_BYTES = 32 * 128;     // 32 rows x 32 cint16 samples
constexpr int SEG_MIN_N = 32 * 32 * (SEG_NW - 1) + 1;  // every warp has >= 1 unit per epoch
constexpr int SEG_TRANS_P = 576;             // transitions per code period (<= 544 for C/A codes)
constexpr int SEG_CLASSES = 8;               // CTA classes by warp slot (CTAs per SM, capped)

struct __align__(64) SegArgs {
    TrackArgs t;
    CUtensorMap tmap;  // ring as [stream][row][32 x u32], SWIZZLE_128B, box 32 x 32 x 1
    // persistent CTAs over work items (chunk j, channel c), chunk-major: item
    // (j, c) runs channel c for up to chunk_epochs epochs once item (j-1, c)
    // has finished (ready[c] == j), so a launch has no wave-quantisation tail
    int* next;          // work-item counter (zeroed before the launch)
    int* ready;         // [n_channels] chunks finished (zeroed before the launch)
    int n_items, n_channels, chunk_epochs;
    int fast_geom;      // seg_geometry_ok: unchecked step-table entries away from ties
    int qgrid;          // every tap offset a multiple of 1/4 chip in [-1, 1]: start chips by the LUT
    int qdirect;        // quarter grid + >= 62 samples per chip: per-run crossings, no step table (QD kernel)
    // gang tickets: the warp scheduler favours a CTA by the age of its warp slots (measured: the CTA in
    // slots 0-3 of an SM runs 2.2x faster than the one in slots 16-19, profiles/r3e_seg_item_trace_chunk32.txt),
    // so CTAs are classed by slot and every class takes whole gang-chunks (one chunk of every channel of
    // one stream): siblings run on equally fast CTAs, start together and stay together, and the stream's
    // window is read from DRAM once.  gang_first == nullptr: single queue of (chunk, channel) items.
    const int* gang_first;        // [n_gangs] first channel of the gang
    const int* gang_count;        // [n_gangs] channels of the gang (<= gang_max)
    int n_gangs, gang_max;
    int* cnext;                   // [SEG_CLASSES] per-class sub-item counters (zeroed before the launch)
    int* ctab;                    // [SEG_CLASSES][ctab_stride] gang-chunk of each class ticket (-1: not yet drawn)
    int ctab_stride;
    const uint32_t* chipw;        // [33][CHIP_EXT / 32 + 1] chip bits per PRN (built once per context)
    unsigned long long* trace;    // optional [n_items][3]: globaltimer at item start / end, smid << 32 | warp slot (L1RXG_SEG_TRACE)
};

template <int T>
struct SegEntry {
    typedef typename std::conditional<(3 * T + 10 <= 32), uint32_t, unsigned long long>::type type;
};

template <int T>
struct SegSmem {
    l1rxg_channel ch;
    EpochConsts c;
    double d[T];
    double sums[2 * T + 2];
    float red[SEG_NW * (2 * T + 2)];
    __align__(16) float2 rot[32];
    __align__(16) float2 rotq[32];  // rot transposed by quarter: rotq[4 t + Q] = rot[8 Q + t]
    uint64_t fbar[SEG_NW][SEG_NBUF];  // per work warp: its unit buffers' TMA completion
    struct {                          // per warp: lane 0's unit stream (kept out of registers)
        long long pos;                // ring position of epoch e's first sample
        int e, k, nwu, e_adm;         // next unit: epoch, warp-unit, units of that epoch; admitted epochs
    } q[SEG_NW];
    uint64_t pbar[2];                 // (cluster exchange: unused, csize == 1)
    l1rxg_epoch_record rec;
    int64_t rec_slot;
    int64_t rec_esh;
    double rec_eenv;
    int pending, stop;
    int item, prn_cached;
    double nco_ph1, nco_cp1;
    uint32_t chipw[CHIP_EXT / 32 + 1];  // bit m % 32 of word m / 32: chip[m] > 0
    int16_t tm[SEG_TRANS_P];  // chip index of the g-th chip transition of one period
#ifndef L1RXG_SEG_NOCUM
    int16_t cum[1024];       // transitions at indices <= r within one period
#endif
    int L;                   // transitions per period
    // quarter-grid start chips: bit t of qlut[4 qq + c] = chip of tap t at
    // a run's first sample, for qq = floor(4 frac(ph)) and c = the chips at
    // floor(ph) - 1 .. + 1 (bits 0..2)
    uint8_t qlut[32];
    // step-table entry pieces of a step at run position q: bits 0-7 the
    // capture-position field, bits 8-9 the tap code (q = 0: no entry); tap k's
    // entry is (entq & 0xff) | (entq >> 8) << (10 + 2 k)
    uint16_t entq[32];
    // QD (direct quarter-crossing) kernel: per-epoch constants in quarter-chip
    // units (x 4 is exact) and the crossing LUT: qdlut[4 c4 + qq], c4 = the
    // chips at floor(ph) - 1 .. + 2, qq = floor(4 ph) & 3; bits [0, T) the
    // taps' start chips, [T, 2T) the taps whose chip flips at the run's first
    // quarter crossing, [2T, 3T) at its second
    struct __align__(16) {
        double cps4, base4;  // 4 cps, 4 base: fma(i, cps4, base4) = 4 fl(fma(i, cps, base)) exactly
        double omb, inv4;    // 1 - base4; 1 / cps4 (estimate)
        int ok;              // cps4 <= 2/31: at most two crossings per run, >= 15 samples apart
    } qd;
    uint32_t qdlut[64];
};

// Per-epoch step table, one entry per 32-sample run of the epoch (runs
// counted from the ring row holding the epoch's first sample):
//   bits [0,4)  q0: the first-half capture position (1..15; 0 = none)
//   bits [4,8)  q1 - 16: the second-half capture position (17..31; 0 = none)
//   bits 8, 9:  half 0 / half 1 claimed by two different positions (ties):
//               every tap stepping in that half takes the slow path
//   bits 10+2k..: tap k's step in the run: 0 none, 1 at 16, 2 at q0, 3 at q1
//   bit 10+2T+k: tap k takes the exact slow path in this run (two steps)
// runs per epoch table: every row a unit of the epoch can cover
__host__ __device__ constexpr int seg_table_runs(int n) { return (((n + 62) >> 5) + 31) / 32 * 32; }

template <int T, bool QD = false>
__host__ __device__ constexpr size_t seg_smem_bytes(int n) {
    // header, step table, then up to 1 KB of padding to the 1024-B aligned unit buffers
    // (L1RXG_SEG_NOPAD: the buffers first, at the 1024-B aligned dynamic base)
    return ((sizeof(SegSmem<T>) + 15) & ~size_t(15)) +
           (QD ? size_t(0)
               : ((static_cast<size_t>(seg_table_runs(n)) * sizeof(typename SegEntry<T>::type) + 15) & ~size_t(15))) +
#ifndef L1RXG_SEG_NOPAD
           1024 +
#endif
           static_cast<size_t>(SEG_NW) * SEG_NBUF * SEG_UNIT_BYTES;
}

// 3-D tensor TMA: box {32 u32, 32 rows, 1 stream} at (0, row, stream).
__device__ __forceinline__ void tma_load_rows(uint32_t dst, const CUtensorMap* map, int row, int strm,
                                              uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(row), "r"(strm), "r"(smem_u32(bar))
        : "memory");
}

// floor(v) for 0 <= v < 2^31: v + 1.5 * 2^52 rounded down leaves floor(v)
// in the low word (one DADD, no F2I).  With v = fl(fma(i, cps, base) + d)
// this is the reference's trunc((int64)(ph + d)) chip index exactly.
__device__ __forceinline__ int floor_idx(double v) {
    return __double2loint(__dadd_rd(v, 6755399441055744.0));
}

// cint16 word -> (re, im) exactly, one I2F.S16 per component (the halves
// selected in the instruction; the format's 1/32768 is folded into the
// rotator table, an exact power of two)
#ifdef L1RXG_SEG_I2FP  // experiment switch: full-rate I2FP on the shifted halves (x 65536)
__device__ __forceinline__ float seg_re(uint32_t w) { return (float)(int)(w << 16); }
__device__ __forceinline__ float seg_im(uint32_t w) { return (float)(int)(w & 0xffff0000u); }
constexpr float SEG_CVT_SCALE = 1.f / (32768.f * 65536.f);
#else
__device__ __forceinline__ float seg_re(uint32_t w) { return (float)(short)(w & 0xffffu); }
__device__ __forceinline__ float seg_im(uint32_t w) { return (float)(short)(w >> 16); }
constexpr float SEG_CVT_SCALE = 1.f / 32768.f;
#endif

// Sample j of the run in row `row` of a 128B-swizzled unit buffer.
__device__ __forceinline__ uint32_t seg_sample(const unsigned char* buf, int row, int j) {
    return *reinterpret_cast<const uint32_t*>(buf + row * 128 + ((((j >> 2) ^ row) & 7) << 4) + ((j & 3) << 2));
}

// Exact per-sample slow path: sum over j in [jlo, jhi) of
// chip[idx(i0 + j, d)] * x_j * conj(rot_j) (un-anchored), the reference's
// chip decision per sample.
__device__ __noinline__ float2 seg_slow_sum(const unsigned char* buf, int row, const float2* rot,
                                            const uint32_t* chipw, double d, int i0, int jlo, int jhi,
                                            double cps, double base) {
    float sr = 0.f, si = 0.f;
    for (int j = jlo; j < jhi; ++j) {
        const uint32_t w = seg_sample(buf, row, j);
        const float xr = seg_re(w), xi = seg_im(w);
        const float2 q = rot[j];
        const float yr = fmaf(xi, q.y, xr * q.x);
        const float yi = fmaf(-xr, q.y, xi * q.x);
        const int m = floor_idx(__dadd_rn(__fma_rn((double)(i0 + j), cps, base), d));
        const float ch = ((chipw[m >> 5] >> (m & 31)) & 1u) ? 1.f : -1.f;
        sr = fmaf(ch, yr, sr);
        si = fmaf(ch, yi, si);
    }
    return make_float2(sr, si);
}

// One run (32 samples of row `lane`), fast path: running sum with the
// captures P(16) (static), P(q0) for q0 in [1, 16), P(q1) for q1 in (16, 32).
// MASK: samples outside [jlo, jhi) (epoch edges) count as zero.
//
// The complex MAC is two packed FFMA2 per sample into one (re, im) register
// pair: (re, im) += (xr, xi) * (c, c), then (re, im) += (xi, xr) * (s, -s)
// -- the swapped operand and the one-sided negation are FFMA2 operand
// modifiers (.LO_HI, .NP) and the rotator component a broadcast scalar, so
// no moves; the same two roundings per component as fmaf(xi, s, fmaf(xr, c,
// acc)) (L1RXG_SEG_SCALAR_FMA restores the four scalar FFMAs).
__device__ __forceinline__ float2 seg_mac(float2 acc, float xr, float xi, float c, float s) {
#ifdef L1RXG_SEG_SCALAR_FMA
    return make_float2(fmaf(xi, s, fmaf(xr, c, acc.x)), fmaf(-xr, s, fmaf(xi, c, acc.y)));
#else
    acc = __ffma2_rn(make_float2(xr, xi), make_float2(c, c), acc);
    return __ffma2_rn(make_float2(xi, xr), make_float2(s, -s), acc);
#endif
}

template <bool MASK>
__device__ __forceinline__ void seg_run(const unsigned char* buf, int lane, const float4* rot4, int q0,
                                        int q1, int jlo, int jhi, float2& p16, float2& c0, float2& c1,
                                        float2& tot) {
    // the two halves as two independent chains A (samples 0..15) and B
    // (16..31), interleaved for ILP: P(16 + j) = P(16) + B(j)
    const unsigned char* rowp = buf + lane * 128;
    const int sw = lane & 7;
    float2 A = make_float2(0.f, 0.f), B = make_float2(0.f, 0.f);
    float2 C0 = make_float2(0.f, 0.f), C1 = make_float2(0.f, 0.f);
#ifdef L1RXG_SEG_SPLIT2
    float2 As = C0, Bs = C0, C0s = C0, C1s = C0;
#endif
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) {
        const uint4 wa4 = *reinterpret_cast<const uint4*>(rowp + ((ch ^ sw) << 4));
        const uint4 wb4 = *reinterpret_cast<const uint4*>(rowp + (((ch + 4) ^ sw) << 4));
        const float4 ra = rot4[2 * ch], rb = rot4[2 * ch + 1];
        const float4 rc_ = rot4[2 * ch + 8], rd = rot4[2 * ch + 9];
        const uint32_t wa[4] = {wa4.x, wa4.y, wa4.z, wa4.w};
        const uint32_t wb[4] = {wb4.x, wb4.y, wb4.z, wb4.w};
        const float ac[4] = {ra.x, ra.z, rb.x, rb.z};
        const float as[4] = {ra.y, ra.w, rb.y, rb.w};
        const float bc[4] = {rc_.x, rc_.z, rd.x, rd.z};
        const float bs[4] = {rc_.y, rc_.w, rd.y, rd.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int j = 4 * ch + t;  // A: sample j, B: sample 16 + j
            uint32_t xa = wa[t], xb = wb[t];
            if (MASK) {
                xa = (j >= jlo && j < jhi) ? xa : 0u;
                xb = (j + 16 >= jlo && j + 16 < jhi) ? xb : 0u;
            }
#ifdef L1RXG_SEG_SPLIT2  // experiment: the two FFMA2 of a sample into separate accumulators (ILP)
            if (j > 0 && j == q0) {
                C0 = A;
                C0s = As;
            }
            if (j > 0 && j + 16 == q1) {
                C1 = B;
                C1s = Bs;
            }
            {
                const float xr = seg_re(xa), xi = seg_im(xa), yr = seg_re(xb), yi = seg_im(xb);
                A = __ffma2_rn(make_float2(xr, xi), make_float2(ac[t], ac[t]), A);
                As = __ffma2_rn(make_float2(xi, xr), make_float2(as[t], -as[t]), As);
                B = __ffma2_rn(make_float2(yr, yi), make_float2(bc[t], bc[t]), B);
                Bs = __ffma2_rn(make_float2(yi, yr), make_float2(bs[t], -bs[t]), Bs);
            }
#else
#ifdef L1RXG_SEG_CAP1  // experiment switch: a capture compare at every position
            if (j > 0 && j == q0)
                C0 = A;
            if (j > 0 && j + 16 == q1)
                C1 = B;
#else  // captures at even positions only (the odd ones add their last sample after the run)
            if ((j & 1) == 0 && j > 0 && j == (q0 & ~1))
                C0 = A;
            if ((j & 1) == 0 && j > 0 && j + 16 == (q1 & ~1))
                C1 = B;
#endif
            A = seg_mac(A, seg_re(xa), seg_im(xa), ac[t], as[t]);
            B = seg_mac(B, seg_re(xb), seg_im(xb), bc[t], bs[t]);
#endif
        }
    }
#ifdef L1RXG_SEG_SPLIT2
    A = make_float2(A.x + As.x, A.y + As.y);
    B = make_float2(B.x + Bs.x, B.y + Bs.y);
    C0 = make_float2(C0.x + C0s.x, C0.y + C0s.y);
    C1 = make_float2(C1.x + C1s.x, C1.y + C1s.y);
#endif
#if !defined(L1RXG_SEG_CAP1) && !defined(L1RXG_SEG_SPLIT2)
    {  // odd capture positions: P(q) = P(q - 1) + the rotated sample q - 1 (masked like the run)
        const int ja = (q0 - 1) & 15, jb = 16 + ((q1 - 1) & 15);
        uint32_t xa = seg_sample(buf, lane, ja), xb = seg_sample(buf, lane, jb);
        xa = (q0 & 1) && (!MASK || (ja >= jlo && ja < jhi)) ? xa : 0u;
        xb = (q1 & 1) && (!MASK || (jb >= jlo && jb < jhi)) ? xb : 0u;
        const float4 r2 = rot4[ja >> 1], r3 = rot4[jb >> 1];
        const float ca = (ja & 1) ? r2.z : r2.x, sa = (ja & 1) ? r2.w : r2.y;
        const float cb = (jb & 1) ? r3.z : r3.x, sb = (jb & 1) ? r3.w : r3.y;
        C0 = seg_mac(C0, seg_re(xa), seg_im(xa), ca, sa);
        C1 = seg_mac(C1, seg_re(xb), seg_im(xb), cb, sb);
    }
#endif
    p16 = A;
    c0 = C0;
    c1 = make_float2(A.x + C1.x, A.y + C1.y);
    tot = make_float2(A.x + B.x, A.y + B.y);
}

#ifdef L1RXG_SEG_CHAINS4
// Four independent chains (quarters of the run: samples 8Q + t, t < 8), for
// more ILP; P(q0) = q0 < 8 ? A(q0) : A(8) + B(q0 - 8), likewise in the
// second half.  rotq holds the rotators transposed by quarter so one
// broadcast LDS.128 gives two quarters' rotators for step t.
template <bool MASK>
__device__ __forceinline__ void seg_run4(const unsigned char* buf, int lane, const float4* rq4, int q0,
                                         int q1, int jlo, int jhi, float2& p16, float2& c0, float2& c1,
                                         float2& tot) {
    const unsigned char* rowp = buf + lane * 128;
    const int sw = lane & 7;
    float2 P[4];
#pragma unroll
    for (int Q = 0; Q < 4; ++Q)
        P[Q] = make_float2(0.f, 0.f);
    float2 CA = P[0], CB = P[0], CC = P[0], CD = P[0];
    const int q1r = q1 - 16;
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // chunk h of each quarter: samples 8Q + 4h + u
        uint4 wq[4];
#pragma unroll
        for (int Q = 0; Q < 4; ++Q)
            wq[Q] = *reinterpret_cast<const uint4*>(rowp + (((2 * Q + h) ^ sw) << 4));
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int t = 4 * h + u;
            const float4 r01 = rq4[2 * t], r23 = rq4[2 * t + 1];
            const float rc[4] = {r01.x, r01.z, r23.x, r23.z};
            const float rs[4] = {r01.y, r01.w, r23.y, r23.w};
            // captures before adding step t: A at q0, B at q0 - 8, C at q1 - 16, D at q1 - 24
            if (t > 0 && t == q0) CA = P[0];
            if (t == q0 - 8) CB = P[1];
            if (t > 0 && t == q1r) CC = P[2];
            if (t == q1r - 8) CD = P[3];
#pragma unroll
            for (int Q = 0; Q < 4; ++Q) {
                const uint32_t wv[4] = {wq[Q].x, wq[Q].y, wq[Q].z, wq[Q].w};
                uint32_t x = wv[u];
                const int j = 8 * Q + t;
                if (MASK)
                    x = (j >= jlo && j < jhi) ? x : 0u;
                P[Q] = seg_mac(P[Q], seg_re(x), seg_im(x), rc[Q], rs[Q]);
            }
        }
    }
    const float2 a8 = P[0];
    const float2 h16 = make_float2(a8.x + P[1].x, a8.y + P[1].y);
    const float2 c24 = make_float2(h16.x + P[2].x, h16.y + P[2].y);
    p16 = h16;
    c0 = q0 < 8 ? CA : make_float2(a8.x + CB.x, a8.y + CB.y);
    c1 = q1r < 8 ? make_float2(h16.x + CC.x, h16.y + CC.y) : make_float2(c24.x + CD.x, c24.y + CD.y);
    tot = make_float2(c24.x + P[3].x, c24.y + P[3].y);
}
#endif

// anchored value z * conj(anchor), anchor = (cos, sin) of theta(i0):
// (fma(zr, c, zi s), fma(zi, c, -(zr s))) -- one FMUL2 (swapped operand,
// one-sided negation) and one FFMA2, the same roundings as the scalar form
__device__ __forceinline__ float2 seg_anchor(float2 z, float ca, float sa) {
#ifdef L1RXG_SEG_SCALAR_FMA
    return make_float2(fmaf(z.x, ca, z.y * sa), fmaf(z.y, ca, -(z.x * sa)));
#else
    return __ffma2_rn(z, make_float2(ca, ca), __fmul2_rn(make_float2(z.y, z.x), make_float2(sa, -sa)));
#endif
}

// 2 p - t (the run sum when the chip flips where p was captured)
__device__ __forceinline__ float2 seg_flip(float2 p, float2 t) {
#ifdef L1RXG_SEG_SCALAR_FMA
    return make_float2(fmaf(2.f, p.x, -t.x), fmaf(2.f, p.y, -t.y));
#else
    return __ffma2_rn(p, make_float2(2.f, 2.f), make_float2(-t.x, -t.y));
#endif
}

// Enters the step of tap k at epoch run position pos (= b + lead).  A step
// at a run's first sample needs no entry (the run's start chip has it).
// checked: one atomic OR of the position and the tap's code whose previous
// word tells whether the half already held another position (-> conflict
// bit) or the tap already stepped in this run (-> its slow bit).  Unchecked
// (a fire-and-forget RED): for steps located away from fp64 ties when the
// geometry rules both out (taps' residues > 15.5 samples apart, > 33 samples
// per chip: steps of different residues are >= 15 samples apart, steps of
// one residue coincide exactly, one tap steps at most once per run).
template <int T>
__device__ __forceinline__ void seg_enter(typename SegEntry<T>::type* tab, int pos, int k, bool checked) {
    typedef typename SegEntry<T>::type E;
    const int r = pos >> 5, q = pos & 31;
    if (q == 0)
        return;
    const int sh = 10 + 2 * k;
    const int h = q >> 4 & (q != 16);  // half 1 for q in 17..31
    const bool mid = q == 16;
    const E qf = mid ? 0 : (E)(q & 15) << (4 * h);
    const E code = mid ? 1 : 2 + h;
    if (!checked) {
        atomicOr(&tab[r], qf | (code << sh));  // result unused: RED
        return;
    }
    const E prev = atomicOr(&tab[r], qf | (code << sh));
    const int pf = (int)((prev >> (4 * h)) & 15);
    const bool conflict = !mid && pf != 0 && pf != (q & 15);
    const bool twice = ((prev >> sh) & 3) != 0;
    if (conflict || twice)  // rare: ties, or two steps of one tap at low sample rates
        atomicOr(&tab[r], (conflict ? (E)1 << (8 + h) : (E)0) | (twice ? (E)1 << (10 + 2 * T + k) : (E)0));
}

// transitions of the PRN's code at chip indices <= m (CodeTables' trans_count)
template <int T>
__device__ __forceinline__ int seg_trans_count(const SegSmem<T>* s, int m) {
    const int p = m / 1023;
#ifdef L1RXG_SEG_NOCUM  // upper bound of r in tm[0, L) by binary search
    const int r = m - p * 1023;
    int lo = 0, hi = s->L;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (s->tm[mid] <= r)
            lo = mid + 1;
        else
            hi = mid;
    }
    return p * s->L + lo;
#else
    return p * s->L + s->cum[m - p * 1023];
#endif
}

// Step table fill for one epoch (every thread, after the loop update): every
// chip transition of every tap with its step inside the epoch, located
// exactly, entered in the run holding it (seg_enter).  The (tap, transition)
// pairs are flattened so every thread gets the same share; transition g of
// the code is chip index p * 1023 + tm[g - p * L].  Each step's estimate
// e = (m - d - base) / cps is within ~1e-10 samples of the reference's
// crossing, so away from ties ceil(e) is the answer (a round-up add of
// 1.5 * 2^52); near one the reference expression decides (tap_boundary);
// entries within 1e-7 samples of a tie are checked.
template <int T>
__device__ __forceinline__ void seg_fill(typename SegEntry<T>::type* tab, const SegSmem<T>* s,
                                        const EpochConsts& c, int lead, int tid, int nthr, bool fast_geom) {
    const int n = c.n, L = s->L;
    const int lane = tid & 31;
    // each warp: lane k < T computes tap k's transition range, all lanes get them
    int g0k = 0, cntk = 0;
    if (lane < T) {
        const double dk = s->d[lane];
        g0k = seg_trans_count(s, tap_index(0, c.cps, c.base, dk));  // transitions in (idx(0), idx(n-1)]
        cntk = seg_trans_count(s, tap_index(n - 1, c.cps, c.base, dk)) - g0k;
    }
    const float inv_L = 1.f / (float)L;  // p = g / L exactly for g < 2^13 (the +0.5 keeps off integers)
#ifdef L1RXG_SEG_FILL_FLAT  // experiment switch: one flattened loop decoding (tap, transition)
    int g0[T], pre[T + 1];
    pre[0] = 0;
#pragma unroll
    for (int k = 0; k < T; ++k) {
        g0[k] = __shfl_sync(0xffffffffu, g0k, k);
        pre[k + 1] = pre[k] + __shfl_sync(0xffffffffu, cntk, k);
    }
    for (int f = tid; f < pre[T]; f += nthr) {
        int k = 0, g = 0;
#pragma unroll
        for (int j = 0; j < T; ++j)
            if (f >= pre[j]) {
                k = j;
                g = g0[j] + (f - pre[j]);
            }
        const int p = (int)(((float)g + 0.5f) * inv_L);
        const int m = p * 1023 + s->tm[g - p * L];
        const double dk = s->d[k];
        const double e = ((double)m + (-dk - c.base)) * c.inv_cps;
        const double dist = fabs(e - rint(e));
        const bool tie = !(dist > 1e-9);
        const int b = tie ? tap_boundary(m, dk, c, 1, n - 1) : __double2loint(__dadd_ru(e, 6755399441055744.0));
        seg_enter<T>(tab, b + lead, k, !(dist > 1e-7) || !fast_geom);
    }
#else
    // one loop per tap (k a compile-time constant inside: no (tap,
    // transition) decode, constant entry shifts), started where the
    // flattened order would put it (thread (pre_k + i) mod nthr takes
    // transition i of tap k) so every thread keeps the same share
    int pre = 0;
#pragma unroll 1  // unrolled (k constant) it ran 5 % fewer instructions but missed the instruction cache
    for (int k = 0; k < T; ++k) {
        const int g0 = __shfl_sync(0xffffffffu, g0k, k);
        const int cnt = __shfl_sync(0xffffffffu, cntk, k);
        const double dk = s->d[k];
        const double off = -dk - c.base;
        int i = tid - pre % nthr;
        if (i < 0)
            i += nthr;
        pre += cnt;
        // transition g = g0 + i is chip p * 1023 + tm[gp], gp = g - p * L,
        // advanced incrementally (nthr < L: at most one period per step)
        int p = (int)(((float)(g0 + i) + 0.5f) * inv_L);
        int gp = g0 + i - p * L;
#ifndef L1RXG_SEG_FILL_SERIAL
        // SEG_FILL_UNR transitions per iteration: the fp64 locate chains
        // (LDS -> I2F.F64 -> DADD -> DMUL -> FRND -> DADD) of different
        // transitions are independent, so they overlap instead of running
        // back to back
        for (; i < cnt; i += SEG_FILL_UNR * nthr) {
            int m[SEG_FILL_UNR];
            bool has[SEG_FILL_UNR];
#pragma unroll
            for (int u = 0; u < SEG_FILL_UNR; ++u) {
                has[u] = i + u * nthr < cnt;
                m[u] = p * 1023 + s->tm[gp];  // gp < L always: in bounds even past cnt
                gp += nthr;
                if (gp >= L) {
                    gp -= L;
                    ++p;
                }
            }
            double dist[SEG_FILL_UNR];
            int b[SEG_FILL_UNR];
#pragma unroll
            for (int u = 0; u < SEG_FILL_UNR; ++u) {
                const double e = ((double)m[u] + off) * c.inv_cps;
                dist[u] = fabs(e - rint(e));
                b[u] = __double2loint(__dadd_ru(e, 6755399441055744.0));
            }
#pragma unroll
            for (int u = 0; u < SEG_FILL_UNR; ++u) {
                if (!has[u])
                    break;
                if (!(dist[u] > 1e-9))  // a tie: the reference expression decides
                    b[u] = tap_boundary(m[u], dk, c, 1, n - 1);
                // checked within 1e-7 of a tie: steps of one residue differ in e by
                // ~1e-11, so a step near a tie and its partner are both checked
                const int pos = b[u] + lead;
                if (!(dist[u] > 1e-7) || !fast_geom)
                    seg_enter<T>(tab, pos, k, true);
                else if (pos & 31) {
                    typedef typename SegEntry<T>::type E;
                    const uint32_t eq = s->entq[pos & 31];
                    atomicOr(&tab[pos >> 5], (E)(eq & 0xffu) | ((E)(eq >> 8) << (10 + 2 * k)));  // result unused: RED
                }
            }
        }
#else
        for (; i < cnt; i += nthr) {
            const int m = p * 1023 + s->tm[gp];
            const double e = ((double)m + off) * c.inv_cps;
            const double dist = fabs(e - rint(e));
            const bool tie = !(dist > 1e-9);
            const int b = tie ? tap_boundary(m, dk, c, 1, n - 1) : __double2loint(__dadd_ru(e, 6755399441055744.0));
            // checked within 1e-7 of a tie: steps of one residue differ in e by
            // ~1e-11, so a step near a tie and its partner are both checked
            const int pos = b + lead;
            if (!(dist > 1e-7) || !fast_geom)
                seg_enter<T>(tab, pos, k, true);
            else if (pos & 31) {
                typedef typename SegEntry<T>::type E;
                const uint32_t eq = s->entq[pos & 31];
                atomicOr(&tab[pos >> 5], (E)(eq & 0xffu) | ((E)(eq >> 8) << (10 + 2 * k)));  // result unused: RED
            }
            gp += nthr;
            if (gp >= L) {
                gp -= L;
                ++p;
            }
        }
#endif
    }
#endif
}

#ifndef L1RXG_SEG_MINB
#define L1RXG_SEG_MINB (SEG_NW == 4 ? 5 : 4)
#endif  // (CTAs per SM the registers are budgeted for)
#ifndef L1RXG_SEG_MINB_QD
#define L1RXG_SEG_MINB_QD (SEG_NW == 4 ? 6 : L1RXG_SEG_MINB)  // QD, 4 warps: 80 registers, six CTAs per SM (+2 %, profiles/r3g)
#endif
// QD = true: the direct quarter-crossing variant (sa.qdirect).  Every tap
// offset is k/4 chip, so fl(ph + d_t) = ph + d_t and every replica step of
// every tap happens where 4 ph(i) = fma(i, 4 cps, 4 base) crosses an integer;
// with >= 62 samples per chip a 32-sample run holds at most two such
// crossings, >= 15 samples apart (never two in one half-run).  Each run
// locates its own crossings (fp64 estimate; within 2^-28 samples of a tie
// the whole run takes the exact per-sample path) and a 64-entry LUT gives
// the taps' start chips and which taps flip at each crossing from the four
// chips around floor(ph): no per-epoch step table, no fill, one barrier
// fewer per epoch, 8 KB less shared memory.  Same captures and the same
// arithmetic as the table path: records are byte-identical away from ties.
template <int T, bool QD = false>
__global__ void __launch_bounds__(SEG_NT, QD ? L1RXG_SEG_MINB_QD : L1RXG_SEG_MINB)
    track_seg_kernel(const __grid_constant__ SegArgs sa) {
    typedef typename SegEntry<T>::type E;
    static_assert(!QD || 3 * T <= 32, "QD packs three T-bit fields into one LUT word");
    const TrackArgs& a = sa.t;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int n = a.n;
    const uint32_t sbase = smem_u32(smem_raw);
    const int truns = QD ? 0 : seg_table_runs(n);
#ifdef L1RXG_SEG_NOPAD
    if (sbase & 1023u)
        __trap();  // the unit buffers need the 1024-B alignment of the 128-B swizzle
    const uint32_t boff = 0;
    const uint32_t hoff = (uint32_t)(SEG_NW * SEG_NBUF * SEG_UNIT_BYTES);
#else
    const uint32_t hoff = 0;
#endif
    SegSmem<T>* s = reinterpret_cast<SegSmem<T>*>(smem_raw + hoff);
    const uint32_t hdr = hoff + (uint32_t)((sizeof(SegSmem<T>) + 15) & ~size_t(15));
    E* tab = reinterpret_cast<E*>(smem_raw + hdr);
#ifndef L1RXG_SEG_NOPAD
    const uint32_t tend = hdr + (uint32_t)((truns * sizeof(E) + 15) & ~size_t(15));
    const uint32_t boff = ((sbase + tend + 1023u) & ~1023u) - sbase;  // unit buffers, 1024-B aligned
#endif
    const float4* rot4 = reinterpret_cast<const float4*>(s->rot);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ctl = SEG_NW - 1;  // also finishes each epoch (metrics, record) before its runs
    constexpr int V = 2 * T + 2;
    const int nh = n / 2;
    const bool noop = a.lc.kernel == L1RXG_KERNEL_NOOP;
    const int64_t R = a.ring_cap;  // multiple of 32
    const float scale = SEG_CVT_SCALE;

    if (tid == 0) {
        for (int w = 0; w < SEG_NW; ++w)
            for (int b = 0; b < SEG_NBUF; ++b)
                mbar_init(&s->fbar[w][b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        s->prn_cached = -1;
    }
    for (int k = tid; k < T; k += blockDim.x)
        s->d[k] = a.taps.offsets_chips[k];
    if (tid < 32) {  // quarter-grid LUT (used when sa.qgrid): floor(ph + d_t) = floor(ph) + ((qq + 4 d_t) >> 2)
        const int qq = tid >> 3, c3 = tid & 7;  // c3 bit 0, 1, 2: the chips at floor(ph) - 1, 0, + 1
        uint32_t pat = 0;
        for (int t = 0; t < T; ++t) {
            const int D = (int)rint(a.taps.offsets_chips[t] * 4.0);
            pat |= ((uint32_t)(c3 >> (1 + ((qq + D) >> 2))) & 1u) << t;
        }
        s->qlut[tid] = (uint8_t)pat;
    }
    if (tid < 32) {  // step-table entry pieces by position (seg_enter's fields)
        const int q = tid;
        const int h = q >> 4 & (q != 16);
        const bool mid = q == 16;
        const uint32_t qf = mid ? 0u : (uint32_t)(q & 15) << (4 * h);
        const uint32_t code = mid ? 1u : 2u + (uint32_t)h;
        s->entq[q] = q == 0 ? (uint16_t)0 : (uint16_t)(qf | (code << 8));
    }
    for (int r = tid; r < truns; r += blockDim.x)
        tab[r] = 0;  // every later epoch leaves the table clean (owners clear their entries)
    if (QD && tid < 64) {  // crossing LUT: chip index of tap t at quarter K = 4 m + qq is m + ((qq + D_t) >> 2)
        const int qq = tid & 3, c4 = tid >> 2;  // c4 bit b: the chip at m - 1 + b
        uint32_t pat = 0;
        for (int t = 0; t < T; ++t) {
            const int D = (int)rint(a.taps.offsets_chips[t] * 4.0);
            const int s0 = (qq + D) >> 2, s1 = (qq + 1 + D) >> 2, s2 = (qq + 2 + D) >> 2;  // -1 .. 2
            const uint32_t b0 = (c4 >> (s0 + 1)) & 1u, b1 = (c4 >> (s1 + 1)) & 1u, b2 = (c4 >> (s2 + 1)) & 1u;
            pat |= b0 << t | (b0 ^ b1) << (T + t) | (b1 ^ b2) << (2 * T + t);
        }
        s->qdlut[tid] = pat;
    }
    // per-warp TMA unit counters: persistent across work items (every item
    // waits for its last copies, so the mbarrier parities continue)
    int issued = 0, consumed = 0;

    for (;;) {
        // ---- next work item
        if (tid == 0) {
            if (sa.gang_first) {
                unsigned wslot;
                asm volatile("mov.u32 %0, %%warpid;" : "=r"(wslot));
                const int k = min((int)(wslot / SEG_NW), SEG_CLASSES - 1);
                const int n_gc = sa.n_items / sa.n_channels * sa.n_gangs;  // gang-chunks of the launch
                int item = sa.n_items;
                for (;;) {
                    const int i = atomicAdd(&sa.cnext[k], 1);
                    const int ticket = i / sa.gang_max, member = i - ticket * sa.gang_max;
                    if (ticket >= sa.ctab_stride)  // (cannot happen: one spare ticket per CTA of the grid)
                        break;
                    volatile int* slot = sa.ctab + (size_t)k * sa.ctab_stride + ticket;
                    int g;
                    if (member == 0) {  // first of its ticket: draws the class's next gang-chunk
                        g = atomicAdd(sa.next, 1);
                        *slot = g;
                    } else {
                        // (published right after its drawer's atomicAdd; bounded so that a broken
                        // invariant ends this CTA -- and is reported by the chunk-order wait -- instead
                        // of hanging the GPU)
                        long long spins = 0;
                        while ((g = *slot) < 0 && ++spins < (1LL << 22))
                            __nanosleep(100);
                        if (g < 0)
                            break;
                    }
                    if (g >= n_gc)
                        break;
                    const int gang = g % sa.n_gangs;
                    if (member >= sa.gang_count[gang])
                        continue;
                    item = (g / sa.n_gangs) * sa.n_channels + sa.gang_first[gang] + member;
                    break;
                }
                s->item = item;
            } else {
                s->item = atomicAdd(sa.next, 1);
            }
        }
        __syncthreads();
        const int item = s->item;
        if (item >= sa.n_items)
            break;
        const int cidx = item % sa.n_channels;
        const int chunk = item / sa.n_channels;
        const int max_e = min(sa.chunk_epochs, a.max_epochs - chunk * sa.chunk_epochs);
        if (tid == 0) {
            s->stop = 0;
            if (chunk > 0) {  // the channel's previous chunk (dequeued earlier, so resident) must be done
                // bounded (~20 s): a broken invariant reports an error instead of hanging the GPU
                long long spins = 0;
                while (*(volatile int*)&sa.ready[cidx] < chunk && ++spins < (1LL << 23))
                    __nanosleep(2000);
                if (spins >= (1LL << 23)) {
                    a.status[cidx] = 2;
                    s->stop = 1;
                }
                __threadfence();
            }
            s->pending = 0;
            if (sa.trace) {
                unsigned long long tn;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
                sa.trace[3 * (size_t)item] = tn;
                unsigned smid, wid;
                asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
                sa.trace[3 * (size_t)item + 2] = ((unsigned long long)smid << 32) | wid;
            }
        }
        __syncthreads();  // (orders the ready wait before every thread's loads)
        {   // state written by another SM: read around L1, every thread a share
            const unsigned long long* src = reinterpret_cast<const unsigned long long*>(a.chans + cidx);
            unsigned long long* dst = reinterpret_cast<unsigned long long*>(&s->ch);
            for (int q = tid; q < (int)(sizeof(l1rxg_channel) / 8); q += blockDim.x)
                dst[q] = __ldcg(src + q);
        }
        __syncthreads();
        if (max_e <= 0 || s->stop) {  // past the launch's epoch budget (or the wait gave up)
            __syncthreads();
            if (tid == 0)
                atomicExch(&sa.ready[cidx], chunk + 1);
            continue;
        }
        const int strm = a.chan_stream[cidx];
        const int64_t avail = a.avail[strm];
        const int64_t off0 = s->ch.sample_offset_next_epoch;
        if (s->prn_cached != s->ch.prn) {  // the PRN's chip bits and transition list
            // stage the code in the (drained) unit buffers; the chip bits come from the context's table
            int8_t* cc = reinterpret_cast<int8_t*>(smem_raw + boff);
            for (int j = tid; j < 1023; j += blockDim.x)
                cc[j] = a.codes[s->ch.prn * 1023 + j];
            for (int q = tid; q <= CHIP_EXT / 32; q += blockDim.x)
                s->chipw[q] = sa.chipw[s->ch.prn * (CHIP_EXT / 32 + 1) + q];
            __syncthreads();
            if (warp == ctl) {  // ballot-scan of the code's transitions
                int running = 0;
                for (int base = 0; base < 1023; base += 32) {
                    const int r = base + lane;
                    const bool t = r < 1023 && cc[r] != cc[(r + 1022) % 1023];
                    const unsigned mask = __ballot_sync(0xffffffffu, t);
                    const int before = __popc(mask & ((1u << lane) - 1u));
                    if (r < 1023) {
                        if (t)
                            s->tm[running + before] = (int16_t)r;
#ifndef L1RXG_SEG_NOCUM
                        s->cum[r] = (int16_t)(running + before + (t ? 1 : 0));
#endif
                    }
                    running += __popc(mask);
                }
                if (lane == 0) {
                    s->L = running;
                    s->prn_cached = s->ch.prn;
                }
            }
            __syncthreads();  // the staging area is a unit buffer again
        }
        if (tid == 0) {
            const l1rxg_channel& ch = s->ch;
            make_consts(s->c, ch.code_phase_chips, ch.code_freq_hz, ch.carrier_doppler_hz,
                        ch.carrier_phase_rad, a.lc.fs, n);
            s->c.inv_cps = fast_rcp(s->c.cps);  // tap_boundary's estimate
            if (QD) {
                s->qd.cps4 = 4.0 * s->c.cps;
                s->qd.base4 = 4.0 * s->c.base;
                s->qd.omb = 1.0 - 4.0 * s->c.base;
                s->qd.inv4 = 0.25 * s->c.inv_cps;
                s->qd.ok = s->c.cps > 0.0 && 4.0 * s->c.cps <= 2.0 / 31.0;
            }
        }
        __syncthreads();
        if (tid < 32) {
            float sn, co;
            sincosf((float)(s->c.w * (double)tid), &sn, &co);
            s->rot[tid] = make_float2(co * scale, sn * scale);
            s->rotq[(tid & 7) * 4 + (tid >> 3)] = make_float2(co * scale, sn * scale);
        }
        // ---- per-work-warp unit stream (uniform across the warp's lanes) ----
        // unit = (epoch ie, warp-unit ik): rows [32 ik, 32 ik + 32) of epoch ie,
        // rows counted from the ring row holding the epoch's first sample
        // epochs whose windows are ingested and still in the ring
        if (lane == 0 && warp < SEG_NW) {
            int e_adm = 0;
            if (!noop && off0 >= 0 && off0 >= avail - R && off0 + n <= avail)
                e_adm = (int)min((int64_t)max_e, (avail - off0 - n) / n + 1);
            const long long pos = e_adm > 0 ? off0 % R : 0;
            s->q[warp].pos = pos;
            s->q[warp].e = 0;
            s->q[warp].k = warp;
            s->q[warp].nwu = (((((int)(pos & 31)) + n + 31) >> 5) + 31) >> 5;
            s->q[warp].e_adm = e_adm;
        }
        // lane 0 issues the warp's next unit (if admitted) and advances its
        // stream; the warp learns whether a copy was issued
        auto issue_one = [&]() -> bool {
            int ok = 0;
            if (lane == 0) {
                auto& Q = s->q[warp];
                if (Q.e < Q.e_adm) {
                    const int b = issued & (SEG_NBUF - 1);
                    uint64_t* bar = &s->fbar[warp][b];
                    mbar_expect_tx(bar, SEG_UNIT_BYTES);
                    tma_load_rows(sbase + boff + (uint32_t)((warp * SEG_NBUF + b) * SEG_UNIT_BYTES), &sa.tmap,
                                  (int)(Q.pos >> 5) + 32 * Q.k, strm, bar);
                    Q.k += SEG_NW;
                    if (Q.k >= Q.nwu) {
                        ++Q.e;
                        Q.k = warp;
                        Q.pos += n;
                        if (Q.pos >= R)
                            Q.pos -= R;
                        Q.nwu = (((((int)(Q.pos & 31)) + n + 31) >> 5) + 31) >> 5;
                    }
                    ok = 1;
                }
            }
            ok = __shfl_sync(0xffffffffu, ok, 0);
            issued += ok;
            return ok != 0;
        };
        if (warp < SEG_NW)
            while (issued < consumed + SEG_NBUF && issue_one()) {
            }
        __syncthreads();

        int e = 0;
        int64_t done = (int64_t)__ldcg(reinterpret_cast<const unsigned long long*>(a.ecount + cidx));
        int rec_i = (int)(done % a.max_records);
        for (;;) {
            const int64_t off = s->ch.sample_offset_next_epoch;
            if (s->ch.state == L1RXG_IDLE || e >= max_e || off + n > avail)
                break;
            if (off < avail - R || off < 0) {  // window already overwritten
                if (tid == 0)
                    a.status[cidx] = 1;
                break;
            }
            // the epoch's NCO constants stay in shared memory (s->c, unchanged
            // until the loop update) rather than in registers across the runs
            const EpochConsts& c = s->c;
            // the step table of this epoch: every thread (the control warp too)
            if (!QD && !noop) {
                seg_fill<T>(tab, s, c, (int)(off & 31), tid, SEG_NT, sa.fast_geom != 0);
                __syncthreads();
            }
            if (warp == ctl) {
                const EpochConsts cc = s->c;
                nco_advance_lanes(s->nco_ph1, s->nco_cp1, cc, s->ch, lane);
                if (s->pending) {
                    finish_epoch<T>(s, a, lane, true);
                    if (lane == 0)
                        s->pending = 0;
                }
            }
            float acc[V];
    #pragma unroll
            for (int v = 0; v < V; ++v)
                acc[v] = 0.f;
            if (warp < SEG_NW) {
                const int lead = (int)(off & 31);
                const int nwu = (((lead + n + 31) >> 5) + 31) >> 5;
                bool snapped = false;
                float hr = 0.f, hi = 0.f;  // first-half prompt (tracking.hpp:265-271)
                const bool qd_ok = !QD || s->qd.ok != 0;
                for (int k = warp; k < nwu && !noop; k += SEG_NW) {
                    const int r = 32 * k + lane;  // the lane's run: epoch run index
                    const int i0 = 32 * r - lead;  // epoch index of its first sample
                    const int jlo = max(0, -i0);
                    const int jhi = max(jlo, min(32, n - i0));
                    E w = 0;
                    uint32_t slow = 0, spat = 0;
                    // QD: crossing positions x1 < x2 (run positions, >= jlo + 1), the LUT word and
                    // whether the run takes the exact per-sample path for every tap
                    int x1 = 0, x2 = 0;
                    bool slow_all = false;
                    if constexpr (QD) {
                        // 4 ph at the run's first counted sample, its floor K0 (quarter index), and
                        // the samples where 4 ph reaches K0 + 1 and K0 + 2: e = (K - base4) / cps4.
                        // z = e + 1.5 * 2^20 holds floor(e) in the high word's low 20 bits and
                        // frac(e) * 2^32 in the low word; the first sample at or past the crossing
                        // is floor(e) + 1 unless e is within 2^-28 of an integer (a tie: the
                        // reference's own rounding decides, so the run goes per-sample)
                        const double q4 = __fma_rn((double)(i0 + jlo), s->qd.cps4, s->qd.base4);
                        const double rk = __dadd_rd(q4, 6755399441055744.0);
                        const int K0 = __double2loint(rk);
                        const double inv4 = s->qd.inv4;
                        const double e1 = __dmul_rn(__dadd_rn(__dsub_rn(rk, 6755399441055744.0), s->qd.omb), inv4);
                        const double z1 = __dadd_rn(e1, 1572864.0);
                        const double z2 = __dadd_rn(z1, inv4);
                        x1 = (__double2hiint(z1) & 0xfffff) - 0x7ffff - i0;
                        x2 = (__double2hiint(z2) & 0xfffff) - 0x7ffff - i0;
                        slow_all = (uint32_t)__double2loint(z1) + 16u < 32u || (uint32_t)__double2loint(z2) + 16u < 32u ||
                                   (x1 >= 16 && x2 <= 31) || !qd_ok;
                        const int m0 = (K0 >> 2) - 2;
                        const uint32_t win = __funnelshift_r(s->chipw[m0 >> 5], s->chipw[(m0 >> 5) + 1], m0 & 31);
                        spat = s->qdlut[((win >> 1) & 15u) * 4u + (uint32_t)(K0 & 3)];
                        // a crossing past the run's last sample flips nothing here
                        if (x1 > 31)
                            spat &= ~(((1u << T) - 1u) << T);
                        if (x2 > 31)
                            spat &= ~(((1u << T) - 1u) << (2 * T));
                    } else {
                        w = tab[r];
                        tab[r] = 0;  // clean for the next epoch (each entry is read once, by its owner)
                        slow = (uint32_t)(w >> (10 + 2 * T)) & ((1u << T) - 1u);
                        if (w & 0x300u) {  // a half with two positions: its steppers take the slow path
        #pragma unroll
                            for (int t = 0; t < T; ++t) {
                                const int code = (int)(w >> (10 + 2 * t)) & 3;
                                if ((code == 2 && (w & 0x100u)) || (code == 3 && (w & 0x200u)))
                                    slow |= 1u << t;
                            }
                        }
                        // start chips of the taps (the reference's chip index at i0)
                        // (the first run of an epoch starts before sample 0: its
                        // start chip is the one at the first sample it counts)
                        const double phs = __fma_rn((double)(i0 + jlo), c.cps, c.base);
                        // |d| <= 1 chip: every tap's index is in [m0, m0 + 4]; the
                        // 32 chip bits from m0 hold them all
                        const int m0 = floor_idx(phs) - 2;
                        const uint32_t win = __funnelshift_r(s->chipw[m0 >> 5], s->chipw[(m0 >> 5) + 1], m0 & 31);
                        // start chips of the taps as bits of `spat` (bit t: the chip of
                        // tap t at the run's first sample, floor(fl(ph + d_t)))
                        spat = 0;
                        bool exact = !sa.qgrid;
                        if (!exact) {
                            // quarter grid: fl(ph + d_t) = ph + d_t exactly (both are
                            // multiples of ulp(ph) < 2^-40), so floor(ph + d_t) =
                            // floor(ph) + ((qq + 4 d_t) >> 2), qq = floor(4 frac(ph)); the
                            // fraction goes to fp32 rounding toward zero (qq exact); within
                            // 1e-6 of a quarter (or of a binade edge) the exact path decides
                            const double fl = __dsub_rn(__dadd_rd(phs, 6755399441055744.0), 6755399441055744.0);
                            const float f4 = __double2float_rz(__dsub_rn(phs, fl)) * 4.f;
                            const int qq = (int)f4;
                            exact = f4 - (float)qq < 1e-6f || (float)(qq + 1) - f4 < 1e-6f;
                            spat = s->qlut[qq * 8 + ((win >> 1) & 7)];
                        }
                        if (exact) {
                            spat = 0;
                            for (int t = 0; t < T; ++t) {
                                const int ms = floor_idx(__dadd_rn(phs, s->d[t]));
                                spat |= ((win >> (ms - m0)) & 1u) << t;
                            }
                        }
                    }
                    // start chip of tap t: its bit moved to bit 31, then +1.0f / -1.0f
                    auto start_chip = [&](int t) -> float {
                        return __uint_as_float(((spat << (31 - t)) & 0x80000000u) ^ 0xBF800000u);
                    };
                    // run anchor e^{-j theta(i0)}, theta as the reference (fma(w, i, phi))
                    const double th = __fma_rn(c.w, (double)i0, c.phi);
                    const double rr = fma(-rint(th * (1.0 / TWO_PI_D)), TWO_PI_D, th);
                    float sa_, ca_;
                    __sincosf((float)rr, &sa_, &ca_);
                    // half-epoch prompt: snapshot of the prompt tap before the
                    // first run that reaches past n/2 (a thread's runs ascend)
                    if (!snapped && i0 + 32 > nh) {
                        snapped = true;
                        // the prompt tap's sums by a weighted sum, not an
                        // index (a dynamic index would put acc in local memory)
                        hr = hi = 0.f;
    #pragma unroll
                        for (int t = 0; t < T; ++t) {
                            const float m = t == a.kp ? 1.f : 0.f;
                            hr = fmaf(m, acc[2 * t], hr);
                            hi = fmaf(m, acc[2 * t + 1], hi);
                        }
                    }
                    // ---- the unit's samples
                    const int b = consumed & (SEG_NBUF - 1);
                    mbar_wait(&s->fbar[warp][b], (uint32_t)((consumed / SEG_NBUF) & 1));
                    const unsigned char* buf = smem_raw + boff + (warp * SEG_NBUF + b) * SEG_UNIT_BYTES;
                    float2 p16, pc0, pc1, tot;
                    // capture positions: first half (1..15), second half (17..31), 0 = none.  QD: the
                    // first crossing in the first half (case A; the second one is then in 16..32), or
                    // no crossing before 16 (the first one takes the second-half capture; position 16
                    // is C1 = 0, i.e. P(16))
                    const bool caseA = QD && x1 <= 15;
                    const int qb = caseA ? x2 : x1;
                    const int q0 = QD ? (caseA ? x1 : 0) : (int)(w & 15);
                    const int q1 = QD ? ((qb >= 17 && qb <= 31) ? qb : 0) : ((w & 0xf0u) ? (int)((w >> 4) & 15) + 16 : 0);
    #ifdef L1RXG_SEG_CHAINS4
                    const float4* rq4 = reinterpret_cast<const float4*>(s->rotq);
                    if (__all_sync(0xffffffffu, jlo == 0 && jhi == 32))
                        seg_run4<false>(buf, lane, rq4, q0, q1, 0, 32, p16, pc0, pc1, tot);
                    else
                        seg_run4<true>(buf, lane, rq4, q0, q1, jlo, jhi, p16, pc0, pc1, tot);
    #else
                    if (__all_sync(0xffffffffu, jlo == 0 && jhi == 32))
                        seg_run<false>(buf, lane, rot4, q0, q1, 0, 32, p16, pc0, pc1, tot);
                    else
                        seg_run<true>(buf, lane, rot4, q0, q1, jlo, jhi, p16, pc0, pc1, tot);
    #endif
                    float2 v0, v1, v2, v3;
                    if constexpr (QD) {
                        // V0 = P(32) (no step); V1 / V2 = the chip flips at the first / second crossing
                        v0 = seg_anchor(tot, ca_, sa_);
                        const float2 w1 = caseA ? pc0 : pc1;
                        v1 = seg_anchor(seg_flip(w1, tot), ca_, sa_);
                        v2 = seg_anchor(seg_flip(pc1, tot), ca_, sa_);
                        v3 = v2;
                        if (slow_all) {  // exact per-sample sums of every tap; the fast combine adds zeros
#pragma unroll 1
                            for (int t = 0; t < T; ++t) {
                                const float2 z = seg_anchor(
                                    seg_slow_sum(buf, lane, s->rot, s->chipw, s->d[t], i0, jlo, jhi, c.cps, c.base),
                                    ca_, sa_);
#pragma unroll
                                for (int u = 0; u < T; ++u) {  // (no dynamic index into acc)
                                    acc[2 * u] += u == t ? z.x : 0.f;
                                    acc[2 * u + 1] += u == t ? z.y : 0.f;
                                }
                            }
                            v0 = v1 = v2 = make_float2(0.f, 0.f);
                        }
                    } else {
                        // tap k's run sum is start_chip * V[code_k]: V0 = P(32) (no step),
                        // V_s = P(q_s) - (P(32) - P(q_s)) (the chip flips at q_s)
                        v0 = seg_anchor(tot, ca_, sa_);
                        v1 = seg_anchor(seg_flip(p16, tot), ca_, sa_);
                        v2 = seg_anchor(seg_flip(pc0, tot), ca_, sa_);
                        v3 = seg_anchor(seg_flip(pc1, tot), ca_, sa_);
                        if (slow) {  // exact per-sample sums replace the fast ones
        #pragma unroll
                            for (int t = 0; t < T; ++t)
                                if ((slow >> t) & 1u) {
                                    const int code = (int)(w >> (10 + 2 * t)) & 3;
                                    const float2 v = code == 0 ? v0 : (code == 1 ? v1 : (code == 2 ? v2 : v3));
                                    const float2 z = seg_anchor(
                                        seg_slow_sum(buf, lane, s->rot, s->chipw, s->d[t], i0, jlo, jhi, c.cps, c.base),
                                        ca_, sa_);
                                    const float cs = start_chip(t);
                                    acc[2 * t] += fmaf(-cs, v.x, z.x);
                                    acc[2 * t + 1] += fmaf(-cs, v.y, z.y);
                                }
                        }
                    }
                    if (i0 < nh && i0 + 32 > nh) {  // the run holding the n/2 split
                        const float2 z = seg_anchor(seg_slow_sum(buf, lane, s->rot, s->chipw, s->d[a.kp], i0,
                                                                 jlo, max(jlo, min(jhi, nh - i0)), c.cps, c.base),
                                                    ca_, sa_);
                        hr += z.x;
                        hi += z.y;
                    }
                    if constexpr (QD) {
    #pragma unroll
                        for (int t = 0; t < T; ++t) {
                            const bool f1 = (spat >> (T + t)) & 1u, f2 = (spat >> (2 * T + t)) & 1u;
                            float2 v = f2 ? v2 : v0;
                            v = f1 ? v1 : v;
                            const float cs = start_chip(t);
                            const float2 at = __ffma2_rn(v, make_float2(cs, cs), make_float2(acc[2 * t], acc[2 * t + 1]));
                            acc[2 * t] = at.x;
                            acc[2 * t + 1] = at.y;
                        }
                    } else {
#ifndef L1RXG_SEG_LDSCOMB  // the tap combine by register selects (measured faster than the LDS variant below)
    #pragma unroll
                    for (int t = 0; t < T; ++t) {
                        const int code = (int)(w >> (10 + 2 * t)) & 3;
                        const float2 lo = (code & 1) ? v1 : v0;
                        const float2 hi2 = (code & 1) ? v3 : v2;
                        const float2 v = (code & 2) ? hi2 : lo;
                        const float cs = start_chip(t);
    #ifdef L1RXG_SEG_SCALAR_FMA
                        acc[2 * t] = fmaf(cs, v.x, acc[2 * t]);
                        acc[2 * t + 1] = fmaf(cs, v.y, acc[2 * t + 1]);
    #else
                        const float2 at = __ffma2_rn(v, make_float2(cs, cs), make_float2(acc[2 * t], acc[2 * t + 1]));
                        acc[2 * t] = at.x;
                        acc[2 * t + 1] = at.y;
    #endif
                    }
#else
                    // experiment (L1RXG_SEG_LDSCOMB, measured -1.7 %): v0..v3 go to
                    // this lane's own row of the consumed unit buffer (thread-private
                    // scratch; slot (4 i + lane) mod 16 puts a warp's 8-byte accesses
                    // on two wavefronts) and every tap loads its value by code -- one
                    // LDS.64 per tap instead of three float2 selects
                    {
                        unsigned char* rowv = smem_raw + boff + (warp * SEG_NBUF + b) * SEG_UNIT_BYTES + lane * 128;
                        *reinterpret_cast<float2*>(rowv + ((lane + 0) & 15) * 8) = v0;
                        *reinterpret_cast<float2*>(rowv + ((lane + 4) & 15) * 8) = v1;
                        *reinterpret_cast<float2*>(rowv + ((lane + 8) & 15) * 8) = v2;
                        *reinterpret_cast<float2*>(rowv + ((lane + 12) & 15) * 8) = v3;
    #pragma unroll
                        for (int t = 0; t < T; ++t) {
                            const int code = (int)(w >> (10 + 2 * t)) & 3;
                            const float2 v = *reinterpret_cast<const float2*>(rowv + ((4 * code + lane) & 15) * 8);
                            const float cs = start_chip(t);
                            const float2 at = __ffma2_rn(v, make_float2(cs, cs), make_float2(acc[2 * t], acc[2 * t + 1]));
                            acc[2 * t] = at.x;
                            acc[2 * t + 1] = at.y;
                        }
                        // these generic writes precede the next TMA into the buffer
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    }
#endif
                    }
                    __syncwarp();
                    ++consumed;
                    if (issued < consumed + SEG_NBUF)
                        issue_one();
                }
                if (!snapped) {
                    hr = hi = 0.f;
    #pragma unroll
                    for (int t = 0; t < T; ++t) {
                        const float m = t == a.kp ? 1.f : 0.f;
                        hr = fmaf(m, acc[2 * t], hr);
                        hi = fmaf(m, acc[2 * t + 1], hi);
                    }
                }
                acc[2 * T] = hr;
                acc[2 * T + 1] = hi;
                warp_partials<V>(acc, s->red, lane, warp);
            }
            __syncthreads();
            if (warp == 0) {
                const EpochConsts cc = s->c;  // this epoch's (warp0_update writes the next one's)
#ifdef L1RXG_SEG_XSKIP_UPDATE  // experiment: bound on hiding the loop update (wrong results)
                if (lane == 0) {
                    s->c.phi = cc.phi;
                    s->c.base = cc.base;
                    s->ch.sample_offset_next_epoch += cc.n;
                    s->ch.epoch_ms_count += 1;
                }
                __syncwarp();
#else
                warp0_update<T>(s, a, cc, off, cidx, done, SEG_NW, lane, 0, e, nullptr, rec_i);
#endif
                if (lane == 0) {
                    s->c.inv_cps = fast_rcp(s->c.cps);
                    if (QD) {
                        s->qd.cps4 = 4.0 * s->c.cps;
                        s->qd.base4 = 4.0 * s->c.base;
                        s->qd.omb = 1.0 - 4.0 * s->c.base;
                        s->qd.inv4 = 0.25 * s->c.inv_cps;
                        s->qd.ok = s->c.cps > 0.0 && 4.0 * s->c.cps <= 2.0 / 31.0;
                    }
                }
                float sn, co;
                sincosf((float)(s->c.w * (double)lane), &sn, &co);
                s->rot[lane] = make_float2(co * scale, sn * scale);
                s->rotq[(lane & 7) * 4 + (lane >> 3)] = make_float2(co * scale, sn * scale);
            }
            __syncthreads();
            if (s->stop)
                break;
            ++e;
            ++done;
            if (++rec_i == a.max_records)
                rec_i = 0;
        }
        __syncthreads();
        if (warp == ctl && s->pending)
            finish_epoch<T>(s, a, lane, true);
        if (warp < SEG_NW) {  // drain this item's prefetched copies (the parities continue)
            for (int u = consumed; u < issued; ++u)
                mbar_wait(&s->fbar[warp][u & (SEG_NBUF - 1)], (uint32_t)((u / SEG_NBUF) & 1));
            consumed = issued;
        }
        __syncthreads();
        {
            const unsigned long long* src = reinterpret_cast<const unsigned long long*>(&s->ch);
            unsigned long long* dst = reinterpret_cast<unsigned long long*>(a.chans + cidx);
            for (int q = tid; q < (int)(sizeof(l1rxg_channel) / 8); q += blockDim.x)
                dst[q] = src[q];
        }
        if (tid == 0) {
            a.ecount[cidx] = done;
            if (sa.trace) {
                unsigned long long tn;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
                sa.trace[3 * (size_t)item + 1] = tn;
            }
        }
        __threadfence();  // records, tap sums and state visible before the chunk is marked done
        __syncthreads();
        if (tid == 0)
            atomicExch(&sa.ready[cidx], chunk + 1);
    }
}

}  // namespace l1rxg
