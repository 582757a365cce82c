// ovlcorr.cuh -- latency-shape tracking kernel with the next epoch's phase A
// overlapped with this epoch's loop update (configs 1-3; sm_100a).
//
// Same contract, phases and results as track_kernel's latency shape
// (correlator.cuh; reference tracking.hpp:226-282 + :520-618), scheduled so
// that the per-sample work of epoch e+1 is off the per-epoch critical path:
//
//   * the loop update of epoch e runs on the control warp (warp0_update is a
//     warp-level function); meanwhile the work warps already compute phase A'
//     of epoch e+1 -- the wiped run-local prefix P'(j) = sum_{t<j} y'_t and
//     its first moment M'(j) = sum_{t<j} t y'_t, y'_t = x_t e^{-j w_e t} --
//     with the rotator table of the CURRENT carrier rate w_e;
//   * when the update has produced w_{e+1}, each run's sums are corrected to
//     the true rate: sum_t x_t e^{-j w t} = P' - j dw M' + O((dw t)^2 / 2),
//     dw = w_{e+1} - w_e, t < RUN = 31 -- below 1e-9 relative for the
//     per-epoch rate changes of a tracking loop (|dw| 30 < 1e-4); larger
//     changes (FLL pull-in) recompute phase A exactly with the new table.
//     The run anchors e^{-j theta(i0)} use the new rate exactly (fp64), so
//     the approximation never spans more than one run;
//   * phase B reads P' - j dw M' at each step (one more LDS.64 and two FFMA
//     per transition).
// The per-epoch chain becomes: update -> per-run anchors and run totals ->
// phase B -> partial sums -> next update.
#pragma once

#include "correlator.cuh"
#include "ingest.cuh"

namespace l1rxg {

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void named_bar_arrive(int id, int count) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// |dw| * RUN above TrackArgs::ovl_dwmax recomputes phase A exactly; the
// host default 1e-3 keeps the second-order term below 5e-7 of the run's
// magnitude (the parity bar is 1e-5).  Env L1RXG_OVL_DWMAX (tests: -1 runs
// the exact recompute every epoch).

// Shared memory of the overlapped kernel: track_kernel's layout (header,
// anchors, 2 sample tiles, cluster exchange slots) sized by the runs of one
// unit (nrun = ceil(len / RUN), not the CTA's work threads), then one P' and
// one M' tile (epoch e's are dead once its phase B is done, before phase A'
// of e+1 starts), per-run totals, double-buffered rotator tables.
__host__ __device__ inline size_t ovl_extra_bytes(int nrun) {
    const size_t cap = (size_t)nrun * RUN;
    return 2 * cap * sizeof(float2) + 2 * (size_t)nrun * sizeof(float2) + 2 * 32 * sizeof(float2) +
           4 * sizeof(double) + 64;
}

// Cluster exchange slots: [2 (epoch parity)][csize][V] fp64 CTA totals.
__host__ __device__ inline size_t ovl_xslot_bytes(int csize, int V) {
    return (2u * (size_t)csize * V * sizeof(double) + 15) & ~size_t(15);
}

// RAW variant (real int8 IF at fs/4, raw byte ring): OVL_NF extra warps turn each
// epoch's unit of raw bytes (bulk copy, 1 B per sample instead of the 8 B of a
// float2 ring) into the float2 tile the work warps read -- the fs/4 mixer and the
// 23-tap half-band FIR of SampleSource (samples.hpp:215-253, if4_fir) -- one
// epoch ahead of phase A', so the ingest pass and its float2 ring are gone.
// Extra shared memory: two raw unit buffers, one float staging row, six mbarriers.
#ifndef L1RXG_OVL_NF
#define L1RXG_OVL_NF 2
#endif
constexpr int OVL_NF = L1RXG_OVL_NF;
__host__ __device__ inline size_t ovl_raw_unit_bytes(int nrun) {  // + copy alignment (16) + staging shift (4)
    return ((size_t)nrun * RUN + 22 + 16 + 12 + 15) & ~size_t(15);
}
__host__ __device__ inline size_t ovl_raw_bytes(int nrun) {
    return 16 + 2 * ovl_raw_unit_bytes(nrun) + 4 * ovl_raw_unit_bytes(nrun) + 8 * 8;
}

// Phase A' of one run: exclusive prefixes P'(j), M'(j) into pp/mp, totals out.
template <bool FULL>
__device__ __forceinline__ void ovl_phase_a(const float2* raw, float2* pp, float2* mp, const float2* rot,
                                            int cnt, float2& ptot, float2& mtot) {
    float pr = 0.f, pi = 0.f, mr = 0.f, mi = 0.f;
#pragma unroll
    for (int j = 0; j < RUN; ++j) {
        pp[j] = make_float2(pr, pi);
        mp[j] = make_float2(mr, mi);
        const float2 x = (FULL || j < cnt) ? raw[j] : make_float2(0.f, 0.f);
        const float2 q = rot[j];
        const float yr = fmaf(x.y, q.y, x.x * q.x);   // x conj(rot): (xr c + xi s,
        const float yi = fmaf(-x.x, q.y, x.y * q.x);  //   xi c - xr s), tracking.hpp:248-249
        pr += yr;
        pi += yi;
        mr = fmaf((float)j, yr, mr);
        mi = fmaf((float)j, yi, mi);
    }
    ptot = make_float2(pr, pi);
    mtot = make_float2(mr, mi);
}

// P - j dw M
__device__ __forceinline__ float2 ovl_corr(float2 p, float2 m, float dw) {
    return make_float2(fmaf(dw, m.y, p.x), fmaf(-dw, m.x, p.y));
}

// One step: acc -= delta * anchor(run(b)) * (P'(b) - j dw M'(b)).
__device__ __forceinline__ void ovl_b_one(PhaseB& pb, const float2* pt, const float2* mt, const float2* anchors,
                                          int u0, int nh, int b, float dlt, float dw) {
    const int off = b - u0;
    const float2 p = ovl_corr(pt[off], mt[off], dw);
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

// Phase B over the tap's transitions (the latency walk of phase_b<T, false>).
template <int T>
__device__ __forceinline__ void ovl_phase_b(PhaseB& pb, const EpochConsts& c, const float2* pt, const float2* mt,
                                            const float2* anchors, const CodeTables& ct, int u0, int len, float dw) {
    if (pb.kt >= T)
        return;
    const int hi = u0 + len - 1;
    const int g0 = pb.g0, cnt = pb.cnt;
    for (int j = pb.jt; j < cnt; j += 2 * pb.gsz) {
        const int j2 = j + pb.gsz;
        const bool two = j2 < cnt;
        const int ga = g0 + j, gb = g0 + (two ? j2 : j);
        const int ma = ct.tm[ga], mb = ct.tm[gb];
        const float da = (float)ct.td[ga], db = (float)ct.td[gb];
        const int ba = tap_boundary(ma, pb.dk, c, u0, hi);
        const int bb = tap_boundary(mb, pb.dk, c, u0, hi);
        ovl_b_one(pb, pt, mt, anchors, u0, c.nh, ba, da, dw);
        if (two)
            ovl_b_one(pb, pt, mt, anchors, u0, c.nh, bb, db, dw);
    }
}

// Run totals after the update (what phase_a adds per run): the run's anchor
// with the true rate, chip_k(last) * anchor * (P'tot - j dw M'tot) per tap,
// and the first-half prompt (tracking.hpp:259-271).
template <int T>
__device__ __forceinline__ void ovl_run_totals(const EpochConsts& c, const CodeTables& ct, const double* d, int kp,
                                               int i0, int cnt, float2 ptot, float2 mtot, const float2* pt,
                                               const float2* mt, float dw, float* acc, float2* anchor_slot) {
    const double th = __fma_rn(c.w, (double)i0, c.phi);
    const double r = fma(-rint(th * (1.0 / TWO_PI_D)), TWO_PI_D, th);
    float sa, ca;
    __sincosf((float)r, &sa, &ca);
    *anchor_slot = make_float2(ca, sa);
    const float2 z0 = ovl_corr(ptot, mtot, dw);
    const float zr = fmaf(z0.x, ca, z0.y * sa);
    const float zi = fmaf(z0.y, ca, -(z0.x * sa));
    const int i_last = i0 + cnt - 1;
    const double dl = (double)i_last;
    float chip_p = 0.f;
#pragma unroll
    for (int k = 0; k < T; ++k) {
        const float ch = (float)ct.chip[__double2int_rz(tap_value(dl, c.cps, c.base, d[k]))];
        acc[2 * k] = fmaf(ch, zr, acc[2 * k]);
        acc[2 * k + 1] = fmaf(ch, zi, acc[2 * k + 1]);
        if (k == kp)
            chip_p = ch;
    }
    if (i_last < c.nh) {
        acc[2 * T] = fmaf(chip_p, zr, acc[2 * T]);
        acc[2 * T + 1] = fmaf(chip_p, zi, acc[2 * T + 1]);
    } else if (i0 < c.nh) {  // the run straddling n/2: chip(nh-1) * P(nh)
        const float ch = (float)ct.chip[tap_index(c.nh - 1, c.cps, c.base, d[kp])];
        const float2 pn = ovl_corr(pt[c.nh - i0], mt[c.nh - i0], dw);
        acc[2 * T] = fmaf(ch, fmaf(pn.x, ca, pn.y * sa), acc[2 * T]);
        acc[2 * T + 1] = fmaf(ch, fmaf(pn.y, ca, -(pn.x * sa)), acc[2 * T + 1]);
    }
}

__device__ __forceinline__ void ovl_fill_rot(float2* rot, double w, int lane) {
    float sn, co;
    sincosf((float)(w * (double)lane), &sn, &co);
    rot[lane] = make_float2(co, sn);
}

// Latency shape only: float2 rings, two sample tiles, one unit per epoch
// (the host selects it), Scalar/Batched kernels (Noop stays on track_kernel).
template <int T, bool RAW>
__global__ void __launch_bounds__(MAX_NT, 1) track_ovl_kernel(TrackArgs a) {
    constexpr int esz = 8;  // tile element: float2 (the RAW variant's ring holds bytes)
    constexpr int A = 2;    // samples per 16-byte bulk-copy granule
    extern __shared__ __align__(16) unsigned char smem_raw[];
    CorrSmem<T>* s = reinterpret_cast<CorrSmem<T>*>(smem_raw);
    const int csize = a.csize;
    const int crank = csize > 1 ? (int)(blockIdx.x % csize) : 0;
    const int cidx = blockIdx.x / csize;
    const bool writer = crank == 0;
    const int strm = a.chan_stream[cidx];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nfir = RAW ? 32 * OVL_NF : 0;  // FIR warps sit after the control warp
    const int nthr = blockDim.x - nfir;
    const int nwarps = (nthr + 31) >> 5;
    const int ctl = nwarps - 1;
    const int nwork = nthr - 32;
    const int nwork_warps = nwarps - 1;
    constexpr int V = 2 * T + 2;
    const int n = a.n;
    const int r0 = csize > 1 ? crank * a.share : 0;
    const int rend = csize > 1 ? min(n, r0 + a.share) : n;
    const int len = rend - r0;  // one unit per epoch
    const int skip = n - len;
    // shared-memory layout unit: rank 0's (largest) unit in every CTA, so the
    // cluster exchange slots sit at the same offset in all of them
    const int nrun = ((csize > 1 ? min(n, a.share) : n) + RUN - 1) / RUN;
    const int cap = nrun * RUN;
    const int64_t avail = a.avail[strm];
    const unsigned char* ring = a.ring + (int64_t)strm * a.ring_stride * (RAW ? 1 : esz);
    float2* anchors = anchors_of(s);
    double* xs = xslots_of(s, nrun, 2, esz);
    unsigned char* xb = reinterpret_cast<unsigned char*>(xs) + ovl_xslot_bytes(csize, V);
    float2* const pm0 = reinterpret_cast<float2*>(xb);  // P' tile [cap]
    float2* const mm0 = pm0 + cap;                       // M' tile [cap]
    float2* ptot = mm0 + cap;
    float2* mtot = ptot + nrun;
    float2* rot2 = mtot + nrun;  // [2][32]
    double* wp = reinterpret_cast<double*>(rot2 + 64);  // [2]: the rate each buffer's P'/M' were made with
    int* ie = reinterpret_cast<int*>(wp + 2);            // [2]: epoch whose copy was issued into each tile
    long long* dn = reinterpret_cast<long long*>(ie + 2); // epochs done (control warp -> writeback)
    // RAW: raw unit buffers [2], float staging row, mbarriers, stop flag
    unsigned char* const rawb = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(dn + 1) + 15) & ~uintptr_t(15));
    const size_t rub = ovl_raw_unit_bytes(nrun);
    float* const xfl = reinterpret_cast<float*>(rawb + 2 * rub);
    uint64_t* const rbar = reinterpret_cast<uint64_t*>(rawb + 6 * rub);  // [2] raw unit landed
    uint64_t* const fbar = rbar + 2;                                     // [2] float2 tile filled
    uint64_t* const ebar = rbar + 4;                                     // [2] float2 tile consumed
    volatile int* const fstop = reinterpret_cast<volatile int*>(rbar + 6);
    const int64_t off0 = a.chans[cidx].sample_offset_next_epoch;
    // (RAW: the 22 samples of FIR history before the window must still be in the ring)
    const bool ring_ok = off0 >= 0 && off0 - (RAW ? 22 : 0) >= avail - a.ring_cap;
    // epoch v's unit into tile v & 1 (range admission only; an Idle channel's
    // speculative copies are drained at exit)
    auto try_issue = [&](int v) {
        const int64_t offv = off0 + (int64_t)v * n;
        if (!ring_ok || v >= a.max_epochs || offv + n > avail)
            return;
        const int b = v & 1;
        const int64_t pos = s->issue_pos;
        issue_unit(s, b, tile_of(s, nrun, b, esz), ring, pos, len, esz);
        ie[b] = v;
        int64_t nxt = pos + len + skip;
        while (nxt >= a.ring_cap)
            nxt -= a.ring_cap;
        s->issue_pos = nxt;
    };
    // ring position of epoch v's unit (the copy's 16-byte alignment slack)
    auto unit_pos = [&](int v) -> int64_t { return (off0 + r0 + (int64_t)v * n) % a.ring_cap; };

    if (tid == 0) {
        s->ch = a.chans[cidx];
        for (int b = 0; b < 2; ++b) {
            mbar_init(&s->bars[b][0], 1);
            mbar_init(&s->bars[b][1], 1);
            mbar_init(&s->pbar[b], 1);
            s->inflight[b] = 0;
            if (RAW) {
                mbar_init(&rbar[b], 1);
                mbar_init(&fbar[b], (uint32_t)nfir);
                mbar_init(&ebar[b], 1);
            }
        }
        if (RAW)
            fstop[0] = fstop[1] = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        s->pending = 0;
        s->stop = 0;
    }
    for (int k = tid; k < T; k += blockDim.x)
        s->d[k] = a.taps.offsets_chips[k];
    if (csize > 1)
        cluster_sync_all();
    __syncthreads();
    PhaseB pb;
    phase_b_init<T>(pb, s->d, a.kp, tid, nwork);
    build_code_tables(s->ct, a.codes, s->ch.prn);
    if (tid == 0) {
        s->issue_pos = ring_ok ? (off0 + r0) % a.ring_cap : 0;
        const l1rxg_channel& ch = s->ch;
        make_consts(s->c, ch.code_phase_chips, ch.code_freq_hz, ch.carrier_doppler_hz, ch.carrier_phase_rad,
                    a.lc.fs, n);
        if (!RAW) {
            try_issue(0);
            try_issue(1);
        }
        wp[0] = s->c.w;
    }
    __syncthreads();
    if (tid < 32)
        ovl_fill_rot(rot2, s->c.w, tid);
    __syncthreads();

    // prologue: phase A' of epoch 0 with its own rate (dw = 0)
    auto phase_a_epoch = [&](int v, const float2* rot) {
        const int b = v & 1;
        const int delta = RAW ? 0 : (int)(unit_pos(v) & (A - 1));
        const int h = A * ((len + delta) / (2 * A));
        const float2* rawt = reinterpret_cast<const float2*>(tile_of(s, nrun, b, esz)) + delta;
        const int i0 = r0 + tid * RUN;
        const int cnt = min(RUN, rend - i0);
        const int r0t = delta + tid * RUN;
        const uint32_t par = (uint32_t)(v >> 1) & 1u;
        if (cnt > 0) {
            if (RAW) {
                mbar_wait(&fbar[b], par);  // the FIR warps filled tile b
            } else {
                if (r0t < h)
                    mbar_wait(&s->bars[b][0], par);
                if (r0t + RUN > h)
                    mbar_wait(&s->bars[b][1], par);
            }
            if (cnt == RUN)
                ovl_phase_a<true>(rawt + tid * RUN, pm0 + tid * RUN, mm0 + tid * RUN, rot, cnt, ptot[tid],
                                  mtot[tid]);
            else
                ovl_phase_a<false>(rawt + tid * RUN, pm0 + tid * RUN, mm0 + tid * RUN, rot, cnt, ptot[tid],
                                   mtot[tid]);
        }
    };
    if (tid == 0)
        *dn = a.ecount[cidx];
    const bool first_ok = ring_ok && a.max_epochs > 0 && off0 + n <= avail && s->ch.state != L1RXG_IDLE;
    if (tid < nwork && first_ok)
        phase_a_epoch(0, rot2);

    int e = 0;
    int64_t done = a.ecount[cidx];
    int rec_i = (int)(done % a.max_records);
    if (RAW && tid >= nthr) {
        // ---- FIR warps: raw unit of epoch v -> float2 tile v & 1, ahead of phase A'
        const int ftid = tid - nthr;
        auto adm = [&](int v) { return first_ok && v < a.max_epochs && off0 + (int64_t)(v + 1) * n <= avail; };
        auto issue_raw = [&](int v) {  // window [pos - 22, pos + len) from the 16-byte boundary below it
            const int64_t pos = (off0 + r0 + (int64_t)v * n) % a.ring_cap;
            const int dl = (int)((pos - 22) & 15);
            const uint32_t bytes = (uint32_t)((dl + len + 22 + 15) & ~15);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&rbar[v & 1], bytes);
            tma_load_1d(rawb + (size_t)(v & 1) * rub, ring + (pos - 22 - dl), bytes, &rbar[v & 1]);
        };
        if (ftid == 0 && adm(0))
            issue_raw(0);
        int pend = adm(0) ? 0 : -1;  // newest epoch whose raw copy was issued
        for (int v = 0; adm(v); ++v) {
            const int b = v & 1;
            named_bar_sync(4, nfir);  // every FIR warp is done with epoch v-1 (raw buffer b^1, staging row)
            if (adm(v + 1)) {
                if (ftid == 0)
                    issue_raw(v + 1);
                pend = v + 1;
            }
            mbar_wait(&rbar[b], (uint32_t)(v >> 1) & 1u);
            const int64_t pos = (off0 + r0 + (int64_t)v * n) % a.ring_cap;
            const int dl = (int)((pos - 22) & 15);
            const unsigned char* rw = rawb + (size_t)b * rub;
            // bytes -> floats, a word at a time, shifted so that sample 4q - 24 of the unit sits at a
            // 16-byte aligned staging index: sample i <-> byte dl + 22 + i <-> float dl + 22 + i + sh
            const int sh = (4 - ((dl + 22) & 3)) & 3;
            for (int j = 4 * ftid; j < dl + len + 22; j += 4 * nfir) {
                const uint32_t w = *reinterpret_cast<const uint32_t*>(rw + j);
                float* o = xfl + j + sh;
                o[0] = (float)(int8_t)(w & 0xffu);
                o[1] = (float)(int8_t)((w >> 8) & 0xffu);
                o[2] = (float)(int8_t)((w >> 16) & 0xffu);
                o[3] = (float)(int8_t)(w >> 24);
            }
            if (ftid == 0) {  // one thread decides (uniformly for the named barrier) whether to go on
                if (v >= 2)
                    mbar_wait(&ebar[b], (uint32_t)((v - 2) >> 1) & 1u);  // epoch v-2 is done with tile b
                fstop[1] = fstop[0];
            }
            named_bar_sync(4, nfir);
            if (fstop[1])
                break;
            float2* tl = reinterpret_cast<float2*>(tile_of(s, nrun, b, esz));
            const int ph0 = (int)((off0 + r0 + (int64_t)v * n) & 3);
            // four consecutive outputs per task from 28 staged floats (samples 4q - 24 .. 4q + 3) held in
            // registers; the mixer phase of output u is (ph0 + u) & 3 for every task
            const float4* x4 = reinterpret_cast<const float4*>(xfl + dl + sh - 2);  // sample -24
            for (int q = ftid; 4 * q < len; q += nfir) {
                float x[28];
#pragma unroll
                for (int k = 0; k < 7; ++k) {
                    const float4 v4 = x4[q + k];
                    x[4 * k] = v4.x;
                    x[4 * k + 1] = v4.y;
                    x[4 * k + 2] = v4.z;
                    x[4 * k + 3] = v4.w;
                }
                float2 y[4];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    y[u] = if4_fir(&x[24 + u], (ph0 + u) & 3);
                if (4 * q + 4 <= len) {
                    float4* o = reinterpret_cast<float4*>(tl + 4 * q);
                    o[0] = make_float4(y[0].x, y[0].y, y[1].x, y[1].y);
                    o[1] = make_float4(y[2].x, y[2].y, y[3].x, y[3].y);
                } else {
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (4 * q + u < len)
                            tl[4 * q + u] = y[u];
                }
            }
            mbar_arrive(&fbar[b]);
            if (pend == v)
                pend = -1;
        }
        if (pend >= 0)  // never leave a bulk copy in flight into freed smem
            mbar_wait(&rbar[pend & 1], (uint32_t)(pend >> 1) & 1u);
    } else if (!first_ok) {  // nothing admitted (also: overwritten window)
        if (tid == 0 && s->ch.state != L1RXG_IDLE && a.max_epochs > 0 && off0 + n <= avail && !ring_ok)
            a.status[cidx] = 1;
    } else if (warp == ctl) {
        // ---- control warp: the loop update of every epoch
        for (;;) {
            const EpochConsts c = s->c;  // epoch e's constants (written by the previous update)
            const int64_t off = s->ch.sample_offset_next_epoch;
            nco_advance_lanes(s->nco_ph1, s->nco_cp1, c, s->ch, lane);
            named_bar_sync(2, nthr);  // X: epoch e's partial sums are in s->red
            warp0_update<T>(s, a, c, off, cidx, done, nwork_warps, lane, crank, e, xs, rec_i);
            const bool stop = s->stop != 0;
            named_bar_arrive(3, nthr);  // Y: epoch e+1's constants (or stop)
            if (s->pending) {           // epoch e's metrics and record, while e+1 correlates
                finish_epoch<T>(s, a, lane, writer);
                __syncwarp();
                if (lane == 0)
                    s->pending = 0;
                __syncwarp();
            }
            if (stop)
                break;
            ++e;
            ++done;
            if (++rec_i == a.max_records)
                rec_i = 0;
            const int64_t offn = off0 + (int64_t)e * n;
            if (e >= a.max_epochs || offn + n > avail)
                break;
        }
        if (lane == 0)
            *dn = done;
    } else {
        // ---- work warps: correlation of epoch e, then phase A' of epoch e+1
        for (;;) {
            if (tid == 0)
                PROF_STAMP(0);  // (profiling builds: CTA 0, thread 0's stage clocks per epoch)
            const int b = e & 1;
            const EpochConsts cc = s->c;
            EpochConsts c = cc;
            c.inv_cps = fast_rcp(c.cps);
            const int u0 = r0;
            float dw = (float)(c.w - wp[b]);
            // work warp 0: this epoch's rotator table (rate w_e), for phase A'
            // of e+1 (published by the barrier after the run totals) and the
            // exact fallback -- off the control warp's update path.  Epoch 0's
            // table is the prologue's (slower warps may still be reading it)
            if (tid < 32 && e > 0)
                ovl_fill_rot(rot2 + 32 * b, c.w, tid);
            if (fabsf(dw) * (float)RUN > a.ovl_dwmax) {  // rate moved too far: exact phase A
                named_bar_sync(1, nwork);
                phase_a_epoch(e, rot2 + 32 * b);
                dw = 0.f;
                named_bar_sync(1, nwork);
            }
            float acc[V];
#pragma unroll
            for (int v = 0; v < V; ++v)
                acc[v] = 0.f;
            phase_b_range<T>(pb, c, s->ct, u0, len);
            {
                const int i0 = u0 + tid * RUN;
                const int cnt = min(RUN, rend - i0);
                if (cnt > 0)
                    ovl_run_totals<T>(c, s->ct, s->d, a.kp, i0, cnt, ptot[tid], mtot[tid], pm0 + tid * RUN,
                                      mm0 + tid * RUN, dw, acc, &anchors[tid]);
            }
            if (tid == 0)
                PROF_STAMP(1);
            named_bar_sync(1, nwork);  // anchors visible
            if (tid == 0)
                PROF_STAMP(2);
            ovl_phase_b<T>(pb, c, pm0, mm0, anchors, s->ct, u0, len, dw);
            phase_b_fold<T>(pb, acc);
            if (tid == 0)
                PROF_STAMP(3);
            warp_partials<V>(acc, s->red, lane, warp);
            named_bar_sync(1, nwork);  // tile b consumed; partials written
            named_bar_arrive(2, nthr);  // X
            if (tid == 0)
                PROF_STAMP(4);
            if (tid == 0) {  // the copy of epoch e+2 into tile b, after X (off the update's path)
                if (RAW) {
                    mbar_arrive(&ebar[b]);  // the FIR warps may refill tile b
                } else {
                    s->inflight[b] = 0;
                    try_issue(e + 2);
                }
            }
            // speculative phase A' of epoch e+1 with this epoch's rate
            const int64_t offn = off0 + (int64_t)(e + 1) * n;
            const bool next_ok = e + 1 < a.max_epochs && offn + n <= avail;
            if (next_ok) {
                phase_a_epoch(e + 1, rot2 + 32 * b);
                if (tid == 0)
                    wp[b ^ 1] = cc.w;
            }
            if (tid == 0)
                PROF_STAMP(5);
            named_bar_sync(3, nthr);  // Y
            if (tid == 0)
                PROF_STAMP(6);
            if (tid == 0)
                PROF_STAMP(7);
            if (s->stop || !next_ok)
                break;
            ++e;
        }
    }
    if (RAW && tid == 0) {  // release FIR warps waiting for a tile no epoch will consume
        fstop[0] = 1;
        mbar_arrive(&ebar[0]);
        mbar_arrive(&ebar[1]);
    }
    __syncthreads();
    if (tid == 0) {
        for (int b = 0; b < 2; ++b)
            if (s->inflight[b]) {  // never leave a bulk copy in flight into freed smem
                const uint32_t par = (uint32_t)(ie[b] >> 1) & 1u;
                mbar_wait(&s->bars[b][0], par);
                mbar_wait(&s->bars[b][1], par);
            }
        if (writer) {
            a.chans[cidx] = s->ch;
            a.ecount[cidx] = *dn;
        }
    }
    if (csize > 1)
        cluster_sync_all();
}

}  // namespace l1rxg
