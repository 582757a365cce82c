// kernels.cuh -- sm_100a device code of the l1rx tracking correlator.
//
// Hot path (reference: /root/reference/proj/include/l1rx):
//   K1 ingest   samples.hpp:177-253   raw int8/int16 -> complex baseband ring
//   K2 correlate tracking.hpp:226-282 carrier wipe + K-tap code replica MAC
//   K3 loop     tracking.hpp:520-618 (+ :459-515) DLL/PLL/FLL + metrics
//
// Correlator algorithm ("boundary-prefix"): the replica
// of tap k is a +/-1 staircase whose steps sit where the reference's fp64
// chip index trunc(fl(fma(i,cps,base)+d_k)) changes.  Each thread owns a
// run of RUN consecutive samples; it wipes the carrier (complex multiply by
// a per-epoch rotator table and a per-run fp64-anchored phasor) and keeps
// the exclusive prefix sums of the wiped samples in shared memory.  A tap's
// sum over the run is then chip(last) * run_total minus, for every chip
// CHANGE inside the run, (chip_after - chip_before) * prefix(boundary).
// Boundaries are located exactly with the reference's own fp64 expression
// (monotone in i), so every chip decision is bit-identical to the
// reference; per-sample work no longer grows with the number of taps.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "l1rxg.h"

namespace l1rxg {

constexpr int RUN = 31;  // samples per thread run; odd -> LDS.64 conflict-free
constexpr double PI_D = 3.14159265358979323846;  // constants.hpp:20
constexpr double TWO_PI_D = 2.0 * PI_D;
constexpr double F_L1_HZ = 1.57542e9;      // constants.hpp:5
constexpr double CHIP_RATE_HZ = 1.023e6;   // constants.hpp:6
constexpr int MAX_NT = 640;                // correlator CTA size cap (<= 102 regs)

// ---------------------------------------------------------------------
// per-epoch NCO constants (tracking.hpp:234-239)
struct EpochConsts {
    double w;        // 2*pi*fD/fs   rad/sample
    double cps;      // code_freq/fs chips/sample
    double inv_cps;
    double base;     // code_phase + 1023
    double phi;      // carrier phase at epoch start
    int n, nh;
};

__device__ __forceinline__ void make_consts(EpochConsts& c, double code_phase,
                                            double code_freq, double doppler,
                                            double phase, double fs, int n) {
    c.w = 2.0 * PI_D * doppler / fs;  // (2*pi*fD)/fs as the reference orders it
    c.cps = code_freq / fs;
    c.inv_cps = 1.0 / c.cps;
    c.base = code_phase + 1023.0;
    c.phi = phase;
    c.n = n;
    c.nh = n / 2;
}

// The reference's replica phase of tap d at sample i (tracking.hpp:251-254
// as compiled: ph = fma(i, cps, base), then ph + d rounded).
__device__ __forceinline__ double tap_value(int i, double cps, double base, double d) {
    return __dadd_rn(__fma_rn((double)i, cps, base), d);
}
__device__ __forceinline__ int tap_index(int i, double cps, double base, double d) {
    return __double2int_rz(tap_value(i, cps, base, d));
}
// First i in [lo, hi] with tap_value(i) >= m, given tap_index(hi) >= m.
__device__ __forceinline__ int tap_boundary(int m, double d, double cps, double inv_cps,
                                            double base, int lo, int hi) {
    const double e = (((double)m - d) - base) * inv_cps;
    int b = (int)ceil(e);
    b = max(lo, min(hi, b));
    const double mm = (double)m;
    while (b > lo && tap_value(b - 1, cps, base, d) >= mm) --b;
    while (b < hi && tap_value(b, cps, base, d) < mm) ++b;
    return b;
}

// fma-free complex multiply x * conj(e^{j a}) with (c, s) = (cos a, sin a):
// (xr c + xi s, xi c - xr s) -- the reference's wipe-off form
// (tracking.hpp:248-249).
__device__ __forceinline__ float2 wipe(float2 x, float c, float s) {
    return make_float2(fmaf(x.x, c, x.y * s), fmaf(x.y, c, -(x.x * s)));
}

// ---------------------------------------------------------------------
// One thread's run: samples [i0, i0+cnt) of the epoch, in shared memory at
// run[0..RUN).  Overwrites run[j] with the exclusive prefix of the wiped
// samples and accumulates the run's contribution of every tap (and of the
// first-half prompt) into acc[2*T+2] (fp32).
// Replica phase at a sample index held as a double (no int->fp64 convert
// on the hot path): same value as tap_value(int).
__device__ __forceinline__ double tap_value_d(double i, double cps, double base, double d) {
    return __dadd_rn(__fma_rn(i, cps, base), d);
}
// First b in [lo, hi] with tap_value(b) >= m (exists: tap_index(hi) >= m);
// fp64 estimate, then exact verification with the reference expression
// (monotone in b), so the boundary is the reference's to the sample.
__device__ __forceinline__ int tap_boundary_d(double m, double d, double cps, double inv_cps,
                                              double base, double lo, double hi) {
    double b = ceil(((m - d) - base) * inv_cps);
    b = fmax(lo, fmin(hi, b));
    while (b > lo && tap_value_d(b - 1.0, cps, base, d) >= m) b -= 1.0;
    while (b < hi && tap_value_d(b, cps, base, d) < m) b += 1.0;
    return __double2int_rz(b);
}

constexpr int CHIP_EXT = 4096;  // chip table extended over m in [0, 4096)

template <int T, bool FULL>
__device__ __forceinline__ void process_run(const EpochConsts& c, float2* run,
                                            const float2* __restrict__ rot,
                                            const float* __restrict__ chipf,
                                            const double* __restrict__ d, int kp,
                                            int i0, int cnt, float* acc) {
    // per-run carrier anchor e^{-j theta(i0)}, theta as the reference
    // computes it (fma(w, i, phi)), reduced to [-pi, pi] in fp64; the fp32
    // phasor's ~4e-7 error is common to the run's 31 samples
    const double di0 = (double)i0;
    const double th = __fma_rn(c.w, di0, c.phi);
    const double r = fma(-rint(th * (1.0 / TWO_PI_D)), TWO_PI_D, th);
    float sa, ca;
    __sincosf((float)r, &sa, &ca);

    float pr = 0.f, pi = 0.f;
#pragma unroll
    for (int j = 0; j < RUN; ++j) {
        const float2 x = (FULL || j < cnt) ? run[j] : make_float2(0.f, 0.f);
        const float2 q = rot[j];
        const float2 z = wipe(x, q.x, q.y);
        run[j] = make_float2(pr, pi);
        pr += z.x;
        pi += z.y;
    }
    const int i_last = i0 + (FULL ? RUN : cnt) - 1;
    const double dlo = di0, dhi = (double)i_last;
    const double dprev = i0 > 0 ? di0 - 1.0 : 0.0;
    const bool straddle = (i0 < c.nh) && (c.nh <= i_last);
#pragma unroll
    for (int k = 0; k < T; ++k) {
        const double dk = d[k];
        const int m_hi = __double2int_rz(tap_value_d(dhi, c.cps, c.base, dk));
        const int m_lo = __double2int_rz(tap_value_d(dprev, c.cps, c.base, dk));
        const float chi = chipf[m_hi];
        float ur = chi * pr, ui = chi * pi;
        // first-half prompt (tracking.hpp:265-271), only where the run
        // straddles n/2
        const bool want_h = (k == kp) && straddle;
        int m_h = 0;
        float hr = 0.f, hi = 0.f;
        if (want_h) {
            m_h = tap_index(c.nh - 1, c.cps, c.base, dk);
            const float chh = chipf[m_h];
            const float2 pn = run[c.nh - i0];
            hr = chh * pn.x;
            hi = chh * pn.y;
        }
        float prev = chipf[m_lo];
        for (int m = m_lo + 1; m <= m_hi; ++m) {
            const float cur = chipf[m];
            const float df = cur - prev;
            prev = cur;
            if (df != 0.f) {
                const int b = tap_boundary_d((double)m, dk, c.cps, c.inv_cps, c.base, dlo, dhi);
                if (b > i0) {
                    const float2 pb = run[b - i0];
                    ur = fmaf(-df, pb.x, ur);
                    ui = fmaf(-df, pb.y, ui);
                    if (want_h && m <= m_h) {
                        hr = fmaf(-df, pb.x, hr);
                        hi = fmaf(-df, pb.y, hi);
                    }
                }
            }
        }
        // rotate by the anchor: U * e^{-j theta0}
        acc[2 * k] += fmaf(ur, ca, ui * sa);
        acc[2 * k + 1] += fmaf(ui, ca, -(ur * sa));
        if (k == kp) {
            if (want_h) {
                acc[2 * T] += fmaf(hr, ca, hi * sa);
                acc[2 * T + 1] += fmaf(hi, ca, -(hr * sa));
            } else if (i_last < c.nh) {
                acc[2 * T] += fmaf(ur, ca, ui * sa);
                acc[2 * T + 1] += fmaf(ui, ca, -(ur * sa));
            }
        }
    }
}

// Per-epoch rotator table rot[j] = (cos wj, sin wj), j < RUN.
__device__ __forceinline__ void fill_rot(float2* rot, double w) {
    const int j = threadIdx.x;
    if (j < RUN) {
        float s, co;
        sincosf((float)(w * (double)j), &s, &co);
        rot[j] = make_float2(co, s);
    }
}

// Cooperative copy of `len` samples into tile[0..len), zero fill to cap.
__device__ __forceinline__ void load_tile(float2* tile, const float2* __restrict__ src,
                                          int len, int cap) {
    for (int i = threadIdx.x; i < cap; i += blockDim.x)
        tile[i] = (i < len) ? __ldg(src + i) : make_float2(0.f, 0.f);
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
// 1-D bulk copy global -> shared (TMA engine), completion counted on bar.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Warp + block reduction of V fp32 partials into fp64 totals in out[V]
// (valid in all threads after the trailing barrier).
template <int V>
__device__ __forceinline__ void block_reduce(float* acc, float* red /*[32][V]*/,
                                             double* out /*[V]*/) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int v = 0; v < V; ++v) {
        float x = acc[v];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0)
            red[warp * V + v] = x;
    }
    __syncthreads();
    if (threadIdx.x < V) {
        double s = 0.0;
        for (int w = 0; w < nwarps; ++w)
            s += (double)red[w * V + threadIdx.x];
        out[threadIdx.x] = s;
    }
    __syncthreads();
}

// ---------------------------------------------------------------------
// K3: loop update on one thread (tracking.hpp:542-601 + :459-515).
struct LoopCfg {
    l1rxg_tracking_cfg cfg;
    int kernel;
    double fs;
};

__device__ __forceinline__ double natural_frequency(double bw, double zeta) {
    return 8.0 * zeta * bw / (4.0 * zeta * zeta + 1.0);  // tracking.hpp:71-73
}

__device__ __forceinline__ double loop_filter(double& integ, double& prev, int& primed,
                                              double err, double bw, double zeta,
                                              double dt) {  // tracking.hpp:75-84
    const double wn = natural_frequency(bw, zeta);
    const double p = primed ? prev : err;
    integ += wn * wn * dt * 0.5 * (err + p);
    prev = err;
    primed = 1;
    return integ + 2.0 * zeta * wn * err;
}

__device__ __forceinline__ double fll_disc(double pi_, double pq, double ci, double cq,
                                           double dt, bool fold) {  // tracking.hpp:113-138
    double cross = pi_ * cq - pq * ci;
    double dot = pi_ * ci + pq * cq;
    if (fold && dot < 0) {
        cross = -cross;
        dot = -dot;
    }
    if (cross == 0.0 && dot == 0.0)
        return 0.0;
    return atan2(cross, dot) / (2.0 * PI_D * dt);
}

// The transcendental pieces of one loop update (and the fmod-based NCO
// advance) are independent of each other.  The tracking kernel evaluates
// them in separate WARPS (divergent lanes of one warp would serialise) via
// loop_piece(), then one thread applies the reference's sequential logic
// (loop_update) -- the same operations in the same order as a
// single-thread update, so the result is identical.
struct LoopPre {
    double e, l;        // |E|, |L|            (tracking.hpp:96-97, 545-546)
    double pll;         // Costas atan         (:104-111)
    double fc, ff;      // FLL coarse / fine   (:113-138)
    double mu_s, cn0;   // C/N0 window result  (:472-498), if the window closes
    double code_phase, carrier_phase, chi;  // NCO advance (:275-280)
};
constexpr int LOOP_PIECES = 6;

__device__ __forceinline__ void advance_nco(double& code_phase, double& carrier_phase,
                                            double& chi, const EpochConsts& c);

__device__ __forceinline__ void loop_piece(int piece, LoopPre& p, const l1rxg_channel& ch,
                                           const l1rxg_corr& o, const LoopCfg& lc,
                                           const EpochConsts& c) {
    const double dt = (double)o.n_samples / lc.fs;
    if (piece == 0) {
        p.e = sqrt(o.ie * o.ie + o.qe * o.qe);
        p.l = sqrt(o.il * o.il + o.ql * o.ql);
    } else if (piece == 1) {
        if (o.ip == 0.0)
            p.pll = (o.qp == 0.0) ? 0.0 : (o.qp > 0 ? PI_D / 2.0 : -PI_D / 2.0);
        else
            p.pll = atan(o.qp / o.ip);
    } else if (piece == 2) {
        p.fc = fll_disc(o.ip_h1, o.qp_h1, o.ip_h2, o.qp_h2, dt / 2.0, false);
    } else if (piece == 3) {
        p.ff = fll_disc(ch.last_ip, ch.last_qp, o.ip, o.qp, dt, true);
    } else if (piece == 5) {
        double cp = ch.code_phase_chips, ph = ch.carrier_phase_rad, chi = ch.chi_chips;
        advance_nco(cp, ph, chi, c);
        p.code_phase = cp;
        p.carrier_phase = ph;
        p.chi = chi;
    } else if (piece == 4) {
        const int m = lc.cfg.cn0_window_ms;
        p.mu_s = ch.mu_smoothed;
        p.cn0 = ch.cn0_dbhz;
        if (ch.win_len + 1 >= m) {
            double nbi = 0, nbq = 0, wbp = 0;
            for (int k = 0; k < m; ++k) {
                const double wi = k < ch.win_len ? ch.win_ip[k] : o.ip;
                const double wq = k < ch.win_len ? ch.win_qp[k] : o.qp;
                const double sg = wi >= 0 ? 1.0 : -1.0;
                nbi += sg * wi;
                nbq += sg * wq;
                wbp += wi * wi + wq * wq;
            }
            const double mu = wbp > 0 ? (nbi * nbi + nbq * nbq) / wbp : 0.0;
            p.mu_s = ch.metrics_valid ? ch.mu_smoothed + 0.2 * (mu - ch.mu_smoothed) : mu;
            const double md = (double)m;
            if (p.mu_s >= md - 1e-9)
                p.cn0 = 65.0;
            else if (p.mu_s <= 1.0)
                p.cn0 = 0.0;
            else
                p.cn0 = 10.0 * log10((p.mu_s - 1.0) / (md - p.mu_s) / 1e-3);
        }
    }
}

// ch: channel state (post NCO advance by the correlator); o: sums.
__device__ void loop_update(l1rxg_channel& ch, const l1rxg_corr& o, const LoopCfg& lc,
                            const LoopPre& p) {
    const l1rxg_tracking_cfg& cfg = lc.cfg;
    const bool noop = lc.kernel == L1RXG_KERNEL_NOOP;
    const double dt = (double)o.n_samples / lc.fs;
    const double e = p.e, l = p.l;
    const double e_env = e + l;
    const double dll_err = (e + l == 0.0) ? 0.0 : 0.5 * (e - l) / (e + l);  // :95-101
    if (e_env == 0.0 && !noop)
        ch.lock_fail_count++;
    const double pll_err = p.pll;  // :104-111
    if (ch.fll_enabled && ch.epochs_since_handoff < (int64_t)cfg.fll_pull_in_ms &&
        ch.carrier_lock_ratio < 0.8 && !noop) {  // :561-576
        if (ch.epochs_since_handoff < (int64_t)cfg.fll_coarse_ms) {
            ch.pll_integrator += 4.0 * cfg.fll_bandwidth_hz * 2.0 * PI_D * p.fc * dt;
        } else if (ch.have_last_prompt) {
            ch.pll_integrator += 4.0 * cfg.fll_bandwidth_hz * 2.0 * PI_D * p.ff * dt;
        }
    }
    const double doppler_cmd = loop_filter(ch.pll_integrator, ch.pll_prev_error, ch.pll_primed,
                                           pll_err, cfg.pll_bandwidth_hz, cfg.pll_damping, dt) /
                               (2.0 * PI_D);
    const double dll_cmd = loop_filter(ch.dll_integrator, ch.dll_prev_error, ch.dll_primed,
                                       dll_err, cfg.dll_bandwidth_hz, cfg.dll_damping, dt);
    ch.carrier_doppler_hz = doppler_cmd;
    ch.code_freq_hz = __fma_rn(CHIP_RATE_HZ, 1.0 + doppler_cmd / F_L1_HZ, dll_cmd);  // :142-147 (fma as compiled)
    ch.last_ip = o.ip;
    ch.last_qp = o.qp;
    ch.have_last_prompt = 1;
    if (ch.state == L1RXG_ACQUIRED)
        ch.state = L1RXG_TRACKING;

    // update_quality_metrics (:459-515)
    const double pwr = o.ip * o.ip + o.qp * o.qp;
    const double clr = pwr > 0 ? (o.ip * o.ip - o.qp * o.qp) / pwr : 0.0;
    const double alpha = 1.0 / (double)cfg.cn0_window_ms;
    ch.carrier_lock_ratio += alpha * (clr - ch.carrier_lock_ratio);
    ch.win_ip[ch.win_len] = o.ip;
    ch.win_qp[ch.win_len] = o.qp;
    ch.win_len++;
    const int m = cfg.cn0_window_ms;
    if (ch.win_len >= m) {  // window sums and the C/N0 map come from lane 4
        ch.win_len = 0;
        ch.mu_smoothed = p.mu_s;
        ch.cn0_dbhz = p.cn0;
        ch.metrics_valid = 1;
    }
    if (ch.metrics_valid &&
        ch.epochs_since_handoff > cfg.fll_pull_in_ms + cfg.cn0_window_ms) {
        if (ch.cn0_dbhz < cfg.cn0_drop_dbhz || ch.carrier_lock_ratio < cfg.carrier_lock_drop)
            ch.lock_fail_count++;
        else
            ch.lock_fail_count = 0;
    }
    if (ch.lock_fail_count > cfg.lock_fail_limit)
        ch.state = L1RXG_IDLE;
    ch.epoch_ms_count++;
    ch.epochs_since_handoff++;
    ch.sample_offset_next_epoch += o.n_samples;
}

// NCO advance over n samples (tracking.hpp:275-280, fma as compiled)
__device__ __forceinline__ void advance_nco(double& code_phase, double& carrier_phase,
                                            double& chi, const EpochConsts& c) {
    carrier_phase = fmod(__fma_rn(c.w, (double)c.n, carrier_phase), 2.0 * PI_D);
    const double adv = __dmul_rn((double)c.n, c.cps);
    code_phase = fmod(__dadd_rn(code_phase, adv), 1023.0);
    chi = __dadd_rn(chi, adv);
}

// ---------------------------------------------------------------------
// Shared-memory layout of the correlator CTA.
template <int T>
struct CorrSmem {
    l1rxg_channel ch;
    EpochConsts c;
    double d[T > 0 ? T : 1];
    double sums[2 * T + 2];
    float red[32 * (2 * T + 2)];
    float2 rot[RUN + 1];
    float chipf[CHIP_EXT];  // chips[m mod 1023] as +/-1.0f, m < CHIP_EXT
    LoopPre pre;
    int flags;
};

// chipf[m] = chips[m mod 1023] (the reference's code_ext idea,
// tracking.hpp:168-173, extended so no modulo is needed on the hot path)
__device__ __forceinline__ void fill_chips(float* chipf, const int8_t* codes, int prn) {
    for (int k = threadIdx.x; k < CHIP_EXT; k += blockDim.x)
        chipf[k] = (float)codes[prn * 1023 + (k % 1023)];
}

template <int T>
__device__ __forceinline__ void run_dispatch(const EpochConsts& c, float2* run, const float2* rot,
                                             const float* chipf, const double* d, int kp, int i0,
                                             int cnt, float* acc) {
    if (cnt == RUN)
        process_run<T, true>(c, run, rot, chipf, d, kp, i0, cnt, acc);
    else
        process_run<T, false>(c, run, rot, chipf, d, kp, i0, cnt, acc);
}

template <int T>
__device__ __forceinline__ float2* tile_of(CorrSmem<T>* s) {
    return reinterpret_cast<float2*>(reinterpret_cast<char*>(s) +
                                     ((sizeof(CorrSmem<T>) + 15) & ~size_t(15)));
}

// Correlates one epoch window (samples src[0..n)) with the consts in
// s->c; leaves fp64 tap sums in s->sums[0..2T) and the first-half prompt
// in s->sums[2T..2T+2).  All threads participate.
template <int T>
__device__ void correlate_epoch(CorrSmem<T>* s, const float2* __restrict__ src, int kp) {
    float2* tile = tile_of(s);
    const EpochConsts c = s->c;
    const int cap = blockDim.x * RUN;
    float acc[2 * T + 2];
#pragma unroll
    for (int v = 0; v < 2 * T + 2; ++v)
        acc[v] = 0.f;
    for (int u0 = 0; u0 < c.n; u0 += cap) {
        const int len = min(cap, c.n - u0);
        load_tile(tile, src + u0, len, cap);
        __syncthreads();
        const int i0 = u0 + threadIdx.x * RUN;
        const int cnt = min(RUN, c.n - i0);
        if (cnt > 0)
            run_dispatch<T>(c, tile + threadIdx.x * RUN, s->rot, s->chipf, s->d, kp, i0, cnt, acc);
        __syncthreads();
    }
    block_reduce<2 * T + 2>(acc, s->red, s->sums);
}

// ---------------------------------------------------------------------
// Kernel arguments for closed-loop tracking.
struct TrackArgs {
    const float2* ring;       // [n_streams][ring_stride]
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
};

// Channel-resident persistent tracking kernel: one CTA per channel loops over
// its epochs with no host round trip.  The epoch window is brought into
// shared memory by the TMA engine (cp.async.bulk, two mbarrier-tracked
// halves); the copy of the next window is issued as soon as the current one
// has been consumed, so it overlaps the block reduction and the loop update.
struct TileLoad {
    int64_t pos;   // ring position of the first sample of the unit
    int delta;     // samples of alignment slack in front (0/1)
    int h;         // split point (samples, even) between the two halves
    int len;       // samples of the unit
};

__device__ __forceinline__ TileLoad plan_load(int64_t abs_first, int len, int64_t R) {
    TileLoad u;
    const int64_t pos = abs_first % R;
    u.delta = (int)(pos & 1);
    u.pos = pos - u.delta;
    u.len = len;
    u.h = 2 * ((len + u.delta) / 4);
    return u;
}

__device__ __forceinline__ void issue_load(const TileLoad& u, float2* tile, const float2* ring,
                                           uint64_t* bars) {
    const uint32_t total = (uint32_t)(((u.len + u.delta) * 8 + 15) & ~15);
    const uint32_t b0 = (uint32_t)u.h * 8u;
    mbar_expect_tx(&bars[0], b0);
    tma_load_1d(tile, ring + u.pos, b0, &bars[0]);
    mbar_expect_tx(&bars[1], total - b0);
    tma_load_1d(tile + u.h, ring + u.pos + u.h, total - b0, &bars[1]);
}

template <int T>
struct TrackSmem {
    CorrSmem<T> cs;
    uint64_t bars[2];
    TileLoad unit;      // the load in flight (or last issued)
    int inflight;       // a unit is in flight into the tile
};

template <int T>
__device__ __forceinline__ float2* track_tile(TrackSmem<T>* s) {
    return reinterpret_cast<float2*>(reinterpret_cast<char*>(s) +
                                     ((sizeof(TrackSmem<T>) + 15) & ~size_t(15)));
}

template <int T>
__global__ void __launch_bounds__(MAX_NT, 1) track_kernel(TrackArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TrackSmem<T>* ts = reinterpret_cast<TrackSmem<T>*>(smem_raw);
    CorrSmem<T>* s = &ts->cs;
    float2* tile = track_tile(ts);
    const int cidx = blockIdx.x;
    const int strm = a.chan_stream[cidx];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = (blockDim.x + 31) >> 5;
    constexpr int V = 2 * T + 2;
    const int cap = blockDim.x * RUN;
    const int n = a.n;
    const int nsub = (n + cap - 1) / cap;
    const bool noop = a.lc.kernel == L1RXG_KERNEL_NOOP;
    const int64_t avail = a.avail[strm];
    const float2* ring = a.ring + (int64_t)strm * a.ring_stride;
    if (threadIdx.x == 0) {
        s->ch = a.chans[cidx];
        mbar_init(&ts->bars[0], 1);
        mbar_init(&ts->bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        ts->inflight = 0;
    }
    for (int k = threadIdx.x; k < T; k += blockDim.x)
        s->d[k] = a.taps.offsets_chips[k];
    __syncthreads();
    fill_chips(s->chipf, a.codes, s->ch.prn);
    // first epoch: consts, rotators and the first tile load
    if (threadIdx.x == 0) {
        const l1rxg_channel& ch = s->ch;
        make_consts(s->c, ch.code_phase_chips, ch.code_freq_hz, ch.carrier_doppler_hz,
                    ch.carrier_phase_rad, a.lc.fs, n);
        const int64_t off = ch.sample_offset_next_epoch;
        if (!noop && ch.state != L1RXG_IDLE && a.max_epochs > 0 && off + n <= avail && off >= 0 &&
            off >= avail - a.ring_cap) {
            ts->unit = plan_load(off, min(cap, n), a.ring_cap);
            issue_load(ts->unit, tile, ring, ts->bars);
            ts->inflight = 1;
        }
    }
    __syncthreads();
    fill_rot(s->rot, s->c.w);
    __syncthreads();

    uint32_t phase = 0;
    int64_t e = 0;
    int64_t done = a.ecount[cidx];
    for (;;) {
        // epoch admission (uniform: every thread reads the same smem state)
        const int64_t off = s->ch.sample_offset_next_epoch;
        if (s->ch.state == L1RXG_IDLE || e >= a.max_epochs || off + n > avail)
            break;
        if (off < avail - a.ring_cap || off < 0) {  // window already overwritten
            if (threadIdx.x == 0)
                a.status[cidx] = 1;
            break;
        }
        const EpochConsts c = s->c;
        float acc[V];
#pragma unroll
        for (int v = 0; v < V; ++v)
            acc[v] = 0.f;
        for (int q = 0; q < nsub; ++q) {
            const int u0 = q * cap;
            const int i0 = u0 + threadIdx.x * RUN;
            const int cnt = min(RUN, n - i0);
            if (!noop) {
                const TileLoad u = ts->unit;
                const int r0 = u.delta + threadIdx.x * RUN;
                if (cnt > 0) {
                    if (r0 < u.h)
                        mbar_wait(&ts->bars[0], phase);
                    if (r0 + RUN > u.h)
                        mbar_wait(&ts->bars[1], phase);
                    run_dispatch<T>(c, tile + r0, s->rot, s->chipf, s->d, a.kp, i0, cnt, acc);
                }
                if (threadIdx.x == 0) {  // every phase completes before the next issue
                    mbar_wait(&ts->bars[0], phase);
                    mbar_wait(&ts->bars[1], phase);
                }
                phase ^= 1u;
            }
            if (q + 1 == nsub) {  // warp-level part of the block reduction
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    float x = acc[v];
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1)
                        x += __shfl_xor_sync(0xffffffffu, x, o);
                    if (lane == 0)
                        s->red[warp * V + v] = x;
                }
            }
            __syncthreads();  // tile consumed
            if (threadIdx.x == 0) {
                ts->inflight = 0;
                if (!noop) {
                    if (q + 1 < nsub) {
                        ts->unit = plan_load(off + (q + 1) * cap, min(cap, n - (q + 1) * cap), a.ring_cap);
                        issue_load(ts->unit, tile, ring, ts->bars);
                        ts->inflight = 1;
                    } else if (s->ch.state != L1RXG_IDLE && e + 1 < a.max_epochs &&
                               off + 2 * (int64_t)n <= avail) {
                        // speculative prefetch of the next epoch's first unit
                        ts->unit = plan_load(off + n, min(cap, n), a.ring_cap);
                        issue_load(ts->unit, tile, ring, ts->bars);
                        ts->inflight = 1;
                    }
                }
            }
            if (q + 1 < nsub)
                __syncthreads();  // publish the next unit
        }
        // ---- loop update: warps 0..PW-1 (PW <= 6) split the independent
        // transcendental pieces, then warp 0 / lane 0 applies them
        const int PW = min(nwarps, LOOP_PIECES);
        if (warp < PW) {
            if (warp == 0) {  // fp64 cross-warp totals
                for (int v = lane; v < V; v += 32) {
                    double sm = 0.0;
                    for (int w = 0; w < nwarps; ++w)
                        sm += (double)s->red[w * V + v];
                    s->sums[v] = sm;
                }
            }
            asm volatile("bar.sync 1, %0;" ::"r"(PW * 32) : "memory");
            l1rxg_corr o;
            o.ie = s->sums[2 * a.ke];
            o.qe = s->sums[2 * a.ke + 1];
            o.ip = s->sums[2 * a.kp];
            o.qp = s->sums[2 * a.kp + 1];
            o.il = s->sums[2 * a.kl];
            o.ql = s->sums[2 * a.kl + 1];
            o.ip_h1 = s->sums[2 * T];
            o.qp_h1 = s->sums[2 * T + 1];
            o.ip_h2 = o.ip - o.ip_h1;
            o.qp_h2 = o.qp - o.qp_h1;
            o.n_samples = c.n;
            o.pad_ = 0;
            if (lane == 0)
                for (int piece = warp; piece < LOOP_PIECES; piece += PW)
                    loop_piece(piece, s->pre, s->ch, o, a.lc, c);
            asm volatile("bar.sync 1, %0;" ::"r"(PW * 32) : "memory");
            const int64_t slot = (int64_t)cidx * a.max_records + (done % a.max_records);
            if (warp == 0 && a.tap_sums && lane < 2 * T)
                a.tap_sums[slot * (2 * T) + lane] = s->sums[lane];
            if (warp == 0 && lane == 0) {
                l1rxg_channel& ch = s->ch;
                const LoopPre pre = s->pre;
                l1rxg_epoch_record r;
                r.sample_offset_start = off;
                r.code_phase_in = ch.code_phase_chips;
                r.code_freq_in = ch.code_freq_hz;
                r.carrier_doppler_in = ch.carrier_doppler_hz;
                r.carrier_phase_in = ch.carrier_phase_rad;
                ch.code_phase_chips = pre.code_phase;
                ch.carrier_phase_rad = pre.carrier_phase;
                ch.chi_chips = pre.chi;
                loop_update(ch, o, a.lc, pre);
            r.epoch_index = ch.epoch_ms_count - 1;
            r.sample_offset_end = ch.sample_offset_next_epoch;
            r.prn = ch.prn;
            r.state = ch.state;
            r.n_samples = c.n;
            r.lock_fail_count = ch.lock_fail_count;
            r.ie = o.ie; r.qe = o.qe; r.ip = o.ip; r.qp = o.qp; r.il = o.il; r.ql = o.ql;
            r.ip_h1 = o.ip_h1; r.qp_h1 = o.qp_h1; r.ip_h2 = o.ip_h2; r.qp_h2 = o.qp_h2;
            r.carrier_doppler_hz = ch.carrier_doppler_hz;
            r.code_freq_hz = ch.code_freq_hz;
            r.code_phase_chips = ch.code_phase_chips;
            r.carrier_phase_rad = ch.carrier_phase_rad;
            r.chi_chips = ch.chi_chips;
            r.cn0_dbhz = ch.cn0_dbhz;
            r.carrier_lock_ratio = ch.carrier_lock_ratio;
            r.dll_integrator = ch.dll_integrator;
            r.pll_integrator = ch.pll_integrator;
            r.mu_smoothed = ch.mu_smoothed;
            r.dll_prev_error = ch.dll_prev_error;
            r.pll_prev_error = ch.pll_prev_error;
                a.recs[slot] = r;
                // next epoch's NCO constants
                make_consts(s->c, ch.code_phase_chips, ch.code_freq_hz, ch.carrier_doppler_hz,
                            ch.carrier_phase_rad, a.lc.fs, n);
            }
            if (warp == 0) {
                __syncwarp();
                fill_rot(s->rot, s->c.w);
            }
        }
        ++e;
        ++done;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (ts->inflight) {  // never leave a bulk copy in flight into freed smem
            mbar_wait(&ts->bars[0], phase);
            mbar_wait(&ts->bars[1], phase);
        }
        a.chans[cidx] = s->ch;
        a.ecount[cidx] = done;
    }
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
    const int j = blockIdx.x;
    const int prn = a.prns[j];
    fill_chips(s->chipf, a.codes, prn);
    for (int k = threadIdx.x; k < T; k += blockDim.x)
        s->d[k] = a.taps.offsets_chips[k];
    if (threadIdx.x == 0) {
        const l1rxg_nco st = a.states[j];
        make_consts(s->c, st.code_phase_chips, st.code_freq_hz, st.carrier_doppler_hz,
                    st.carrier_phase_rad, a.fs, a.n);
    }
    __syncthreads();
    fill_rot(s->rot, s->c.w);
    if (a.kernel != L1RXG_KERNEL_NOOP) {
        correlate_epoch<T>(s, a.samples + (int64_t)j * a.n, a.kp);
    } else {
        if (threadIdx.x < 2 * T + 2)
            s->sums[threadIdx.x] = 0.0;
        __syncthreads();
    }
    if (threadIdx.x < 2 * T)
        a.tap_sums[(int64_t)j * 2 * T + threadIdx.x] = s->sums[threadIdx.x];
    if (threadIdx.x == 0) {
        l1rxg_nco st = a.states[j];
        advance_nco(st.code_phase_chips, st.carrier_phase_rad, st.chi_chips, s->c);
        a.states[j] = st;
        l1rxg_corr o;
        o.ie = s->sums[2 * a.ke];
        o.qe = s->sums[2 * a.ke + 1];
        o.ip = s->sums[2 * a.kp];
        o.qp = s->sums[2 * a.kp + 1];
        o.il = s->sums[2 * a.kl];
        o.ql = s->sums[2 * a.kl + 1];
        o.ip_h1 = s->sums[2 * T];
        o.qp_h1 = s->sums[2 * T + 1];
        o.ip_h2 = o.ip - o.ip_h1;
        o.qp_h2 = o.qp - o.qp_h1;
        o.n_samples = a.n;
        o.pad_ = 0;
        a.corr[j] = o;
    }
}

// ---------------------------------------------------------------------
// K1 ingest.  Ring write: sample g -> ring[g mod R] (+ apron copy).
__device__ __forceinline__ void ring_put(float2* ring, int64_t R, int64_t apron,
                                         int64_t pos, float2 v) {
    ring[pos] = v;
    if (pos < apron)
        ring[R + pos] = v;
}

// Int8RealIF at IF = fs/4: the mixer step is exactly -pi/2, so
// mixed(g) = v(g)/128 * {1, -j, -1, j}[g mod 4]; the FIR output
// 2*sum_t h[t] mixed(g-t) (samples.hpp:234-240) is a 23-tap real
// convolution per output phase with coefficient tables cre/cim[4][23]
// folded on the host (includes the 2/128 scale).
__constant__ float c_if4_re[4][23];
__constant__ float c_if4_im[4][23];

constexpr int ING_TPB = 256;
constexpr int ING_OUT_PER_THREAD = 4;
constexpr int ING_TILE = ING_TPB * ING_OUT_PER_THREAD;  // outputs per block

// raw: bytes of samples [g0, g0+count); hist: the 22 bytes before g0
// (zeros at stream start); writes hist_out = the last 22 bytes of the run.
__global__ void __launch_bounds__(ING_TPB) ingest_if4_kernel(
    const int8_t* __restrict__ raw, const int8_t* __restrict__ hist, int8_t* hist_out,
    int64_t g0, int64_t count, float2* ring, int64_t R, int64_t apron, int64_t pos0,
    int64_t* avail_slot) {
    __shared__ float v[ING_TILE + 24];
    const int64_t t0 = (int64_t)blockIdx.x * ING_TILE;  // run-relative first output
    // inputs t0-22 .. t0+ING_TILE-1
    for (int k = threadIdx.x; k < ING_TILE + 22; k += ING_TPB) {
        const int64_t idx = t0 - 22 + k;
        int8_t b = 0;
        if (idx < 0)
            b = hist[22 + idx];
        else if (idx < count)
            b = raw[idx];
        v[k] = (float)b;
    }
    __syncthreads();
    const int q = threadIdx.x * ING_OUT_PER_THREAD;
#pragma unroll
    for (int u = 0; u < ING_OUT_PER_THREAD; ++u) {
        const int64_t idx = t0 + q + u;
        if (idx >= count)
            break;
        const int ph = (int)((g0 + idx) & 3);
        float re = 0.f, im = 0.f;
#pragma unroll
        for (int t = 0; t < 23; ++t) {
            const float x = v[q + u + 22 - t];
            re = fmaf(c_if4_re[ph][t], x, re);
            im = fmaf(c_if4_im[ph][t], x, im);
        }
        int64_t pos = pos0 + idx;
        if (pos >= R)
            pos -= R;
        ring_put(ring, R, apron, pos, make_float2(re, im));
    }
    if (blockIdx.x == 0 && threadIdx.x < 22) {
        const int64_t idx = count - 22 + threadIdx.x;
        hist_out[threadIdx.x] = idx >= 0 ? raw[idx] : hist[22 + idx];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && avail_slot)
        *avail_slot = g0 + count;
}

// Generic real IF: pass 1, mixer at the global index in fp64
// (samples.hpp:217-226) into mixed[22 + i]; mixed[0..22) holds history.
__global__ void mix_generic_kernel(const int8_t* __restrict__ raw, int64_t g0, int64_t count,
                                   double w, float2* mixed) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count)
        return;
    const double vv = (double)raw[i] / 128.0;
    double s, c;
    sincos(w * (double)(g0 + i), &s, &c);
    mixed[22 + i] = make_float2((float)(vv * c), (float)(vv * s));
}

// pass 2: out(g) = 2 sum_t h[t] mixed(g - t)
__constant__ float c_halfband2[23];
__global__ void fir_generic_kernel(const float2* __restrict__ mixed, int64_t count, float2* ring,
                                   int64_t R, int64_t apron, int64_t pos0, float2* hist_out,
                                   int64_t* avail_slot, int64_t avail_value) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) {
        float re = 0.f, im = 0.f;
#pragma unroll
        for (int t = 0; t < 23; ++t) {
            const float2 m = mixed[22 + i - t];
            re = fmaf(c_halfband2[t], m.x, re);
            im = fmaf(c_halfband2[t], m.y, im);
        }
        int64_t pos = pos0 + i;
        if (pos >= R)
            pos -= R;
        ring_put(ring, R, apron, pos, make_float2(re, im));
    }
    if (blockIdx.x == 0 && threadIdx.x < 22)
        hist_out[threadIdx.x] = mixed[count + threadIdx.x];
    if (blockIdx.x == 0 && threadIdx.x == 0 && avail_slot)
        *avail_slot = avail_value;
}

// Complex int8 / int16 decode (samples.hpp:188-205).
__global__ void decode_iq_kernel(const void* __restrict__ raw, int fmt, int64_t count,
                                 float2* ring, int64_t R, int64_t apron, int64_t pos0,
                                 int64_t* avail_slot, int64_t avail_value) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) {
        float2 v;
        if (fmt == L1RXG_FMT_INT8_IQ) {
            const char2 b = reinterpret_cast<const char2*>(raw)[i];
            v = make_float2((float)b.x * (1.0f / 128.0f), (float)b.y * (1.0f / 128.0f));
        } else {
            const short2 b = reinterpret_cast<const short2*>(raw)[i];
            v = make_float2((float)b.x * (1.0f / 32768.0f), (float)b.y * (1.0f / 32768.0f));
        }
        int64_t pos = pos0 + i;
        if (pos >= R)
            pos -= R;
        ring_put(ring, R, apron, pos, v);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && avail_slot)
        *avail_slot = avail_value;
}

// complex<double> -> float2 (per-call path)
__global__ void cf64_to_f32_kernel(const double2* __restrict__ in, float2* out, int64_t count) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) {
        const double2 x = in[i];
        out[i] = make_float2((float)x.x, (float)x.y);
    }
}

}  // namespace l1rxg
