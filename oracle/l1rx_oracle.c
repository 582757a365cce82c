/*
 * oracle/l1rx_oracle.c -- TEST INFRASTRUCTURE: the CPU oracle.
 *
 * A plain-C restatement of the reference's hot path (l1rx,
 * /root/reference/proj/include/l1rx), written from its semantics, used
 * ONLY as the checker by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg.  The product (libl1rxg.so) never links or calls it.
 *
 * Parity pin: tests/test_oracle.py checks every function here against the
 * reference itself (oracle/_ref/libl1rx_ref.so, built from the unmodified
 * headers) and against the golden fixtures in tests/golden/ generated from
 * it (tests/golden/make_golden.py), plus the reference's own known-answer
 * tests restated (test_cacode.cpp, test_tracking.cpp, test_samples.cpp).
 *
 * Floating point: built with -ffp-contract=off; every multiply-add that
 * the reference's Release build (g++ -O3 -march=native) contracts into an
 * FMA is written as an explicit fma() so chip decisions and NCO state
 * advance are bit-identical to the reference (verified by objdump of the
 * reference build: ph = fma(i, cps, base), theta = fma(w, i, phi),
 * carrier advance = fma(w, n, phi); tracking.hpp:244-280).
 *
 * Builder extensions (NOT reference code, labelled where they occur):
 *   - the K-tap correlator (orc_correlate with n_taps != 3), whose 3-tap
 *     E/P/L instance is the reference expression bit for bit;
 *   - the multi-threaded closed-loop driver orc_track_run (the reference
 *     pipeline caps at 12 channels, pipeline.hpp:769).
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "l1rxg.h"

#define PI_D 3.14159265358979323846 /* constants.hpp:20 */
#define F_L1_HZ 1.57542e9           /* constants.hpp:5  */
#define CHIP_RATE_HZ 1.023e6        /* constants.hpp:6  */

static __thread char g_err[256];
const char* orc_last_error(void) { return g_err; }
static int fail(int code, const char* msg) {
    strncpy(g_err, msg, sizeof g_err - 1);
    g_err[sizeof g_err - 1] = 0;
    return code;
}

/* ---- C/A codes: cacode.hpp:20-64 ------------------------------------ */
/* G2 phase-select tap pairs per PRN (IS-GPS-200 Table 3-I), cacode.hpp:24-30 */
static const int k_g2_taps[33][2] = {
    {0, 0},  {2, 6}, {3, 7}, {4, 8},  {5, 9}, {1, 9},  {2, 10}, {1, 8}, {2, 9},
    {3, 10}, {2, 3}, {3, 4}, {5, 6},  {6, 7}, {7, 8},  {8, 9},  {9, 10}, {1, 4},
    {2, 5},  {3, 6}, {4, 7}, {5, 8},  {6, 9}, {1, 3},  {4, 6},  {5, 7},  {6, 8},
    {7, 9},  {8, 10}, {1, 6}, {2, 7}, {3, 8}, {4, 9},
};

/* Registers as 10-bit words, bit j = stage j+1.  G1 = x^10+x^3+1,
 * G2 = x^10+x^9+x^8+x^6+x^3+x^2+1; chip = 1 - 2*(g1_out ^ g2_out). */
int orc_ca_code(int prn, int8_t* out) {
    if (prn < 1 || prn > 32)
        return fail(L1RXG_ERANGE, "PRN must be in 1..32");
    unsigned g1 = 0x3FF, g2 = 0x3FF;
    const int t1 = k_g2_taps[prn][0] - 1, t2 = k_g2_taps[prn][1] - 1;
    for (int i = 0; i < 1023; ++i) {
        const unsigned o1 = (g1 >> 9) & 1u;
        const unsigned o2 = ((g2 >> t1) ^ (g2 >> t2)) & 1u;
        out[i] = (int8_t)(1 - 2 * (int)(o1 ^ o2));
        const unsigned f1 = ((g1 >> 2) ^ (g1 >> 9)) & 1u;
        const unsigned f2 =
            ((g2 >> 1) ^ (g2 >> 2) ^ (g2 >> 5) ^ (g2 >> 7) ^ (g2 >> 8) ^ (g2 >> 9)) & 1u;
        g1 = ((g1 << 1) | f1) & 0x3FF;
        g2 = ((g2 << 1) | f2) & 0x3FF;
    }
    return 0;
}

static int8_t g_codes[33][1023];
static pthread_once_t g_codes_once = PTHREAD_ONCE_INIT;
static void init_codes(void) {
    for (int p = 1; p <= 32; ++p)
        orc_ca_code(p, g_codes[p]);
}
static const int8_t* code_of(int prn) {
    pthread_once(&g_codes_once, init_codes);
    return g_codes[prn];
}

/* resample_code_into (cacode.hpp:66-83): out[i] = chips[floor(phase +
 * i*rate) mod 1023]. */
int orc_resample_code(int prn, double fs, double code_phase, double code_freq,
                      int n, int8_t* out) {
    if (prn < 1 || prn > 32)
        return fail(L1RXG_ERANGE, "PRN must be in 1..32");
    if (code_freq <= 0.0)
        return fail(L1RXG_EINVAL, "code_freq_hz must be positive");
    if (n <= 0)
        return fail(L1RXG_EINVAL, "n_samples must be positive");
    const int8_t* c = code_of(prn);
    const double rate = code_freq / fs;
    for (int i = 0; i < n; ++i) {
        int64_t idx = (int64_t)floor(fma((double)i, rate, code_phase));
        idx %= 1023;
        if (idx < 0)
            idx += 1023;
        out[i] = c[idx];
    }
    return 0;
}

/* ---- ingest: samples.hpp:85-253 ------------------------------------- */
/* detail::halfband_taps: 23-tap Hamming-windowed sinc, cutoff fs/4, unit
 * DC gain (samples.hpp:89-108). */
void orc_halfband_taps(double* h) {
    double sum = 0.0;
    for (int n = 0; n < 23; ++n) {
        const double k = (double)(n - 11);
        double v = (n == 11) ? 0.5 : sin(PI_D * k / 2.0) / (PI_D * k);
        v *= 0.54 - 0.46 * cos(2.0 * PI_D * n / 22.0);
        h[n] = v;
        sum += v;
    }
    for (int n = 0; n < 23; ++n)
        h[n] /= sum;
}

typedef struct {
    int32_t format;
    int32_t pad_;
    double fs, if_hz;
    int64_t consumed;   /* input_samples_consumed_ (samples.hpp:261) */
    double hist[2 * 22]; /* fir_history_ (samples.hpp:258), oldest first */
} orc_ingest_state;

int orc_ingest_state_size(void) { return (int)sizeof(orc_ingest_state); }

void orc_ingest_init(orc_ingest_state* st, int format, double fs, double if_hz) {
    memset(st, 0, sizeof *st);
    st->format = format;
    st->fs = fs;
    st->if_hz = if_hz;
}

/* read_samples (samples.hpp:177-211) + downconvert (:215-253) over a byte
 * run.  Block framing does not change the values (history and the global
 * mixer index are carried), so any chunking gives the same stream. */
int64_t orc_ingest(orc_ingest_state* st, const uint8_t* raw, int64_t nbytes,
                   double* iq) {
    if (st->format == L1RXG_FMT_INT8_IQ) {
        const int64_t n = nbytes / 2;
        for (int64_t i = 0; i < n; ++i) {
            iq[2 * i] = (int8_t)raw[2 * i] / 128.0;
            iq[2 * i + 1] = (int8_t)raw[2 * i + 1] / 128.0;
        }
        return n;
    }
    if (st->format == L1RXG_FMT_INT16_IQ) {
        const int64_t n = nbytes / 4;
        for (int64_t i = 0; i < n; ++i) {
            const int16_t a = (int16_t)((uint16_t)raw[4 * i] | ((uint16_t)raw[4 * i + 1] << 8));
            const int16_t b = (int16_t)((uint16_t)raw[4 * i + 2] | ((uint16_t)raw[4 * i + 3] << 8));
            iq[2 * i] = a / 32768.0;
            iq[2 * i + 1] = b / 32768.0;
        }
        return n;
    }
    /* Int8RealIF: mixer at -IF (global index), then the half-band FIR with
     * carried history, output x2. */
    double h[23];
    orc_halfband_taps(h);
    const int64_t n = nbytes;
    const double w = -2.0 * PI_D * st->if_hz / st->fs;
    double* mixed = (double*)malloc((size_t)(n + 22) * 2 * sizeof(double));
    memcpy(mixed, st->hist, sizeof st->hist);
    for (int64_t i = 0; i < n; ++i) {
        const double v = (int8_t)raw[i] / 128.0;
        const double ph = w * (double)(st->consumed + i);
        mixed[2 * (22 + i)] = v * cos(ph);
        mixed[2 * (22 + i) + 1] = v * sin(ph);
    }
    st->consumed += n;
    for (int64_t i = 0; i < n; ++i) {
        double ar = 0.0, ai = 0.0;
        for (int t = 0; t < 23; ++t) {
            const double* p = &mixed[2 * (i + 22 - t)];
            ar = fma(h[t], p[0], ar);
            ai = fma(h[t], p[1], ai);
        }
        iq[2 * i] = 2.0 * ar;
        iq[2 * i + 1] = 2.0 * ai;
    }
    memcpy(st->hist, &mixed[2 * n], sizeof st->hist); /* last 22 mixed */
    free(mixed);
    return n;
}

/* ---- correlator: tracking.hpp:226-282 (K-tap generalisation) --------- */
static void advance(l1rxg_nco* st, double w, double cps, int n) {
    /* tracking.hpp:275-280 */
    st->carrier_phase_rad = fmod(fma(w, (double)n, st->carrier_phase_rad), 2.0 * PI_D);
    const double adv = (double)n * cps;
    st->code_phase_chips = fmod(st->code_phase_chips + adv, 1023.0);
    st->chi_chips += adv;
}

/* Reference contract of correlate_epoch_scalar on K taps: tap k's replica
 * chip at sample i is chips[trunc(fl(fma(i, cps, base) + offsets[k])) mod
 * 1023] with base = code_phase + 1023; the 3-tap instance with offsets
 * (+s/2, 0, -s/2) is the reference expression.  tap_sums[2k], [2k+1] =
 * sum of wr*chip, wi*chip; half sums on the prompt tap split at n/2. */
int orc_correlate(int kernel, const double* iq, int n, l1rxg_nco* st, int prn,
                  const l1rxg_taps* taps, double fs, double* tap_sums,
                  l1rxg_corr* out) {
    if (n <= 0)
        return fail(L1RXG_EINVAL, "empty epoch view");
    if (prn < 1 || prn > 32)
        return fail(L1RXG_ERANGE, "PRN must be in 1..32");
    const int K = taps->n_taps;
    const double w = 2.0 * PI_D * st->carrier_doppler_hz / fs;
    const double cps = st->code_freq_hz / fs;
    memset(out, 0, sizeof *out);
    out->n_samples = n;
    if (tap_sums)
        memset(tap_sums, 0, sizeof(double) * 2 * (size_t)K);
    if (kernel == L1RXG_KERNEL_NOOP) {
        advance(st, w, cps, n);
        return 0;
    }
    const int8_t* c = code_of(prn);
    const double base = st->code_phase_chips + 1023.0;
    const int nh = n / 2, kp = taps->prompt;
    double acc[2 * L1RXG_MAX_TAPS] = {0};
    double h1r = 0, h1i = 0, h2r = 0, h2i = 0;
    for (int i = 0; i < n; ++i) {
        const double th = fma(w, (double)i, st->carrier_phase_rad);
        const double cs = cos(th), sn = sin(th);
        const double xr = iq[2 * i], xi = iq[2 * i + 1];
        const double wr = xr * cs + xi * sn;
        const double wi = xi * cs - xr * sn;
        const double ph = fma((double)i, cps, base);
        for (int k = 0; k < K; ++k) {
            const int64_t idx = (int64_t)(ph + taps->offsets_chips[k]);
            const double chip = c[idx % 1023];
            acc[2 * k] += wr * chip;
            acc[2 * k + 1] += wi * chip;
            if (k == kp) {
                if (i < nh) {
                    h1r += wr * chip;
                    h1i += wi * chip;
                } else {
                    h2r += wr * chip;
                    h2i += wi * chip;
                }
            }
        }
    }
    out->ie = acc[2 * taps->early];
    out->qe = acc[2 * taps->early + 1];
    out->ip = acc[2 * kp];
    out->qp = acc[2 * kp + 1];
    out->il = acc[2 * taps->late];
    out->ql = acc[2 * taps->late + 1];
    out->ip_h1 = h1r;
    out->qp_h1 = h1i;
    out->ip_h2 = h2r;
    out->qp_h2 = h2i;
    if (tap_sums)
        memcpy(tap_sums, acc, sizeof(double) * 2 * (size_t)K);
    advance(st, w, cps, n);
    return 0;
}

/* ---- loop: tracking.hpp:65-147 --------------------------------------- */
static double natural_frequency(double bw, double zeta) {
    return 8.0 * zeta * bw / (4.0 * zeta * zeta + 1.0);
}

double orc_loop_filter_update(double* integ, double* prev, int32_t* primed,
                              double err, double bw, double zeta, double dt) {
    const double wn = natural_frequency(bw, zeta);
    const double p = *primed ? *prev : err;
    *integ += wn * wn * dt * 0.5 * (err + p);
    *prev = err;
    *primed = 1;
    return *integ + 2.0 * zeta * wn * err;
}

double orc_dll_discriminator(const l1rxg_corr* o) {
    const double e = sqrt(o->ie * o->ie + o->qe * o->qe);
    const double l = sqrt(o->il * o->il + o->ql * o->ql);
    if (e + l == 0.0)
        return 0.0;
    return 0.5 * (e - l) / (e + l);
}

double orc_pll_discriminator(double ip, double qp) {
    if (ip == 0.0) {
        if (qp == 0.0)
            return 0.0;
        return qp > 0 ? PI_D / 2.0 : -PI_D / 2.0;
    }
    return atan(qp / ip);
}

double orc_fll_discriminator(double pi_, double pq, double ci, double cq,
                             double dt) {
    const double cross = pi_ * cq - pq * ci;
    const double dot = pi_ * ci + pq * cq;
    if (cross == 0.0 && dot == 0.0)
        return 0.0;
    return atan2(cross, dot) / (2.0 * PI_D * dt);
}

double orc_fll_discriminator_di(double pi_, double pq, double ci, double cq,
                                double dt) {
    double cross = pi_ * cq - pq * ci;
    double dot = pi_ * ci + pq * cq;
    if (dot < 0) {
        cross = -cross;
        dot = -dot;
    }
    if (cross == 0.0 && dot == 0.0)
        return 0.0;
    return atan2(cross, dot) / (2.0 * PI_D * dt);
}

double orc_carrier_aid(double doppler, double dll) {
    return fma(CHIP_RATE_HZ, 1.0 + doppler / F_L1_HZ, dll); /* contracted as compiled */
}

/* update_quality_metrics (tracking.hpp:459-515) */
void orc_update_quality_metrics(l1rxg_channel* ch, const l1rxg_corr* o,
                                const l1rxg_tracking_cfg* cfg) {
    const double pwr = o->ip * o->ip + o->qp * o->qp;
    const double clr = pwr > 0 ? (o->ip * o->ip - o->qp * o->qp) / pwr : 0.0;
    const double alpha = 1.0 / (double)cfg->cn0_window_ms;
    ch->carrier_lock_ratio += alpha * (clr - ch->carrier_lock_ratio);
    const int m = cfg->cn0_window_ms;
    double nbi = 0, nbq = 0, wbp = 0;
    int full = 0;
    if (m <= L1RXG_WIN_MAX) {
        ch->win_ip[ch->win_len] = o->ip;
        ch->win_qp[ch->win_len] = o->qp;
        ch->win_len++;
        if (ch->win_len >= m) {
            for (int k = 0; k < m; ++k) {
                const double sg = ch->win_ip[k] >= 0 ? 1.0 : -1.0;
                nbi += sg * ch->win_ip[k];
                nbq += sg * ch->win_qp[k];
                wbp += ch->win_ip[k] * ch->win_ip[k] + ch->win_qp[k] * ch->win_qp[k];
            }
            full = 1;
        }
    } else {
        /* windows longer than the POD's arrays: the same sums accumulated in
           push order (win_ip[0], win_qp[0], win_ip[1]) -- the reference's
           loop over the window vectors sums in exactly this order */
        if (ch->win_len > 0) {
            nbi = ch->win_ip[0];
            nbq = ch->win_qp[0];
            wbp = ch->win_ip[1];
        }
        const double sg = o->ip >= 0 ? 1.0 : -1.0;
        nbi += sg * o->ip;
        nbq += sg * o->qp;
        wbp += o->ip * o->ip + o->qp * o->qp;
        ch->win_len++;
        full = ch->win_len >= m;
        if (!full) {
            ch->win_ip[0] = nbi;
            ch->win_qp[0] = nbq;
            ch->win_ip[1] = wbp;
        }
    }
    if (full) {
        ch->win_len = 0;
        const double mu = wbp > 0 ? (nbi * nbi + nbq * nbq) / wbp : 0.0;
        ch->mu_smoothed = ch->metrics_valid ? ch->mu_smoothed + 0.2 * (mu - ch->mu_smoothed) : mu;
        const double md = (double)m;
        if (ch->mu_smoothed >= md - 1e-9)
            ch->cn0_dbhz = 65.0;
        else if (ch->mu_smoothed <= 1.0)
            ch->cn0_dbhz = 0.0;
        else
            ch->cn0_dbhz = 10.0 * log10((ch->mu_smoothed - 1.0) / (md - ch->mu_smoothed) / 1e-3);
        ch->metrics_valid = 1;
    }
    if (ch->metrics_valid &&
        ch->epochs_since_handoff > cfg->fll_pull_in_ms + cfg->cn0_window_ms) {
        if (ch->cn0_dbhz < cfg->cn0_drop_dbhz || ch->carrier_lock_ratio < cfg->carrier_lock_drop)
            ch->lock_fail_count++;
        else
            ch->lock_fail_count = 0;
    }
    if (ch->lock_fail_count > cfg->lock_fail_limit)
        ch->state = L1RXG_IDLE; /* nav reset happens on the host consumer */
}

/* track_epoch (tracking.hpp:520-618) with the K-tap correlator. */
int orc_track_epoch(l1rxg_channel* ch, const double* iq, int n,
                    const l1rxg_tracking_cfg* cfg, const l1rxg_taps* taps,
                    double fs, int kernel, l1rxg_epoch_record* rec,
                    double* tap_sums) {
    if (ch->state == L1RXG_IDLE)
        return fail(L1RXG_ELOGIC, "track_epoch on an idle channel");
    l1rxg_nco nco = {ch->code_phase_chips, ch->code_freq_hz,
                     ch->carrier_doppler_hz, ch->carrier_phase_rad, ch->chi_chips};
    const l1rxg_nco in = nco;
    const int64_t start = ch->sample_offset_next_epoch;
    const double chi_at_start = ch->chi_chips;
    (void)chi_at_start; /* nav::on_prompt input; nav runs on the host */
    l1rxg_corr o;
    int rc = orc_correlate(kernel, iq, n, &nco, ch->prn, taps, fs, tap_sums, &o);
    if (rc)
        return rc;
    ch->code_phase_chips = nco.code_phase_chips;
    ch->carrier_phase_rad = nco.carrier_phase_rad;
    ch->chi_chips = nco.chi_chips;
    const double dt = (double)o.n_samples / fs;

    const double e_env = sqrt(o.ie * o.ie + o.qe * o.qe) + sqrt(o.il * o.il + o.ql * o.ql);
    const double dll_err = orc_dll_discriminator(&o);
    if (e_env == 0.0 && kernel != L1RXG_KERNEL_NOOP)
        ch->lock_fail_count++;
    const double pll_err = orc_pll_discriminator(o.ip, o.qp);

    if (ch->fll_enabled && ch->epochs_since_handoff < (int64_t)cfg->fll_pull_in_ms &&
        ch->carrier_lock_ratio < 0.8 && kernel != L1RXG_KERNEL_NOOP) {
        if (ch->epochs_since_handoff < (int64_t)cfg->fll_coarse_ms) {
            const double f = orc_fll_discriminator(o.ip_h1, o.qp_h1, o.ip_h2, o.qp_h2, dt / 2.0);
            ch->pll_integrator += 4.0 * cfg->fll_bandwidth_hz * 2.0 * PI_D * f * dt;
        } else if (ch->have_last_prompt) {
            const double f = orc_fll_discriminator_di(ch->last_ip, ch->last_qp, o.ip, o.qp, dt);
            ch->pll_integrator += 4.0 * cfg->fll_bandwidth_hz * 2.0 * PI_D * f * dt;
        }
    }
    const double doppler_cmd =
        orc_loop_filter_update(&ch->pll_integrator, &ch->pll_prev_error, &ch->pll_primed,
                               pll_err, cfg->pll_bandwidth_hz, cfg->pll_damping, dt) /
        (2.0 * PI_D);
    const double dll_cmd =
        orc_loop_filter_update(&ch->dll_integrator, &ch->dll_prev_error, &ch->dll_primed,
                               dll_err, cfg->dll_bandwidth_hz, cfg->dll_damping, dt);
    ch->carrier_doppler_hz = doppler_cmd;
    ch->code_freq_hz = orc_carrier_aid(doppler_cmd, dll_cmd);
    ch->last_ip = o.ip;
    ch->last_qp = o.qp;
    ch->have_last_prompt = 1;
    if (ch->state == L1RXG_ACQUIRED)
        ch->state = L1RXG_TRACKING;
    orc_update_quality_metrics(ch, &o, cfg);
    ch->epoch_ms_count++;
    ch->epochs_since_handoff++;
    ch->sample_offset_next_epoch += o.n_samples;

    if (rec) {
        memset(rec, 0, sizeof *rec);
        rec->epoch_index = ch->epoch_ms_count - 1;
        rec->sample_offset_start = start;
        rec->sample_offset_end = ch->sample_offset_next_epoch;
        rec->prn = ch->prn;
        rec->state = ch->state;
        rec->n_samples = o.n_samples;
        rec->lock_fail_count = ch->lock_fail_count;
        rec->code_phase_in = in.code_phase_chips;
        rec->code_freq_in = in.code_freq_hz;
        rec->carrier_doppler_in = in.carrier_doppler_hz;
        rec->carrier_phase_in = in.carrier_phase_rad;
        rec->ie = o.ie; rec->qe = o.qe; rec->ip = o.ip; rec->qp = o.qp;
        rec->il = o.il; rec->ql = o.ql;
        rec->ip_h1 = o.ip_h1; rec->qp_h1 = o.qp_h1;
        rec->ip_h2 = o.ip_h2; rec->qp_h2 = o.qp_h2;
        rec->carrier_doppler_hz = ch->carrier_doppler_hz;
        rec->code_freq_hz = ch->code_freq_hz;
        rec->code_phase_chips = ch->code_phase_chips;
        rec->carrier_phase_rad = ch->carrier_phase_rad;
        rec->chi_chips = ch->chi_chips;
        rec->cn0_dbhz = ch->cn0_dbhz;
        rec->carrier_lock_ratio = ch->carrier_lock_ratio;
        rec->dll_integrator = ch->dll_integrator;
        rec->pll_integrator = ch->pll_integrator;
        rec->mu_smoothed = ch->mu_smoothed;
        rec->dll_prev_error = ch->dll_prev_error;
        rec->pll_prev_error = ch->pll_prev_error;
    }
    return 0;
}

/* init_channel_from_acquisition (tracking.hpp:622-650) */
void orc_init_channel(l1rxg_channel* ch, int prn, double doppler,
                      int64_t acq_start, int code_delay, int64_t start_offset,
                      double fs) {
    memset(ch, 0, sizeof *ch);
    ch->prn = prn;
    ch->state = L1RXG_ACQUIRED;
    ch->carrier_doppler_hz = doppler;
    ch->code_freq_hz = orc_carrier_aid(doppler, 0.0);
    ch->pll_integrator = 2.0 * PI_D * doppler;
    ch->fll_enabled = 1;
    const int64_t spm = llround(fs / 1000.0);
    const int64_t boundary = acq_start + code_delay;
    int64_t start = boundary;
    if (start < start_offset) {
        const int64_t gap = start_offset - boundary;
        start = boundary + ((gap + spm - 1) / spm) * spm;
    }
    ch->sample_offset_next_epoch = start;
    const double cps = ch->code_freq_hz / fs;
    ch->code_phase_chips = fmod((double)(start - boundary) * cps, 1023.0);
    ch->chi_chips = ch->code_phase_chips;
}

void orc_default_cfg(l1rxg_tracking_cfg* c) {
    memset(c, 0, sizeof *c);
    c->epoch_ms = 1;
    c->el_spacing_chips = 0.5;
    c->dll_bandwidth_hz = 2.0;
    c->dll_damping = 0.707;
    c->pll_bandwidth_hz = 25.0;
    c->pll_damping = 0.707;
    c->fll_bandwidth_hz = 15.0;
    c->fll_pull_in_ms = 400;
    c->fll_coarse_ms = 100;
    c->cn0_window_ms = 20;
    c->lock_fail_limit = 50;
    c->cn0_drop_dbhz = 28.0;
    c->carrier_lock_drop = 0.6;
}

/* ---- closed-loop driver (builder extension) -------------------------- */
/* Runs each channel over a complex<double> buffer per stream until its
 * next window leaves the buffer, the channel goes Idle or max_epochs is
 * reached, like run_closed_loop (test_tracking.cpp:368-399); channels are
 * spread over `threads` POSIX threads like ChannelPool. */
typedef struct {
    l1rxg_channel* chans;
    const int32_t* chan_stream;
    const double* const* streams;
    const int64_t* stream_len;
    int n_channels, n;
    const l1rxg_tracking_cfg* cfg;
    const l1rxg_taps* taps;
    double fs;
    int kernel;
    int64_t max_epochs;
    l1rxg_epoch_record* recs; /* [channel][max_epochs] or NULL */
    double* tap_sums;         /* [channel][max_epochs][2K] or NULL */
    int64_t* done;
    int next;
    pthread_mutex_t mu;
} run_job;

static void* run_worker(void* arg) {
    run_job* j = (run_job*)arg;
    const int K = j->taps->n_taps;
    for (;;) {
        pthread_mutex_lock(&j->mu);
        const int c = j->next++;
        pthread_mutex_unlock(&j->mu);
        if (c >= j->n_channels)
            return NULL;
        l1rxg_channel* ch = &j->chans[c];
        const double* s = j->streams[j->chan_stream[c]];
        const int64_t len = j->stream_len[j->chan_stream[c]];
        int64_t e = 0;
        while (e < j->max_epochs && ch->state != L1RXG_IDLE &&
               ch->sample_offset_next_epoch + j->n <= len) {
            l1rxg_epoch_record* r = j->recs ? &j->recs[(int64_t)c * j->max_epochs + e] : NULL;
            double* ts = j->tap_sums ? &j->tap_sums[((int64_t)c * j->max_epochs + e) * 2 * K] : NULL;
            orc_track_epoch(ch, s + 2 * ch->sample_offset_next_epoch, j->n, j->cfg, j->taps,
                            j->fs, j->kernel, r, ts);
            ++e;
        }
        j->done[c] = e;
    }
}

int orc_track_run(l1rxg_channel* chans, const int32_t* chan_stream, int n_channels,
                  const double* const* streams, const int64_t* stream_len, int n,
                  const l1rxg_tracking_cfg* cfg, const l1rxg_taps* taps, double fs,
                  int kernel, int64_t max_epochs, int threads,
                  l1rxg_epoch_record* recs, double* tap_sums, int64_t* done) {
    run_job j = {chans, chan_stream, streams, stream_len, n_channels, n, cfg, taps, fs,
                 kernel, max_epochs, recs, tap_sums, done, 0, PTHREAD_MUTEX_INITIALIZER};
    if (threads < 1)
        threads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    for (int t = 0; t < threads; ++t)
        pthread_create(&th[t], NULL, run_worker, &j);
    for (int t = 0; t < threads; ++t)
        pthread_join(th[t], NULL);
    free(th);
    return 0;
}

/* ---- search grid: acquisition.hpp:38-50,114-222 (config 5) ---------- */
/* wipe_carrier (acquisition.hpp:170-182): rotation recurrence anchored at
 * the global buffer index, renormalised every 1024 samples. */
static void wipe_carrier(const double* in, int64_t n, int64_t global_start,
                         double f, double fs, double* out) {
    const double w = -2.0 * PI_D * f / fs;
    const double ph0 = w * (double)global_start;
    double cr = cos(ph0), ci = sin(ph0);
    const double rr = cos(w), ri = sin(w);
    for (int64_t i = 0; i < n; ++i) {
        const double xr = in[2 * i], xi = in[2 * i + 1];
        out[2 * i] = xr * cr - xi * ci;
        out[2 * i + 1] = xr * ci + xi * cr;
        const double nr = cr * rr - ci * ri;
        const double ni = cr * ri + ci * rr;
        cr = nr;
        ci = ni;
        if ((i & 1023) == 1023) {
            const double a = hypot(cr, ci);
            cr /= a;
            ci /= a;
        }
    }
}

/* acquire_pcs plane cells (acquisition.hpp:189-222) evaluated directly in
 * the time domain at the requested delays: cell[b][j] = sum over 1-ms
 * segments s of N * |sum_n wiped_s[n] * code[(n - d_j) mod N]| with
 * d_j = j*delay_step (FFTW's inverse is unnormalised, fft.hpp:17-19, so
 * the FFT path carries the factor N).  iq holds n_seg*N complex samples. */
int orc_search_grid(const double* iq, int N, int n_seg, int prn, double fs,
                    const double* bins, int n_bins, int delay_step, int n_delays,
                    double* plane) {
    if (prn < 1 || prn > 32)
        return fail(L1RXG_ERANGE, "PRN must be in 1..32");
    int8_t* code = (int8_t*)malloc((size_t)N);
    orc_resample_code(prn, fs, 0.0, CHIP_RATE_HZ, N, code);
    double* wiped = (double*)malloc(sizeof(double) * 2 * (size_t)N);
    memset(plane, 0, sizeof(double) * (size_t)n_bins * (size_t)n_delays);
    for (int b = 0; b < n_bins; ++b)
        for (int s = 0; s < n_seg; ++s) {
            wipe_carrier(iq + 2 * (int64_t)s * N, N, (int64_t)s * N, bins[b], fs, wiped);
            for (int j = 0; j < n_delays; ++j) {
                const int d = j * delay_step;
                double ar = 0, ai = 0;
                for (int nn = 0; nn < N; ++nn) {
                    int idx = nn - d;
                    if (idx < 0)
                        idx += N;
                    ar += wiped[2 * nn] * code[idx];
                    ai += wiped[2 * nn + 1] * code[idx];
                }
                plane[(int64_t)b * n_delays + j] += (double)N * hypot(ar, ai);
            }
        }
    free(wiped);
    free(code);
    return 0;
}
