// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE, not product code.
//
// A thin extern "C" veneer over the UNMODIFIED reference headers
// (/root/reference/proj/include/l1rx/*.hpp), compiled in place by
// oracle/Makefile into oracle/_ref/libl1rx_ref.so.  Nothing of the reference
// is copied here: every numeric result below is computed by the reference's
// own inline functions.  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference leg may load the resulting library.
//
// The POD types come from include/l1rxg.h so the reference, the C
// restatement (oracle/l1rx_oracle.c) and the GPU library share one layout.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <deque>
#include <fstream>
#include <functional>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <unistd.h>
#include <vector>

#include "l1rx/cacode.hpp"
#include "l1rx/samples.hpp"
#include "l1rx/simsource.hpp"
#include "l1rx/tracking.hpp"

#include "l1rxg.h"

using namespace l1rx;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return L1RXG_EINVAL;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return L1RXG_ERANGE;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return L1RXG_ELOGIC;
    } catch (const std::exception& e) {
        g_err = e.what();
        return L1RXG_ECUDA;
    }
}

TrackingConfig to_cfg(const l1rxg_tracking_cfg* c) {
    TrackingConfig cfg;
    if (!c)
        return cfg;
    cfg.epoch_ms = c->epoch_ms;
    cfg.el_spacing_chips = c->el_spacing_chips;
    cfg.dll_bandwidth_hz = c->dll_bandwidth_hz;
    cfg.dll_damping = c->dll_damping;
    cfg.pll_bandwidth_hz = c->pll_bandwidth_hz;
    cfg.pll_damping = c->pll_damping;
    cfg.fll_bandwidth_hz = c->fll_bandwidth_hz;
    cfg.fll_pull_in_ms = c->fll_pull_in_ms;
    cfg.fll_coarse_ms = c->fll_coarse_ms;
    cfg.cn0_window_ms = c->cn0_window_ms;
    cfg.lock_fail_limit = c->lock_fail_limit;
    cfg.cn0_drop_dbhz = c->cn0_drop_dbhz;
    cfg.carrier_lock_drop = c->carrier_lock_drop;
    return cfg;
}

void to_state(const l1rxg_channel& p, ChannelState& ch) {
    ch.prn = p.prn;
    ch.state = static_cast<ChannelRunState>(p.state);
    ch.code_phase_chips = p.code_phase_chips;
    ch.code_freq_hz = p.code_freq_hz;
    ch.carrier_doppler_hz = p.carrier_doppler_hz;
    ch.carrier_phase_rad = p.carrier_phase_rad;
    ch.chi_chips = p.chi_chips;
    ch.dll_filter.integrator = p.dll_integrator;
    ch.dll_filter.prev_error = p.dll_prev_error;
    ch.dll_filter.primed = p.dll_primed != 0;
    ch.pll_filter.integrator = p.pll_integrator;
    ch.pll_filter.prev_error = p.pll_prev_error;
    ch.pll_filter.primed = p.pll_primed != 0;
    ch.fll_enabled = p.fll_enabled != 0;
    ch.last_ip = p.last_ip;
    ch.last_qp = p.last_qp;
    ch.have_last_prompt = p.have_last_prompt != 0;
    ch.epoch_ms_count = p.epoch_ms_count;
    ch.epochs_since_handoff = p.epochs_since_handoff;
    ch.cn0_dbhz = p.cn0_dbhz;
    ch.carrier_lock_ratio = p.carrier_lock_ratio;
    ch.lock_fail_count = p.lock_fail_count;
    ch.metrics_valid = p.metrics_valid != 0;
    ch.sample_offset_next_epoch = p.sample_offset_next_epoch;
    ch.mu_smoothed = p.mu_smoothed;
    ch.win_ip.assign(p.win_ip, p.win_ip + p.win_len);
    ch.win_qp.assign(p.win_qp, p.win_qp + p.win_len);
}

void from_state(const ChannelState& ch, l1rxg_channel& p) {
    std::memset(&p, 0, sizeof p);
    p.prn = ch.prn;
    p.state = static_cast<int32_t>(ch.state);
    p.code_phase_chips = ch.code_phase_chips;
    p.code_freq_hz = ch.code_freq_hz;
    p.carrier_doppler_hz = ch.carrier_doppler_hz;
    p.carrier_phase_rad = ch.carrier_phase_rad;
    p.chi_chips = ch.chi_chips;
    p.dll_integrator = ch.dll_filter.integrator;
    p.dll_prev_error = ch.dll_filter.prev_error;
    p.dll_primed = ch.dll_filter.primed;
    p.pll_integrator = ch.pll_filter.integrator;
    p.pll_prev_error = ch.pll_filter.prev_error;
    p.pll_primed = ch.pll_filter.primed;
    p.fll_enabled = ch.fll_enabled;
    p.last_ip = ch.last_ip;
    p.last_qp = ch.last_qp;
    p.have_last_prompt = ch.have_last_prompt;
    p.epoch_ms_count = ch.epoch_ms_count;
    p.epochs_since_handoff = ch.epochs_since_handoff;
    p.cn0_dbhz = ch.cn0_dbhz;
    p.carrier_lock_ratio = ch.carrier_lock_ratio;
    p.lock_fail_count = ch.lock_fail_count;
    p.metrics_valid = ch.metrics_valid;
    p.sample_offset_next_epoch = ch.sample_offset_next_epoch;
    p.mu_smoothed = ch.mu_smoothed;
    p.win_len = static_cast<int32_t>(
        std::min<std::size_t>(ch.win_ip.size(), L1RXG_WIN_MAX));
    for (int k = 0; k < p.win_len; ++k) {
        p.win_ip[k] = ch.win_ip[static_cast<std::size_t>(k)];
        p.win_qp[k] = ch.win_qp[static_cast<std::size_t>(k)];
    }
}

void set_nco(ChannelState& ch, const l1rxg_nco* st) {
    ch.code_phase_chips = st->code_phase_chips;
    ch.code_freq_hz = st->code_freq_hz;
    ch.carrier_doppler_hz = st->carrier_doppler_hz;
    ch.carrier_phase_rad = st->carrier_phase_rad;
    ch.chi_chips = st->chi_chips;
}

void get_nco(const ChannelState& ch, l1rxg_nco* st) {
    st->code_phase_chips = ch.code_phase_chips;
    st->code_freq_hz = ch.code_freq_hz;
    st->carrier_doppler_hz = ch.carrier_doppler_hz;
    st->carrier_phase_rad = ch.carrier_phase_rad;
    st->chi_chips = ch.chi_chips;
}

void put_corr(const CorrelatorOutputs& o, l1rxg_corr* out) {
    out->ie = o.ie;
    out->qe = o.qe;
    out->ip = o.ip;
    out->qp = o.qp;
    out->il = o.il;
    out->ql = o.ql;
    out->ip_h1 = o.ip_h1;
    out->qp_h1 = o.qp_h1;
    out->ip_h2 = o.ip_h2;
    out->qp_h2 = o.qp_h2;
    out->n_samples = o.n_samples;
    out->pad_ = 0;
}

CorrelatorOutputs run_kernel(int kernel, std::span<const cplx> view,
                             ChannelState& ch, const CaCode& code,
                             const TrackingConfig& cfg, double fs) {
    switch (kernel) {
    case L1RXG_KERNEL_SCALAR:
        return correlate_epoch_scalar(view, ch, code, cfg, fs);
    case L1RXG_KERNEL_BATCHED:
        return correlate_epoch_batched(view, ch, code, cfg, fs);
    default:
        return correlate_epoch_noop(view, ch, fs);
    }
}

KernelKind kind_of(int kernel) {
    switch (kernel) {
    case L1RXG_KERNEL_SCALAR: return KernelKind::Scalar;
    case L1RXG_KERNEL_BATCHED: return KernelKind::Batched;
    default: return KernelKind::Noop;
    }
}

void fill_record(const ChannelState& ch, const CorrelatorOutputs& o,
                 const TrackingEpochOutput& teo, const l1rxg_nco& in,
                 int64_t start, l1rxg_epoch_record* r) {
    std::memset(r, 0, sizeof *r);
    r->epoch_index = teo.epoch_index;
    r->sample_offset_start = start;
    r->sample_offset_end = teo.sample_offset_end;
    r->prn = teo.prn;
    r->state = static_cast<int32_t>(teo.state);
    r->n_samples = o.n_samples;
    r->lock_fail_count = ch.lock_fail_count;
    r->code_phase_in = in.code_phase_chips;
    r->code_freq_in = in.code_freq_hz;
    r->carrier_doppler_in = in.carrier_doppler_hz;
    r->carrier_phase_in = in.carrier_phase_rad;
    r->ie = o.ie;
    r->qe = o.qe;
    r->ip = o.ip;
    r->qp = o.qp;
    r->il = o.il;
    r->ql = o.ql;
    r->ip_h1 = o.ip_h1;
    r->qp_h1 = o.qp_h1;
    r->ip_h2 = o.ip_h2;
    r->qp_h2 = o.qp_h2;
    r->carrier_doppler_hz = teo.carrier_doppler_hz;
    r->code_freq_hz = teo.code_freq_hz;
    r->code_phase_chips = teo.code_phase_chips;
    r->carrier_phase_rad = ch.carrier_phase_rad;
    r->chi_chips = teo.chi_chips;
    r->cn0_dbhz = teo.cn0_dbhz;
    r->carrier_lock_ratio = teo.carrier_lock_ratio;
    r->dll_integrator = ch.dll_filter.integrator;
    r->pll_integrator = ch.pll_filter.integrator;
    r->mu_smoothed = ch.mu_smoothed;
    r->dll_prev_error = ch.dll_filter.prev_error;
    r->pll_prev_error = ch.pll_filter.prev_error;
}

// One tracking step of the reference on a channel (track_epoch,
// tracking.hpp:520-618), also capturing the CorrelatorOutputs it used by
// running the same deterministic kernel on a copy first.
void step(ChannelState& ch, std::span<const cplx> view,
          const TrackingConfig& cfg, double fs, int kernel,
          l1rxg_epoch_record* rec) {
    const CaCode& code = ca_code_table().at(static_cast<std::size_t>(ch.prn));
    l1rxg_nco in{};
    get_nco(ch, &in);
    const int64_t start = ch.sample_offset_next_epoch;
    CorrelatorOutputs o;
    if (rec) {
        ChannelState copy = ch;
        o = run_kernel(kernel, view, copy, code, cfg, fs);
    }
    const auto teo = track_epoch(ch, view, code, cfg, fs, kind_of(kernel));
    if (rec)
        fill_record(ch, o, teo, in, start, rec);
}

} // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_ca_code(int prn, int8_t* out) {
    return guarded([&] {
        const auto code = generate_ca_code(prn);
        std::memcpy(out, code.chips.data(), 1023);
    });
}

void ref_halfband_taps(double* out) {
    const auto& h = detail::halfband_taps();
    std::copy(h.begin(), h.end(), out);
}

// SampleSource over a file (samples.hpp:114-265): reads every block of
// block_ms and concatenates the complex<double> samples.  Returns the
// number of samples written (<= max_samples) or -status.
int64_t ref_read_source(const char* path, int format, double fs, double if_hz,
                        int block_ms, double* iq_out, int64_t max_samples) {
    int64_t got = 0;
    const int rc = guarded([&] {
        SourceConfig cfg;
        cfg.locator = path;
        cfg.format.kind = static_cast<SampleKind>(
            format == L1RXG_FMT_INT8_IQ      ? 0
            : format == L1RXG_FMT_INT16_IQ   ? 1
                                             : 2);
        cfg.format.if_frequency_hz = if_hz;
        cfg.sample_rate_hz = fs;
        cfg.block_length_ms = block_ms;
        SampleSource src(cfg);
        while (auto blk = src.read_block()) {
            for (const auto& s : blk->samples) {
                if (got >= max_samples)
                    return;
                iq_out[2 * got] = s.real();
                iq_out[2 * got + 1] = s.imag();
                ++got;
            }
        }
    });
    return rc ? -rc : got;
}

int ref_validate_source(int format, double fs, double if_hz, int block_ms) {
    return guarded([&] {
        SourceConfig cfg;
        cfg.format.kind = static_cast<SampleKind>(
            format == L1RXG_FMT_INT8_IQ      ? 0
            : format == L1RXG_FMT_INT16_IQ   ? 1
                                             : 2);
        cfg.format.if_frequency_hz = if_hz;
        cfg.sample_rate_hz = fs;
        cfg.block_length_ms = block_ms;
        validate(cfg);
    });
}

// correlate_epoch_{scalar,batched,noop} (tracking.hpp:226-452)
int ref_correlate(int kernel, const double* iq, int n, l1rxg_nco* st,
                  int prn, double el_spacing, double fs, l1rxg_corr* out) {
    return guarded([&] {
        ChannelState ch;
        ch.prn = prn;
        ch.state = ChannelRunState::Tracking;
        set_nco(ch, st);
        TrackingConfig cfg;
        cfg.el_spacing_chips = el_spacing;
        const CaCode& code = ca_code_table().at(static_cast<std::size_t>(prn));
        const auto view = std::span<const cplx>(
            reinterpret_cast<const cplx*>(iq), static_cast<std::size_t>(n));
        const auto o = run_kernel(kernel, view, ch, code, cfg, fs);
        get_nco(ch, st);
        put_corr(o, out);
    });
}

// track_epoch on a POD channel (state copied in and out).
int ref_track_epoch(l1rxg_channel* chp, const double* iq, int n,
                    const l1rxg_tracking_cfg* cfgp, double fs, int kernel,
                    l1rxg_epoch_record* rec) {
    return guarded([&] {
        ChannelState ch;
        to_state(*chp, ch);
        const auto cfg = to_cfg(cfgp);
        const auto view = std::span<const cplx>(
            reinterpret_cast<const cplx*>(iq), static_cast<std::size_t>(n));
        step(ch, view, cfg, fs, kernel, rec);
        from_state(ch, *chp);
    });
}

// Closed loop over one buffer for one channel, like run_closed_loop
// (test_tracking.cpp:368-399): steps while a full epoch of samples remains
// and the channel is not Idle.  Returns the epochs run.
int64_t ref_track_buffer(l1rxg_channel* chp, const double* iq,
                         int64_t n_total, int n, const l1rxg_tracking_cfg* cfgp,
                         double fs, int kernel, int64_t max_epochs,
                         l1rxg_epoch_record* recs) {
    int64_t done = 0;
    const int rc = guarded([&] {
        ChannelState ch;
        to_state(*chp, ch);
        const auto cfg = to_cfg(cfgp);
        while (done < max_epochs &&
               ch.sample_offset_next_epoch + n <= n_total &&
               ch.state != ChannelRunState::Idle) {
            const auto view = std::span<const cplx>(
                reinterpret_cast<const cplx*>(iq) + ch.sample_offset_next_epoch,
                static_cast<std::size_t>(n));
            step(ch, view, cfg, fs, kernel, recs ? recs + done : nullptr);
            ++done;
        }
        from_state(ch, *chp);
    });
    return rc ? -rc : done;
}

// init_channel_from_acquisition (tracking.hpp:622-650)
void ref_init_channel(l1rxg_channel* chp, int prn, double doppler_hz,
                      int64_t acq_buffer_start, int code_delay_samples,
                      int64_t start_offset_samples, double fs) {
    ChannelState ch;
    init_channel_from_acquisition(ch, prn, doppler_hz, acq_buffer_start,
                                  code_delay_samples, start_offset_samples,
                                  fs);
    from_state(ch, *chp);
}

void ref_default_cfg(l1rxg_tracking_cfg* c) {
    TrackingConfig d;
    std::memset(c, 0, sizeof *c);
    c->epoch_ms = d.epoch_ms;
    c->el_spacing_chips = d.el_spacing_chips;
    c->dll_bandwidth_hz = d.dll_bandwidth_hz;
    c->dll_damping = d.dll_damping;
    c->pll_bandwidth_hz = d.pll_bandwidth_hz;
    c->pll_damping = d.pll_damping;
    c->fll_bandwidth_hz = d.fll_bandwidth_hz;
    c->fll_pull_in_ms = d.fll_pull_in_ms;
    c->fll_coarse_ms = d.fll_coarse_ms;
    c->cn0_window_ms = d.cn0_window_ms;
    c->lock_fail_limit = d.lock_fail_limit;
    c->cn0_drop_dbhz = d.cn0_drop_dbhz;
    c->carrier_lock_drop = d.carrier_lock_drop;
}

// discriminators / filters (tracking.hpp:65-147) for unit-level goldens
double ref_dll_discriminator(const l1rxg_corr* c) {
    CorrelatorOutputs o;
    o.ie = c->ie; o.qe = c->qe; o.il = c->il; o.ql = c->ql;
    return dll_discriminator(o);
}
double ref_pll_discriminator(double ip, double qp) {
    CorrelatorOutputs o;
    o.ip = ip; o.qp = qp;
    return pll_discriminator(o);
}
double ref_fll_discriminator(double a, double b, double c, double d, double dt) {
    return fll_discriminator(a, b, c, d, dt);
}
double ref_fll_discriminator_di(double a, double b, double c, double d, double dt) {
    return fll_discriminator_data_insensitive(a, b, c, d, dt);
}
double ref_carrier_aid(double doppler, double dll) {
    return carrier_aid_code_freq(doppler, dll);
}
double ref_loop_filter_update(double* integ, double* prev, int* primed,
                              double err, double bw, double damp, double dt) {
    LoopFilterState st;
    st.integrator = *integ; st.prev_error = *prev; st.primed = *primed != 0;
    const double r = loop_filter_update(st, err, bw, damp, dt);
    *integ = st.integrator; *prev = st.prev_error; *primed = st.primed;
    return r;
}

// SimStream complex-baseband synthesis (simsource.hpp:198-378): nsv
// satellites in raw mode; writes duration_s*fs complex samples.
int64_t ref_sim_baseband(int nsv, const int* prns, const double* cn0,
                         const double* doppler, const double* doppler_rate,
                         const double* delay_chips, const double* phase0,
                         double duration_s, double fs, int noise,
                         uint64_t seed, double* iq_out, int64_t max_samples) {
    int64_t got = 0;
    const int rc = guarded([&] {
        SimScenario sc;
        for (int k = 0; k < nsv; ++k) {
            SimSatellite sv;
            sv.prn = prns[k];
            sv.cn0_dbhz = cn0[k];
            sv.doppler_hz = doppler[k];
            sv.doppler_rate_hz_per_s = doppler_rate ? doppler_rate[k] : 0.0;
            sv.code_delay_chips = delay_chips[k];
            sv.initial_carrier_phase_rad = phase0 ? phase0[k] : 0.0;
            sc.satellites.push_back(sv);
        }
        sc.duration_s = duration_s;
        sc.sample_rate_hz = fs;
        sc.noise_enabled = noise != 0;
        sc.seed = seed;
        SimStream stream(sc);
        while (auto blk = stream.next_block())
            for (const auto& s : *blk) {
                if (got >= max_samples)
                    return;
                iq_out[2 * got] = s.real();
                iq_out[2 * got + 1] = s.imag();
                ++got;
            }
    });
    return rc ? -rc : got;
}

// ---------------------------------------------------------------------
// CPU baseline: the reference receiver's tracking path on host cores.
// Mirrors Receiver (pipeline.hpp:326-805) minus acquisition / nav / PVT,
// which need FFTW or are off the hot path: one producer thread running
// SampleSource::read_block (samples.hpp:136-172, incl. the real-IF
// downconvert) into a bounded queue (BlockQueue, pipeline.hpp:30-86), and
// the consumer appending to the sliding window and running track_epoch for
// every runnable channel per 1-ms round on a worker pool (ChannelPool,
// pipeline.hpp:91-151).  Timings: wall time of the whole run and the sum of
// tracking-round wall times (bench_tracking's tracking_ns,
// pipeline.hpp:576-598).
int ref_bench_pipeline(const char* path, int format, double fs, double if_hz,
                       int n_channels, const l1rxg_channel* init,
                       const l1rxg_tracking_cfg* cfgp, int kernel, int threads,
                       int64_t max_rounds, double* wall_s, double* tracking_s,
                       int64_t* channel_epochs, l1rxg_channel* final_out) {
    return guarded([&] {
        SourceConfig scfg;
        scfg.locator = path;
        scfg.format.kind = static_cast<SampleKind>(
            format == L1RXG_FMT_INT8_IQ      ? 0
            : format == L1RXG_FMT_INT16_IQ   ? 1
                                             : 2);
        scfg.format.if_frequency_hz = if_hz;
        scfg.sample_rate_hz = fs;
        SampleSource source(scfg);
        const auto cfg = to_cfg(cfgp);
        const auto spm = static_cast<int64_t>(std::llround(fs / 1000.0));

        std::vector<ChannelState> chans(static_cast<std::size_t>(n_channels));
        for (int c = 0; c < n_channels; ++c)
            to_state(init[c], chans[static_cast<std::size_t>(c)]);

        // bounded block queue (producer/consumer, pipeline.hpp:30-86)
        std::deque<SampleBlock> q;
        std::mutex mu;
        std::condition_variable cv_put, cv_get;
        bool closed = false;
        bool abort_run = false;
        const std::size_t cap = 32;
        const auto t_start = std::chrono::steady_clock::now();
        std::thread producer([&] {
            for (;;) {
                {
                    std::lock_guard<std::mutex> lk(mu);
                    if (abort_run)
                        break;
                }
                auto blk = source.read_block();
                if (!blk)
                    break;
                std::unique_lock<std::mutex> lk(mu);
                cv_put.wait(lk, [&] { return q.size() < cap || abort_run; });
                if (abort_run)
                    break;
                q.push_back(std::move(*blk));
                cv_get.notify_one();
            }
            std::lock_guard<std::mutex> lk(mu);
            closed = true;
            cv_get.notify_all();
        });

        // worker pool with index hand-out (ChannelPool, pipeline.hpp:91-151)
        const int nw = std::max(1, threads);
        std::vector<std::thread> workers;
        std::mutex pmu;
        std::condition_variable pcv, pdone;
        std::function<void(int)> task;
        int next = 0, total = 0, finished = 0;
        int64_t generation = 0;
        bool stop = false;
        for (int w = 0; w < nw; ++w)
            workers.emplace_back([&] {
                int64_t seen = 0;
                for (;;) {
                    int idx;
                    {
                        std::unique_lock<std::mutex> lk(pmu);
                        pcv.wait(lk, [&] {
                            return stop || (generation != seen && next < total);
                        });
                        if (stop)
                            return;
                        idx = next++;
                        if (next >= total)
                            seen = generation;
                    }
                    task(idx);
                    std::lock_guard<std::mutex> lk(pmu);
                    if (++finished == total)
                        pdone.notify_all();
                }
            });
        auto pool_run = [&](int n, std::function<void(int)> fn) {
            {
                std::lock_guard<std::mutex> lk(pmu);
                task = std::move(fn);
                next = 0;
                total = n;
                finished = 0;
                ++generation;
            }
            pcv.notify_all();
            std::unique_lock<std::mutex> lk(pmu);
            pdone.wait(lk, [&] { return finished == total; });
        };

        std::vector<cplx> window;
        int64_t window_base = 0;
        int64_t rounds = 0;
        double track_acc = 0;
        int64_t ce = 0;
        std::vector<int> runnable;
        for (;;) {
            SampleBlock blk;
            {
                std::unique_lock<std::mutex> lk(mu);
                cv_get.wait(lk, [&] { return !q.empty() || closed; });
                if (q.empty())
                    break;
                blk = std::move(q.front());
                q.pop_front();
                cv_put.notify_one();
            }
            // append_to_window (pipeline.hpp:432-447)
            if (window.empty())
                window_base = blk.receiver_time_offset_samples;
            window.insert(window.end(), blk.samples.begin(), blk.samples.end());
            const int64_t wend = window_base + static_cast<int64_t>(window.size());
            const int64_t keep = wend - 6 * spm - static_cast<int64_t>(blk.count());
            if (keep > window_base) {
                window.erase(window.begin(), window.begin() + (keep - window_base));
                window_base = keep;
            }
            const int64_t ms_in_block = static_cast<int64_t>(blk.count()) / spm;
            for (int64_t m = 0; m < ms_in_block && rounds < max_rounds; ++m) {
                const int64_t round_end = blk.receiver_time_offset_samples + (m + 1) * spm;
                runnable.clear();
                for (int c = 0; c < n_channels; ++c) {
                    auto& ch = chans[static_cast<std::size_t>(c)];
                    if (ch.state == ChannelRunState::Idle)
                        continue;
                    if (ch.sample_offset_next_epoch + spm <= round_end &&
                        ch.sample_offset_next_epoch >= window_base)
                        runnable.push_back(c);
                }
                ++rounds;
                if (runnable.empty())
                    continue;
                const auto t0 = std::chrono::steady_clock::now();
                pool_run(static_cast<int>(runnable.size()), [&](int i) {
                    auto& ch = chans[static_cast<std::size_t>(runnable[static_cast<std::size_t>(i)])];
                    const auto view = std::span<const cplx>(
                        window.data() + (ch.sample_offset_next_epoch - window_base),
                        static_cast<std::size_t>(spm));
                    track_epoch(ch, view,
                                ca_code_table()[static_cast<std::size_t>(ch.prn)],
                                cfg, fs, kind_of(kernel));
                });
                const auto t1 = std::chrono::steady_clock::now();
                track_acc += std::chrono::duration<double>(t1 - t0).count();
                ce += static_cast<int64_t>(runnable.size());
            }
            if (rounds >= max_rounds)
                break;
        }
        {
            std::lock_guard<std::mutex> lk(mu);
            abort_run = true;
            q.clear();
        }
        cv_put.notify_all();
        producer.join();
        {
            std::lock_guard<std::mutex> lk(pmu);
            stop = true;
        }
        pcv.notify_all();
        for (auto& w : workers)
            w.join();
        const auto t_end = std::chrono::steady_clock::now();
        *wall_s = std::chrono::duration<double>(t_end - t_start).count();
        *tracking_s = track_acc;
        *channel_epochs = ce;
        if (final_out)
            for (int c = 0; c < n_channels; ++c)
                from_state(chans[static_cast<std::size_t>(c)], final_out[c]);
    });
}

} // extern "C"
