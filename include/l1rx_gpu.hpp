// l1rx_gpu.hpp -- header-only C++ adapter: the GPU correlator behind the
// reference's own types and signatures (drop-in for l1rx, proj/include/l1rx).
//
//   #include "l1rx/tracking.hpp"   // the reference
//   #include "l1rx_gpu.hpp"        // this adapter (links libl1rxg.so)
//
//   auto out = l1rx::gpu::correlate_epoch_gpu(view, ch, code, cfg, fs);
//
// correlate_epoch_gpu has exactly the signature and contract of
// correlate_epoch_scalar / _batched (tracking.hpp:226-230, 288-292): one
// epoch of complex<double> samples, the three NCO fields of ChannelState
// advanced in place with the same fmod forms (:275-280), CorrelatorOutputs
// returned, std::invalid_argument on an empty view (:232-233),
// std::out_of_range on a bad PRN (cacode.hpp:38-39).  Re-entrant across
// threads (each call takes the context's per-call lock).
//
// GpuTracker wraps the closed-loop tracker (l1rxg_tracker_*): it replaces
// Receiver::tracking_round's per-channel track_epoch fan-out
// (pipeline.hpp:563-610) with one device-resident loop per channel and
// returns TrackingEpochOutput-equivalent records; see INTEGRATION.md.
#pragma once

#include <cstring>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "l1rx/tracking.hpp"
#include "l1rxg.h"

namespace l1rx::gpu {

// Maps an l1rxg_status to the reference's exception types.
inline void check(int rc) {
    if (rc == L1RXG_OK)
        return;
    const std::string msg = l1rxg_last_error();
    switch (rc) {
    case L1RXG_EINVAL: throw std::invalid_argument(msg);
    case L1RXG_ELOGIC: throw std::logic_error(msg);
    case L1RXG_ERANGE: throw std::out_of_range(msg);
    default: throw std::runtime_error(msg);
    }
}

// One context per process (device 0 unless set before first use).
inline int& device_ordinal() {
    static int dev = 0;
    return dev;
}

inline l1rxg_ctx* context() {
    static l1rxg_ctx* ctx = nullptr;
    static std::once_flag once;
    std::call_once(once, [] { check(l1rxg_create(device_ordinal(), &ctx)); });
    return ctx;
}

inline l1rxg_tracking_cfg to_c(const TrackingConfig& c) {
    l1rxg_tracking_cfg o{};
    o.epoch_ms = c.epoch_ms;
    o.el_spacing_chips = c.el_spacing_chips;
    o.dll_bandwidth_hz = c.dll_bandwidth_hz;
    o.dll_damping = c.dll_damping;
    o.pll_bandwidth_hz = c.pll_bandwidth_hz;
    o.pll_damping = c.pll_damping;
    o.fll_bandwidth_hz = c.fll_bandwidth_hz;
    o.fll_pull_in_ms = c.fll_pull_in_ms;
    o.fll_coarse_ms = c.fll_coarse_ms;
    o.cn0_window_ms = c.cn0_window_ms;
    o.lock_fail_limit = c.lock_fail_limit;
    o.cn0_drop_dbhz = c.cn0_drop_dbhz;
    o.carrier_lock_drop = c.carrier_lock_drop;
    return o;
}

// Drop-in for correlate_epoch_scalar / correlate_epoch_batched.
inline CorrelatorOutputs correlate_epoch_gpu(std::span<const cplx> view, ChannelState& ch,
                                             const CaCode& code, const TrackingConfig& cfg,
                                             double sample_rate_hz) {
    if (view.empty())
        throw std::invalid_argument("empty epoch view");  // tracking.hpp:232-233
    l1rxg_nco st{ch.code_phase_chips, ch.code_freq_hz, ch.carrier_doppler_hz,
                 ch.carrier_phase_rad, ch.chi_chips};
    l1rxg_corr o{};
    check(l1rxg_correlate_epoch(context(), L1RXG_KERNEL_SCALAR,
                                reinterpret_cast<const double*>(view.data()),
                                static_cast<int>(view.size()), &st, code.prn,
                                cfg.el_spacing_chips, sample_rate_hz, &o));
    ch.code_phase_chips = st.code_phase_chips;
    ch.carrier_phase_rad = st.carrier_phase_rad;
    ch.chi_chips = st.chi_chips;
    CorrelatorOutputs out;
    out.ie = o.ie;
    out.qe = o.qe;
    out.ip = o.ip;
    out.qp = o.qp;
    out.il = o.il;
    out.ql = o.ql;
    out.ip_h1 = o.ip_h1;
    out.qp_h1 = o.qp_h1;
    out.ip_h2 = o.ip_h2;
    out.qp_h2 = o.qp_h2;
    out.n_samples = o.n_samples;
    return out;
}

// ChannelState <-> l1rxg_channel (NavDecodeState stays on the host).
// window_ms > L1RXG_WIN_MAX: the C/N0 window travels as its running sums
// (see l1rxg_channel in l1rxg.h), accumulated in the reference's order
inline l1rxg_channel to_c(const ChannelState& ch, int window_ms = 0) {
    l1rxg_channel p;
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
    p.pll_integrator = ch.pll_filter.integrator;
    p.pll_prev_error = ch.pll_filter.prev_error;
    p.dll_primed = ch.dll_filter.primed;
    p.pll_primed = ch.pll_filter.primed;
    p.fll_enabled = ch.fll_enabled;
    p.have_last_prompt = ch.have_last_prompt;
    p.last_ip = ch.last_ip;
    p.last_qp = ch.last_qp;
    p.epoch_ms_count = ch.epoch_ms_count;
    p.epochs_since_handoff = ch.epochs_since_handoff;
    p.cn0_dbhz = ch.cn0_dbhz;
    p.carrier_lock_ratio = ch.carrier_lock_ratio;
    p.mu_smoothed = ch.mu_smoothed;
    p.lock_fail_count = ch.lock_fail_count;
    p.metrics_valid = ch.metrics_valid;
    p.sample_offset_next_epoch = ch.sample_offset_next_epoch;
    p.win_len = static_cast<int32_t>(ch.win_ip.size());
    if (window_ms > L1RXG_WIN_MAX) {
        double nbi = 0, nbq = 0, wbp = 0;
        for (std::size_t k = 0; k < ch.win_ip.size(); ++k) {
            const double sg = ch.win_ip[k] >= 0 ? 1.0 : -1.0;
            nbi += sg * ch.win_ip[k];
            nbq += sg * ch.win_qp[k];
            wbp += ch.win_ip[k] * ch.win_ip[k] + ch.win_qp[k] * ch.win_qp[k];
        }
        p.win_ip[0] = nbi;
        p.win_qp[0] = nbq;
        p.win_ip[1] = wbp;
        return p;
    }
    for (std::size_t k = 0; k < ch.win_ip.size() && k < L1RXG_WIN_MAX; ++k) {
        p.win_ip[k] = ch.win_ip[k];
        p.win_qp[k] = ch.win_qp[k];
    }
    return p;
}

// window_ms > L1RXG_WIN_MAX: the device state holds the open window's sums,
// not its samples, so the reference-side window restarts empty (its C/N0
// estimate resumes at the next full window)
inline void from_c(const l1rxg_channel& p, ChannelState& ch, int window_ms = 0) {
    ch.state = static_cast<ChannelRunState>(p.state);
    ch.code_phase_chips = p.code_phase_chips;
    ch.code_freq_hz = p.code_freq_hz;
    ch.carrier_doppler_hz = p.carrier_doppler_hz;
    ch.carrier_phase_rad = p.carrier_phase_rad;
    ch.chi_chips = p.chi_chips;
    ch.dll_filter.integrator = p.dll_integrator;
    ch.dll_filter.prev_error = p.dll_prev_error;
    ch.dll_filter.primed = p.dll_primed;
    ch.pll_filter.integrator = p.pll_integrator;
    ch.pll_filter.prev_error = p.pll_prev_error;
    ch.pll_filter.primed = p.pll_primed;
    ch.fll_enabled = p.fll_enabled;
    ch.have_last_prompt = p.have_last_prompt;
    ch.last_ip = p.last_ip;
    ch.last_qp = p.last_qp;
    ch.epoch_ms_count = p.epoch_ms_count;
    ch.epochs_since_handoff = p.epochs_since_handoff;
    ch.cn0_dbhz = p.cn0_dbhz;
    ch.carrier_lock_ratio = p.carrier_lock_ratio;
    ch.mu_smoothed = p.mu_smoothed;
    ch.lock_fail_count = p.lock_fail_count;
    ch.metrics_valid = p.metrics_valid;
    ch.sample_offset_next_epoch = p.sample_offset_next_epoch;
    if (window_ms > L1RXG_WIN_MAX) {
        ch.win_ip.clear();
        ch.win_qp.clear();
        return;
    }
    ch.win_ip.assign(p.win_ip, p.win_ip + p.win_len);
    ch.win_qp.assign(p.win_qp, p.win_qp + p.win_len);
}

// Closed-loop tracking of a set of channels on one raw sample stream.
class GpuTracker {
public:
    GpuTracker(SampleKind kind, double fs, double if_hz, const std::vector<ChannelState>& chans,
               const TrackingConfig& cfg = {}, int64_t ring_samples = 0, int max_records = 4096) {
        l1rxg_tracker_desc d{};
        d.format = kind == SampleKind::Int8ComplexInterleaved   ? L1RXG_FMT_INT8_IQ
                   : kind == SampleKind::Int16ComplexInterleaved ? L1RXG_FMT_INT16_IQ
                                                                 : L1RXG_FMT_INT8_REAL_IF;
        d.kernel = L1RXG_KERNEL_SCALAR;
        d.sample_rate_hz = fs;
        d.if_frequency_hz = if_hz;
        d.n_streams = 1;
        d.n_channels = static_cast<int32_t>(chans.size());
        const int64_t spm = static_cast<int64_t>(fs / 1000.0 + 0.5);
        d.ring_samples = ring_samples > 0 ? ring_samples : 256 * spm;
        d.max_records = max_records;
        l1rxg_epl_taps(cfg.el_spacing_chips, &d.taps);
        d.cfg = to_c(cfg);
        std::vector<l1rxg_channel> c;
        for (const auto& ch : chans)
            c.push_back(to_c(ch, cfg.cn0_window_ms));
        window_ms_ = cfg.cn0_window_ms;
        std::vector<int32_t> s(chans.size(), 0);
        check(l1rxg_tracker_create(context(), &d, c.data(), s.data(), &trk_));
        n_ = chans.size();
    }
    ~GpuTracker() { l1rxg_tracker_destroy(trk_); }
    GpuTracker(const GpuTracker&) = delete;
    GpuTracker& operator=(const GpuTracker&) = delete;

    // raw recording bytes in the samples-module format (samples.hpp:22-40)
    void push(const void* bytes, int64_t nbytes) { check(l1rxg_tracker_push(trk_, 0, bytes, nbytes)); }
    void run(int max_epochs = -1) { check(l1rxg_tracker_run(trk_, max_epochs)); }
    void channels(std::vector<ChannelState>& out) {
        std::vector<l1rxg_channel> c(n_);
        check(l1rxg_tracker_channels(trk_, c.data()));
        out.resize(n_);
        for (std::size_t k = 0; k < n_; ++k) {
            out[k].prn = c[k].prn;
            from_c(c[k], out[k], window_ms_);
        }
    }
    std::vector<l1rxg_epoch_record> records(int channel, int64_t e0, int64_t count) {
        std::vector<l1rxg_epoch_record> r(static_cast<std::size_t>(count));
        check(l1rxg_tracker_records(trk_, channel, e0, count, r.data(), nullptr));
        return r;
    }

private:
    l1rxg_tracker* trk_ = nullptr;
    int window_ms_ = 0;
    std::size_t n_ = 0;
};

// Host navigation-data consumer over the GPU's epoch records (SURVEY.md 8(f)
// item 1): the reference's own nav::on_prompt (navdata.hpp:607-625), fed the
// values track_epoch would have passed it (tracking.hpp:596-597): the epoch's
// prompt I, its epoch index and chi at the START of the epoch (the previous
// record's chi, or the hand-off value for the first).  Legal off the device
// because nav state never feeds the loops; a record with state Idle is where
// the reference would have reset it (tracking.hpp:511-514).
inline void replay_nav(NavDecodeState& st, const std::vector<l1rxg_epoch_record>& recs,
                       double& chi_at_start) {
    for (const auto& r : recs) {
        nav::on_prompt(st, r.ip, r.epoch_index, chi_at_start);
        chi_at_start = r.chi_chips;
        if (r.state == L1RXG_IDLE)
            st = NavDecodeState{};
    }
}

}  // namespace l1rx::gpu
