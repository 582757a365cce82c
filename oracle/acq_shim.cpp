// acq_shim.cpp -- TEST INFRASTRUCTURE: C entry points over the UNMODIFIED
// reference acquisition (/root/reference/proj/include/l1rx/acquisition.hpp,
// fft.hpp) compiled against cuFFTW (oracle/fftw_cufftw/fftw3.h).  Built by
// oracle/Makefile into oracle/_ref/libl1rx_acq_ref.so; used only by tests/
// and bench.py's reference legs as the checker for the config-5 search grid
// and the acquisition hand-off.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "l1rx/acquisition.hpp"
#include "l1rxg.h"

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

void to_result(const l1rx::AcquisitionResult& r, l1rxg_acq_result* out) {
    out->prn = r.prn;
    out->detected = r.detected ? 1 : 0;
    out->ratio = r.ratio;
    out->doppler_hz = r.doppler_hz;
    out->code_delay_samples = r.code_delay_samples;
    out->code_delay_chips = r.code_delay_chips;
}

l1rx::AcqConfig make_cfg(double dmin, double dmax, double dstep, int integration_ms, double threshold) {
    l1rx::AcqConfig cfg;
    cfg.doppler_min_hz = dmin;
    cfg.doppler_max_hz = dmax;
    cfg.doppler_step_hz = dstep;
    cfg.integration_ms = integration_ms;
    cfg.threshold_ratio = threshold;
    return cfg;
}
}  // namespace

extern "C" {

const char* acq_last_error(void) { return g_err.c_str(); }

// doppler_bins (acquisition.hpp:38-50); returns the bin count (<= cap written)
int acq_doppler_bins(double dmin, double dmax, double dstep, int integration_ms, double* out, int cap) {
    int n = -1;
    const int rc = guarded([&] {
        const auto b = l1rx::doppler_bins(make_cfg(dmin, dmax, dstep, integration_ms, 2.0));
        n = static_cast<int>(b.size());
        for (int i = 0; i < n && i < cap; ++i)
            out[i] = b[static_cast<std::size_t>(i)];
    });
    return rc ? -rc : n;
}

// acquire_pcs (acquisition.hpp:189-222), the reference entry point itself
int acq_acquire_pcs(const double* iq, int64_t n, int prn, double fs, double dmin, double dmax, double dstep,
                    int integration_ms, double threshold, l1rxg_acq_result* out) {
    return guarded([&] {
        std::span<const l1rx::cplx> buf(reinterpret_cast<const l1rx::cplx*>(iq), static_cast<std::size_t>(n));
        to_result(l1rx::acquire_pcs(buf, prn, make_cfg(dmin, dmax, dstep, integration_ms, threshold), fs), out);
    });
}

// acquire_fast (acquisition.hpp:227-262)
int acq_acquire_fast(const double* iq, int64_t n, int prn, double fs, double dmin, double dmax, double dstep,
                     int integration_ms, double threshold, l1rxg_acq_result* out) {
    return guarded([&] {
        std::span<const l1rx::cplx> buf(reinterpret_cast<const l1rx::cplx*>(iq), static_cast<std::size_t>(n));
        to_result(l1rx::acquire_fast(buf, prn, make_cfg(dmin, dmax, dstep, integration_ms, threshold), fs), out);
    });
}

// The acquire_pcs plane (acquisition.hpp:196-219; the plane is internal to
// acquire_pcs, so its loop is restated here over the reference's own
// detail::conj_code_spectrum, detail::wipe_carrier and Fft): cells[b][d]
// for every sample delay d < N = fs/1000, |.| summed over n_seg segments.
int acq_pcs_plane(const double* iq, int n_seg, int prn, double fs, const double* bins, int n_bins,
                  double* cells) {
    return guarded([&] {
        const auto seg = static_cast<std::size_t>(std::llround(fs / 1000.0));
        const auto* x = reinterpret_cast<const l1rx::cplx*>(iq);
        std::span<const l1rx::cplx> buffer(x, seg * static_cast<std::size_t>(n_seg));
        const auto code_spec = l1rx::detail::conj_code_spectrum(prn, fs, seg);
        std::vector<l1rx::cplx> wiped(seg), spec(seg), corr(seg);
        std::memset(cells, 0, sizeof(double) * seg * static_cast<std::size_t>(n_bins));
        for (int b = 0; b < n_bins; ++b) {
            double* row = cells + static_cast<std::size_t>(b) * seg;
            for (int s = 0; s < n_seg; ++s) {
                l1rx::detail::wipe_carrier(buffer.subspan(static_cast<std::size_t>(s) * seg, seg),
                                           static_cast<std::size_t>(s) * seg, bins[b], fs, wiped);
                l1rx::Fft::forward(wiped, spec);
                for (std::size_t i = 0; i < seg; ++i)
                    spec[i] *= code_spec[i];
                l1rx::Fft::inverse(spec, corr);
                for (std::size_t i = 0; i < seg; ++i)
                    row[i] += std::abs(corr[i]);
            }
        }
    });
}

// detail::pick_peak (acquisition.hpp:114-149) over a caller plane
int acq_pick_peak(const double* cells, int n_bins, int n_delays, const double* bins, int prn, double fs,
                  double threshold, l1rxg_acq_result* out) {
    return guarded([&] {
        l1rx::detail::AcqPlane plane;
        plane.cells.assign(cells, cells + static_cast<std::size_t>(n_bins) * n_delays);
        plane.n_delays = static_cast<std::size_t>(n_delays);
        plane.bins.assign(bins, bins + n_bins);
        to_result(l1rx::detail::pick_peak(plane, prn, fs, threshold), out);
    });
}

}  // extern "C"
