// gpu_receiver.cpp -- a GPU receiver front end over the C ABI only
// (include/l1rxg.h; no CUDA or reference headers needed): cold-start
// acquisition on the tensor-core search grid, the reference's peak rule and
// channel hand-off, then closed-loop tracking of a recording streamed from
// disk through pinned, double-buffered pushes -- SURVEY.md 8(f) items 2-3
// (GPU acquisition hand-off; receiver integration with paced mode and
// overflow accounting, the analogue of the paper's Table 6 real-time run).
//
//   gpu_receiver FILE FORMAT FS_HZ IF_HZ [--acq-ms N] [--chunk-ms N]
//                [--paced] [--max-ms N]
//   FORMAT: int8_real_if | int8_iq | int16_iq
//
// Prints one JSON object per detected channel and a summary object.
// Reference behaviour mirrored: acquisition.hpp:114-149 (pick_peak: peak
// cell, runner-up outside +-1 chip, threshold ratio 2.0) and
// tracking.hpp:622-650 (init_channel_from_acquisition) through the library's
// l1rxg_pick_peak / l1rxg_init_channel, pipeline.hpp:388-428 (block reader +
// paced mode with overflow counting).
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "l1rxg.h"

namespace {

void die(const char* what) {
    std::fprintf(stderr, "gpu_receiver: %s: %s\n", what, l1rxg_last_error());
    std::exit(2);
}
#define OK(x)            \
    do {                 \
        if ((x) != 0)    \
            die(#x);     \
    } while (0)

constexpr double kChipRate = 1.023e6;

}  // namespace

int main(int argc, char** argv) {
    if (argc < 5) {
        std::fprintf(stderr, "usage: %s FILE FORMAT FS_HZ IF_HZ [--acq-ms N] [--chunk-ms N] [--paced] [--max-ms N]\n",
                     argv[0]);
        return 1;
    }
    const char* path = argv[1];
    const std::string fmt_s = argv[2];
    const double fs = std::atof(argv[3]), if_hz = std::atof(argv[4]);
    int acq_ms = 10, chunk_ms = 100, max_ms = 1 << 30;
    bool paced = false;
    for (int k = 5; k < argc; ++k) {
        const std::string a = argv[k];
        if (a == "--acq-ms" && k + 1 < argc)
            acq_ms = std::atoi(argv[++k]);
        else if (a == "--chunk-ms" && k + 1 < argc)
            chunk_ms = std::atoi(argv[++k]);
        else if (a == "--max-ms" && k + 1 < argc)
            max_ms = std::atoi(argv[++k]);
        else if (a == "--paced")
            paced = true;
    }
    const int fmt = fmt_s == "int8_real_if" ? L1RXG_FMT_INT8_REAL_IF
                    : fmt_s == "int16_iq"   ? L1RXG_FMT_INT16_IQ
                                            : L1RXG_FMT_INT8_IQ;
    const int bps = fmt == L1RXG_FMT_INT8_REAL_IF ? 1 : fmt == L1RXG_FMT_INT16_IQ ? 4 : 2;
    const int64_t n = std::llround(fs / 1000.0);
    const int spc = static_cast<int>(std::llround(fs / kChipRate / 2.0));

    FILE* f = std::fopen(path, "rb");
    if (!f) {
        std::perror(path);
        return 1;
    }
    std::fseek(f, 0, SEEK_END);
    const int64_t file_bytes = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    const int64_t total_ms = std::min<int64_t>(file_bytes / (n * bps), max_ms);

    l1rxg_ctx* ctx = nullptr;
    OK(l1rxg_create(0, &ctx));

    // ---- cold start: the search grid over the first acq_ms blocks
    std::vector<uint8_t> acq(static_cast<size_t>(acq_ms * n * bps));
    if (std::fread(acq.data(), 1, acq.size(), f) != acq.size())
        die("short recording");
    std::vector<int32_t> prns(32);
    for (int p = 0; p < 32; ++p)
        prns[p] = p + 1;
    std::vector<double> bins;
    for (double b = -5000.0; b <= 5000.0 + 1e-9; b += 500.0)
        bins.push_back(b);
    const int n_delays = 2 * 1023;
    std::vector<double> plane(static_cast<size_t>(32) * bins.size() * n_delays);
    auto t0 = std::chrono::steady_clock::now();
    OK(l1rxg_search_grid(ctx, fmt, acq.data(), 0, static_cast<int64_t>(acq.size()), fs, if_hz, acq_ms,
                         prns.data(), 32, bins.data(), static_cast<int>(bins.size()), spc, n_delays,
                         plane.data()));
    const double acq_wall_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    std::vector<l1rxg_channel> chans;
    for (int p = 0; p < 32; ++p) {
        // the reference's peak rule and hand-off, from the library (one
        // implementation, pinned to acquisition.hpp:114-149 and
        // tracking.hpp:622-650 by tests/test_acquisition_ref.py, test_oracle.py)
        l1rxg_acq_result d;
        OK(l1rxg_pick_peak(plane.data() + static_cast<size_t>(p) * bins.size() * n_delays,
                           static_cast<int>(bins.size()), n_delays, bins.data(), spc, p + 1, fs,
                           2.0 /* AcqConfig::threshold_ratio, acquisition.hpp:23 */, &d));
        if (d.detected) {
            l1rxg_channel ch;
            OK(l1rxg_init_channel(d.prn, d.doppler_hz, 0, d.code_delay_samples, 0, fs, &ch));
            chans.push_back(ch);
        }
    }
    if (chans.empty()) {
        std::printf("{\"summary\": {\"detected\": 0}}\n");
        return 0;
    }

    // ---- tracking: stream the recording from its start in chunk_ms pieces
    l1rxg_tracker_desc desc;
    std::memset(&desc, 0, sizeof desc);
    desc.format = fmt;
    desc.kernel = L1RXG_KERNEL_SCALAR;
    desc.sample_rate_hz = fs;
    desc.if_frequency_hz = if_hz;
    desc.n_streams = 1;
    desc.n_channels = static_cast<int32_t>(chans.size());
    desc.ring_samples = static_cast<int64_t>(3 * chunk_ms + 8) * n;
    desc.max_records = 4 * chunk_ms;
    desc.cta_mode = L1RXG_CTA_AUTO;
    l1rxg_default_tracking_cfg(&desc.cfg);
    l1rxg_epl_taps(desc.cfg.el_spacing_chips, &desc.taps);
    std::vector<int32_t> cs(chans.size(), 0);
    l1rxg_tracker* trk = nullptr;
    OK(l1rxg_tracker_create(ctx, &desc, chans.data(), cs.data(), &trk));
    const int64_t chunk_bytes = chunk_ms * n * bps;
    void* pinned[2] = {nullptr, nullptr};
    OK(l1rxg_host_alloc(ctx, chunk_bytes, &pinned[0]));
    OK(l1rxg_host_alloc(ctx, chunk_bytes, &pinned[1]));
    std::fseek(f, 0, SEEK_SET);
    int64_t overflows = 0, ms_done = 0;
    const auto start = std::chrono::steady_clock::now();
    for (int k = 0; ms_done < total_ms; ++k) {
        const int64_t ms = std::min<int64_t>(chunk_ms, total_ms - ms_done);
        void* buf = pinned[k & 1];
        // the previous push from this buffer has been copied once the push
        // two chunks ago is done: sync keeps the double buffer safe
        if (k >= 2)
            OK(l1rxg_tracker_sync(trk));
        if (std::fread(buf, 1, static_cast<size_t>(ms * n * bps), f) != static_cast<size_t>(ms * n * bps))
            break;
        OK(l1rxg_tracker_push(trk, 0, buf, ms * n * bps));
        OK(l1rxg_tracker_run(trk, -1));
        ms_done += ms;
        if (paced) {  // hold real time; a chunk finishing late is an overflow (pipeline.hpp:412-428)
            const auto due = start + std::chrono::milliseconds(ms_done);
            if (std::chrono::steady_clock::now() > due + std::chrono::milliseconds(chunk_ms))
                ++overflows;
            std::this_thread::sleep_until(due);
        }
    }
    OK(l1rxg_tracker_sync(trk));
    const double wall_s =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
    std::vector<l1rxg_channel> out(chans.size());
    std::vector<int64_t> epochs(chans.size());
    OK(l1rxg_tracker_channels(trk, out.data()));
    OK(l1rxg_tracker_epoch_counts(trk, epochs.data()));
    int64_t ch_epochs = 0;
    for (size_t c = 0; c < out.size(); ++c) {
        ch_epochs += epochs[c];
        std::printf("{\"prn\": %d, \"state\": %d, \"epochs\": %lld, \"doppler_hz\": %.3f, \"cn0_dbhz\": %.2f, "
                    "\"carrier_lock_ratio\": %.4f, \"code_freq_hz\": %.4f}\n",
                    out[c].prn, out[c].state, static_cast<long long>(epochs[c]), out[c].carrier_doppler_hz,
                    out[c].cn0_dbhz, out[c].carrier_lock_ratio, out[c].code_freq_hz);
    }
    std::printf("{\"summary\": {\"detected\": %zu, \"recording_ms\": %lld, \"acquisition_wall_ms\": %.2f, "
                "\"tracking_wall_s\": %.4f, \"real_time_factor\": %.2f, \"channel_epochs_per_s\": %.0f, "
                "\"paced\": %s, \"overflows\": %lld}}\n",
                chans.size(), static_cast<long long>(ms_done), acq_wall_ms, wall_s,
                (ms_done / 1000.0) / wall_s, ch_epochs / wall_s, paced ? "true" : "false",
                static_cast<long long>(overflows));
    l1rxg_host_free(ctx, pinned[0]);
    l1rxg_host_free(ctx, pinned[1]);
    l1rxg_tracker_destroy(trk);
    l1rxg_destroy(ctx);
    std::fclose(f);
    return 0;
}
