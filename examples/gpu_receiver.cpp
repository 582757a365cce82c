// gpu_receiver.cpp -- a GPU receiver front end over the C ABI only
// (include/l1rxg.h; no CUDA or reference headers needed): cold-start
// acquisition on the tensor-core search grid, the reference's peak rule and
// channel hand-off, then closed-loop tracking of a recording streamed from
// disk through pinned, double-buffered pushes -- SURVEY.md 8(f) items 2-3
// (GPU acquisition hand-off; receiver integration with paced mode and
// overflow accounting, the analogue of the paper's Table 6 real-time run).
//
//   gpu_receiver FILE FORMAT FS_HZ IF_HZ [--acq-ms N] [--chunk-ms N]
//                [--paced] [--max-ms N] [--queue N] [--consumer-delay-ms N]
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
#include <condition_variable>
#include <deque>
#include <mutex>
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
        std::fprintf(stderr, "usage: %s FILE FORMAT FS_HZ IF_HZ [--acq-ms N] [--chunk-ms N] [--paced] [--max-ms N] "
                             "[--queue N] [--consumer-delay-ms N]\n",
                     argv[0]);
        return 1;
    }
    const char* path = argv[1];
    const std::string fmt_s = argv[2];
    const double fs = std::atof(argv[3]), if_hz = std::atof(argv[4]);
    int acq_ms = 10, chunk_ms = 100, max_ms = 1 << 30, queue_cap = 4, consumer_delay_ms = 0;
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
        else if (a == "--queue" && k + 1 < argc)
            queue_cap = std::max(1, std::atoi(argv[++k]));
        else if (a == "--consumer-delay-ms" && k + 1 < argc)  // test hook: a slow consumer
            consumer_delay_ms = std::atoi(argv[++k]);
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
    // ---- streaming: a producer thread reads the recording in chunk_ms blocks
    // into a bounded queue of pinned buffers (BlockQueue, pipeline.hpp:30-86);
    // paced, it releases each block at its stream time (samples.hpp:162-170)
    // and a block that finds the queue full is dropped and counted as an
    // overflow, the run marked degraded (pipeline.hpp:393-397: never silent
    // loss) -- the consumer pushes zeros in its place, so sample accounting and
    // every later epoch's timing stay exact.  Offline, the producer blocks.
    const int64_t chunk_bytes = chunk_ms * n * bps;
    const int n_buf = queue_cap + 1;  // queue slots + the one being consumed
    std::vector<void*> pinned(static_cast<size_t>(n_buf), nullptr);
    for (auto& pb : pinned)
        OK(l1rxg_host_alloc(ctx, chunk_bytes, &pb));
    void* zeros = nullptr;
    OK(l1rxg_host_alloc(ctx, chunk_bytes, &zeros));
    std::memset(zeros, 0, static_cast<size_t>(chunk_bytes));
    struct Item {
        int buf;        // pinned buffer, or -1: a dropped block (zeros)
        int64_t bytes;
    };
    std::mutex mu;
    std::condition_variable cv_item, cv_free;
    std::deque<Item> q;
    std::vector<int> free_bufs;
    for (int k = 0; k < n_buf; ++k)
        free_bufs.push_back(k);
    bool closed = false;
    int64_t overflows = 0;
    std::fseek(f, 0, SEEK_SET);
    const auto start = std::chrono::steady_clock::now();
    std::thread producer([&] {
        std::vector<unsigned char> tmp(static_cast<size_t>(chunk_bytes));
        for (int64_t done = 0; done < total_ms;) {
            const int64_t ms = std::min<int64_t>(chunk_ms, total_ms - done);
            const size_t want = static_cast<size_t>(ms * n * bps);
            if (std::fread(tmp.data(), 1, want, f) != want)
                break;
            done += ms;
            if (paced)  // the block is due at its stream time
                std::this_thread::sleep_until(start + std::chrono::milliseconds(done));
            std::unique_lock<std::mutex> lk(mu);
            if (!paced)
                cv_free.wait(lk, [&] { return !free_bufs.empty() && (int)q.size() < queue_cap; });
            if (free_bufs.empty() || (int)q.size() >= queue_cap) {  // paced: try_push failed
                ++overflows;
                q.push_back({-1, static_cast<int64_t>(want)});  // a gap marker, not data
                cv_item.notify_one();
                continue;
            }
            const int b = free_bufs.back();
            free_bufs.pop_back();
            std::memcpy(pinned[static_cast<size_t>(b)], tmp.data(), want);
            q.push_back({b, static_cast<int64_t>(want)});
            cv_item.notify_one();
        }
        std::lock_guard<std::mutex> lk(mu);
        closed = true;
        cv_item.notify_all();
    });
    int64_t ms_done = 0;
    for (;;) {
        Item it;
        {
            std::unique_lock<std::mutex> lk(mu);
            cv_item.wait(lk, [&] { return !q.empty() || closed; });
            if (q.empty())
                break;
            it = q.front();
            q.pop_front();
        }
        OK(l1rxg_tracker_push(trk, 0, it.buf >= 0 ? pinned[static_cast<size_t>(it.buf)] : zeros, it.bytes));
        OK(l1rxg_tracker_run(trk, -1));
        OK(l1rxg_tracker_sync(trk));  // the pinned buffer's copy is done: back to the pool
        ms_done += it.bytes / (n * bps);
        if (consumer_delay_ms > 0)
            std::this_thread::sleep_for(std::chrono::milliseconds(consumer_delay_ms));
        if (it.buf >= 0) {
            std::lock_guard<std::mutex> lk(mu);
            free_bufs.push_back(it.buf);
            cv_free.notify_one();
        }
    }
    producer.join();
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
                "\"paced\": %s, \"overflows\": %lld, \"degraded\": %s, \"queue\": %d}}\n",
                chans.size(), static_cast<long long>(ms_done), acq_wall_ms, wall_s,
                (ms_done / 1000.0) / wall_s, ch_epochs / wall_s, paced ? "true" : "false",
                static_cast<long long>(overflows), overflows > 0 ? "true" : "false", queue_cap);
    for (auto pb : pinned)
        l1rxg_host_free(ctx, pb);
    l1rxg_host_free(ctx, zeros);
    l1rxg_tracker_destroy(trk);
    l1rxg_destroy(ctx);
    std::fclose(f);
    return 0;
}
