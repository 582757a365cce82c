/*
 * l1rxg.h -- C ABI of the B200-native tracking correlator (libl1rxg.so).
 *
 * This is the drop-in boundary for the hot path of the l1rx GPS L1 C/A
 * receiver (reference: /root/reference/proj, "l1rx").  Every entry point
 * replaces one reference interface; the file:line it replaces is cited on
 * each declaration.  Nothing here throws: every function returns an
 * l1rxg_status and l1rxg_last_error() gives the (thread-local) message.
 * The status codes map 1:1 onto the reference's exception types so a C++
 * adapter (include/l1rx_gpu.hpp) can re-throw exactly what the reference
 * throws:
 *
 *   L1RXG_EINVAL  -> std::invalid_argument   (e.g. tracking.hpp:232-233)
 *   L1RXG_ELOGIC  -> std::logic_error        (tracking.hpp:526-527)
 *   L1RXG_ERANGE  -> std::out_of_range       (cacode.hpp:38-39)
 *   L1RXG_ECUDA / L1RXG_ENOMEM -> std::runtime_error
 *
 * Plain pointers and sizes only; no torch or C++ types cross this ABI.
 * All POD structs are 8-byte aligned, little-endian x86-64 layout; their
 * field order is part of the ABI (checked by tests/test_abi.py).
 */
#ifndef L1RXG_H
#define L1RXG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define L1RXG_ABI_VERSION 2
#define L1RXG_CODE_LENGTH 1023
#define L1RXG_MAX_TAPS 16
#define L1RXG_WIN_MAX 64

typedef enum {
    L1RXG_OK = 0,
    L1RXG_EINVAL = 1,
    L1RXG_ELOGIC = 2,
    L1RXG_ERANGE = 3,
    L1RXG_ECUDA = 4,
    L1RXG_ENOMEM = 5
} l1rxg_status;

/* KernelKind (tracking.hpp:60).  Scalar and Batched select the same GPU
 * correlator (both are restatements of one contract); Noop advances the
 * NCO state only (tracking.hpp:434-452). */
typedef enum {
    L1RXG_KERNEL_SCALAR = 0,
    L1RXG_KERNEL_BATCHED = 1,
    L1RXG_KERNEL_NOOP = 2
} l1rxg_kernel_kind;

/* SampleKind (samples.hpp:22-26) plus the in-memory complex formats the
 * per-call path accepts. */
typedef enum {
    L1RXG_FMT_INT8_IQ = 0,      /* Int8ComplexInterleaved, /128        */
    L1RXG_FMT_INT16_IQ = 1,     /* Int16ComplexInterleaved LE, /32768  */
    L1RXG_FMT_INT8_REAL_IF = 2, /* Int8RealIF: mixer + half-band FIR    */
    L1RXG_FMT_CF64 = 3          /* already-decoded complex<double>      */
} l1rxg_format;

/* ChannelRunState (tracking.hpp:59). */
typedef enum {
    L1RXG_IDLE = 0,
    L1RXG_ACQUIRED = 1,
    L1RXG_TRACKING = 2
} l1rxg_run_state;

/* NCO fields of ChannelState (tracking.hpp:181-185). */
typedef struct {
    double code_phase_chips;
    double code_freq_hz;
    double carrier_doppler_hz;
    double carrier_phase_rad;
    double chi_chips;
} l1rxg_nco;

/* CorrelatorOutputs (tracking.hpp:19-23). */
typedef struct {
    double ie, qe, ip, qp, il, ql;
    double ip_h1, qp_h1, ip_h2, qp_h2;
    int32_t n_samples;
    int32_t pad_;
} l1rxg_corr;

/* TrackingConfig (tracking.hpp:25-45). */
typedef struct {
    int32_t epoch_ms;
    int32_t pad0_;
    double el_spacing_chips;
    double dll_bandwidth_hz;
    double dll_damping;
    double pll_bandwidth_hz;
    double pll_damping;
    double fll_bandwidth_hz;
    int32_t fll_pull_in_ms;
    int32_t fll_coarse_ms;
    int32_t cn0_window_ms;
    int32_t lock_fail_limit;
    double cn0_drop_dbhz;
    double carrier_lock_drop;
} l1rxg_tracking_cfg;

/* Replica tap set.  The reference has exactly three taps
 * (E/P/L = +s/2, 0, -s/2; tracking.hpp:237,252-254).  Multi-tap
 * correlators (spoofing monitor, wideband batch) are the builder's K-tap
 * generalisation: tap k uses chip index trunc(fl(ph + offsets[k])), whose
 * 3-tap instance is the reference expression bit for bit.  early / prompt /
 * late name the taps that drive the DLL, the PLL/FLL and the half-epoch
 * prompt sums.  n_counted is how many taps (the first n_counted) count
 * towards the sample-tap metric; extra loop-only taps follow them. */
typedef struct {
    int32_t n_taps;
    int32_t n_counted;
    int32_t early;
    int32_t prompt;
    int32_t late;
    int32_t pad_;
    double offsets_chips[L1RXG_MAX_TAPS];
} l1rxg_taps;

/* Full ChannelState (tracking.hpp:177-207) as POD, minus NavDecodeState
 * (host-side consumer) and KernelScratch.  The C/N0
 * window vectors (tracking.hpp:203) are a fixed array of win_len entries;
 * for cn0_window_ms > L1RXG_WIN_MAX the window carries its running sums
 * instead (win_ip[0] = sum sign(ip) ip, win_qp[0] = sum sign(ip) qp,
 * win_ip[1] = sum ip^2 + qp^2 over its win_len epochs, accumulated in push
 * order -- the reference's sums bit for bit). */
typedef struct {
    int32_t prn;
    int32_t state; /* l1rxg_run_state */
    double code_phase_chips;
    double code_freq_hz;
    double carrier_doppler_hz;
    double carrier_phase_rad;
    double chi_chips;
    double dll_integrator;
    double dll_prev_error;
    double pll_integrator;
    double pll_prev_error;
    int32_t dll_primed;
    int32_t pll_primed;
    int32_t fll_enabled;
    int32_t have_last_prompt;
    double last_ip;
    double last_qp;
    int64_t epoch_ms_count;
    int64_t epochs_since_handoff;
    double cn0_dbhz;
    double carrier_lock_ratio;
    double mu_smoothed;
    int32_t lock_fail_count;
    int32_t metrics_valid;
    int64_t sample_offset_next_epoch;
    int32_t win_len;
    int32_t pad_;
    double win_ip[L1RXG_WIN_MAX];
    double win_qp[L1RXG_WIN_MAX];
} l1rxg_channel;

/* One tracked epoch of one channel: TrackingEpochOutput
 * (tracking.hpp:209-222) plus the correlator inputs/outputs, so a host
 * consumer (nav decode, telemetry) and the per-epoch replay check can use
 * it without touching the device. */
typedef struct {
    int64_t epoch_index;          /* TrackingEpochOutput::epoch_index     */
    int64_t sample_offset_start;  /* window start (input)                 */
    int64_t sample_offset_end;    /* TrackingEpochOutput::sample_offset_end */
    int32_t prn;
    int32_t state;                /* after the update                      */
    int32_t n_samples;
    int32_t lock_fail_count;
    /* NCO at epoch start: the correlator's inputs */
    double code_phase_in, code_freq_in, carrier_doppler_in, carrier_phase_in;
    /* CorrelatorOutputs (E/P/L = taps.early/prompt/late) */
    double ie, qe, ip, qp, il, ql, ip_h1, qp_h1, ip_h2, qp_h2;
    /* state after the loop update */
    double carrier_doppler_hz, code_freq_hz, code_phase_chips;
    double carrier_phase_rad, chi_chips, cn0_dbhz, carrier_lock_ratio;
    double dll_integrator, pll_integrator, mu_smoothed;
    double dll_prev_error, pll_prev_error;
} l1rxg_epoch_record;

typedef struct l1rxg_ctx l1rxg_ctx;
typedef struct l1rxg_tracker l1rxg_tracker;

/* ---- library --------------------------------------------------------- */
int l1rxg_abi_version(void);
const char* l1rxg_last_error(void);
/* Fills cfg with TrackingConfig{} defaults (tracking.hpp:25-45). */
void l1rxg_default_tracking_cfg(l1rxg_tracking_cfg* cfg);
/* E/P/L taps for el_spacing (tracking.hpp:237). */
void l1rxg_epl_taps(double el_spacing_chips, l1rxg_taps* taps);

/* generate_ca_code (cacode.hpp:37-64): chips in +/-1 form. */
int l1rxg_ca_code(int prn, int8_t* chips_out /* 1023 */);
/* detail::halfband_taps (samples.hpp:89-108). */
void l1rxg_halfband_taps(double* taps_out /* 23 */);

/* ---- context (one per device) ---------------------------------------- */
int l1rxg_create(int device, l1rxg_ctx** out);
int l1rxg_destroy(l1rxg_ctx* ctx);
/* pinned host buffers for the double-buffered H2D ingest ring */
int l1rxg_host_alloc(l1rxg_ctx* ctx, int64_t bytes, void** out);
int l1rxg_host_free(l1rxg_ctx* ctx, void* p);

/* ---- per-call compatibility path ------------------------------------- */
/* correlate_epoch_scalar / _batched / _noop (tracking.hpp:226-230,
 * 288-292, 434-436): one epoch of n complex<double> samples (interleaved
 * re,im), NCO state advanced in place (tracking.hpp:275-280),
 * CorrelatorOutputs returned.  n == 0 -> L1RXG_EINVAL ("empty epoch view").
 * Re-entrant: each calling host thread gets its own CUDA stream and device
 * buffers (created on its first call, freed by l1rxg_destroy), so the
 * reference's ChannelPool workers (pipeline.hpp:584-588) call it
 * concurrently, one channel each. */
int l1rxg_correlate_epoch(l1rxg_ctx* ctx, int kernel, const double* iq,
                          int n, l1rxg_nco* state_inout, int prn,
                          double el_spacing_chips, double sample_rate_hz,
                          l1rxg_corr* out);

/* Open-loop batch: n_jobs independent channel-epochs of n samples each
 * (job j reads iq + 2*n*j), K taps.  tap_sums_out[j*2K + 2k + {0,1}] = I/Q
 * of tap k; corr_out[j] carries E/P/L + half-epoch prompt sums.  NCO
 * states are advanced in place exactly as the reference does. */
int l1rxg_correlate_batch(l1rxg_ctx* ctx, const double* iq, int n,
                          int n_jobs, l1rxg_nco* states_inout,
                          const int32_t* prns, const l1rxg_taps* taps,
                          double sample_rate_hz, double* tap_sums_out,
                          l1rxg_corr* corr_out);

/* ---- closed-loop tracking (the performance path) --------------------- */
/* track_epoch (tracking.hpp:520-618) + update_quality_metrics (:459-515)
 * run on device between 1-ms epochs for every channel; replaces the
 * Receiver::tracking_round fan-out (pipeline.hpp:563-610).  Channels are
 * bound to one of n_streams independent sample streams (recordings). */
typedef struct {
    int32_t format;            /* l1rxg_format (not CF64)              */
    int32_t kernel;            /* l1rxg_kernel_kind                     */
    double sample_rate_hz;
    double if_frequency_hz;    /* Int8RealIF only                       */
    int32_t n_streams;
    int32_t n_channels;
    int64_t ring_samples;      /* per-stream device ring capacity       */
    int32_t max_records;       /* per-channel record ring capacity      */
    /* CTA shape: 0 = auto.  L1RXG_CTA_LATENCY: each channel's epoch split
     * over a thread-block cluster of up to 16 CTAs (one per SM; the CTAs
     * exchange fp64 partial sums through distributed shared memory and all
     * run the same loop update) -- few channels, the per-epoch critical path
     * is what matters; L1RXG_CTA_SINGLE: the latency shape with one CTA per
     * channel; L1RXG_CTA_THROUGHPUT: narrow CTAs, four resident per SM, so
     * one channel's serial loop update overlaps the others' correlation
     * (many channels).  Auto picks throughput when n_channels >= 2 x SMs.
     * L1RXG_CTA_SEGMENT: the throughput shape's segment correlator over a
     * raw complex-int16 ring (no decode pass; per-warp TMA tensor copies;
     * the run sums captured in registers instead of a shared-memory prefix
     * tile); complex int16 only, fs >= 3.073 MHz.  Auto picks it for the
     * throughput shape on complex int16 recordings whose chips span > 33
     * samples with tap residues > 15.5 samples apart (BASELINE config 4). */
    int32_t cta_mode;
    /* Latency shape: CTAs per channel cluster (0 = auto, 1..16). */
    int32_t cluster_size;
    /* 1: keep complex int recordings raw in the ring (2/4 B per sample,
     * converted in the correlator); 0: decode to float2 (default). */
    int32_t ring_raw;
    l1rxg_taps taps;
    l1rxg_tracking_cfg cfg;
} l1rxg_tracker_desc;

#define L1RXG_CTA_AUTO 0
#define L1RXG_CTA_LATENCY 1
#define L1RXG_CTA_THROUGHPUT 2
#define L1RXG_CTA_SINGLE 3
#define L1RXG_CTA_SEGMENT 4

int l1rxg_tracker_create(l1rxg_ctx* ctx, const l1rxg_tracker_desc* desc,
                         const l1rxg_channel* channels,
                         const int32_t* channel_stream,
                         l1rxg_tracker** out);
int l1rxg_tracker_destroy(l1rxg_tracker* trk);
/* Appends raw recording bytes (host memory; pinned is fastest) to stream
 * s: async H2D into the device ring, then on-device ingest (decode, or
 * the reference's fs/4 mixer + half-band FIR with carried history,
 * samples.hpp:215-253).  Replaces SampleSource::read_block +
 * BlockQueue (samples.hpp:136-211, pipeline.hpp:388-404). */
int l1rxg_tracker_push(l1rxg_tracker* trk, int stream, const void* bytes,
                       int64_t nbytes);
/* Same, from bytes already resident in device memory. */
int l1rxg_tracker_push_device(l1rxg_tracker* trk, int stream,
                              const void* dev_bytes, int64_t nbytes);
/* Host-memory variant: one pitched H2D copy (host stream s at
 * bytes + s * stride_bytes) into the staging block, then the strided
 * device push.  Asynchronous like l1rxg_tracker_push. */
int l1rxg_tracker_push_strided(l1rxg_tracker* trk, const void* bytes,
                               int64_t nbytes_per_stream, int64_t stride_bytes);
/* Appends nbytes_per_stream to EVERY stream in one launch: stream s reads
 * dev_bytes + s * stride_bytes (device memory).  All streams must be at the
 * same sample count (the batched-recordings case, BASELINE config 4: one
 * SampleSource per recording, samples.hpp:136-211, fed in lock step). */
int l1rxg_tracker_push_device_strided(l1rxg_tracker* trk, const void* dev_bytes,
                                      int64_t nbytes_per_stream,
                                      int64_t stride_bytes);
/* Segment correlator (cta_mode SEGMENT) only: the trackers' rings become
 * complex-int16 recordings already resident in device memory (stream s at
 * dev_bytes + s * stride_bytes, samples_per_stream samples each, a multiple
 * of 32; 16-byte aligned base and stride): every sample is available at
 * once and no ingest pass runs (the correlator reads the recordings in
 * place by TMA).  The streams must be empty (fresh or reset); reset keeps
 * the attachment.  Replaces SampleSource over a file already read
 * (samples.hpp:136-211) for batch re-processing. */
int l1rxg_tracker_attach_device(l1rxg_tracker* trk, const void* dev_bytes,
                                int64_t samples_per_stream, int64_t stride_bytes);
/* Ends an attachment: the tracker reads its own ring again, every stream
 * restarts empty (pushes are refused while recordings are attached). */
int l1rxg_tracker_detach(l1rxg_tracker* trk);
/* Runs every channel over every epoch whose 1-ms window is fully
 * ingested (at most max_epochs per channel; <0 = unbounded).  Async. */
int l1rxg_tracker_run(l1rxg_tracker* trk, int max_epochs);
int l1rxg_tracker_sync(l1rxg_tracker* trk);
/* Channel states and per-channel epoch counts after sync. */
int l1rxg_tracker_channels(l1rxg_tracker* trk, l1rxg_channel* out);
int l1rxg_tracker_epoch_counts(l1rxg_tracker* trk, int64_t* out);
/* Records of channel c, epochs [e0, e0+count) (must still be in the
 * per-channel record ring), and the per-tap sums (2 doubles per tap). */
int l1rxg_tracker_records(l1rxg_tracker* trk, int channel, int64_t e0,
                          int64_t count, l1rxg_epoch_record* out,
                          double* tap_sums_out);
/* All records of the ring, channel-major [channel][max_records], into a
 * device buffer (for an NCCL gather) or host buffer. */
int l1rxg_tracker_records_raw(l1rxg_tracker* trk, void* dst, int dst_is_device,
                              int64_t* bytes_out);
/* Restarts every stream at sample 0 (empty ring, zero FIR history, like a
 * fresh SampleSource) and resets the channels to `channels` with zero epoch
 * counts: one more pass over a recording without reallocating.  channels ==
 * NULL restores the channels given to l1rxg_tracker_create (a device-side
 * copy: no host transfer). */
int l1rxg_tracker_reset(l1rxg_tracker* trk, const l1rxg_channel* channels);
/* The CUDA stream (cudaStream_t) the tracker's kernels run on, so a caller
 * can bracket work with its own events. */
void* l1rxg_tracker_stream(l1rxg_tracker* trk);
/* Reads back ingested baseband samples [s0, s0+count) of stream s as
 * interleaved doubles (ingest parity checks against SampleSource). */
int l1rxg_tracker_read_samples(l1rxg_tracker* trk, int stream, int64_t s0,
                               int64_t count, double* iq_out);
/* Milliseconds of device time of the last run() (CUDA events on the
 * tracker's stream), split into ingest and tracking kernels. */
int l1rxg_tracker_timing(l1rxg_tracker* trk, double* ingest_ms,
                         double* track_ms, int64_t* kernel_launches);

/* ---- search grid (config 5) ------------------------------------------ */
/* acquire_pcs plane semantics (acquisition.hpp:170-222): for each PRN and
 * Doppler bin, carrier wipe anchored at the global sample index, circular
 * correlation with the zero-order-hold code at delays d = 8k... given by
 * delay_step, |.| accumulated over n_blocks 1-ms blocks, scaled by N like
 * FFTW's unnormalised inverse (fft.hpp:17-19).  Input is the raw stream. */
int l1rxg_search_grid(l1rxg_ctx* ctx, int format, const void* bytes,
                      int bytes_on_device, int64_t nbytes,
                      double sample_rate_hz, double if_frequency_hz,
                      int n_blocks, const int32_t* prns, int n_prns,
                      const double* doppler_bins_hz, int n_bins,
                      int delay_step, int n_delays, double* plane_out);
/* Same plane into float32 or float64 (plane_f32 = 1 / 0) at host or device
 * memory (plane_on_device): the GPU converts and trims the plane, so a pinned
 * host buffer or a device buffer (e.g. for an NCCL gather) receives it with
 * one copy.  l1rxg_search_grid = float64, host. */
int l1rxg_search_grid_ex(l1rxg_ctx* ctx, int format, const void* bytes,
                         int bytes_on_device, int64_t nbytes,
                         double sample_rate_hz, double if_frequency_hz,
                         int n_blocks, const int32_t* prns, int n_prns,
                         const double* doppler_bins_hz, int n_bins,
                         int delay_step, int n_delays, void* plane_out,
                         int plane_f32, int plane_on_device);
/* Device time of the last l1rxg_search_grid: ingest + fold, correlation. */
int l1rxg_search_grid_timing(l1rxg_ctx* ctx, double* ingest_fold_ms,
                             double* corr_ms);

/* ---- acquisition hand-off (host functions, no GPU needed) -------------- */
/* AcquisitionResult (acquisition.hpp:52-59). */
typedef struct {
    int32_t prn;
    int32_t detected;
    double ratio;
    double doppler_hz;
    int32_t code_delay_samples;
    int32_t pad_;
    double code_delay_chips;
} l1rxg_acq_result;

/* detail::pick_peak (acquisition.hpp:114-149) over one PRN's plane
 * cells[bin][k] whose delays are d = k * delay_step samples (delay_step 1:
 * the reference's full plane; the search grid's half-chip plane: delay_step
 * = samples per half chip): peak cell; runner-up over every bin outside
 * +-ceil(fs / chip rate) samples of the peak delay, with circular distance
 * on the n_delays * delay_step sample axis; detected = ratio >= threshold. */
int l1rxg_pick_peak(const double* cells, int n_bins, int n_delays, const double* bins,
                    int delay_step, int prn, double sample_rate_hz,
                    double threshold_ratio, l1rxg_acq_result* out);
/* init_channel_from_acquisition (tracking.hpp:622-650). */
int l1rxg_init_channel(int prn, double doppler_hz, int64_t acq_buffer_start,
                       int64_t code_delay_samples, int64_t start_offset_samples,
                       double sample_rate_hz, l1rxg_channel* out);

/* ---- scenario synthesizer (test and benchmark corpora) ----------------- */
/* SimSatellite in raw mode (simsource.hpp:24-40). */
typedef struct {
    double code_delay_chips;
    double doppler_hz;
    double doppler_rate_hz_per_s;
    double initial_carrier_phase_rad;
    double cn0_dbhz;
    int32_t prn;
    int32_t pad_;
} l1rxg_sim_sv;

/* SimStream::next_block + generate_recording (simsource.hpp:194-413) on the
 * GPU for n_rec recordings at once: recording r has the n_sv satellites
 * svs[r * n_sv ...], milliseconds [ms0, ms0 + n_ms) are written as raw bytes
 * of `format` (int8/int16 IQ; int8 real IF at if_hz is a builder extension)
 * to dev_out + r * rec_stride_bytes (device memory).  Noise (noise != 0) is
 * Philox4x32-10 keyed by (seed, r) and counted by sample index, so any
 * chunking of a recording gives the same bytes.  Synchronous. */
int l1rxg_simulate(l1rxg_ctx* ctx, const l1rxg_sim_sv* svs, int n_sv, int n_rec,
                   double sample_rate_hz, double if_frequency_hz, int format,
                   int64_t ms0, int n_ms, uint64_t seed, int noise,
                   void* dev_out, int64_t rec_stride_bytes);

#ifdef __cplusplus
}
#endif

#endif /* L1RXG_H */
