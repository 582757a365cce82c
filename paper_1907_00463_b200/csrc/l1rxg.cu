// l1rxg.cu -- host runtime (C++) and C ABI of the B200 tracking correlator.
//
// One context per device owns the C/A code table (33 x 1023 int8, built
// once like ca_code_table(), cacode.hpp:99-107), two CUDA streams (compute
// and H2D copy) and scratch buffers.  A tracker owns per-stream device
// rings of complex baseband (float2) fed by the ingest kernels, the channel
// states, and per-channel epoch-record rings.  See include/l1rxg.h for the
// reference interface each entry point replaces.
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <mutex>
#include <string>
#include <vector>

#include "correlator.cuh"
#include "ingest.cuh"
#include "search.cuh"
#include "ovlcorr.cuh"
#include "segcorr.cuh"
#include "gridmma.cuh"
#include "simgen.cuh"
#include "l1rxg.h"

using namespace l1rxg;

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CK(expr)                                                                 \
    do {                                                                         \
        cudaError_t e_ = (expr);                                                 \
        if (e_ != cudaSuccess)                                                   \
            return set_err(e_ == cudaErrorMemoryAllocation ? L1RXG_ENOMEM        \
                                                           : L1RXG_ECUDA,        \
                           std::string(#expr) + ": " + cudaGetErrorString(e_));  \
    } while (0)

// ---- C/A code generation (cacode.hpp:20-64), host side ---------------
const int k_g2_taps[33][2] = {
    {0, 0},  {2, 6}, {3, 7}, {4, 8},  {5, 9}, {1, 9},  {2, 10}, {1, 8}, {2, 9},
    {3, 10}, {2, 3}, {3, 4}, {5, 6},  {6, 7}, {7, 8},  {8, 9},  {9, 10}, {1, 4},
    {2, 5},  {3, 6}, {4, 7}, {5, 8},  {6, 9}, {1, 3},  {4, 6},  {5, 7},  {6, 8},
    {7, 9},  {8, 10}, {1, 6}, {2, 7}, {3, 8}, {4, 9},
};

void gold_code(int prn, int8_t* out) {
    // G1 = x^10+x^3+1, G2 = x^10+x^9+x^8+x^6+x^3+x^2+1 as 10-bit shift
    // registers (bit j = stage j+1), G2 output from the phase-select taps.
    unsigned g1 = 0x3FF, g2 = 0x3FF;
    const int t1 = k_g2_taps[prn][0] - 1, t2 = k_g2_taps[prn][1] - 1;
    for (int i = 0; i < 1023; ++i) {
        const unsigned o = ((g1 >> 9) ^ (g2 >> t1) ^ (g2 >> t2)) & 1u;
        out[i] = static_cast<int8_t>(1 - 2 * static_cast<int>(o));
        const unsigned f1 = ((g1 >> 2) ^ (g1 >> 9)) & 1u;
        const unsigned f2 = ((g2 >> 1) ^ (g2 >> 2) ^ (g2 >> 5) ^ (g2 >> 7) ^ (g2 >> 8) ^ (g2 >> 9)) & 1u;
        g1 = ((g1 << 1) | f1) & 0x3FF;
        g2 = ((g2 << 1) | f2) & 0x3FF;
    }
}

void halfband(double* h) {  // samples.hpp:89-108
    double sum = 0.0;
    for (int n = 0; n < 23; ++n) {
        const double k = static_cast<double>(n - 11);
        double v = (n == 11) ? 0.5 : std::sin(PI_D * k / 2.0) / (PI_D * k);
        v *= 0.54 - 0.46 * std::cos(2.0 * PI_D * n / 22.0);
        h[n] = v;
        sum += v;
    }
    for (int n = 0; n < 23; ++n)
        h[n] /= sum;
}

std::once_flag g_const_once;
int g_const_rc = 0;

int upload_constants() {
    std::call_once(g_const_once, [] {
        double h[23];
        halfband(h);
        float re[4][23], im[4][23], h2[23];
        // mixed(g) = v/128 * P[g mod 4], P = {1, -j, -1, j}
        const double pr[4] = {1, 0, -1, 0}, pi[4] = {0, -1, 0, 1};
        for (int r = 0; r < 4; ++r)
            for (int t = 0; t < 23; ++t) {
                const int p = ((r - t) % 4 + 4) % 4;
                re[r][t] = static_cast<float>(2.0 * h[t] / 128.0 * pr[p]);
                im[r][t] = static_cast<float>(2.0 * h[t] / 128.0 * pi[p]);
            }
        for (int t = 0; t < 23; ++t)
            h2[t] = static_cast<float>(2.0 * h[t]);
        If4Fir f{};
        for (int k = 0; k < 12; ++k)
            f.a[k] = re[0][2 * k];
        f.c = im[0][11];
        for (int r = 0; r < 4; ++r) {
            const float big = (r & 1) ? im[r][0] : re[r][0];
            const float cc = (r & 1) ? re[r][11] : im[r][11];
            if (std::fabs(big) != std::fabs(f.a[0]) || std::fabs(cc) != std::fabs(f.c))
                g_const_rc = 1;
            f.big_neg |= (big != f.a[0] ? 1u : 0u) << r;
            f.c_neg |= (cc != f.c ? 1u : 0u) << r;
        }
        if (cudaMemcpyToSymbol(c_if4f, &f, sizeof f) != cudaSuccess)
            g_const_rc = 1;
        if (cudaMemcpyToSymbol(c_halfband2, h2, sizeof h2) != cudaSuccess)
            g_const_rc = 1;
    });
    return g_const_rc;
}

// instantiated tap counts; a request for K taps runs the smallest T >= K
// with the extra taps padded (their sums are discarded)
const int k_inst[] = {3, 5, 7, 9, 11, 13, 16};
int pick_T(int K) {
    for (int t : k_inst)
        if (t >= K)
            return t;
    return -1;
}

// Block size: enough RUN-sample runs to cover the epoch in the fewest
// sub-tiles of at most 768 threads (<= 190 KB of shared tile).
int pick_threads(int n, int* subtiles, int max_nt = MAX_NT) {
    const int k = (n + max_nt * RUN - 1) / (max_nt * RUN);
    const int runs = (n + k * RUN - 1) / (k * RUN);
    int nt = ((runs + 31) / 32) * 32;
    nt = std::max(64, std::min(max_nt, nt));
    if (subtiles)
        *subtiles = (n + nt * RUN - 1) / (nt * RUN);
    return nt;
}

// header + anchors[nwork] + nbuf sample tiles of nwork*RUN samples of esz
// bytes (+ bulk-copy slack) + for raw sample kinds the float2 prefix tile
template <int T>
size_t smem_bytes(int nwork, int nbuf = 1, int esz = 8) {
    return corr_smem_header<T>() + static_cast<size_t>(anchors_len(nwork)) * sizeof(float2) +
           static_cast<size_t>(nbuf) * tile_bytes(nwork, esz) +
           (esz == 8 ? 0 : static_cast<size_t>(nwork) * RUN * sizeof(float2));
}

// ring element size per recording format: real IF is filtered to float2;
// complex int recordings are decoded to float2 too unless the descriptor's
// ring_raw keeps them raw (2/4 B per sample, converted in the correlator:
// fewer ring and shared-memory bytes, but the separate prefix tile costs
// shared-memory capacity -- measured slower for the throughput shape)
int ring_esz(int fmt, int raw) {
    if (!raw)
        return 8;
    return fmt == L1RXG_FMT_INT16_IQ ? 4 : fmt == L1RXG_FMT_INT8_IQ ? 2 : 8;
}

// Loop-filter constants precomputed with the reference's operation order
// (tracking.hpp:71-92, 466, 542).
LoopCfg make_loop_cfg(const l1rxg_tracking_cfg& cfg, int kernel, double fs, int n) {
    LoopCfg lc{};
    lc.cfg = cfg;
    lc.kernel = kernel;
    lc.fs = fs;
    lc.dt = static_cast<double>(n) / fs;
    auto wn = [](double bw, double z) { return 8.0 * z * bw / (4.0 * z * z + 1.0); };
    const double wp = wn(cfg.pll_bandwidth_hz, cfg.pll_damping);
    const double wd = wn(cfg.dll_bandwidth_hz, cfg.dll_damping);
    lc.pll_k1 = wp * wp * lc.dt * 0.5;
    lc.pll_k2 = 2.0 * cfg.pll_damping * wp;
    lc.dll_k1 = wd * wd * lc.dt * 0.5;
    lc.dll_k2 = 2.0 * cfg.dll_damping * wd;
    lc.fll_k = 4.0 * cfg.fll_bandwidth_hz * 2.0 * PI_D;
    lc.alpha = 1.0 / static_cast<double>(cfg.cn0_window_ms);
    lc.inv_fll_c = 1.0 / (2.0 * PI_D * (lc.dt / 2.0));
    lc.inv_fll_f = 1.0 / (2.0 * PI_D * lc.dt);
    return lc;
}

template <int T, int SK, bool THR>
int launch_track_sk(const TrackArgs& a, int n_ch, int nt, cudaStream_t s) {
    // the control warp owns no tile runs; + the cluster exchange slots
    const size_t sm = smem_bytes<T>(nt - 32, a.nbuf, Samp<SK>::esz) +
                      (a.csize > 1 ? 2u * a.csize * (2 * T + 2) * sizeof(double) : 0);
    CK(cudaFuncSetAttribute(track_kernel<T, SK, THR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    CK(cudaFuncSetAttribute(track_kernel<T, SK, THR>, cudaFuncAttributePreferredSharedMemoryCarveout,
                            cudaSharedmemCarveoutMaxShared));
    if (a.csize <= 1) {
        track_kernel<T, SK, THR><<<n_ch, nt, sm, s>>>(a);
    } else {  // one thread-block cluster of csize CTAs per channel
        if (a.csize > 8)
            CK(cudaFuncSetAttribute(track_kernel<T, SK, THR>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(n_ch * a.csize));
        cfg.blockDim = dim3(static_cast<unsigned>(nt));
        cfg.dynamicSmemBytes = sm;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = static_cast<unsigned>(a.csize);
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, track_kernel<T, SK, THR>, a));
    }
    CK(cudaGetLastError());
    return 0;
}

template <int T, bool THR>
int launch_track_thr(const TrackArgs& a, int n_ch, int nt, cudaStream_t s, int sk) {
    switch (sk) {
    case SK_I16: return launch_track_sk<T, SK_I16, THR>(a, n_ch, nt, s);
    case SK_I8: return launch_track_sk<T, SK_I8, THR>(a, n_ch, nt, s);
    default: return launch_track_sk<T, SK_F32, THR>(a, n_ch, nt, s);
    }
}
// Overlapped latency kernel (ovlcorr.cuh): float2 rings, two tiles, one unit
// per epoch, and its P'/M' tiles within the shared-memory budget.  Returns
// -1 when not applicable (the caller then runs track_kernel).
// Shared memory of track_ovl_kernel<T, RAW> for nt main threads (0: does not fit / not applicable).
template <int T>
size_t ovl_smem(const TrackArgs& a, int nt, bool raw) {
    const int len = a.csize > 1 ? std::min(a.n, a.share) : a.n;  // rank 0's unit: the largest
    if (len > (nt - 32) * RUN)
        return 0;
    const int nrun = (len + RUN - 1) / RUN;  // the kernel's layout unit
    const size_t xsl = ovl_xslot_bytes(a.csize, 2 * T + 2);
    const size_t sm = smem_bytes<T>(nrun, 2, 8) + xsl + ovl_extra_bytes(nrun) + (raw ? ovl_raw_bytes(nrun) : 0);
    return sm > 227u * 1024u ? 0 : sm;
}

template <int T, bool RAW>
int launch_ovl_k(const TrackArgs& a, int n_ch, int nt, cudaStream_t s, bool check_only) {
    const size_t sm = ovl_smem<T>(a, nt, RAW);
    const int block = nt + (RAW ? 32 * OVL_NF : 0);
    if (!sm || block > MAX_NT)
        return -1;
    CK(cudaFuncSetAttribute(track_ovl_kernel<T, RAW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    CK(cudaFuncSetAttribute(track_ovl_kernel<T, RAW>, cudaFuncAttributePreferredSharedMemoryCarveout,
                            cudaSharedmemCarveoutMaxShared));
    // the P'/M' tiles must not cost co-residency: every CTA of the launch
    // resident at once, as with track_kernel (measured: config 3's paired
    // CTAs at one per SM run 2.3x slower)
    int per_sm = 0, nsm = 148, dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, track_ovl_kernel<T, RAW>, block, sm));
    if (static_cast<long long>(n_ch) * a.csize > static_cast<long long>(per_sm) * nsm)
        return -1;
    if (check_only)
        return 0;
    if (a.csize <= 1) {
        track_ovl_kernel<T, RAW><<<n_ch, block, sm, s>>>(a);
    } else {
        if (a.csize > 8)
            CK(cudaFuncSetAttribute(track_ovl_kernel<T, RAW>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(n_ch * a.csize));
        cfg.blockDim = dim3(static_cast<unsigned>(block));
        cfg.dynamicSmemBytes = sm;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = static_cast<unsigned>(a.csize);
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, track_ovl_kernel<T, RAW>, a));
    }
    CK(cudaGetLastError());
    return 0;
}

// Overlapped latency kernel (ovlcorr.cuh): float2 rings (or the raw real-IF
// byte ring, sk == SK_R8), two tiles, one unit per epoch, and its P'/M' tiles
// within the shared-memory budget.  Returns -1 when not applicable (the caller
// then runs track_kernel; a raw real-IF ring is only created when it applies).
template <int T>
int launch_ovl(const TrackArgs& a, int n_ch, int nt, cudaStream_t s, int sk, bool check_only = false) {
    static const char* ev = std::getenv("L1RXG_OVL");
    if ((ev && ev[0] == '0') || a.thr || (sk != SK_F32 && sk != SK_R8) || a.nbuf != 2 ||
        a.lc.kernel == L1RXG_KERNEL_NOOP)
        return -1;
    return sk == SK_R8 ? launch_ovl_k<T, true>(a, n_ch, nt, s, check_only)
                       : launch_ovl_k<T, false>(a, n_ch, nt, s, check_only);
}
// create-time probe: would the RAW variant run this tracker's shape?
template <int T>
int ovl_raw_applicable(const TrackArgs& a, int n_ch, int nt) {
    return launch_ovl<T>(a, n_ch, nt, nullptr, SK_R8, true);
}

// How many clusters of K CTAs (nt threads each) can be resident at once for
// the latency kernels launch_track may pick (the smaller of track_kernel's
// and the overlapped kernel's count).  Clusters of more than 8 CTAs are
// limited by how many fit a GPC, not by the SM count, so the auto cluster
// rule checks this before it keeps K = 16.
template <int T>
int cluster_capacity(int K, int nt, int nbuf, int len) {
    auto cap = [&](const void* fn, size_t sm) -> int {
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess ||
            (K > 8 && cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)) {
            cudaGetLastError();
            return 0;
        }
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(K));
        cfg.blockDim = dim3(static_cast<unsigned>(nt));
        cfg.dynamicSmemBytes = sm;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = static_cast<unsigned>(K);
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nc = 0;
        if (cudaOccupancyMaxActiveClusters(&nc, fn, &cfg) != cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
        return nc;
    };
    const size_t xs = 2u * K * (2 * T + 2) * sizeof(double);
    int c = cap(reinterpret_cast<const void*>(track_kernel<T, SK_F32, false>),
                smem_bytes<T>(nt - 32, nbuf, 8) + xs);
    const int nrun = (len + RUN - 1) / RUN;
    const size_t sm_ovl = smem_bytes<T>(nrun, 2, 8) + ovl_xslot_bytes(K, 2 * T + 2) + ovl_extra_bytes(nrun);
    if (nbuf == 2 && sm_ovl <= 227u * 1024u)
        c = std::min(c, cap(reinterpret_cast<const void*>(track_ovl_kernel<T, false>), sm_ovl));
    return c;
}

int cluster_capacity_T(int T, int K, int nt, int nbuf, int len) {
    switch (T) {
    case 3: return cluster_capacity<3>(K, nt, nbuf, len);
    case 5: return cluster_capacity<5>(K, nt, nbuf, len);
    case 7: return cluster_capacity<7>(K, nt, nbuf, len);
    case 9: return cluster_capacity<9>(K, nt, nbuf, len);
    case 11: return cluster_capacity<11>(K, nt, nbuf, len);
    case 13: return cluster_capacity<13>(K, nt, nbuf, len);
    default: return cluster_capacity<16>(K, nt, nbuf, len);
    }
}

template <int T>
int launch_track(const TrackArgs& a, int n_ch, int nt, cudaStream_t s, int sk) {
    if (!a.thr) {
        const int rc = launch_ovl<T>(a, n_ch, nt, s, sk);
        if (rc != -1)
            return rc;
    }
    if (sk == SK_R8)
        return set_err(L1RXG_EINVAL, "raw real-IF ring without the overlapped kernel (L1RXG_OVL changed after create?)");
    return a.thr ? launch_track_thr<T, true>(a, n_ch, nt, s, sk)
                 : launch_track_thr<T, false>(a, n_ch, nt, s, sk);
}

// Segment correlator: persistent CTAs over (chunk, channel) work items.
template <int T, bool QD>
int launch_seg_k(const SegArgs& sa, cudaStream_t s) {
    const size_t sm = seg_smem_bytes<T, QD>(sa.t.n);
    CK(cudaFuncSetAttribute(track_seg_kernel<T, QD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    CK(cudaFuncSetAttribute(track_seg_kernel<T, QD>, cudaFuncAttributePreferredSharedMemoryCarveout,
                            cudaSharedmemCarveoutMaxShared));
    // persistent: as many CTAs as fit, each looping over work items
    int per_sm = 0, nsm = 148, dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, track_seg_kernel<T, QD>, SEG_NT, sm));
    int grid = std::max(1, std::min(sa.n_items, std::max(1, per_sm) * nsm));
    if (const char* ev = std::getenv("L1RXG_SEG_GRID"))  // tests: many work items per CTA
        grid = std::max(1, std::min(grid, std::atoi(ev)));
    track_seg_kernel<T, QD><<<grid, SEG_NT, sm, s>>>(sa);
    CK(cudaGetLastError());
    return 0;
}
template <int T>
int launch_seg(const SegArgs& sa, int n_ch, cudaStream_t s) {
    (void)n_ch;
    if constexpr (3 * T <= 32 && T <= 9) {  // (the quarter grid has at most 9 distinct taps)
        if (sa.qdirect)
            return launch_seg_k<T, true>(sa, s);
    }
    return launch_seg_k<T, false>(sa, s);
}

template <int T>
int launch_jobs(const JobArgs& a, int n_jobs, int nt, cudaStream_t s) {
    const size_t sm = smem_bytes<T>(nt, 1, 8);
    CK(cudaFuncSetAttribute(correlate_jobs_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    correlate_jobs_kernel<T><<<n_jobs, nt, sm, s>>>(a);
    CK(cudaGetLastError());
    return 0;
}

#define DISPATCH_T(T_, FN, ...)            \
    switch (T_) {                          \
    case 3: return FN<3>(__VA_ARGS__);     \
    case 5: return FN<5>(__VA_ARGS__);     \
    case 7: return FN<7>(__VA_ARGS__);     \
    case 9: return FN<9>(__VA_ARGS__);     \
    case 11: return FN<11>(__VA_ARGS__);   \
    case 13: return FN<13>(__VA_ARGS__);   \
    case 16: return FN<16>(__VA_ARGS__);   \
    default: return set_err(L1RXG_EINVAL, "unsupported tap count"); \
    }

// Segment correlator fast-path geometry (track_seg_kernel is exact for any
// geometry; outside this one most runs would take its per-sample slow
// path): a chip spans more than 33 samples (at most one replica step per
// tap in a 32-sample run) and distinct tap residues (offsets mod 1 chip)
// are more than 15.5 samples apart (one dynamic capture per half-run).
bool seg_geometry_ok(const l1rxg_tracker_desc* d) {
    const double spc = d->sample_rate_hz / CHIP_RATE_HZ;
    if (spc <= 33.0)
        return false;
    std::vector<double> r;
    for (int k = 0; k < d->taps.n_taps; ++k)
        r.push_back(d->taps.offsets_chips[k] - std::floor(d->taps.offsets_chips[k]));
    std::sort(r.begin(), r.end());
    std::vector<double> u;
    for (double x : r)
        if (u.empty() || x - u.back() > 1e-9)
            u.push_back(x);
    if (u.size() > 1 && 1.0 + u.front() - u.back() < 1e-9)
        u.pop_back();  // 0 and 1 - eps are one residue
    double gap = 1.0;
    for (size_t k = 0; k < u.size(); ++k)
        gap = std::min(gap, (k + 1 < u.size() ? u[k + 1] : 1.0 + u[0]) - u[k]);
    return gap * spc > 15.5;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no
// libcuda link dependency).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// Complex-int16 streams as a 3-D tensor of u32 samples for the segment
// correlator: {32 samples, rows per stream, streams} (stream s at
// base + s * stride_bytes), box 32 x 32 rows x 1, 128-byte swizzle.
int encode_ring_map(CUtensorMap* map, void* ring, int64_t rows, int64_t stride_bytes, int n_streams) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p)
            return set_err(L1RXG_ECUDA, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    cuuint64_t dims[3] = {32, static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(n_streams)};
    cuuint64_t strides[2] = {128, static_cast<cuuint64_t>(stride_bytes)};
    cuuint32_t box[3] = {32, 32, 1};
    cuuint32_t es[3] = {1, 1, 1};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, ring, dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return set_err(L1RXG_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return 0;
}

// 2-D uint8 tensor {cols, rows} (row pitch = cols bytes), box {box_cols,
// box_rows}, 128-byte swizzle: the search grid's digit rows for K4c.
int encode_u8_2d(CUtensorMap* map, void* base, int64_t cols, int64_t rows, int box_cols, int box_rows) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p)
            return set_err(L1RXG_ECUDA, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols)};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
    cuuint32_t es[2] = {1, 1};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return set_err(L1RXG_ECUDA, "cuTensorMapEncodeTiled (grid digits) failed (" + std::to_string((int)r) + ")");
    return 0;
}

int validate_taps(const l1rxg_taps* t) {
    if (!t || t->n_taps < 1 || t->n_taps > L1RXG_MAX_TAPS)
        return set_err(L1RXG_EINVAL, "n_taps must be in 1..16");
    for (int k : {t->early, t->prompt, t->late})
        if (k < 0 || k >= t->n_taps)
            return set_err(L1RXG_EINVAL, "early/prompt/late must index a tap");
    for (int k = 0; k < t->n_taps; ++k)
        if (!(std::fabs(t->offsets_chips[k]) <= 1.0))
            return set_err(L1RXG_EINVAL, "tap offsets must be within +/-1 chip");
    return 0;
}

// tracking.hpp:47-57
int validate_cfg(const l1rxg_tracking_cfg* c) {
    if (c->el_spacing_chips <= 0 || c->el_spacing_chips > 1)
        return set_err(L1RXG_EINVAL, "el_spacing_chips must be in (0,1]");
    if (c->dll_bandwidth_hz <= 0 || c->pll_bandwidth_hz <= 0 || c->fll_bandwidth_hz <= 0)
        return set_err(L1RXG_EINVAL, "loop bandwidths must be positive");
    if (c->epoch_ms != 1)
        return set_err(L1RXG_EINVAL, "only 1 ms epochs are supported");
    if (c->cn0_window_ms < 2)
        return set_err(L1RXG_EINVAL, "cn0_window_ms must be >= 2");
    return 0;
}

l1rxg_taps padded_taps(const l1rxg_taps& t, int T) {
    l1rxg_taps p = t;
    for (int k = t.n_taps; k < T; ++k)
        p.offsets_chips[k] = t.offsets_chips[t.prompt];
    return p;
}

struct DevBuf {
    void* p = nullptr;
    size_t n = 0;
    int ensure(size_t bytes) {
        if (bytes <= n)
            return 0;
        if (p)
            cudaFree(p);
        p = nullptr;
        n = 0;
        CK(cudaMalloc(&p, bytes));
        n = bytes;
        return 0;
    }
    void release() {
        if (p)
            cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

}  // namespace

// Per-thread state of the per-call path (l1rxg_correlate_epoch/_batch): its
// own stream and device buffers, so calls from many host threads -- the
// reference's ChannelPool workers, pipeline.hpp:584-588 -- run concurrently.
struct CallScratch {
    cudaStream_t s = nullptr;
    DevBuf iq64, iq32, states, prns, sums, corr;
    std::vector<double> hsums;
};

struct l1rxg_ctx {
    int device = 0;
    uint64_t id = 0;  // unique per context (keys the threads' CallScratch)
    cudaStream_t compute = nullptr, copy = nullptr;
    int8_t* d_codes = nullptr;
    uint32_t* d_chipw = nullptr;  // [33][CHIP_EXT / 32 + 1]: bit m % 32 of word m / 32 = chip[m mod 1023] > 0
    DevBuf iq64, iq32, states, prns, sums, corr;
    std::mutex scratch_mu;                    // guards `scratch` (registration, destroy)
    std::vector<CallScratch*> scratch;        // every thread's per-call state
    DevBuf graw, gbase, gF, gplane, gbins, gprns, ghist;  // search grid scratch
    DevBuf gsim;  // simulator scenario
    DevBuf gA, gMt, gC;                                   // tensor-core grid: operands, products
    DevBuf gQ, gS;                                        // K4c: int8 digit rows, row steps
    DevBuf gout;                                          // the trimmed, converted plane
    std::vector<int32_t> gMt_prns;                        // PRNs whose circulants gMt holds
    cublasHandle_t blas = nullptr;
    cudaEvent_t gev[3] = {nullptr, nullptr, nullptr};
    double grid_ms[2] = {0, 0};
    std::mutex mu;  // serialises the search grid and simulator scratch
    int64_t launches = 0;
};

struct StreamRing {
    unsigned char* ring = nullptr;  // R + apron samples of esz bytes
    int64_t pushed = 0;      // samples ingested
    int8_t* hist8[2] = {nullptr, nullptr};
    float2* histf[2] = {nullptr, nullptr};
    int hist_cur = 0;
};

struct l1rxg_tracker {
    l1rxg_ctx* ctx = nullptr;
    l1rxg_tracker_desc d{};
    int T = 3;
    int nt = 64;
    int nbuf = 1;
    int csize = 1;   // CTAs per channel (cluster) in the latency shape
    int thr = 0;     // throughput shape
    int seg = 0;     // segment correlator (track_seg_kernel) over a raw cint16 ring
    CUtensorMap tmap{};  // seg: the ring as [stream][row][32 samples] for TMA tensor copies
    int64_t att_samples = 0;  // seg: > 0 while device recordings are attached in place of the ring
    int* d_segq = nullptr;    // seg: work-item counter + per-channel chunks done + class counters
    int* d_gangs = nullptr;   // seg: [2][n_gangs] first channel and channel count of each gang (same-stream run)
    int n_gangs = 0, gang_max = 0;
    DevBuf seg_ctab;          // seg: per-class ticket table of a launch
    int share = 0;   // samples of each epoch per cluster CTA
    int64_t R = 0, apron = 0;
    int64_t pad = 0; // raw real-IF ring: bytes in front of every stream's ring (mirror of its tail)
    int rawif = 0;   // raw real-IF byte ring filtered inside the overlapped kernel (no ingest pass)
    int esz = 8;     // ring element bytes (ring_esz)
    std::vector<StreamRing> streams;
    unsigned char* d_ring = nullptr;
    int64_t* d_avail = nullptr;
    unsigned char* d_hist = nullptr;  // every stream's FIR histories, one allocation (zeroed by reset)
    size_t hist_bytes = 0;
    l1rxg_channel* d_chans = nullptr;
    l1rxg_channel* d_chans0 = nullptr;  // the channels given at creation (reset(NULL) restores them)
    int32_t* d_chan_stream = nullptr;
    l1rxg_epoch_record* d_recs = nullptr;
    double* d_tapsums = nullptr;
    int64_t* d_ecount = nullptr;
    int32_t* d_status = nullptr;
    DevBuf staging[2];
    DevBuf mixed;
    cudaEvent_t ev_copy[2] = {nullptr, nullptr}, ev_used[2] = {nullptr, nullptr};
    int stage_cur = 0;
    struct Timed {
        cudaEvent_t a, b;
        int kind;  // 0 ingest, 1 track
    };
    std::vector<Timed> timed;
    std::vector<cudaEvent_t> ev_pool;
    int64_t launches = 0;
};

namespace {

// This thread's per-call state for context c (created on first use).
CallScratch* call_scratch(l1rxg_ctx* c) {
    thread_local std::vector<std::pair<uint64_t, CallScratch*>> mine;
    for (auto& e : mine)
        if (e.first == c->id)
            return e.second;
    auto* cs = new CallScratch();
    if (cudaStreamCreateWithFlags(&cs->s, cudaStreamNonBlocking) != cudaSuccess) {
        delete cs;
        return nullptr;
    }
    {
        std::lock_guard<std::mutex> lk(c->scratch_mu);
        c->scratch.push_back(cs);
    }
    mine.emplace_back(c->id, cs);
    return cs;
}

cudaEvent_t get_event(l1rxg_tracker* t) {
    if (!t->ev_pool.empty()) {
        cudaEvent_t e = t->ev_pool.back();
        t->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

int ingest_launch(l1rxg_tracker* t, int s, const void* dev_bytes, int64_t nsamp,
                  cudaStream_t st) {
    StreamRing& r = t->streams[static_cast<size_t>(s)];
    const int64_t g0 = r.pushed;
    const int64_t pos0 = g0 % t->R;
    int64_t* slot = t->d_avail + s;
    const int fmt = t->d.format;
    cudaEvent_t a = get_event(t), b = get_event(t);
    cudaEventRecord(a, st);
    if (fmt == L1RXG_FMT_INT8_REAL_IF) {
        const double w = -2.0 * PI_D * t->d.if_frequency_hz / t->d.sample_rate_hz;
        if (t->rawif) {  // the bytes themselves; the overlapped kernel's FIR warps filter them
            const unsigned blocks = static_cast<unsigned>((nsamp + 255) / 256);
            copy_rawif_kernel<<<blocks, 256, 0, st>>>(static_cast<const int8_t*>(dev_bytes), nsamp,
                                                      reinterpret_cast<int8_t*>(r.ring), t->R, t->apron, pos0,
                                                      slot, g0 + nsamp);
            t->launches += 1;
        } else if (w == -PI_D / 2.0) {
            const int cur = r.hist_cur;
            const int64_t blocks = (nsamp + ING_TILE - 1) / ING_TILE;
            ingest_if4_kernel<<<(unsigned)blocks, ING_TPB, 0, st>>>(
                static_cast<const int8_t*>(dev_bytes), r.hist8[cur], r.hist8[cur ^ 1], g0, nsamp,
                reinterpret_cast<float2*>(r.ring), t->R, t->apron, pos0, slot);
            r.hist_cur ^= 1;
            t->launches += 1;
        } else {
            if (t->mixed.ensure(static_cast<size_t>(nsamp + 22) * sizeof(float2)))
                return L1RXG_ENOMEM;
            float2* mixed = static_cast<float2*>(t->mixed.p);
            const int cur = r.hist_cur;
            CK(cudaMemcpyAsync(mixed, r.histf[cur], 22 * sizeof(float2), cudaMemcpyDeviceToDevice, st));
            const unsigned blocks = static_cast<unsigned>((nsamp + 255) / 256);
            mix_generic_kernel<<<blocks, 256, 0, st>>>(static_cast<const int8_t*>(dev_bytes), g0,
                                                       nsamp, w, mixed);
            fir_generic_kernel<<<blocks, 256, 0, st>>>(mixed, nsamp, reinterpret_cast<float2*>(r.ring),
                                                       t->R, t->apron, pos0, r.histf[cur ^ 1], slot,
                                                       g0 + nsamp);
            r.hist_cur ^= 1;
            t->launches += 2;
        }
    } else {
        const unsigned blocks = static_cast<unsigned>((nsamp + 255) / 256);
        if (t->esz == 8)
            decode_iq_kernel<<<blocks, 256, 0, st>>>(dev_bytes, fmt, nsamp,
                                                     reinterpret_cast<float2*>(r.ring), t->R, t->apron,
                                                     pos0, slot, g0 + nsamp);
        else if (fmt == L1RXG_FMT_INT16_IQ)
            copy_raw_kernel<uint32_t><<<blocks, 256, 0, st>>>(
                static_cast<const uint32_t*>(dev_bytes), nsamp, reinterpret_cast<uint32_t*>(r.ring),
                t->R, t->apron, pos0, slot, g0 + nsamp);
        else
            copy_raw_kernel<uint16_t><<<blocks, 256, 0, st>>>(
                static_cast<const uint16_t*>(dev_bytes), nsamp, reinterpret_cast<uint16_t*>(r.ring),
                t->R, t->apron, pos0, slot, g0 + nsamp);
        t->launches += 1;
    }
    CK(cudaGetLastError());
    cudaEventRecord(b, st);
    t->timed.push_back({a, b, 0});
    r.pushed += nsamp;
    return 0;
}

// pushes write the tracker's own ring: refused while recordings are attached
// (the kernels read the attachment through the tensor map, not the ring)
int refuse_if_attached(const l1rxg_tracker* t) {
    if (t->att_samples > 0)
        return set_err(L1RXG_EINVAL, "push on a tracker with attached device recordings "
                                     "(l1rxg_tracker_detach first)");
    return 0;
}

int bytes_per_sample(int fmt) {
    switch (fmt) {
    case L1RXG_FMT_INT8_IQ: return 2;
    case L1RXG_FMT_INT16_IQ: return 4;
    case L1RXG_FMT_INT8_REAL_IF: return 1;
    default: return 0;
    }
}

}  // namespace

extern "C" {

int l1rxg_abi_version(void) { return L1RXG_ABI_VERSION; }
const char* l1rxg_last_error(void) { return g_err.c_str(); }

void l1rxg_default_tracking_cfg(l1rxg_tracking_cfg* c) {
    std::memset(c, 0, sizeof *c);
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

void l1rxg_epl_taps(double el_spacing, l1rxg_taps* t) {
    std::memset(t, 0, sizeof *t);
    t->n_taps = 3;
    t->n_counted = 3;
    t->early = 0;
    t->prompt = 1;
    t->late = 2;
    t->offsets_chips[0] = el_spacing / 2.0;
    t->offsets_chips[1] = 0.0;
    t->offsets_chips[2] = -el_spacing / 2.0;
}

int l1rxg_ca_code(int prn, int8_t* out) {
    if (prn < 1 || prn > 32)
        return set_err(L1RXG_ERANGE, "PRN must be in 1..32");
    gold_code(prn, out);
    return 0;
}

void l1rxg_halfband_taps(double* out) { halfband(out); }

int l1rxg_create(int device, l1rxg_ctx** out) {
    if (!out)
        return set_err(L1RXG_EINVAL, "null out");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev)
        return set_err(L1RXG_EINVAL, "no such CUDA device");
    CK(cudaSetDevice(device));
    if (upload_constants())
        return set_err(L1RXG_ECUDA, "constant upload failed");
    auto* c = new l1rxg_ctx();
    static std::atomic<uint64_t> next_id{1};
    c->id = next_id++;
    c->device = device;
    std::vector<int8_t> codes(33 * 1023, 0);
    for (int p = 1; p <= 32; ++p)
        gold_code(p, codes.data() + p * 1023);
    cudaError_t e = cudaMalloc(&c->d_codes, codes.size());
    if (e == cudaSuccess)
        e = cudaMemcpy(c->d_codes, codes.data(), codes.size(), cudaMemcpyHostToDevice);
    {
        constexpr int W = CHIP_EXT / 32 + 1;
        std::vector<uint32_t> cw(33 * W, 0u);
        for (int p = 1; p <= 32; ++p)
            for (int q = 0; q < W; ++q)
                for (int b = 0; b < 32; ++b)
                    cw[p * W + q] |= (codes[p * 1023 + (32 * q + b) % 1023] > 0 ? 1u : 0u) << b;
        if (e == cudaSuccess)
            e = cudaMalloc(&c->d_chipw, cw.size() * 4);
        if (e == cudaSuccess)
            e = cudaMemcpy(c->d_chipw, cw.data(), cw.size() * 4, cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess)
        e = cudaStreamCreateWithFlags(&c->compute, cudaStreamNonBlocking);
    if (e == cudaSuccess)
        e = cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete c;
        return set_err(L1RXG_ECUDA, std::string("context init: ") + cudaGetErrorString(e));
    }
    *out = c;
    return 0;
}

int l1rxg_destroy(l1rxg_ctx* c) {
    if (!c)
        return 0;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    for (auto e : c->gev)
        if (e)
            cudaEventDestroy(e);
    for (DevBuf* b : {&c->gsim, &c->iq64, &c->iq32, &c->states, &c->prns, &c->sums, &c->corr, &c->graw,
                      &c->gbase, &c->gF, &c->gplane, &c->gbins, &c->gprns, &c->ghist, &c->gA,
                      &c->gMt, &c->gC, &c->gQ, &c->gS, &c->gout})
        b->release();
    for (CallScratch* cs : c->scratch) {
        for (DevBuf* b : {&cs->iq64, &cs->iq32, &cs->states, &cs->prns, &cs->sums, &cs->corr})
            b->release();
        cudaStreamDestroy(cs->s);
        delete cs;
    }
    if (c->blas)
        cublasDestroy(c->blas);
    cudaFree(c->d_codes);
    cudaFree(c->d_chipw);
    cudaStreamDestroy(c->compute);
    cudaStreamDestroy(c->copy);
    delete c;
    return 0;
}

int l1rxg_host_alloc(l1rxg_ctx* c, int64_t bytes, void** out) {
    if (!c || !out || bytes <= 0)
        return set_err(L1RXG_EINVAL, "bad host_alloc arguments");
    CK(cudaSetDevice(c->device));
    CK(cudaHostAlloc(out, static_cast<size_t>(bytes), cudaHostAllocPortable));
    return 0;
}

int l1rxg_host_free(l1rxg_ctx* c, void* p) {
    (void)c;
    CK(cudaFreeHost(p));
    return 0;
}

int l1rxg_correlate_batch(l1rxg_ctx* c, const double* iq, int n, int n_jobs,
                          l1rxg_nco* states, const int32_t* prns, const l1rxg_taps* taps,
                          double fs, double* tap_sums, l1rxg_corr* corr_out) {
    if (!c)
        return set_err(L1RXG_EINVAL, "null context");
    if (n <= 0)
        return set_err(L1RXG_EINVAL, "empty epoch view");  // tracking.hpp:232-233
    if (n > MAXSUB * (MAX_NT - 32) * RUN)
        return set_err(L1RXG_EINVAL, "epoch longer than the correlator supports (fs <= 150 MHz)");
    if (n_jobs <= 0)
        return 0;
    if (int rc = validate_taps(taps))
        return rc;
    if (!(fs > 0))
        return set_err(L1RXG_EINVAL, "sample_rate_hz must be positive");
    for (int j = 0; j < n_jobs; ++j) {
        if (prns[j] < 1 || prns[j] > 32)
            return set_err(L1RXG_ERANGE, "PRN must be in 1..32");  // cacode.hpp:38-39
        const l1rxg_nco& st = states[j];
        // replica chip indices must stay inside the extended chip table
        if (!(st.code_freq_hz > 0) || !(st.code_phase_chips >= 0.0) ||
            !(st.code_phase_chips + 1023.0 + n * (st.code_freq_hz / fs) + 2.0 < (double)CHIP_EXT))
            return set_err(L1RXG_EINVAL, "code NCO state out of the correlator's domain "
                                         "(0 <= code_phase, code_freq > 0, replica span < 4096 chips)");
    }
    CK(cudaSetDevice(c->device));
    CallScratch* cs = call_scratch(c);
    if (!cs)
        return set_err(L1RXG_ECUDA, "per-thread stream creation failed");
    const int T = pick_T(taps->n_taps);
    const size_t ns = static_cast<size_t>(n) * n_jobs;
    if (cs->iq64.ensure(ns * 16) || cs->iq32.ensure(ns * 8) ||
        cs->states.ensure(sizeof(l1rxg_nco) * n_jobs) || cs->prns.ensure(4 * (size_t)n_jobs) ||
        cs->sums.ensure(sizeof(double) * 2 * T * (size_t)n_jobs) ||
        cs->corr.ensure(sizeof(l1rxg_corr) * n_jobs))
        return L1RXG_ENOMEM;
    cudaStream_t s = cs->s;
    CK(cudaMemcpyAsync(cs->iq64.p, iq, ns * 16, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(cs->states.p, states, sizeof(l1rxg_nco) * n_jobs, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(cs->prns.p, prns, 4 * (size_t)n_jobs, cudaMemcpyHostToDevice, s));
    cf64_to_f32_kernel<<<(unsigned)((ns + 255) / 256), 256, 0, s>>>(
        static_cast<const double2*>(cs->iq64.p), static_cast<float2*>(cs->iq32.p), (int64_t)ns);
    CK(cudaGetLastError());
    JobArgs a{};
    a.samples = static_cast<const float2*>(cs->iq32.p);
    a.states = static_cast<l1rxg_nco*>(cs->states.p);
    a.prns = static_cast<const int32_t*>(cs->prns.p);
    a.codes = c->d_codes;
    a.tap_sums = static_cast<double*>(cs->sums.p);
    a.corr = static_cast<l1rxg_corr*>(cs->corr.p);
    a.n = n;
    a.kp = taps->prompt;
    a.ke = taps->early;
    a.kl = taps->late;
    a.kernel = L1RXG_KERNEL_SCALAR;
    a.fs = fs;
    a.taps = padded_taps(*taps, T);
    const int nt = pick_threads(n, nullptr);
    int rc = 0;
    auto go = [&]() -> int { DISPATCH_T(T, launch_jobs, a, n_jobs, nt, s); };
    rc = go();
    if (rc)
        return rc;
    CK(cudaMemcpyAsync(states, cs->states.p, sizeof(l1rxg_nco) * n_jobs, cudaMemcpyDeviceToHost, s));
    cs->hsums.resize(static_cast<size_t>(2 * T) * n_jobs);
    CK(cudaMemcpyAsync(cs->hsums.data(), cs->sums.p, cs->hsums.size() * 8, cudaMemcpyDeviceToHost, s));
    if (corr_out)
        CK(cudaMemcpyAsync(corr_out, cs->corr.p, sizeof(l1rxg_corr) * n_jobs, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (tap_sums)
        for (int j = 0; j < n_jobs; ++j)
            std::memcpy(tap_sums + (size_t)j * 2 * taps->n_taps, cs->hsums.data() + (size_t)j * 2 * T,
                        sizeof(double) * 2 * taps->n_taps);
    return 0;
}

int l1rxg_correlate_epoch(l1rxg_ctx* c, int kernel, const double* iq, int n,
                          l1rxg_nco* st, int prn, double el_spacing, double fs,
                          l1rxg_corr* out) {
    if (n <= 0)
        return set_err(L1RXG_EINVAL, "empty epoch view");  // tracking.hpp:232-233
    if (kernel == L1RXG_KERNEL_NOOP) {  // tracking.hpp:434-452: state only
        const double w = 2.0 * PI_D * st->carrier_doppler_hz / fs;
        st->carrier_phase_rad = std::fmod(std::fma(w, (double)n, st->carrier_phase_rad), 2.0 * PI_D);
        const double adv = static_cast<double>(n) * st->code_freq_hz / fs;
        st->code_phase_chips = std::fmod(st->code_phase_chips + adv, 1023.0);
        st->chi_chips += adv;
        std::memset(out, 0, sizeof *out);
        out->n_samples = n;
        return 0;
    }
    l1rxg_taps t;
    l1rxg_epl_taps(el_spacing, &t);
    int32_t p = prn;
    return l1rxg_correlate_batch(c, iq, n, 1, st, &p, &t, fs, nullptr, out);
}

// ---- tracker -----------------------------------------------------------

int l1rxg_tracker_create(l1rxg_ctx* c, const l1rxg_tracker_desc* d, const l1rxg_channel* chans,
                         const int32_t* chan_stream, l1rxg_tracker** out) {
    if (!c || !d || !out || (!chans && d->n_channels > 0))
        return set_err(L1RXG_EINVAL, "null argument");
    if (bytes_per_sample(d->format) == 0)
        return set_err(L1RXG_EINVAL, "tracker format must be int8_iq, int16_iq or int8_real_if");
    if (!(d->sample_rate_hz >= 2.046e6))  // samples.hpp:61-76
        return set_err(L1RXG_EINVAL, "sample_rate_hz must be >= 2.046 MHz to cover the C/A main lobe");
    const bool is_if = d->format == L1RXG_FMT_INT8_REAL_IF;
    if (is_if && d->if_frequency_hz <= 0.0)
        return set_err(L1RXG_EINVAL, "if_frequency_hz required for Int8RealIF format");
    if (!is_if && d->if_frequency_hz != 0.0)
        return set_err(L1RXG_EINVAL, "if_frequency_hz must be 0 for complex-baseband formats");
    if (d->if_frequency_hz >= d->sample_rate_hz / 2.0)
        return set_err(L1RXG_EINVAL, "if_frequency_hz must be < fs/2");
    if (int rc = validate_taps(&d->taps))
        return rc;
    if (int rc = validate_cfg(&d->cfg))
        return rc;
    if (d->cta_mode < L1RXG_CTA_AUTO || d->cta_mode > L1RXG_CTA_SEGMENT)
        return set_err(L1RXG_EINVAL, "unknown cta_mode");
    if (d->cluster_size < 0 || d->cluster_size > 16 || (d->ring_raw != 0 && d->ring_raw != 1))
        return set_err(L1RXG_EINVAL, "cluster_size must be in 0..16, ring_raw 0 or 1");
    if (d->n_streams < 1 || d->n_channels < 0 || d->max_records < 1)
        return set_err(L1RXG_EINVAL, "n_streams >= 1, n_channels >= 0, max_records >= 1");
    const int n = static_cast<int>(std::llround(d->sample_rate_hz / 1000.0));
    if (d->ring_samples < 2 * (int64_t)n)
        return set_err(L1RXG_EINVAL, "ring_samples must hold at least two epochs");
    if (n > MAXSUB * (MAX_NT - 32) * RUN)
        return set_err(L1RXG_EINVAL, "epoch longer than the correlator supports (fs <= 150 MHz)");
    if (d->cta_mode == L1RXG_CTA_SEGMENT && (d->format != L1RXG_FMT_INT16_IQ || n < SEG_MIN_N))
        return set_err(L1RXG_EINVAL, "the segment correlator takes complex int16 at fs >= 3.073 MHz");
    for (int k = 0; k < d->n_channels; ++k) {
        if (chan_stream[k] < 0 || chan_stream[k] >= d->n_streams)
            return set_err(L1RXG_EINVAL, "channel bound to a missing stream");
        if (chans[k].prn < 1 || chans[k].prn > 32)
            return set_err(L1RXG_ERANGE, "PRN must be in 1..32");
        if (!(chans[k].code_phase_chips >= 0.0) || !(chans[k].code_phase_chips < 1023.0) ||
            !(chans[k].code_freq_hz > 0) || !(chans[k].code_freq_hz < 1.1 * CHIP_RATE_HZ))
            return set_err(L1RXG_EINVAL, "channel code NCO out of domain");
        if (chans[k].win_len < 0 || chans[k].win_len >= d->cfg.cn0_window_ms)  // (sums mode: any count < m)
            return set_err(L1RXG_EINVAL, "channel C/N0 window length out of range");
    }
    CK(cudaSetDevice(c->device));
    auto* t = new l1rxg_tracker();
    t->ctx = c;
    t->d = *d;
    t->T = pick_T(d->taps.n_taps);
    // correlation warps + one control warp (see track_kernel)
    {
        int nsm = 148;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device);
        const bool thr = d->cta_mode == L1RXG_CTA_THROUGHPUT ||
                         (d->cta_mode == L1RXG_CTA_AUTO && d->n_channels >= 2 * nsm);
        // segment correlator: on request, or for the auto throughput shape on
        // complex int16 recordings where its fast path is the common case
        static const char* ev_seg = std::getenv("L1RXG_SEG");
        const bool seg = d->cta_mode == L1RXG_CTA_SEGMENT ||
                         (d->cta_mode == L1RXG_CTA_AUTO && thr && d->format == L1RXG_FMT_INT16_IQ &&
                          n >= SEG_MIN_N && seg_geometry_ok(d) && !(ev_seg && ev_seg[0] == '0'));
        // latency: up to 19 correlation warps + the control warp, one CTA
        // per SM, one tile (the copy overlaps the loop update).
        // throughput: 5 correlation warps + the control warp and two tiles
        // (copy of unit u+2 overlaps unit u+1), ~110 KB of shared memory ->
        // two CTAs per SM, so one CTA's serial loop update overlaps the
        // other's correlation
        if (seg) {
            t->seg = 1;
            t->thr = 1;
            t->nt = SEG_NT;
            t->nbuf = SEG_NBUF;
        } else if (thr) {
            static const char* ev_nw = std::getenv("L1RXG_THR_NWORK");
            static const char* ev_nb = std::getenv("L1RXG_THR_NBUF");
            // 128 correlation threads (float2 ring: ~51 KB) or 96 (raw samples
            // + prefix tile: ~55 KB) keep four CTAs per SM
            int mx = ev_nw ? std::atoi(ev_nw) : (ring_esz(d->format, d->ring_raw) == 8 ? 128 : 96);
            while ((n + mx * RUN - 1) / (mx * RUN) > MAXSUB)
                mx += 32;
            t->nt = pick_threads(n, nullptr, mx) + 32;
            t->nbuf = ev_nb ? std::atoi(ev_nb) : 1;
            t->thr = 1;
        } else {
            // latency shape: split each channel's epoch over a cluster of K
            // CTAs (one per SM) while the channels x K fit the SMs and each
            // CTA keeps >= 1024 samples; K = 1 is the single-CTA path
            static const char* ev_cl = std::getenv("L1RXG_CLUSTER");
            int K = 1;
            if (d->cta_mode == L1RXG_CTA_SINGLE) {
                K = 1;
            } else if (d->cluster_size > 0) {
                K = d->cluster_size;
            } else if (ev_cl) {
                K = std::max(1, std::min(16, std::atoi(ev_cl)));
            } else {
                // CTAs with <= 4096 samples are small enough to pair up on an
                // SM (measured: config 3's 32 channels run 6 % faster as
                // 8-CTA clusters, two CTAs per SM, than as 4-CTA clusters);
                // at one CTA per SM a share down to 32 runs still pays
                // (config 1, overlapped kernel: 16-CTA cluster +3 % over 8)
                while (K < 16) {
                    const int per = n / (K * 2);
                    const int ctas = d->n_channels * K * 2;
                    if (!(ctas <= nsm ? per >= 32 * RUN
                                      : per >= 1024 && per <= 4096 && ctas <= 2 * nsm))
                        break;
                    // 16-CTA clusters only up to 96 CTAs (measured, 16.368 MHz
                    // real IF: 4 and 6 channels +3 % over K = 8, 8 and 9
                    // channels -1.5 %; profiles/r2b,r2c_cluster_ab.txt)
                    if (2 * K > 8 && d->n_channels * 2 * K > 96)
                        break;
                    K *= 2;
                }
            }
            const bool auto_k = d->cta_mode != L1RXG_CTA_SINGLE && d->cluster_size == 0 && !ev_cl;
            for (;;) {
                const int share = ((n + K * RUN - 1) / (K * RUN)) * RUN;
                while (K > 1 && (K - 1) * share >= n)
                    --K;
                t->csize = K;
                t->share = K > 1 ? share : n;
                t->nt = pick_threads(t->share, nullptr, MAX_NT - 32) + 32;
                {   // phase B deals the work threads to the taps, so more threads than runs shorten its walk:
                    // measured (profiles/r3l_lat_nwork.txt, 16.368 MHz) E/P/L at one CTA per SM: 160-224 work
                    // threads, about one transition per thread, -3.7 % per epoch (128 and 256 are no gain: more
                    // warps cost barrier and reduction time); 13 taps at two CTAs per SM: 160, -2 %
                    // (L1RXG_LAT_NWORK overrides the minimum)
                    static const char* ev_nw = std::getenv("L1RXG_LAT_NWORK");
                    int min_nw = 0;
                    if ((t->T <= 5 && d->n_channels * K <= nsm && t->share >= 1500) ||
                        (t->T >= 11 && d->n_channels * K > nsm))
                        min_nw = 160;
                    if (ev_nw)
                        min_nw = std::atoi(ev_nw);
                    if (min_nw > 0)
                        t->nt = std::max(t->nt, std::min(MAX_NT, (min_nw + 31) / 32 * 32 + 32));
                }
                // a second tile when it fits: the copy of epoch e+1 is then issued
                // while epoch e is still being correlated (a full epoch ahead)
                static const char* ev_nb1 = std::getenv("L1RXG_LAT_NBUF");
                const size_t two = static_cast<size_t>(t->nt - 32) * RUN * 2 * sizeof(float2) + 40000;
                t->nbuf = ev_nb1 ? std::atoi(ev_nb1) : (two <= 200000 ? 2 : 1);
                // non-portable cluster sizes: every channel's cluster must be
                // resident at once (GPC-limited), else fall back to 8
                if (!auto_k || K <= 8 ||
                    cluster_capacity_T(t->T, K, t->nt, t->nbuf, std::min(n, t->share)) >= d->n_channels)
                    break;
                K = 8;
            }
        }
    }
    t->R = d->ring_samples;
    t->esz = ring_esz(d->format, d->ring_raw);
    {   // raw real-IF byte ring filtered by the overlapped kernel's FIR warps (RAW variant), opt-in with
        // L1RXG_OVL_RAWIF=1: it removes the ingest pass and the float2 ring (config 2: 1.36 GB -> ~0.2 GB of
        // DRAM traffic per 10 000 blocks), but the FIR warps share the SM with the per-epoch critical path and
        // the latency-bound epoch gets 4 % longer (profiles/r3e_rawif_ab.txt), so the float2 ring stays default
        static const char* ev_raw = std::getenv("L1RXG_OVL_RAWIF");
        const double w = -2.0 * PI_D * d->if_frequency_hz / d->sample_rate_hz;
        if (!t->seg && !t->thr && d->format == L1RXG_FMT_INT8_REAL_IF && w == -PI_D / 2.0 &&
            ev_raw && ev_raw[0] == '1' && d->n_channels > 0) {
            TrackArgs pa{};
            pa.n = n;
            pa.csize = t->csize;
            pa.share = t->share;
            pa.nbuf = t->nbuf;
            pa.thr = 0;
            pa.lc.kernel = d->kernel;
            auto probe = [&]() -> int { DISPATCH_T(t->T, ovl_raw_applicable, pa, d->n_channels, t->nt); };
            if (probe() == 0) {
                t->rawif = 1;
                t->esz = 1;
                t->pad = RAWIF_PAD;
            }
            cudaGetLastError();
        }
    }
    if (t->seg) {
        // raw cint16 in rows of 32 samples: R and the apron whole rows; the
        // apron covers an epoch plus the last unit's row overhang
        t->esz = 4;
        t->R = (t->R + 31) / 32 * 32;
        t->apron = (n + 2048 + 31) / 32 * 32;
    } else {
        // apron >= one epoch (+ bulk-copy slack); R + apron a multiple of the
        // samples per 16 bytes keeps every stream's ring 16-byte aligned for TMA
        const int64_t A = 16 / t->esz;
        t->apron = n + 64;
        t->apron += (A - (t->R + t->apron) % A) % A;
    }
    t->streams.resize(static_cast<size_t>(d->n_streams));
    auto fail = [&](cudaError_t e) {
        l1rxg_tracker_destroy(t);
        return set_err(e == cudaErrorMemoryAllocation ? L1RXG_ENOMEM : L1RXG_ECUDA,
                       std::string("tracker alloc: ") + cudaGetErrorString(e));
    };
    cudaError_t e;
    const int64_t stride = t->R + t->apron + t->pad;
    if ((e = cudaMalloc(&t->d_ring, static_cast<size_t>(t->esz) * static_cast<size_t>(stride) * t->streams.size())) !=
        cudaSuccess)
        return fail(e);
    if (t->rawif)  // the pad in front of the head reads as the zero FIR history of a stream's start
        cudaMemset(t->d_ring, 0, static_cast<size_t>(stride) * t->streams.size());
    for (size_t k = 0; k < t->streams.size(); ++k)
        t->streams[k].ring = t->d_ring + (static_cast<int64_t>(k) * stride + t->pad) * t->esz;
    if (t->seg && (e = cudaMalloc(&t->d_segq, 4 * (1 + static_cast<size_t>(std::max(1, d->n_channels)) + SEG_CLASSES))) != cudaSuccess)
        return fail(e);
    if (t->seg && d->n_channels > 0) {  // gangs: runs of consecutive channels on the same stream
        std::vector<int> first, count;
        for (int c = 0; c < d->n_channels; ++c) {
            if (c > 0 && chan_stream[c] == chan_stream[c - 1])
                count.back() += 1;
            else {
                first.push_back(c);
                count.push_back(1);
            }
        }
        t->n_gangs = static_cast<int>(first.size());
        t->gang_max = *std::max_element(count.begin(), count.end());
        first.insert(first.end(), count.begin(), count.end());
        if ((e = cudaMalloc(&t->d_gangs, 4 * first.size())) != cudaSuccess)
            return fail(e);
        cudaMemcpy(t->d_gangs, first.data(), 4 * first.size(), cudaMemcpyHostToDevice);
    }
    if (t->seg) {
        if (int rc = encode_ring_map(&t->tmap, t->d_ring, stride / 32, stride * 4, d->n_streams)) {
            const std::string msg = g_err;
            l1rxg_tracker_destroy(t);
            return set_err(rc, msg);
        }
    }
    {  // per stream: two int8 histories (32 B) and two float2 histories (256 B)
        const size_t per = 2 * 32 + 2 * 32 * sizeof(float2);
        t->hist_bytes = per * t->streams.size();
        if ((e = cudaMalloc(&t->d_hist, t->hist_bytes)) != cudaSuccess)
            return fail(e);
        cudaMemset(t->d_hist, 0, t->hist_bytes);
        for (size_t q = 0; q < t->streams.size(); ++q) {
            unsigned char* b = t->d_hist + q * per;
            auto& r = t->streams[q];
            r.histf[0] = reinterpret_cast<float2*>(b);
            r.histf[1] = reinterpret_cast<float2*>(b + 32 * sizeof(float2));
            r.hist8[0] = reinterpret_cast<int8_t*>(b + 64 * sizeof(float2));
            r.hist8[1] = reinterpret_cast<int8_t*>(b + 64 * sizeof(float2) + 32);
        }
    }
    const size_t C = static_cast<size_t>(std::max(1, d->n_channels));
    const size_t nrec = C * static_cast<size_t>(d->max_records);
    if ((e = cudaMalloc(&t->d_avail, 8 * t->streams.size())) != cudaSuccess ||
        (e = cudaMalloc(&t->d_chans, sizeof(l1rxg_channel) * C)) != cudaSuccess ||
        (e = cudaMalloc(&t->d_chans0, sizeof(l1rxg_channel) * C)) != cudaSuccess ||
        (e = cudaMalloc(&t->d_chan_stream, 4 * C)) != cudaSuccess ||
        (e = cudaMalloc(&t->d_recs, sizeof(l1rxg_epoch_record) * nrec)) != cudaSuccess ||
        (e = cudaMalloc(&t->d_tapsums, sizeof(double) * 2 * t->T * nrec)) != cudaSuccess ||
        (e = cudaMalloc(&t->d_ecount, 8 * C)) != cudaSuccess ||
        (e = cudaMalloc(&t->d_status, 4 * C)) != cudaSuccess)
        return fail(e);
    cudaMemset(t->d_avail, 0, 8 * t->streams.size());
    cudaMemset(t->d_recs, 0, sizeof(l1rxg_epoch_record) * nrec);  // unused record slots read as zeros
    cudaMemset(t->d_ecount, 0, 8 * C);
    cudaMemset(t->d_status, 0, 4 * C);
    if (d->n_channels > 0) {
        cudaMemcpy(t->d_chans, chans, sizeof(l1rxg_channel) * d->n_channels, cudaMemcpyHostToDevice);
        cudaMemcpy(t->d_chans0, chans, sizeof(l1rxg_channel) * d->n_channels, cudaMemcpyHostToDevice);
        cudaMemcpy(t->d_chan_stream, chan_stream, 4 * (size_t)d->n_channels, cudaMemcpyHostToDevice);
    }
    for (int k = 0; k < 2; ++k) {
        cudaEventCreateWithFlags(&t->ev_copy[k], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&t->ev_used[k], cudaEventDisableTiming);
    }
    if ((e = cudaDeviceSynchronize()) != cudaSuccess)
        return fail(e);
    *out = t;
    return 0;
}

int l1rxg_tracker_destroy(l1rxg_tracker* t) {
    if (!t)
        return 0;
    cudaSetDevice(t->ctx->device);
    cudaDeviceSynchronize();
    cudaFree(t->d_ring);
    cudaFree(t->d_segq);
    cudaFree(t->d_gangs);
    t->seg_ctab.release();
    cudaFree(t->d_hist);
    cudaFree(t->d_avail);
    cudaFree(t->d_chans);
    cudaFree(t->d_chans0);
    cudaFree(t->d_chan_stream);
    cudaFree(t->d_recs);
    cudaFree(t->d_tapsums);
    cudaFree(t->d_ecount);
    cudaFree(t->d_status);
    for (int k = 0; k < 2; ++k) {
        t->staging[k].release();
        if (t->ev_copy[k]) cudaEventDestroy(t->ev_copy[k]);
        if (t->ev_used[k]) cudaEventDestroy(t->ev_used[k]);
    }
    t->mixed.release();
    for (auto& x : t->timed) {
        cudaEventDestroy(x.a);
        cudaEventDestroy(x.b);
    }
    for (auto e : t->ev_pool)
        cudaEventDestroy(e);
    delete t;
    return 0;
}

int l1rxg_tracker_push_device(l1rxg_tracker* t, int s, const void* dev_bytes, int64_t nbytes) {
    if (!t || s < 0 || s >= (int)t->streams.size())
        return set_err(L1RXG_EINVAL, "bad stream");
    if (int rc = refuse_if_attached(t))
        return rc;
    const int bps = bytes_per_sample(t->d.format);
    if (nbytes <= 0)
        return 0;
    if (nbytes % bps)
        return set_err(L1RXG_EINVAL, "byte count is not a whole number of samples");
    const int64_t nsamp = nbytes / bps;
    if (nsamp > t->R - t->nt)
        return set_err(L1RXG_EINVAL, "push larger than the device ring");
    CK(cudaSetDevice(t->ctx->device));
    return ingest_launch(t, s, dev_bytes, nsamp, t->ctx->compute);
}

int l1rxg_tracker_push_device_strided(l1rxg_tracker* t, const void* dev_bytes,
                                      int64_t nbytes_per_stream, int64_t stride_bytes) {
    if (!t || !dev_bytes)
        return set_err(L1RXG_EINVAL, "null argument");
    if (int rc = refuse_if_attached(t))
        return rc;
    const int bps = bytes_per_sample(t->d.format);
    if (nbytes_per_stream <= 0)
        return 0;
    if (nbytes_per_stream % bps || stride_bytes % bps)
        return set_err(L1RXG_EINVAL, "byte count or stride is not a whole number of samples");
    if (stride_bytes < nbytes_per_stream)
        return set_err(L1RXG_EINVAL, "stride shorter than the per-stream chunk");
    const int64_t nsamp = nbytes_per_stream / bps;
    if (nsamp > t->R - t->nt)
        return set_err(L1RXG_EINVAL, "push larger than the device ring");
    CK(cudaSetDevice(t->ctx->device));
    if (t->d.format == L1RXG_FMT_INT8_REAL_IF) {  // FIR history per stream: one launch each
        for (size_t s = 0; s < t->streams.size(); ++s)
            if (int rc = ingest_launch(t, static_cast<int>(s),
                                       static_cast<const uint8_t*>(dev_bytes) + s * stride_bytes,
                                       nsamp, t->ctx->compute))
                return rc;
        return 0;
    }
    const int64_t g0 = t->streams[0].pushed;
    for (const auto& r : t->streams)
        if (r.pushed != g0)
            return set_err(L1RXG_EINVAL, "strided push needs every stream at the same sample count");
    cudaStream_t st = t->ctx->compute;
    cudaEvent_t a = get_event(t), b = get_event(t);
    cudaEventRecord(a, st);
    const dim3 grid(static_cast<unsigned>((nsamp + 255) / 256), static_cast<unsigned>(t->streams.size()));
    const int64_t pos0 = g0 % t->R;
    if (t->esz == 8 && t->d.format == L1RXG_FMT_INT16_IQ && (pos0 & 1) == 0 && (t->R & 1) == 0 &&
        (t->apron & 1) == 0 && (nsamp & 1) == 0 && (stride_bytes & 7) == 0 &&
        (reinterpret_cast<uintptr_t>(dev_bytes) & 7) == 0) {
        const dim3 g2(static_cast<unsigned>((nsamp / 2 + 255) / 256), static_cast<unsigned>(t->streams.size()));
        decode_i16x2_strided_kernel<<<g2, 256, 0, st>>>(static_cast<const uint8_t*>(dev_bytes), stride_bytes,
                                                        nsamp / 2, reinterpret_cast<float2*>(t->d_ring),
                                                        t->R + t->apron, t->R, t->apron, pos0, t->d_avail,
                                                        g0 + nsamp);
    } else if (t->esz == 8)
        decode_iq_strided_kernel<<<grid, 256, 0, st>>>(static_cast<const uint8_t*>(dev_bytes), stride_bytes,
                                                       t->d.format, nsamp,
                                                       reinterpret_cast<float2*>(t->d_ring),
                                                       t->R + t->apron, t->R, t->apron, g0 % t->R,
                                                       t->d_avail, g0 + nsamp);
    else if (t->d.format == L1RXG_FMT_INT16_IQ)
        copy_raw_strided_kernel<uint32_t><<<grid, 256, 0, st>>>(
            static_cast<const uint8_t*>(dev_bytes), stride_bytes, nsamp,
            reinterpret_cast<uint32_t*>(t->d_ring), t->R + t->apron, t->R, t->apron, g0 % t->R,
            t->d_avail, g0 + nsamp);
    else
        copy_raw_strided_kernel<uint16_t><<<grid, 256, 0, st>>>(
            static_cast<const uint8_t*>(dev_bytes), stride_bytes, nsamp,
            reinterpret_cast<uint16_t*>(t->d_ring), t->R + t->apron, t->R, t->apron, g0 % t->R,
            t->d_avail, g0 + nsamp);
    CK(cudaGetLastError());
    cudaEventRecord(b, st);
    t->timed.push_back({a, b, 0});
    t->launches += 1;
    for (auto& r : t->streams)
        r.pushed += nsamp;
    return 0;
}

int l1rxg_tracker_push_strided(l1rxg_tracker* t, const void* bytes, int64_t nbytes_per_stream,
                               int64_t stride_bytes) {
    if (!t || !bytes)
        return set_err(L1RXG_EINVAL, "null argument");
    if (int rc = refuse_if_attached(t))
        return rc;
    if (nbytes_per_stream <= 0)
        return 0;
    const int bps = bytes_per_sample(t->d.format);
    if (nbytes_per_stream % bps || stride_bytes % bps)
        return set_err(L1RXG_EINVAL, "byte count or stride is not a whole number of samples");
    if (stride_bytes < nbytes_per_stream)
        return set_err(L1RXG_EINVAL, "stride shorter than the per-stream chunk");
    if (nbytes_per_stream / bps > t->R - t->nt)
        return set_err(L1RXG_EINVAL, "push larger than the device ring");
    if (t->d.format != L1RXG_FMT_INT8_REAL_IF)
        for (const auto& r : t->streams)
            if (r.pushed != t->streams[0].pushed)
                return set_err(L1RXG_EINVAL, "strided push needs every stream at the same sample count");
    CK(cudaSetDevice(t->ctx->device));
    const size_t ns = t->streams.size();
    const int k = t->stage_cur;
    t->stage_cur ^= 1;
    if (t->staging[k].ensure(static_cast<size_t>(nbytes_per_stream) * ns))
        return L1RXG_ENOMEM;
    CK(cudaStreamWaitEvent(t->ctx->copy, t->ev_used[k], 0));
    // one pitched copy gathers every stream's chunk into a dense staging block
    CK(cudaMemcpy2DAsync(t->staging[k].p, static_cast<size_t>(nbytes_per_stream), bytes,
                         static_cast<size_t>(stride_bytes), static_cast<size_t>(nbytes_per_stream), ns,
                         cudaMemcpyHostToDevice, t->ctx->copy));
    CK(cudaEventRecord(t->ev_copy[k], t->ctx->copy));
    CK(cudaStreamWaitEvent(t->ctx->compute, t->ev_copy[k], 0));
    if (int rc = l1rxg_tracker_push_device_strided(t, t->staging[k].p, nbytes_per_stream,
                                                   nbytes_per_stream))
        return rc;
    CK(cudaEventRecord(t->ev_used[k], t->ctx->compute));
    return 0;
}

int l1rxg_tracker_attach_device(l1rxg_tracker* t, const void* dev_bytes, int64_t samples_per_stream,
                                int64_t stride_bytes) {
    if (!t || !dev_bytes)
        return set_err(L1RXG_EINVAL, "null argument");
    if (!t->seg)
        return set_err(L1RXG_EINVAL, "attach needs the segment correlator (cta_mode SEGMENT)");
    if (samples_per_stream <= 0 || samples_per_stream % 32 || stride_bytes < samples_per_stream * 4 ||
        stride_bytes % 16 || (reinterpret_cast<uintptr_t>(dev_bytes) & 15))
        return set_err(L1RXG_EINVAL, "attach: whole 32-sample rows, 16-byte aligned base and stride");
    for (const auto& r : t->streams)
        if (r.pushed != 0)
            return set_err(L1RXG_EINVAL, "attach: the tracker's streams must be empty");
    CK(cudaSetDevice(t->ctx->device));
    CK(cudaStreamSynchronize(t->ctx->compute));
    // the recordings become the rings: one tensor over them, no wrap (the
    // capacity is the whole recording), every sample available
    CUtensorMap m{};
    if (int rc = encode_ring_map(&m, const_cast<void*>(dev_bytes), samples_per_stream / 32, stride_bytes,
                                 static_cast<int>(t->streams.size())))
        return rc;
    t->tmap = m;
    t->att_samples = samples_per_stream;
    for (auto& r : t->streams)
        r.pushed = samples_per_stream;
    std::vector<int64_t> av(t->streams.size(), samples_per_stream);
    CK(cudaMemcpy(t->d_avail, av.data(), 8 * av.size(), cudaMemcpyHostToDevice));
    return 0;
}

int l1rxg_tracker_detach(l1rxg_tracker* t) {
    if (!t)
        return set_err(L1RXG_EINVAL, "null tracker");
    if (t->att_samples == 0)
        return 0;
    CK(cudaSetDevice(t->ctx->device));
    CK(cudaStreamSynchronize(t->ctx->compute));
    // the tensor map describes the tracker's own ring again; streams restart empty
    const int64_t stride = t->R + t->apron;
    CUtensorMap m{};
    if (int rc = encode_ring_map(&m, t->d_ring, stride / 32, stride * 4, static_cast<int>(t->streams.size())))
        return rc;
    t->tmap = m;
    t->att_samples = 0;
    for (auto& r : t->streams)
        r.pushed = 0;
    CK(cudaMemset(t->d_avail, 0, 8 * t->streams.size()));
    return 0;
}

int l1rxg_tracker_push(l1rxg_tracker* t, int s, const void* bytes, int64_t nbytes) {
    if (!t || s < 0 || s >= (int)t->streams.size())
        return set_err(L1RXG_EINVAL, "bad stream");
    if (int rc = refuse_if_attached(t))
        return rc;
    const int bps = bytes_per_sample(t->d.format);
    if (nbytes <= 0)
        return 0;
    if (nbytes % bps)
        return set_err(L1RXG_EINVAL, "byte count is not a whole number of samples");
    if (nbytes / bps > t->R - t->nt)
        return set_err(L1RXG_EINVAL, "push larger than the device ring");
    CK(cudaSetDevice(t->ctx->device));
    // double-buffered staging: copy k+1 overlaps ingest/track of k
    const int k = t->stage_cur;
    t->stage_cur ^= 1;
    if (t->staging[k].ensure(static_cast<size_t>(nbytes)))
        return L1RXG_ENOMEM;
    CK(cudaStreamWaitEvent(t->ctx->copy, t->ev_used[k], 0));
    CK(cudaMemcpyAsync(t->staging[k].p, bytes, static_cast<size_t>(nbytes), cudaMemcpyHostToDevice,
                       t->ctx->copy));
    CK(cudaEventRecord(t->ev_copy[k], t->ctx->copy));
    CK(cudaStreamWaitEvent(t->ctx->compute, t->ev_copy[k], 0));
    if (int rc = ingest_launch(t, s, t->staging[k].p, nbytes / bps, t->ctx->compute))
        return rc;
    CK(cudaEventRecord(t->ev_used[k], t->ctx->compute));
    return 0;
}

int l1rxg_tracker_run(l1rxg_tracker* t, int max_epochs) {
    if (!t)
        return set_err(L1RXG_EINVAL, "null tracker");
    if (t->d.n_channels == 0)
        return 0;
    CK(cudaSetDevice(t->ctx->device));
    TrackArgs a{};
    a.ring = t->d_ring + t->pad * t->esz;
    a.ring_stride = t->R + t->apron + t->pad;
    a.ring_cap = t->att_samples > 0 ? t->att_samples : t->R;
    a.avail = t->d_avail;
    a.chans = t->d_chans;
    a.chan_stream = t->d_chan_stream;
    a.recs = t->d_recs;
    a.tap_sums = t->d_tapsums;
    a.ecount = t->d_ecount;
    a.status = t->d_status;
    a.codes = t->ctx->d_codes;
    a.max_records = t->d.max_records;
    a.max_epochs = max_epochs < 0 ? 0x7fffffff : max_epochs;
    a.n = static_cast<int>(std::llround(t->d.sample_rate_hz / 1000.0));
    a.kp = t->d.taps.prompt;
    a.ke = t->d.taps.early;
    a.kl = t->d.taps.late;
    a.taps = padded_taps(t->d.taps, t->T);
    a.lc = make_loop_cfg(t->d.cfg, t->d.kernel, t->d.sample_rate_hz, a.n);
    a.nbuf = t->nbuf;
    a.csize = t->csize;
    a.share = t->share;
    a.thr = t->thr;
    static const char* ev_dw = std::getenv("L1RXG_OVL_DWMAX");
    a.ovl_dwmax = ev_dw ? static_cast<float>(std::atof(ev_dw)) : 1e-3f;
    cudaStream_t st = t->ctx->compute;
    cudaEvent_t e0 = get_event(t), e1 = get_event(t);
    cudaEventRecord(e0, st);
    // L1RXG_PROF=1: stage clocks of CTA 0's first 64 epochs, averaged to stderr
    static const bool prof = std::getenv("L1RXG_PROF") != nullptr;
    long long* dprof = nullptr;
    if (prof) {
        CK(cudaMalloc(&dprof, 4 * 64 * 8 * sizeof(long long)));
        CK(cudaMemsetAsync(dprof, 0, 4 * 64 * 8 * sizeof(long long), st));
    }
    a.prof = dprof;
    const int sk = t->rawif ? SK_R8 : t->esz == 4 ? SK_I16 : t->esz == 2 ? SK_I8 : SK_F32;
    SegArgs sa;
    auto go = [&]() -> int {
        if (t->seg) {
            sa.t = a;
            sa.tmap = t->tmap;
            // work items: chunks of the launch's epochs per channel, so the
            // persistent CTAs end together (no wave-quantisation tail)
            int64_t most = t->att_samples;
            for (const auto& r : t->streams)
                most = std::max(most, r.pushed);
            const int64_t max_e = std::min<int64_t>(a.max_epochs, most / a.n + 1);
            // gang tickets when streams are shared (L1RXG_SEG_GANGS=0: the single item queue); with them a
            // work item is 16 epochs (measured at full size, profiles/r3f_seg_gang_tickets.txt: DRAM reads 1.14x
            // the unique bytes; 32 epochs 1.7x, 64 epochs 3.6x, same time), else an eighth of the launch
            // (L1RXG_SEG_CHUNK overrides)
            static const char* ev_gangs = std::getenv("L1RXG_SEG_GANGS");
            static const char* ev_chunk = std::getenv("L1RXG_SEG_CHUNK");
            const bool use_gangs = t->gang_max > 1 && !(ev_gangs && ev_gangs[0] == '0');
            int chunk = ev_chunk ? std::max(1, std::atoi(ev_chunk))
                        : use_gangs ? 16
                                    : static_cast<int>(std::max<int64_t>(16, (max_e + 7) / 8));
            // very long launches: at most ~4 M gang-chunks (the ticket table is 32 B per gang-chunk)
            if (use_gangs && (max_e + chunk - 1) / chunk * t->n_gangs > (4LL << 20))
                chunk = static_cast<int>((max_e * t->n_gangs + (4LL << 20) - 1) / (4LL << 20));
            const int64_t nchunk = std::max<int64_t>(1, (max_e + chunk - 1) / chunk);
            const int64_t items = nchunk * t->d.n_channels;
            if (items > 0x7fffffff)
                return set_err(L1RXG_EINVAL, "too many work items in one run");
            sa.next = t->d_segq;
            sa.ready = t->d_segq + 1;
            sa.n_items = static_cast<int>(items);
            sa.n_channels = t->d.n_channels;
            sa.chunk_epochs = chunk;
            sa.fast_geom = seg_geometry_ok(&t->d) ? 1 : 0;
            sa.qgrid = 1;  // start-chip LUT when every (padded) tap offset is k/4 chip, |k| <= 4
            for (int k = 0; k < t->T; ++k) {
                const double q4 = a.taps.offsets_chips[k] * 4.0;
                if (!(q4 == std::rint(q4) && std::fabs(q4) <= 4.0))
                    sa.qgrid = 0;
            }
            if (const char* ev = std::getenv("L1RXG_SEG_QGRID"))  // tests: force the exact per-tap path
                sa.qgrid = sa.qgrid && ev[0] != '0';
            // direct quarter-crossing kernel (no step table): the quarter grid at >= 62 samples
            // per chip (nominal rate with 0.1 % margin; the device re-checks every epoch's rate)
            sa.qdirect = sa.qgrid && sa.fast_geom && t->T <= 9 && a.n < 500000 &&
                         4.0 * CHIP_RATE_HZ / t->d.sample_rate_hz * 1.001 <= 2.0 / 31.0;
            if (const char* ev = std::getenv("L1RXG_SEG_QDIRECT"))  // tests: force the step-table kernel
                sa.qdirect = sa.qdirect && ev[0] != '0';
            CK(cudaMemsetAsync(t->d_segq, 0, 4 * (1 + static_cast<size_t>(t->d.n_channels) + SEG_CLASSES), st));
            sa.gang_first = nullptr;
            sa.gang_count = nullptr;
            sa.n_gangs = t->n_gangs;
            sa.gang_max = t->gang_max;
            sa.cnext = t->d_segq + 1 + t->d.n_channels;
            sa.ctab = nullptr;
            sa.ctab_stride = 0;
            if (use_gangs && nchunk * t->n_gangs < 0x3fffffff) {
                sa.ctab_stride = static_cast<int>(nchunk * t->n_gangs) + 1024;
                const size_t tb = 4 * static_cast<size_t>(SEG_CLASSES) * sa.ctab_stride;
                if (t->seg_ctab.ensure(tb))
                    return L1RXG_ENOMEM;
                CK(cudaMemsetAsync(t->seg_ctab.p, 0xff, tb, st));
                sa.ctab = static_cast<int*>(t->seg_ctab.p);
                sa.gang_first = t->d_gangs;
                sa.gang_count = t->d_gangs + t->n_gangs;
            }
            sa.chipw = t->ctx->d_chipw;
            // L1RXG_SEG_TRACE=<file>: globaltimer at every work item's start and end, written as
            // "item channel chunk start_ns end_ns smid warp_slot" lines after the launch (diagnostics)
            static const char* ev_trace = std::getenv("L1RXG_SEG_TRACE");
            sa.trace = nullptr;
            if (ev_trace) {
                CK(cudaMalloc(&sa.trace, 24 * static_cast<size_t>(items)));
                CK(cudaMemsetAsync(sa.trace, 0, 24 * static_cast<size_t>(items), st));
                if (int rc = [&]() -> int { DISPATCH_T(t->T, launch_seg, sa, t->d.n_channels, st); }())
                    return rc;
                std::vector<unsigned long long> h(3 * static_cast<size_t>(items));
                CK(cudaMemcpyAsync(h.data(), sa.trace, 24 * static_cast<size_t>(items), cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                cudaFree(sa.trace);
                if (FILE* f = std::fopen(ev_trace, "w")) {
                    for (int64_t i = 0; i < items; ++i)
                        std::fprintf(f, "%lld %lld %lld %llu %llu %llu %llu\n", (long long)i,
                                     (long long)(i % t->d.n_channels), (long long)(i / t->d.n_channels), h[3 * i],
                                     h[3 * i + 1], h[3 * i + 2] >> 32, h[3 * i + 2] & 0xffffffffull);
                    std::fclose(f);
                }
                return 0;
            }
            DISPATCH_T(t->T, launch_seg, sa, t->d.n_channels, st);
        }
        DISPATCH_T(t->T, launch_track, a, t->d.n_channels, t->nt, st, sk);
    };
    if (int rc = go())
        return rc;
    t->launches += 1;
    cudaEventRecord(e1, st);
    t->timed.push_back({e0, e1, 1});
    if (prof) {
        long long h[4 * 64 * 8];
        CK(cudaMemcpyAsync(h, dprof, sizeof h, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        cudaFree(dprof);
        double acc[8] = {0}, pc[8] = {0}, arr[8] = {0};
        int cnt = 0;
        for (int e = 2; e < 64; ++e) {
            if (h[e * 8 + 7] == 0 || h[e * 8] == 0)
                continue;
            for (int k = 1; k < 8; ++k)
                acc[k] += static_cast<double>(h[e * 8 + k] - h[e * 8 + k - 1]);
            acc[0] += static_cast<double>(h[e * 8 + 7] - h[e * 8]);
            for (int k = 0; k < 8; ++k)
                pc[k] += static_cast<double>(h[512 + e * 8 + k]);
            for (int k = 1; k < 8; ++k)
                arr[k] += static_cast<double>(h[1024 + e * 8 + k] - h[1024 + e * 8 + k - 1]);
            ++cnt;
        }
        if (cnt)
            std::fprintf(stderr,
                         "[l1rxg prof] cycles/epoch %.0f | A %.0f | barA %.0f | B+red %.0f | "
                         "totals %.0f | pieces %.0f | apply %.0f | bar %.0f\n",
                         acc[0] / cnt, acc[1] / cnt, acc[2] / cnt, acc[3] / cnt, acc[4] / cnt,
                         acc[5] / cnt, acc[6] / cnt, acc[7] / cnt);
        if (cnt)
            std::fprintf(stderr,
                         "[l1rxg prof] per epoch, summed over units (thread 0): A+wait %.0f | "
                         "barrier A %.0f | B+partials %.0f | consumed barrier %.0f | "
                         "issue+publish %.0f\n",
                         pc[0] / cnt, pc[1] / cnt, pc[2] / cnt, pc[3] / cnt, pc[4] / cnt);
        if (cnt)
            std::fprintf(stderr,
                         "[l1rxg prof] warp-0 update: totals %.0f | cluster exchange %.0f | "
                         "operands %.0f | atan2/sqrt/fmod %.0f | shuffles+pre %.0f | loop_fast %.0f "
                         "| division %.0f | consts %.0f\n",
                         arr[1] / cnt, arr[2] / cnt, 0.0, arr[3] / cnt, arr[4] / cnt, arr[5] / cnt,
                         arr[6] / cnt, arr[7] / cnt);
        {
            double ph[8] = {0};
            int c2 = 0;
            for (int e = 2; e < 64; ++e) {
                if (h[1536 + e * 8] == 0)
                    continue;
                for (int k = 1; k < 8; ++k)
                    if (h[1536 + e * 8 + k])
                        ph[k] += static_cast<double>(h[1536 + e * 8 + k] - h[1536 + e * 8 + k - 1]);
                ++c2;
            }
            if (c2)
                std::fprintf(stderr,
                             "[l1rxg prof] phase A (thread 0, last unit): consts %.0f | range %.0f | "
                             "tile wait %.0f | phase A %.0f | own-copy wait %.0f\n",
                             ph[1] / c2, ph[2] / c2, ph[3] / c2, ph[4] / c2, ph[5] / c2);
        }
    }
    return 0;
}

int l1rxg_tracker_sync(l1rxg_tracker* t) {
    if (!t)
        return set_err(L1RXG_EINVAL, "null tracker");
    CK(cudaSetDevice(t->ctx->device));
    CK(cudaStreamSynchronize(t->ctx->copy));
    CK(cudaStreamSynchronize(t->ctx->compute));
    std::vector<int32_t> status(static_cast<size_t>(std::max(1, t->d.n_channels)));
    if (t->d.n_channels > 0) {
        CK(cudaMemcpy(status.data(), t->d_status, 4 * status.size(), cudaMemcpyDeviceToHost));
        for (int k = 0; k < t->d.n_channels; ++k) {
            if (status[static_cast<size_t>(k)] == 2)
                return set_err(L1RXG_ECUDA, "segment correlator: a work item timed out waiting for its "
                                            "channel's previous chunk");
            if (status[static_cast<size_t>(k)])
                return set_err(L1RXG_EINVAL, "ring overrun: a channel's window was overwritten "
                                             "before it was tracked (ring_samples too small)");
        }
    }
    return 0;
}

int l1rxg_tracker_channels(l1rxg_tracker* t, l1rxg_channel* out) {
    if (int rc = l1rxg_tracker_sync(t))
        return rc;
    if (t->d.n_channels > 0)
        CK(cudaMemcpy(out, t->d_chans, sizeof(l1rxg_channel) * t->d.n_channels, cudaMemcpyDeviceToHost));
    return 0;
}

int l1rxg_tracker_epoch_counts(l1rxg_tracker* t, int64_t* out) {
    if (int rc = l1rxg_tracker_sync(t))
        return rc;
    if (t->d.n_channels > 0)
        CK(cudaMemcpy(out, t->d_ecount, 8 * (size_t)t->d.n_channels, cudaMemcpyDeviceToHost));
    return 0;
}

int l1rxg_tracker_records(l1rxg_tracker* t, int ch, int64_t e0, int64_t count,
                          l1rxg_epoch_record* out, double* tap_sums_out) {
    if (!t || ch < 0 || ch >= t->d.n_channels)
        return set_err(L1RXG_EINVAL, "bad channel");
    if (int rc = l1rxg_tracker_sync(t))
        return rc;
    int64_t done = 0;
    CK(cudaMemcpy(&done, t->d_ecount + ch, 8, cudaMemcpyDeviceToHost));
    const int64_t M = t->d.max_records;
    if (e0 < 0 || count < 0 || e0 + count > done || e0 < done - M)
        return set_err(L1RXG_EINVAL, "records not available (outside the record ring)");
    const int K = t->d.taps.n_taps, T = t->T;
    std::vector<double> sums;
    for (int64_t e = e0; e < e0 + count;) {
        const int64_t slot = e % M;
        const int64_t run = std::min<int64_t>(count - (e - e0), M - slot);
        const size_t base = static_cast<size_t>(ch) * M + slot;
        if (out)
            CK(cudaMemcpy(out + (e - e0), t->d_recs + base, sizeof(l1rxg_epoch_record) * run,
                          cudaMemcpyDeviceToHost));
        if (tap_sums_out) {
            sums.resize(static_cast<size_t>(run) * 2 * T);
            CK(cudaMemcpy(sums.data(), t->d_tapsums + base * 2 * T, sums.size() * 8,
                          cudaMemcpyDeviceToHost));
            for (int64_t q = 0; q < run; ++q)
                std::memcpy(tap_sums_out + (e - e0 + q) * 2 * K, sums.data() + q * 2 * T,
                            sizeof(double) * 2 * K);
        }
        e += run;
    }
    return 0;
}

int l1rxg_tracker_records_raw(l1rxg_tracker* t, void* dst, int dst_is_device, int64_t* bytes_out) {
    if (!t)
        return set_err(L1RXG_EINVAL, "null tracker");
    const size_t bytes = sizeof(l1rxg_epoch_record) * static_cast<size_t>(std::max(1, t->d.n_channels)) *
                         static_cast<size_t>(t->d.max_records);
    if (bytes_out)
        *bytes_out = static_cast<int64_t>(bytes);
    if (!dst)
        return 0;
    CK(cudaSetDevice(t->ctx->device));
    CK(cudaMemcpyAsync(dst, t->d_recs, bytes,
                       dst_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                       t->ctx->compute));
    CK(cudaStreamSynchronize(t->ctx->compute));
    return 0;
}

int l1rxg_tracker_reset(l1rxg_tracker* t, const l1rxg_channel* chans) {
    if (!t)
        return set_err(L1RXG_EINVAL, "null argument");
    CK(cudaSetDevice(t->ctx->device));
    CK(cudaStreamSynchronize(t->ctx->copy));
    CK(cudaStreamSynchronize(t->ctx->compute));
    const size_t C = static_cast<size_t>(std::max(1, t->d.n_channels));
    cudaStream_t st = t->ctx->compute;
    if (t->att_samples > 0) {  // attached recordings stay fully available
        std::vector<int64_t> av(t->streams.size(), t->att_samples);
        CK(cudaMemcpyAsync(t->d_avail, av.data(), 8 * av.size(), cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
    } else {
        CK(cudaMemsetAsync(t->d_avail, 0, 8 * t->streams.size(), st));
    }
    CK(cudaMemsetAsync(t->d_ecount, 0, 8 * C, st));
    CK(cudaMemsetAsync(t->d_status, 0, 4 * C, st));
    for (auto& r : t->streams) {
        r.pushed = t->att_samples;  // attached: every recorded sample stays available
        r.hist_cur = 0;
    }
    CK(cudaMemsetAsync(t->d_hist, 0, t->hist_bytes, st));  // every stream's FIR history, one memset
    if (t->rawif)  // and the raw rings' front pads
        CK(cudaMemset2DAsync(t->d_ring, static_cast<size_t>(t->R + t->apron + t->pad), 0,
                             static_cast<size_t>(t->pad), t->streams.size(), st));
    if (t->d.n_channels > 0) {
        if (chans)
            CK(cudaMemcpyAsync(t->d_chans, chans, sizeof(l1rxg_channel) * t->d.n_channels,
                               cudaMemcpyHostToDevice, st));
        else  // the creation-time channels, device to device
            CK(cudaMemcpyAsync(t->d_chans, t->d_chans0, sizeof(l1rxg_channel) * t->d.n_channels,
                               cudaMemcpyDeviceToDevice, st));
    }
    CK(cudaStreamSynchronize(st));
    return 0;
}

void* l1rxg_tracker_stream(l1rxg_tracker* t) { return t ? static_cast<void*>(t->ctx->compute) : nullptr; }

int l1rxg_tracker_read_samples(l1rxg_tracker* t, int s, int64_t s0, int64_t count, double* iq_out) {
    if (!t || s < 0 || s >= (int)t->streams.size())
        return set_err(L1RXG_EINVAL, "bad stream");
    if (int rc = l1rxg_tracker_sync(t))
        return rc;
    const StreamRing& r = t->streams[static_cast<size_t>(s)];
    if (s0 < 0 || count < 0 || s0 + count > r.pushed || s0 < r.pushed - t->R)
        return set_err(L1RXG_EINVAL, "samples not in the ring");
    if (t->rawif) {  // the baseband the FIR warps see: the same if4_fir over the ring's bytes
        if (s0 >= 22 && s0 - 22 < r.pushed - t->R)
            return set_err(L1RXG_EINVAL, "samples (with their FIR history) not in the ring");
        if (count == 0)
            return 0;
        float2* dout = nullptr;
        CK(cudaMalloc(&dout, sizeof(float2) * static_cast<size_t>(count)));
        rawif_window_kernel<<<static_cast<unsigned>((count + 255) / 256), 256>>>(
            reinterpret_cast<const int8_t*>(r.ring), t->R, s0, count, dout);
        std::vector<float2> h(static_cast<size_t>(count));
        const cudaError_t ce = cudaMemcpy(h.data(), dout, sizeof(float2) * h.size(), cudaMemcpyDeviceToHost);
        cudaFree(dout);
        if (ce != cudaSuccess)
            return set_err(L1RXG_ECUDA, cudaGetErrorString(ce));
        for (int64_t k = 0; k < count; ++k) {
            iq_out[2 * k] = h[static_cast<size_t>(k)].x;
            iq_out[2 * k + 1] = h[static_cast<size_t>(k)].y;
        }
        return 0;
    }
    const int esz = t->esz;
    std::vector<unsigned char> tmp(static_cast<size_t>(count) * esz);
    for (int64_t k = 0; k < count;) {
        const int64_t pos = (s0 + k) % t->R;
        const int64_t run = std::min(count - k, t->R - pos);
        CK(cudaMemcpy(tmp.data() + k * esz, r.ring + pos * esz, static_cast<size_t>(esz) * run,
                      cudaMemcpyDeviceToHost));
        k += run;
    }
    // the ring holds the SampleSource outputs (samples.hpp:188-253): float2
    // after the IF front end, raw complex ints otherwise (decoded here)
    for (int64_t k = 0; k < count; ++k) {
        const unsigned char* p = tmp.data() + k * esz;
        if (esz == 8) {
            float v[2];
            std::memcpy(v, p, 8);
            iq_out[2 * k] = v[0];
            iq_out[2 * k + 1] = v[1];
        } else if (esz == 4) {
            int16_t v[2];
            std::memcpy(v, p, 4);
            iq_out[2 * k] = static_cast<double>(static_cast<float>(v[0]) * (1.0f / 32768.0f));
            iq_out[2 * k + 1] = static_cast<double>(static_cast<float>(v[1]) * (1.0f / 32768.0f));
        } else {
            const int8_t v0 = static_cast<int8_t>(p[0]), v1 = static_cast<int8_t>(p[1]);
            iq_out[2 * k] = static_cast<double>(static_cast<float>(v0) * (1.0f / 128.0f));
            iq_out[2 * k + 1] = static_cast<double>(static_cast<float>(v1) * (1.0f / 128.0f));
        }
    }
    return 0;
}

int l1rxg_tracker_timing(l1rxg_tracker* t, double* ingest_ms, double* track_ms, int64_t* launches) {
    if (!t)
        return set_err(L1RXG_EINVAL, "null tracker");
    CK(cudaSetDevice(t->ctx->device));
    double ing = 0, trk = 0;
    for (auto& x : t->timed) {
        CK(cudaEventSynchronize(x.b));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, x.a, x.b));
        (x.kind == 0 ? ing : trk) += ms;
        t->ev_pool.push_back(x.a);
        t->ev_pool.push_back(x.b);
    }
    t->timed.clear();
    if (ingest_ms) *ingest_ms = ing;
    if (track_ms) *track_ms = trk;
    if (launches) *launches = t->launches;
    t->launches = 0;
    return 0;
}

int l1rxg_search_grid(l1rxg_ctx* c, int format, const void* bytes, int bytes_on_device,
                      int64_t nbytes, double fs, double if_hz, int n_blocks, const int32_t* prns,
                      int n_prns, const double* bins, int n_bins, int delay_step, int n_delays,
                      double* plane_out) {
    return l1rxg_search_grid_ex(c, format, bytes, bytes_on_device, nbytes, fs, if_hz, n_blocks, prns, n_prns, bins,
                                n_bins, delay_step, n_delays, plane_out, 0, 0);
}

int l1rxg_search_grid_ex(l1rxg_ctx* c, int format, const void* bytes, int bytes_on_device,
                         int64_t nbytes, double fs, double if_hz, int n_blocks, const int32_t* prns,
                         int n_prns, const double* bins, int n_bins, int delay_step, int n_delays,
                         void* plane_out, int plane_f32, int plane_on_device) {
    if (!c || !bytes || !prns || !bins || !plane_out)
        return set_err(L1RXG_EINVAL, "null argument");
    const int bps = bytes_per_sample(format);
    if (bps == 0)
        return set_err(L1RXG_EINVAL, "format must be int8_iq, int16_iq or int8_real_if");
    // the direct half-chip identity needs an integer number of samples per
    // half chip, and delays on that grid (config 5: 8 samples at 16.368 MHz)
    const double spc_d = fs / CHIP_RATE_HZ / 2.0;
    const int spc = static_cast<int>(std::llround(spc_d));
    if (spc < 1 || std::fabs(spc_d - spc) > 1e-9)
        return set_err(L1RXG_EINVAL, "search grid needs fs = 2*k*1.023 MHz (integer samples per half chip)");
    if (delay_step != spc)
        return set_err(L1RXG_EINVAL, "search grid delay_step must be half a chip (fs/2.046 MHz samples)");
    const int N = 2 * GRID_CHIPS * spc;
    if (n_delays < 1 || n_delays > 2 * GRID_CHIPS)
        return set_err(L1RXG_EINVAL, "n_delays must be in 1..2046");
    if (n_blocks < 1 || n_blocks > 24)
        return set_err(L1RXG_EINVAL, "n_blocks must be in 1..24");
    if (n_prns < 1 || n_bins < 1)
        return set_err(L1RXG_EINVAL, "need at least one PRN and one Doppler bin");
    for (int k = 0; k < n_prns; ++k)
        if (prns[k] < 1 || prns[k] > 32)
            return set_err(L1RXG_ERANGE, "PRN must be in 1..32");
    const bool is_if = format == L1RXG_FMT_INT8_REAL_IF;
    if (is_if && !(if_hz > 0.0 && if_hz < fs / 2.0))
        return set_err(L1RXG_EINVAL, "if_frequency_hz required in (0, fs/2) for Int8RealIF");
    const int64_t nsamp = static_cast<int64_t>(n_blocks) * N;
    if (nbytes < nsamp * bps)
        return set_err(L1RXG_EINVAL, "not enough bytes for n_blocks 1-ms blocks");
    std::lock_guard<std::mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->compute;
    if (!c->gev[0])
        for (auto& e : c->gev)
            CK(cudaEventCreate(&e));
    if (c->gbase.ensure(sizeof(float2) * (nsamp + 64)) || c->gF.ensure(sizeof(float2) * 2 * GRID_CHIPS * n_bins * n_blocks) ||
        c->gplane.ensure(sizeof(float) * 2 * GRID_CHIPS * n_bins * n_prns) || c->gbins.ensure(8 * n_bins) ||
        c->gprns.ensure(4 * n_prns) || c->ghist.ensure(64 * sizeof(float2)))
        return L1RXG_ENOMEM;
    const void* raw = bytes;
    if (!bytes_on_device) {
        if (c->graw.ensure(static_cast<size_t>(nsamp * bps)))
            return L1RXG_ENOMEM;
        CK(cudaMemcpyAsync(c->graw.p, bytes, nsamp * bps, cudaMemcpyHostToDevice, st));
        raw = c->graw.p;
    }
    CK(cudaMemcpyAsync(c->gbins.p, bins, 8 * n_bins, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(c->gprns.p, prns, 4 * n_prns, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(c->ghist.p, 0, 64 * sizeof(float2), st));
    float2* base = static_cast<float2*>(c->gbase.p);
    CK(cudaEventRecord(c->gev[0], st));
    // K1 ingest of the n_blocks blocks (a flat ring: R = nsamp, no apron)
    if (is_if) {
        const double w = -2.0 * PI_D * if_hz / fs;
        if (w == -PI_D / 2.0) {
            const unsigned blocks = static_cast<unsigned>((nsamp + ING_TILE - 1) / ING_TILE);
            ingest_if4_kernel<<<blocks, ING_TPB, 0, st>>>(
                static_cast<const int8_t*>(raw), static_cast<const int8_t*>(c->ghist.p),
                static_cast<int8_t*>(c->ghist.p) + 32, 0, nsamp, base, nsamp, 0, 0, nullptr);
        } else {
            DevBuf& mixed = c->iq32;  // reuse as float2 scratch
            if (mixed.ensure(sizeof(float2) * (nsamp + 22)))
                return L1RXG_ENOMEM;
            float2* mx = static_cast<float2*>(mixed.p);
            CK(cudaMemsetAsync(mx, 0, 22 * sizeof(float2), st));
            const unsigned blocks = static_cast<unsigned>((nsamp + 255) / 256);
            mix_generic_kernel<<<blocks, 256, 0, st>>>(static_cast<const int8_t*>(raw), 0, nsamp, w, mx);
            fir_generic_kernel<<<blocks, 256, 0, st>>>(mx, nsamp, base, nsamp, 0, 0,
                                                       static_cast<float2*>(c->ghist.p), nullptr, 0);
        }
    } else {
        const unsigned blocks = static_cast<unsigned>((nsamp + 255) / 256);
        decode_iq_kernel<<<blocks, 256, 0, st>>>(raw, format, nsamp, base, nsamp, 0, 0, nullptr, 0);
    }
    CK(cudaGetLastError());
    grid_fold_kernel<<<n_bins * n_blocks, 256, 2 * GRID_CHIPS * sizeof(float2), st>>>(
        base, N, spc, static_cast<const double*>(c->gbins.p), fs, n_blocks,
        static_cast<float2*>(c->gF.p));
    CK(cudaGetLastError());
    CK(cudaEventRecord(c->gev[1], st));
    const char* ev_fp32 = std::getenv("L1RXG_GRID_FP32");  // per call: tests compare the paths
    const char* ev_path = std::getenv("L1RXG_GRID");          // "mma" (default) | "gemm" (cuBLAS) | "fp32"
    const bool use_fp32 = (ev_fp32 && std::atoi(ev_fp32)) || (ev_path && std::strcmp(ev_path, "fp32") == 0);
    const bool use_gemm = !use_fp32 && ev_path && std::strcmp(ev_path, "gemm") == 0;
    if (!use_fp32 && !use_gemm) {  // K4c: hand-written tcgen05 int8 GEMM + fused |.| epilogue
        const int G = n_bins * 2;
        const int NR = gm_rows(n_blocks);
        if (c->gQ.ensure(static_cast<size_t>(G) * NR * 1024) || c->gS.ensure(sizeof(float) * G * n_blocks))
            return L1RXG_ENOMEM;
        CK(cudaMemsetAsync(c->gQ.p, 0, static_cast<size_t>(G) * NR * 1024, st));  // padding rows
        grid_digits_kernel<<<G * n_blocks, 256, 0, st>>>(static_cast<const float2*>(c->gF.p), n_blocks, NR,
                                                         static_cast<int8_t*>(c->gQ.p), static_cast<float*>(c->gS.p));
        CK(cudaGetLastError());
        GridMmaArgs ga;
        std::memset(&ga, 0, sizeof ga);
        if (int rc = encode_u8_2d(&ga.bmap, c->gQ.p, 1024, static_cast<int64_t>(G) * NR, GM_KB, NR))
            return rc;
        ga.codes = c->d_codes;
        ga.prns = static_cast<const int32_t*>(c->gprns.p);
        ga.scales = static_cast<const float*>(c->gS.p);
        ga.plane = static_cast<float*>(c->gplane.p);
        ga.n_prns = n_prns;
        ga.n_groups = G;
        ga.n_seg = n_blocks;
        ga.n_rows = NR;
        ga.out_scale = static_cast<float>(N);
        // shape knobs (defaults measured, DESIGN.md section 3 K4c)
        const char* ev_a = std::getenv("L1RXG_GRID_A");    // "smem" | "tmem"
        const char* ev_ks = std::getenv("L1RXG_GRID_KS");  // K blocks per stage
        const char* ev_epi = std::getenv("L1RXG_GRID_EPI");
        // measured (profiles/r2k_grid_shapes.txt, config 5): A in TMEM with 4 K
        // blocks per stage 0.306 ms; A in shared memory (2 per stage) 0.332 ms
        ga.a_smem = ev_a ? (std::strcmp(ev_a, "smem") == 0) : 0;
        ga.ks = ev_ks ? std::max(1, std::min(4, std::atoi(ev_ks))) : 4;
        if (ga.ks == 3)
            ga.ks = 2;
        ga.epi = ev_epi ? std::atoi(ev_epi) != 0 : 1;
        if (gm_stages(NR, ga.ks, ga.a_smem) < 2)
            return set_err(L1RXG_EINVAL, "search grid: too many blocks for the B ring");
        const size_t sm = gm_smem_bytes_rt(NR, ga.ks, ga.a_smem);
        int nsm = 148;
        CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
        const int units = n_prns * GM_TILES * G;
        auto launch = [&](auto kern) -> int {
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            kern<<<std::min(nsm, units), GM_THREADS, sm, st>>>(ga);
            CK(cudaGetLastError());
            return 0;
        };
        int lrc = 0;
        if (ga.a_smem)
            lrc = ga.ks == 1 ? launch(grid_mma_kernel<true, 1>) : ga.ks == 2 ? launch(grid_mma_kernel<true, 2>)
                                                                             : launch(grid_mma_kernel<true, 4>);
        else
            lrc = ga.ks == 1 ? launch(grid_mma_kernel<false, 1>) : ga.ks == 2 ? launch(grid_mma_kernel<false, 2>)
                                                                              : launch(grid_mma_kernel<false, 4>);
        if (lrc)
            return lrc;
        c->launches += 3;
    } else if (use_fp32) {  // FP32-pipe circulant correlation (reference kernel)
        const size_t sm = 2 * 1024 * sizeof(float) + sizeof(float2) * GRID_CHIPS * n_blocks;
        CK(cudaFuncSetAttribute(grid_corr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        grid_corr_kernel<<<n_prns * n_bins * 2, GRID_TPB, sm, st>>>(
            static_cast<const float2*>(c->gF.p), c->d_codes, static_cast<const int32_t*>(c->gprns.p),
            n_bins, n_blocks, static_cast<float>(N), static_cast<float*>(c->gplane.p));
        CK(cudaGetLastError());
    } else {  // tensor cores: one bf16x3 GEMM per PRN (search.cuh K4b)
        const int n_vec = n_bins * n_blocks * 2;
        const int rows = 2 * n_vec;
        const void* mt_before = c->gMt.p;
        if (c->gA.ensure(sizeof(__nv_bfloat16) * static_cast<size_t>(rows) * GRID_KS) ||
            c->gMt.ensure(sizeof(__nv_bfloat16) * static_cast<size_t>(n_prns) * GRID_K * GRID_KS) ||
            c->gC.ensure(sizeof(float) * static_cast<size_t>(n_prns) * rows * GRID_K))
            return L1RXG_ENOMEM;
        if (c->gMt.p != mt_before)
            c->gMt_prns.clear();  // reallocated: contents gone
        if (!c->blas) {
            if (cublasCreate(&c->blas) != CUBLAS_STATUS_SUCCESS)
                return set_err(L1RXG_ECUDA, "cublasCreate failed");
        }
        cublasSetStream(c->blas, st);
        grid_split_kernel<<<n_vec, 256, 0, st>>>(static_cast<const float2*>(c->gF.p), n_vec,
                                                 static_cast<__nv_bfloat16*>(c->gA.p));
        // the circulant code matrices depend only on the PRN list: built once
        // per list and kept with the context
        const std::vector<int32_t> want(prns, prns + n_prns);
        if (c->gMt_prns != want) {
            c->gMt_prns.clear();
            grid_circ_kernel<<<dim3(GRID_KS, n_prns), 256, 0, st>>>(
                c->d_codes, static_cast<const int32_t*>(c->gprns.p),
                static_cast<__nv_bfloat16*>(c->gMt.p));
            CK(cudaGetLastError());
            c->gMt_prns = want;
        }
        const float one = 1.f, zero = 0.f;
        // column-major: C_p (GRID_K x rows) = Mt_p (GRID_K x GRID_KS) * A (GRID_KS x rows)
        const cublasStatus_t bs = cublasGemmStridedBatchedEx(
            c->blas, CUBLAS_OP_N, CUBLAS_OP_N, GRID_K, rows, GRID_KS, &one, c->gMt.p, CUDA_R_16BF,
            GRID_K, static_cast<long long>(GRID_K) * GRID_KS, c->gA.p, CUDA_R_16BF, GRID_KS, 0, &zero,
            c->gC.p, CUDA_R_32F, GRID_K, static_cast<long long>(rows) * GRID_K, n_prns,
            CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
        if (bs != CUBLAS_STATUS_SUCCESS)
            return set_err(L1RXG_ECUDA, "cublasGemmStridedBatchedEx failed");
        grid_mag_kernel<<<dim3(n_bins * 2, n_prns), 256, 0, st>>>(
            static_cast<const float*>(c->gC.p), rows, n_bins, n_blocks, static_cast<float>(N),
            static_cast<float*>(c->gplane.p));
        CK(cudaGetLastError());
        c->launches += 3;
    }
    CK(cudaEventRecord(c->gev[2], st));
    // the plane trimmed to n_delays and converted on the GPU, one copy out
    const int64_t cells = static_cast<int64_t>(n_bins) * n_prns * n_delays;
    const size_t ebytes = plane_f32 ? sizeof(float) : sizeof(double);
    void* dst = plane_out;
    if (!plane_on_device) {
        if (c->gout.ensure(static_cast<size_t>(cells) * ebytes))
            return L1RXG_ENOMEM;
        dst = c->gout.p;
    }
    grid_plane_out_kernel<<<static_cast<unsigned>((cells + 255) / 256), 256, 0, st>>>(
        static_cast<const float*>(c->gplane.p), n_delays, cells, dst, plane_f32);
    CK(cudaGetLastError());
    if (!plane_on_device)
        CK(cudaMemcpyAsync(plane_out, dst, static_cast<size_t>(cells) * ebytes, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    float ms0 = 0, ms1 = 0;
    cudaEventElapsedTime(&ms0, c->gev[0], c->gev[1]);
    cudaEventElapsedTime(&ms1, c->gev[1], c->gev[2]);
    c->grid_ms[0] = ms0;
    c->grid_ms[1] = ms1;
    c->launches += 4;
    return 0;
}

int l1rxg_pick_peak(const double* cells, int n_bins, int n_delays, const double* bins, int delay_step, int prn,
                    double fs, double threshold_ratio, l1rxg_acq_result* out) {
    if (!cells || !bins || !out || n_bins < 1 || n_delays < 1 || delay_step < 1 || !(fs > 0))
        return set_err(L1RXG_EINVAL, "bad pick_peak arguments");
    const int64_t cells_n = static_cast<int64_t>(n_bins) * n_delays;
    int64_t best = 0;  // first maximum in row-major order, as the reference's strict '>'
    for (int64_t i = 1; i < cells_n; ++i)
        if (cells[i] > cells[best])
            best = i;
    const int64_t pk = best % n_delays, pb = best / n_delays;
    // distances on the sample axis (n_delays * delay_step samples, circular)
    const int64_t n = static_cast<int64_t>(n_delays) * delay_step;
    const int64_t chip_samples = static_cast<int64_t>(std::ceil(fs / CHIP_RATE_HZ));
    double runner = 0;
    for (int64_t b = 0; b < n_bins; ++b)
        for (int64_t k = 0; k < n_delays; ++k) {
            int64_t dist = (k > pk ? k - pk : pk - k) * delay_step;
            dist = std::min(dist, n - dist);
            if (dist <= chip_samples)
                continue;
            runner = std::max(runner, cells[b * n_delays + k]);
        }
    out->prn = prn;
    out->ratio = runner > 0 ? cells[best] / runner : std::numeric_limits<double>::infinity();
    out->detected = out->ratio >= threshold_ratio ? 1 : 0;
    out->doppler_hz = bins[pb];
    out->code_delay_samples = static_cast<int32_t>(pk * delay_step);
    out->pad_ = 0;
    out->code_delay_chips = static_cast<double>(pk * delay_step) * CHIP_RATE_HZ / fs;
    return 0;
}

int l1rxg_init_channel(int prn, double doppler_hz, int64_t acq_buffer_start, int64_t code_delay_samples,
                       int64_t start_offset_samples, double fs, l1rxg_channel* out) {
    if (!out)
        return set_err(L1RXG_EINVAL, "null out");
    if (prn < 1 || prn > 32)
        return set_err(L1RXG_ERANGE, "PRN must be in 1..32");
    if (!(fs > 0))
        return set_err(L1RXG_EINVAL, "sample_rate_hz must be positive");
    l1rxg_channel ch;
    std::memset(&ch, 0, sizeof ch);  // ChannelState{} (tracking.hpp:626)
    ch.prn = prn;
    ch.state = L1RXG_ACQUIRED;
    ch.carrier_doppler_hz = doppler_hz;
    ch.code_freq_hz = CHIP_RATE_HZ * (1.0 + doppler_hz / F_L1_HZ) + 0.0;  // carrier_aided_code_freq(f, 0)
    ch.pll_integrator = 2.0 * PI_D * doppler_hz;
    ch.fll_enabled = 1;
    const int64_t spm = std::llround(fs / 1000.0);
    const int64_t boundary = acq_buffer_start + code_delay_samples;
    int64_t start = boundary;
    if (start < start_offset_samples) {  // the first code boundary at or after the start offset
        const int64_t gap = start_offset_samples - boundary;
        start = boundary + ((gap + spm - 1) / spm) * spm;
    }
    ch.sample_offset_next_epoch = start;
    const double cps = ch.code_freq_hz / fs;
    ch.code_phase_chips = std::fmod(static_cast<double>(start - boundary) * cps, 1023.0);
    ch.chi_chips = ch.code_phase_chips;
    *out = ch;
    return 0;
}

int l1rxg_search_grid_timing(l1rxg_ctx* c, double* ingest_fold_ms, double* corr_ms) {
    if (!c)
        return set_err(L1RXG_EINVAL, "null context");
    if (ingest_fold_ms) *ingest_fold_ms = c->grid_ms[0];
    if (corr_ms) *corr_ms = c->grid_ms[1];
    return 0;
}

// ---- scenario synthesizer (SimStream raw mode, simsource.hpp:194-413) ----
int l1rxg_simulate(l1rxg_ctx* c, const l1rxg_sim_sv* svs, int n_sv, int n_rec, double fs, double if_hz,
                   int format, int64_t ms0, int n_ms, uint64_t seed, int noise, void* dev_out,
                   int64_t rec_stride_bytes) {
    if (!c || (!svs && n_sv > 0) || !dev_out)
        return set_err(L1RXG_EINVAL, "null argument");
    if (n_sv < 0 || n_sv > SIM_MAX_SV || n_rec < 1 || n_ms < 1 || ms0 < 0)
        return set_err(L1RXG_EINVAL, "n_sv must be in 0..32, n_rec and n_ms >= 1, ms0 >= 0");
    const int n = static_cast<int>(std::llround(fs / 1000.0));
    if (!(fs > 0) || std::fabs(fs / 1000.0 - n) > 1e-9)  // simsource.hpp:203-206
        return set_err(L1RXG_EINVAL, "simulator requires an integer number of samples per ms");
    if (format != L1RXG_FMT_INT8_IQ && format != L1RXG_FMT_INT16_IQ && format != L1RXG_FMT_INT8_REAL_IF)
        return set_err(L1RXG_EINVAL, "format must be int8_iq, int16_iq or int8_real_if");
    const int bps = bytes_per_sample(format);
    if (rec_stride_bytes < static_cast<int64_t>(n_ms) * n * bps)
        return set_err(L1RXG_EINVAL, "rec_stride_bytes shorter than one recording");
    std::vector<SimSvDev> h(static_cast<size_t>(n_rec) * std::max(1, n_sv));
    for (int r = 0; r < n_rec; ++r)
        for (int k = 0; k < n_sv; ++k) {
            const l1rxg_sim_sv& v = svs[static_cast<size_t>(r) * n_sv + k];
            if (v.prn < 1 || v.prn > 32)
                return set_err(L1RXG_ERANGE, "PRN must be in 1..32");
            SimSvDev& d = h[static_cast<size_t>(r) * n_sv + k];
            d.delay_s = v.code_delay_chips / CHIP_RATE_HZ;
            d.fd_over_l1 = v.doppler_hz / F_L1_HZ;
            d.rate_over_l1 = v.doppler_rate_hz_per_s / F_L1_HZ;
            d.phase0 = v.initial_carrier_phase_rad;
            d.amp = (noise ? 0.25 : 1.0) * std::sqrt(std::pow(10.0, v.cn0_dbhz / 10.0) / fs);  // :237-239
            d.prn = v.prn;
            d.pad = 0;
        }
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->compute;
    if (c->gsim.ensure(h.size() * sizeof(SimSvDev)))
        return L1RXG_ENOMEM;
    CK(cudaMemcpyAsync(c->gsim.p, h.data(), h.size() * sizeof(SimSvDev), cudaMemcpyHostToDevice, st));
    const dim3 grid(static_cast<unsigned>(n_ms), static_cast<unsigned>(n_rec));
    simgen_kernel<<<grid, 256, 0, st>>>(static_cast<const SimSvDev*>(c->gsim.p), n_sv, c->d_codes, n, fs, if_hz,
                                        ms0, format, static_cast<unsigned long long>(seed), noise ? 1 : 0,
                                        static_cast<unsigned char*>(dev_out), rec_stride_bytes);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return 0;
}

}  // extern "C"
