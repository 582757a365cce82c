// Micro-benchmark: latency of the per-epoch loop update (warp0_update) on one
// warp in isolation (no cluster), cycles per call.  nvcc ... -I include -I csrc
#include <cstdio>
#include "correlator.cuh"
using namespace l1rxg;
__global__ void k(TrackArgs a, long long* cyc) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    CorrSmem<3>* s = reinterpret_cast<CorrSmem<3>*>(smem_raw);
    const int lane = threadIdx.x;
    if (lane == 0) {
        memset(&s->ch, 0, sizeof(s->ch));
        s->ch.state = L1RXG_TRACKING;
        s->ch.code_freq_hz = 1.023e6; s->ch.carrier_doppler_hz = 1200.0;
        s->ch.epochs_since_handoff = 1000; s->ch.carrier_lock_ratio = 0.95;
        s->ch.fll_enabled = 1; s->ch.pll_primed = 1; s->ch.dll_primed = 1; s->ch.have_last_prompt = 1;
        s->ch.last_ip = 1000.0; s->ch.last_qp = 10.0;
        make_consts(s->c, 100.25, 1.023e6, 1200.0, 0.3, a.lc.fs, a.n);
        s->nco_ph1 = 0.1; s->nco_cp1 = 200.5;
    }
    for (int v = lane; v < 32 * 8; v += 32) s->red[v] = 1.0f + 0.01f * v;
    __syncwarp();
    const EpochConsts c = s->c;
    long long t0 = clock64();
    for (int it = 0; it < 100; ++it) {
        warp0_update<3>(s, a, c, 0, 0, it, 19, lane, 0, it, nullptr, 0);
        s->ch.state = L1RXG_TRACKING;
        s->stop = 0;
    }
    long long t1 = clock64();
    if (lane == 0) cyc[0] = (t1 - t0) / 100;
}
#ifdef L1RXG_PROFILE
static const char* W[] = {"totals", "cluster", "operands", "atan2/sqrt", "pre", "loop_fast", "div", "consts"};
#endif
int main() {
    TrackArgs a{};
    a.n = 16368; a.kp = 1; a.ke = 0; a.kl = 2; a.max_records = 16; a.csize = 1;
    a.lc.fs = 16.368e6; a.lc.dt = 1e-3; a.lc.pll_k1 = 0.1; a.lc.pll_k2 = 0.2;
    a.lc.dll_k1 = 0.01; a.lc.dll_k2 = 0.02; a.lc.fll_k = 1.0; a.lc.inv_fll_c = 1.0; a.lc.inv_fll_f = 1.0;
    a.lc.cfg.fll_pull_in_ms = 400; a.lc.cfg.fll_coarse_ms = 100;
    long long* c; cudaMalloc(&c, 8);
    long long* prof = nullptr;
#ifdef L1RXG_PROFILE
    cudaMalloc(&prof, 4 * 64 * 8 * 8); cudaMemset(prof, 0, 4 * 64 * 8 * 8);
#endif
    a.prof = prof;
    const size_t sm = sizeof(CorrSmem<3>) + 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<1, 32, sm>>>(a, c); k<<<1, 32, sm>>>(a, c);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("warp0_update: %lld cycles per call (err %s)\n", h, cudaGetErrorString(cudaGetLastError()));
#ifdef L1RXG_PROFILE
    long long hp[4 * 64 * 8];
    cudaMemcpy(hp, prof, sizeof hp, cudaMemcpyDeviceToHost);
    double acc[8] = {0}; int n = 0;
    for (int e = 2; e < 64; ++e) { for (int k = 1; k < 8; ++k) acc[k] += hp[1024 + e * 8 + k] - hp[1024 + e * 8 + k - 1]; ++n; }
    for (int k = 1; k < 8; ++k) printf("  %-12s %.0f\n", W[k], acc[k] / n);
#endif
    return 0;
}
