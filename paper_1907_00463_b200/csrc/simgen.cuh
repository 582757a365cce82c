// simgen.cuh -- K0: on-device scenario synthesizer for the benchmark corpora.
//
// Restates the reference simulator's raw mode (SimStream, simsource.hpp:
// 194-331) and its recording quantisation (generate_recording,
// simsource.hpp:387-413) as one kernel over many seeded recordings:
//   * effective delay tau(t) = delay / chip_rate - (fD t + rate t^2 / 2) / f_L1
//     (:344-352); per 1-ms block the transmit chip count and the carrier
//     phase are interpolated linearly between the block edges (:262-284),
//     chip = code[floor(c0 + i dc) mod 1023] (:296-302);
//   * amplitude A = sigma sqrt(10^(CN0/10) / fs), sigma = 0.25 with noise,
//     1 without (:237-239);
//   * per-SV waveforms summed before the noise (superposition, :309-312);
//     complex AWGN of sigma / sqrt(2) per component (:325-327);
//   * quantisation lround + clamp to int16 / int8 (:393-413).
// Differences, by design: the carrier is cos/sin of the interpolated phase
// (the reference rotates a phasor, renormalised every 1024 samples, :292-307
// -- the same phase to ~1e-12 rad); the noise is Philox4x32-10 keyed by
// (seed, recording) and counted by sample index with Box-Muller pairs, so any
// chunking of a recording gives the same bytes (the reference draws one
// sequential stream).  Builder extension (as simsource.py): real-IF int8
// output Re{s(n) e^{+j 2 pi IF n / fs}} + N(0, sigma^2 / 4).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace l1rxg {

constexpr int SIM_MAX_SV = 32;

struct SimSvDev {
    double delay_s;    // code_delay_chips / chip_rate
    double fd_over_l1; // doppler / f_L1 (cycles of delay per second)
    double rate_over_l1;
    double phase0;
    double amp;
    int prn;
    int pad;
};

// Philox4x32-10 (Salmon et al. 2011), one block of four 32-bit outputs.
__device__ __forceinline__ uint4 philox4x32(uint4 ctr, uint2 key) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, ctr.x), lo0 = 0xD2511F53u * ctr.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, ctr.z), lo1 = 0xCD9E8D57u * ctr.z;
        ctr = make_uint4(hi1 ^ ctr.y ^ key.x, lo1, hi0 ^ ctr.w ^ key.y, lo0);
        key.x += 0x9E3779B9u;
        key.y += 0xBB67AE85u;
    }
    return ctr;
}

// two standard normals from two 32-bit uniforms (Box-Muller, fp32)
__device__ __forceinline__ float2 box_muller(uint32_t a, uint32_t b) {
    const float u1 = ((float)a + 1.0f) * 2.3283064365386963e-10f;  // (0, 1]
    const float u2 = (float)b * 2.3283064365386963e-10f;
    const float r = sqrtf(-2.0f * __logf(u1));
    float s, c;
    sincospif(2.0f * u2, &s, &c);
    return make_float2(r * c, r * s);
}

__device__ __forceinline__ long q_lround(double v) {  // std::lround
    return (long)(v + (v >= 0.0 ? 0.5 : -0.5));
}

// One CTA per (recording, 1-ms block): the block's per-SV chip count and
// carrier phase at the edges in shared memory, then the block's samples.
// format: 0 int8 IQ, 1 int16 IQ, 2 int8 real IF.
__global__ void __launch_bounds__(256) simgen_kernel(const SimSvDev* __restrict__ svs, int n_sv,
                                                     const int8_t* __restrict__ codes, int n, double fs,
                                                     double if_hz, int64_t ms0, int format,
                                                     unsigned long long seed, int noise,
                                                     unsigned char* out, int64_t rec_stride) {
    constexpr double CHIP = 1.023e6, F_L1 = 1.57542e9, PI = 3.14159265358979323846;
    __shared__ double c0s[SIM_MAX_SV], dcs[SIM_MAX_SV], th0s[SIM_MAX_SV], dths[SIM_MAX_SV];
    __shared__ float amps[SIM_MAX_SV];
    __shared__ int8_t code_s[SIM_MAX_SV][1023];
    const int rec = blockIdx.y;
    const int64_t ms = ms0 + blockIdx.x;
    const SimSvDev* sv = svs + (int64_t)rec * n_sv;
    if (threadIdx.x < n_sv) {
        const SimSvDev p = sv[threadIdx.x];
        const double t0 = (double)ms * 1e-3, t1 = t0 + 1e-3;
        const double tau0 = p.delay_s - (p.fd_over_l1 * t0 + 0.5 * p.rate_over_l1 * t0 * t0);
        const double tau1 = p.delay_s - (p.fd_over_l1 * t1 + 0.5 * p.rate_over_l1 * t1 * t1);
        const double off = 6.0;  // tow_start - nav_encode_start
        const double c0 = (t0 + off - tau0) * CHIP, c1 = (t1 + off - tau1) * CHIP;
        c0s[threadIdx.x] = c0;
        dcs[threadIdx.x] = (c1 - c0) / (double)n;
        const double th0 = p.phase0 - 2.0 * PI * F_L1 * tau0;
        const double th1 = p.phase0 - 2.0 * PI * F_L1 * tau1;
        th0s[threadIdx.x] = th0;
        dths[threadIdx.x] = (th1 - th0) / (double)n;
        amps[threadIdx.x] = (float)p.amp;
    }
    for (int k = threadIdx.x; k < n_sv * 1023; k += blockDim.x) {
        const int s_ = k / 1023, j = k - s_ * 1023;
        code_s[s_][j] = codes[sv[s_].prn * 1023 + j];
    }
    __syncthreads();
    const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32) ^ (uint32_t)rec * 0x9E3779B9u);
    const int64_t g0 = (int64_t)blockIdx.x * n;  // first sample of the block in this launch
    unsigned char* dst = out + (int64_t)rec * rec_stride;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double re = 0.0, im = 0.0;
        for (int s_ = 0; s_ < n_sv; ++s_) {
            const double chips = fma((double)i, dcs[s_], c0s[s_]);
            const int64_t ic = (int64_t)chips;
            const double ch = (double)code_s[s_][(int)(ic % 1023)];
            // carrier phase reduced in fp64, cos/sin in fp32 (amplitude ~1e-2)
            const double th = fma((double)i, dths[s_], th0s[s_]);
            const double r = th - 2.0 * PI * rint(th * (1.0 / (2.0 * PI)));
            float sn, cs;
            __sincosf((float)r, &sn, &cs);
            re = fma((double)(amps[s_] * cs), ch, re);
            im = fma((double)(amps[s_] * sn), ch, im);
        }
        const int64_t gs = (ms0 * n) + g0 + i;  // sample index in the recording
        if (format == 2) {  // real IF
            const double ph = 2.0 * PI * if_hz / fs * (double)gs;
            double v = re * cos(ph) - im * sin(ph);
            if (noise) {
                const uint4 w = philox4x32(make_uint4((uint32_t)gs, (uint32_t)(gs >> 32), 0x5eedu, 0u), key);
                v += 0.125 * (double)box_muller(w.x, w.y).x;
            }
            long q = q_lround(v * 128.0);
            q = q < -127 ? -127 : (q > 127 ? 127 : q);
            reinterpret_cast<int8_t*>(dst)[gs - ms0 * n] = (int8_t)q;
        } else {
            if (noise) {
                const uint4 w = philox4x32(make_uint4((uint32_t)gs, (uint32_t)(gs >> 32), 0x5eedu, 0u), key);
                const float2 z = box_muller(w.x, w.y);
                const double sg = 0.25 / 1.4142135623730951;
                re += sg * (double)z.x;
                im += sg * (double)z.y;
            }
            const double scale = format == 1 ? 32768.0 : 128.0;
            const long lim = format == 1 ? 32767 : 127;
            long qr = q_lround(re * scale), qi = q_lround(im * scale);
            qr = qr < -lim ? -lim : (qr > lim ? lim : qr);
            qi = qi < -lim ? -lim : (qi > lim ? lim : qi);
            const int64_t o = gs - ms0 * n;
            if (format == 1) {
                reinterpret_cast<short2*>(dst)[o] = make_short2((short)qr, (short)qi);
            } else {
                reinterpret_cast<char2*>(dst)[o] = make_char2((char)qr, (char)qi);
            }
        }
    }
}

}  // namespace l1rxg
