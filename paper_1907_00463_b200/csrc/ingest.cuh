// ingest.cuh -- K1: raw recording bytes -> complex baseband ring (sm_100a).
//
// Reference: SampleSource::read_samples / downconvert (samples.hpp:177-253):
// int8 / int16 complex decode (/128, /32768) and, for Int8RealIF, the
// complex mixer at -IF on the global sample index followed by the 23-tap
// half-band FIR (Hamming-windowed sinc, cutoff fs/4, unit DC gain, x2)
// with a 22-sample history carried across blocks.  One pass per stream
// sample, shared by every channel that tracks the stream.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "l1rxg.h"

namespace l1rxg {

// ---------------------------------------------------------------------
// K1 ingest.  Ring write: sample g -> ring[g mod R] (+ apron copy).
__device__ __forceinline__ void ring_put(float2* ring, int64_t R, int64_t apron,
                                         int64_t pos, float2 v) {
    ring[pos] = v;
    if (pos < apron)
        ring[R + pos] = v;
}

// Int8RealIF at IF = fs/4: the mixer step is exactly -pi/2, so
// mixed(g) = v(g)/128 * {1, -j, -1, j}[g mod 4]; the FIR output
// 2*sum_t h[t] mixed(g-t) (samples.hpp:234-240) is a 23-tap real
// convolution per output phase with coefficient tables cre/cim[4][23]
// folded on the host (includes the 2/128 scale).
// The same filter with its structure used: of the 46 products per output
// only 13 matter -- the mixer zeroes one component of every sample, and the
// half-band taps at odd t != 11 are 1e-17 (sin(m pi) in floating point).
// For g = ph mod 4 the component fed by the even taps is
//   B = sum_{k<12} a[k] v(g - 2k),  a[k] = 2 h[2k] / 128 * (-1)^k  (phase 0's signs),
// negated for the phases in big_neg, and the other component is c * v(g - 11),
// negated for the phases in c_neg; even phases give (re, im) = (B, C), odd
// phases (C, B).  Same ascending-t FMA chain as the full tables minus the
// terms below 1e-15 of the result.  One definition for the ingest kernel
// (float2 rings) and the FIR warps of the overlapped kernel (raw rings).
struct If4Fir {
    float a[12];
    float c;
    uint32_t big_neg, c_neg;
};
__constant__ If4Fir c_if4f;

// x[0] = v(g), x[-t] = v(g - t) as floats (the raw int8 values); ph = g & 3.
__device__ __forceinline__ float2 if4_fir(const float* x, int ph) {
    float b = 0.f;
#pragma unroll
    for (int k = 0; k < 12; ++k)
        b = fmaf(c_if4f.a[k], x[-2 * k], b);
    float c = c_if4f.c * x[-11];
    b = (c_if4f.big_neg >> ph) & 1u ? -b : b;
    c = (c_if4f.c_neg >> ph) & 1u ? -c : c;
    return (ph & 1) ? make_float2(c, b) : make_float2(b, c);
}

constexpr int ING_TPB = 256;
constexpr int ING_OUT_PER_THREAD = 4;
constexpr int ING_TILE = ING_TPB * ING_OUT_PER_THREAD;  // outputs per block

// raw: bytes of samples [g0, g0+count); hist: the 22 bytes before g0
// (zeros at stream start); writes hist_out = the last 22 bytes of the run.
// A block stages its 1024 + 24 input samples as floats (sample t0 - 24 + k at
// v[k]); a thread then holds the 28 samples of four consecutive outputs in
// registers (seven LDS.128) and stores the outputs as two 16-byte vectors
// where the ring position allows it.
__global__ void __launch_bounds__(ING_TPB) ingest_if4_kernel(
    const int8_t* __restrict__ raw, const int8_t* __restrict__ hist, int8_t* hist_out,
    int64_t g0, int64_t count, float2* ring, int64_t R, int64_t apron, int64_t pos0,
    int64_t* avail_slot) {
    __shared__ __align__(16) float v[ING_TILE + 24];
    const int64_t t0 = (int64_t)blockIdx.x * ING_TILE;  // run-relative first output
    for (int k = threadIdx.x; k < ING_TILE + 24; k += ING_TPB) {
        const int64_t idx = t0 - 24 + k;
        int8_t b = 0;
        if (idx < 0)
            b = idx >= -22 ? hist[22 + idx] : (int8_t)0;
        else if (idx < count)
            b = raw[idx];
        v[k] = (float)b;
    }
    __syncthreads();
    const int q = threadIdx.x * ING_OUT_PER_THREAD;
    const int64_t idx0 = t0 + q;
    if (idx0 < count) {
        float x[28];
        const float4* v4 = reinterpret_cast<const float4*>(v + q);
#pragma unroll
        for (int k = 0; k < 7; ++k) {
            const float4 f = v4[k];
            x[4 * k] = f.x;
            x[4 * k + 1] = f.y;
            x[4 * k + 2] = f.z;
            x[4 * k + 3] = f.w;
        }
        const int ph0 = (int)((g0 + idx0) & 3);
        float2 y[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            y[u] = if4_fir(&x[24 + u], (ph0 + u) & 3);
        int64_t pos = pos0 + idx0;
        if (pos >= R)
            pos -= R;
        if (idx0 + 4 <= count && pos + 4 <= R && ((pos | R) & 1) == 0) {
            const float4 a = make_float4(y[0].x, y[0].y, y[1].x, y[1].y);
            const float4 b = make_float4(y[2].x, y[2].y, y[3].x, y[3].y);
            float4* o = reinterpret_cast<float4*>(ring + pos);
            o[0] = a;
            o[1] = b;
            if (pos + 4 <= apron) {
                float4* m = reinterpret_cast<float4*>(ring + R + pos);
                m[0] = a;
                m[1] = b;
            } else if (pos < apron) {
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (pos + u < apron)
                        ring[R + pos + u] = y[u];
            }
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (idx0 + u >= count)
                    break;
                int64_t p = pos + u;
                if (p >= R)
                    p -= R;
                ring_put(ring, R, apron, p, y[u]);
            }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < 22) {
        const int64_t idx = count - 22 + threadIdx.x;
        hist_out[threadIdx.x] = idx >= 0 ? raw[idx] : hist[22 + idx];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && avail_slot)
        *avail_slot = g0 + count;
}

// Raw real-IF ring (overlapped kernel with FIR warps): the bytes themselves,
// ring[g mod R], the head mirrored behind the tail (apron) and the last
// RAWIF_PAD bytes mirrored in front of the head, so every window
// [pos - 22, pos + n) is contiguous.  The pad reads zero at stream start.
constexpr int RAWIF_PAD = 32;
__global__ void copy_rawif_kernel(const int8_t* __restrict__ src, int64_t count, int8_t* ring, int64_t R,
                                  int64_t apron, int64_t pos0, int64_t* avail_slot, int64_t avail_value) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) {
        const int8_t v = src[i];
        int64_t pos = pos0 + i;
        if (pos >= R)
            pos -= R;
        ring[pos] = v;
        if (pos < apron)
            ring[R + pos] = v;
        if (pos >= R - RAWIF_PAD)
            ring[pos - R] = v;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && avail_slot)
        *avail_slot = avail_value;
}
// Baseband samples [g0, g0 + count) of a raw real-IF ring (read_samples).
__global__ void rawif_window_kernel(const int8_t* __restrict__ ring, int64_t R, int64_t g0, int64_t count,
                                    float2* out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count)
        return;
    float x[23];
#pragma unroll
    for (int t = 0; t < 23; ++t) {
        const int64_t g = g0 + i - t;
        x[22 - t] = g >= 0 ? (float)ring[g % R] : 0.f;
    }
    out[i] = if4_fir(&x[22], (int)((g0 + i) & 3));
}

// Generic real IF: pass 1, mixer at the global index in fp64
// (samples.hpp:217-226) into mixed[22 + i]; mixed[0..22) holds history.
__global__ void mix_generic_kernel(const int8_t* __restrict__ raw, int64_t g0, int64_t count,
                                   double w, float2* mixed) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count)
        return;
    const double vv = (double)raw[i] / 128.0;
    double s, c;
    sincos(w * (double)(g0 + i), &s, &c);
    mixed[22 + i] = make_float2((float)(vv * c), (float)(vv * s));
}

// pass 2: out(g) = 2 sum_t h[t] mixed(g - t)
__constant__ float c_halfband2[23];
__global__ void fir_generic_kernel(const float2* __restrict__ mixed, int64_t count, float2* ring,
                                   int64_t R, int64_t apron, int64_t pos0, float2* hist_out,
                                   int64_t* avail_slot, int64_t avail_value) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) {
        float re = 0.f, im = 0.f;
#pragma unroll
        for (int t = 0; t < 23; ++t) {
            const float2 m = mixed[22 + i - t];
            re = fmaf(c_halfband2[t], m.x, re);
            im = fmaf(c_halfband2[t], m.y, im);
        }
        int64_t pos = pos0 + i;
        if (pos >= R)
            pos -= R;
        ring_put(ring, R, apron, pos, make_float2(re, im));
    }
    if (blockIdx.x == 0 && threadIdx.x < 22)
        hist_out[threadIdx.x] = mixed[count + threadIdx.x];
    if (blockIdx.x == 0 && threadIdx.x == 0 && avail_slot)
        *avail_slot = avail_value;
}

// Complex int8 / int16 decode (samples.hpp:188-205).
__global__ void decode_iq_kernel(const void* __restrict__ raw, int fmt, int64_t count,
                                 float2* ring, int64_t R, int64_t apron, int64_t pos0,
                                 int64_t* avail_slot, int64_t avail_value) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) {
        float2 v;
        if (fmt == L1RXG_FMT_INT8_IQ) {
            const char2 b = reinterpret_cast<const char2*>(raw)[i];
            v = make_float2((float)b.x * (1.0f / 128.0f), (float)b.y * (1.0f / 128.0f));
        } else {
            const short2 b = reinterpret_cast<const short2*>(raw)[i];
            v = make_float2((float)b.x * (1.0f / 32768.0f), (float)b.y * (1.0f / 32768.0f));
        }
        int64_t pos = pos0 + i;
        if (pos >= R)
            pos -= R;
        ring_put(ring, R, apron, pos, v);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && avail_slot)
        *avail_slot = avail_value;
}

// The same decode for many streams in one launch (blockIdx.y = stream):
// stream s reads raw + s * raw_stride bytes and writes ring + s * ring_stride.
__global__ void decode_iq_strided_kernel(const uint8_t* __restrict__ raw, int64_t raw_stride, int fmt,
                                         int64_t count, float2* ring, int64_t ring_stride, int64_t R,
                                         int64_t apron, int64_t pos0, int64_t* avail,
                                         int64_t avail_value) {
    const int s = blockIdx.y;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint8_t* rs = raw + (int64_t)s * raw_stride;
    float2* rg = ring + (int64_t)s * ring_stride;
    if (i < count) {
        float2 v;
        if (fmt == L1RXG_FMT_INT8_IQ) {
            const char2 b = reinterpret_cast<const char2*>(rs)[i];
            v = make_float2((float)b.x * (1.0f / 128.0f), (float)b.y * (1.0f / 128.0f));
        } else {
            const short2 b = reinterpret_cast<const short2*>(rs)[i];
            v = make_float2((float)b.x * (1.0f / 32768.0f), (float)b.y * (1.0f / 32768.0f));
        }
        int64_t pos = pos0 + i;
        if (pos >= R)
            pos -= R;
        ring_put(rg, R, apron, pos, v);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0)
        avail[s] = avail_value;
}

// Fast path of the strided cint16 decode: two samples per thread (one 8-byte
// load, one 16-byte store), for even ring positions, even R and an even
// apron (then a pair never straddles the wrap or the apron edge).
__global__ void decode_i16x2_strided_kernel(const uint8_t* __restrict__ raw, int64_t raw_stride,
                                            int64_t npairs, float2* ring, int64_t ring_stride,
                                            int64_t R, int64_t apron, int64_t pos0, int64_t* avail,
                                            int64_t avail_value) {
    const int s = blockIdx.y;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint2* rs = reinterpret_cast<const uint2*>(raw + (int64_t)s * raw_stride);
    float2* rg = ring + (int64_t)s * ring_stride;
    if (i < npairs) {
        const uint2 w = __ldcs(rs + i);  // streamed once
        const float k = 1.0f / 32768.0f;
        const float4 v = make_float4((float)(short)(w.x & 0xffffu) * k, (float)((int)w.x >> 16) * k,
                                     (float)(short)(w.y & 0xffffu) * k, (float)((int)w.y >> 16) * k);
        int64_t pos = pos0 + 2 * i;
        if (pos >= R)
            pos -= R;
        *reinterpret_cast<float4*>(rg + pos) = v;
        if (pos < apron)
            *reinterpret_cast<float4*>(rg + R + pos) = v;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0)
        avail[s] = avail_value;
}

// Complex int8 / int16 recordings are kept RAW in the tracker's ring (E =
// uint16_t or uint32_t per sample; the correlator converts while it wipes,
// with the /128 or /32768 scale folded exactly into its rotator table): the
// push is a copy into ring position pos (+ the apron mirror).
template <typename E>
__global__ void copy_raw_kernel(const E* __restrict__ src, int64_t count, E* ring, int64_t R,
                                int64_t apron, int64_t pos0, int64_t* avail_slot,
                                int64_t avail_value) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) {
        const E v = src[i];
        int64_t pos = pos0 + i;
        if (pos >= R)
            pos -= R;
        ring[pos] = v;
        if (pos < apron)
            ring[R + pos] = v;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && avail_slot)
        *avail_slot = avail_value;
}
// The same for every stream of a tracker in one launch (blockIdx.y = stream).
template <typename E>
__global__ void copy_raw_strided_kernel(const uint8_t* __restrict__ src, int64_t src_stride_bytes,
                                        int64_t count, E* ring, int64_t ring_stride, int64_t R,
                                        int64_t apron, int64_t pos0, int64_t* avail,
                                        int64_t avail_value) {
    const int s = blockIdx.y;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const E* sp = reinterpret_cast<const E*>(src + (int64_t)s * src_stride_bytes);
    E* rg = ring + (int64_t)s * ring_stride;
    if (i < count) {
        const E v = sp[i];
        int64_t pos = pos0 + i;
        if (pos >= R)
            pos -= R;
        rg[pos] = v;
        if (pos < apron)
            rg[R + pos] = v;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0)
        avail[s] = avail_value;
}

// complex<double> -> float2 (per-call path)
__global__ void cf64_to_f32_kernel(const double2* __restrict__ in, float2* out, int64_t count) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) {
        const double2 x = in[i];
        out[i] = make_float2((float)x.x, (float)x.y);
    }
}

}  // namespace l1rxg
