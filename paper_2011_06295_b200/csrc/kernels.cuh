// Device kernels of the sm_100a direct sparse convolution engine.
//
// Semantics (reference _kernels.py:53-85, engine.py:68-87): for every output
//   o = bias[k];  for t in row k, in colidx (= (c, r, s)) order:
//       o = o (+) v_t (x) x[n, c_t, e*stride + r_t - pad, f*stride + s_t - pad]
// with the multiply and the add rounded separately (exact mode) and 0 for
// taps that fall into the zero padding.  f16 storage upcasts to f32 and the
// product of two f16 numbers is exact in f32, so a single FFMA is bit-equal
// to the reference there.  f64 computes in f64 (generic kernel).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace scb {

// Opt a kernel into the full dynamic shared memory on the CURRENT device.  The
// attribute is per (function, device), so `lim` is a per-launcher array indexed by
// device: a process driving several GPUs sets it once on each (benign race:
// idempotent).  Returns cudaErrorInvalidValue if `smem` exceeds the limit.
template <typename K>
inline cudaError_t dyn_smem_ok(K kern, size_t smem, int (&lim)[64]) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    if (lim[dev] == 0) {
        cudaFuncAttributes fa;
        if ((e = cudaFuncGetAttributes(&fa, kern)) != cudaSuccess) return e;
        const int l = 227 * 1024 - (int)fa.sharedSizeBytes;
        if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, l)) != cudaSuccess) return e;
        lim[dev] = l;
    }
    return (int)smem > lim[dev] ? cudaErrorInvalidValue : cudaSuccess;
}

enum { MODE_EXACT = 0, MODE_FMA = 1,
       MODE_HALF2 = 2 };  // f16 opt-in fast mode: half2 accumulators, HFMA2 (tolerance 1e-2)
enum { WF_F32 = 0, WF_F16 = 1, WF_CB4 = 2, WF_LIN16 = 3, WF_AFF16 = 4 };
// how the tiled kernel dispatches a tap to its unrolled MAC block (gen_taploop.py)
enum { DISPATCH_JUMP = 0,   // brx.idx jump table, one indirect branch per tap
       DISPATCH_MASK = 1,   // per-channel KT x 16-bit masks walked in order
       DISPATCH_WIDE = 2,   // (direct kind) column tiles of tw for any row width
       DISPATCH_ONED = 3 }; // (direct kind) 1D rows: tiles of th*tw columns, H = R = 1

// Activation fake-quant (quantize.py:332-338, affine int quantize.py:122-138): clip in
// the activation dtype, code = clamp(rint((c - mu) / step)) in f64, mu + code*step in
// f64, one round to the activation dtype.  Separate IEEE roundings as numpy does.
struct ActQuant {
    float lo, hi;         // clip bounds rounded to the activation dtype (f32 / f16 values)
    double dlo, dhi;      // ... as f64 (f64 activations)
    double mu, step, clo, chi;
};
__device__ __forceinline__ double fq_code(double c, const ActQuant& q) {
    double r = rint(__ddiv_rn(__dsub_rn(c, q.mu), q.step));
    return fmin(fmax(r, q.clo), q.chi);
}
__device__ __forceinline__ double fq_value(double code, const ActQuant& q) {
    return __dadd_rn(q.mu, __dmul_rn(code, q.step));
}
__device__ __forceinline__ float fq_f32(float a, const ActQuant& q) {
    const float c = fminf(fmaxf(a, q.lo), q.hi);
    return __double2float_rn(fq_value(fq_code((double)c, q), q));
}
__device__ __forceinline__ __half fq_f16(__half a, const ActQuant& q) {
    const float c = fminf(fmaxf(__half2float(a), q.lo), q.hi);  // exact: f16 values in f32
    return __double2half(fq_value(fq_code((double)c, q), q));
}
__device__ __forceinline__ double fq_f64(double a, const ActQuant& q) {
    return fq_value(fq_code(fmin(fmax(a, q.dlo), q.dhi), q), q);
}

// fake-quant of an epilogue value in its storage type, returned as the (exact) float of the
// stored value: f32 directly, f16 via one round to half first (the reference's f16 profile)
template <typename T>
__device__ __forceinline__ float fq_store(float o, const ActQuant& q);
template <>
__device__ __forceinline__ float fq_store<float>(float o, const ActQuant& q) { return fq_f32(o, q); }
template <>
__device__ __forceinline__ float fq_store<__half>(float o, const ActQuant& q) {
    return __half2float(fq_f16(__float2half_rn(o), q));
}

// ReLU in the storage dtype (store.py:284 applies np.maximum(., 0) to the conv output AFTER
// it was rounded to the activation dtype): for f16 a tiny negative sum rounds to -0.0 and
// stays -0.0.  Returns the exact float of the value to store.
template <typename T>
__device__ __forceinline__ float relu_io(float o);
template <>
__device__ __forceinline__ float relu_io<float>(float o) { return o < 0.f ? 0.f : o; }
template <>
__device__ __forceinline__ float relu_io<__half>(float o) {
    const float r = __half2float(__float2half_rn(o));
    return r < 0.f ? 0.f : r;
}

template <int MODE>
__device__ __forceinline__ float mac1(float acc, float v, float x) {
    if constexpr (MODE == MODE_EXACT) return __fadd_rn(acc, __fmul_rn(v, x));
    else return __fmaf_rn(v, x, acc);
}

struct Tap {          // one nonzero of the device tap program
    uint32_t meta;    // case index kk*R*S + r*S + s
    uint32_t payload; // f32 bits | f16 bits | int16 code | 4-bit codebook index
};

struct QuantAux {
    float cb[16];     // codebook table (CB4)
    float scale;      // 2^-frac (LIN16)
    double step;      // affine symmetric step (AFF16, quantize.py:99-138)
    unsigned short cb16[16];  // CB4 table as f16 bits (f16-storage kernels)
};

// Compact f16 tap (4 bytes): bits 0..15 = element offset in the stage window,
// bits 16..31 = payload decoded IN REGISTER by the weight format:
//   WF_F16   f16 bits of the value
//   WF_CB4   4-bit codebook index -> cb16[] (the reference's Codebook.decode, quantize.py:209-210)
//   WF_LIN16 int16 code x 2^-frac, exact in f32, then f16 (quantize_fixed + astype, quantize.py:64-71,275)
//   WF_AFF16 int16 code: f16(f64(code) * step) -- dequantize_affine_int in f64 then astype(f16)
//            (quantize.py:137-138, 279-283), one direct f64 -> f16 rounding like numpy
template <int WF>
__device__ __forceinline__ unsigned short tap_f16(unsigned payload, const unsigned short* cbt, float scale,
                                                  double step) {
    if constexpr (WF == WF_F16) {
        return (unsigned short)payload;
    } else if constexpr (WF == WF_CB4) {
        return cbt[payload & 15u];
    } else if constexpr (WF == WF_LIN16) {
        return __half_as_ushort(__float2half_rn((float)(short)payload * scale));
    } else {
        static_assert(WF == WF_AFF16, "f16 tap format");
        return __half_as_ushort(__double2half(__dmul_rn((double)(short)payload, step)));
    }
}

struct GenericParams {
    const void* x;
    const void* bias;       // compute dtype (f32, or f64 for f64), may be null
    void* y;
    const void* values;     // native values (f32/f64/f16)
    const int32_t* dec;     // flat kernel index c*R*S + r*S + s per tap (any extent: < C*R*S <= 2^31)
    const int32_t* rowptr;
    int n, c, h, w, k, e, f, stride, pad;
    int kr, ks;             // kernel extent R, S (decode of dec)
    uint32_t flags;
};

struct TiledParams {
    const void* x;
    const float* bias;      // f32 compute dtype, may be null
    void* y;
    const int32_t* tap_ptr; // [G][C+1] absolute tap offsets
    const Tap* taps;        // (c, kk, r, s)-ordered taps per group, two slack slots at the end
    const uint32_t* masks;  // DISPATCH_MASK: [G][C][KT/2] 16-bit tap masks per kk
    QuantAux q;
    int n, c, h, w, k, e, f, pad;
    int imgs, bh, bw, cc, wk;   // launch shape
    int wp;                     // pixel warps per warp group
    int row;                    // smem row pitch (elements)
    int stage_el;               // elements per pipeline stage
    int chunk;                  // cp.async size in bytes (16, 8 or 4)
    int tap_cap;                // tap entries per (stage, warp group) in shared memory
    int n_ey, n_fx, kblocks, groups;
    uint32_t flags;
};

}  // namespace scb
