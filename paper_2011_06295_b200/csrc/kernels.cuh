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
#include <cstdint>

namespace scb {

// ------------------------------------------------------------------------
// arithmetic policies
// ------------------------------------------------------------------------
enum { MODE_EXACT = 0, MODE_FMA = 1 };

template <int MODE>
__device__ __forceinline__ float mac1(float acc, float v, float x) {
    if constexpr (MODE == MODE_EXACT) return __fadd_rn(acc, __fmul_rn(v, x));
    else return __fmaf_rn(v, x, acc);
}

__device__ __forceinline__ unsigned long long pack2(float2 a) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
    return r;
}
__device__ __forceinline__ float2 unpack2(unsigned long long r) {
    float2 a;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
    return a;
}

// Two MACs sharing one weight, two images packed in a register pair.
// Exact: one packed FMUL2 then two scalar FADDs (ptxas fuses a packed add
// after a packed mul into FFMA2, which would break bit-exactness; the scalar
// adds are kept separate -- tests/test_sass.py checks the SASS).
template <int MODE>
__device__ __forceinline__ void mac2(float2& acc, unsigned long long vv, float2 x) {
    if constexpr (MODE == MODE_EXACT) {
        unsigned long long p;
        asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(p) : "l"(vv), "l"(pack2(x)));
        float2 pr = unpack2(p);
        acc.x = __fadd_rn(acc.x, pr.x);
        acc.y = __fadd_rn(acc.y, pr.y);
    } else {
        unsigned long long a = pack2(acc), r;
        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pack2(x)), "l"(vv), "l"(a));
        acc = unpack2(r);
    }
}

// ------------------------------------------------------------------------
// weight payload decode (in-register dequantisation)
// ------------------------------------------------------------------------
enum { WF_F32 = 0, WF_F16 = 1, WF_CB4 = 2, WF_LIN16 = 3 };

struct Tap {          // one nonzero of the device tap program
    uint32_t meta;    // case index kk*R*S + r*S + s
    uint32_t payload; // f32 bits | f16 bits | int16 code | 4-bit codebook index
};

struct QuantAux {
    float cb[16];     // codebook table (CB4)
    float scale;      // 2^-frac (LIN16)
};

template <int WF>
__device__ __forceinline__ float decode_w(uint32_t payload, const QuantAux& q) {
    if constexpr (WF == WF_F32) return __uint_as_float(payload);
    else if constexpr (WF == WF_F16) return __half2float(__ushort_as_half((unsigned short)payload));
    else if constexpr (WF == WF_CB4) return q.cb[payload & 15u];
    else return (float)(int)(short)(payload & 0xffffu) * q.scale;
}

// ------------------------------------------------------------------------
// kernel parameter blocks
// ------------------------------------------------------------------------
struct GenericParams {
    const void* x;
    const void* bias;       // may be null
    void* y;
    const void* values;     // native values (f32/f64/f16)
    const int32_t* dec;     // packed (c << 12) | (r << 6) | s per tap
    const int32_t* rowptr;
    int n, c, h, w, k, e, f, stride, pad;
    uint32_t flags;
};

struct TiledParams {
    const void* x;
    const void* bias;       // may be null
    void* y;
    const int32_t* tap_ptr; // [G][C+1] absolute tap offsets
    const Tap* taps;
    QuantAux q;
    int n, c, h, w, k, e, f, pad;
    int imgs, bh, bw, cc, wk;   // launch shape
    int wp;                     // pixel warps per warp group
    int row;                    // smem row pitch in pixels
    int tap_cap;                // taps per (warp group, stage)
    int n_ey, n_fx, kblocks, groups;
    uint32_t flags;
};

}  // namespace scb
