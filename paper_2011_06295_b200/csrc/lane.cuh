// Image-lane position-class kernel (kind 7, sm_100a) for small output planes.
//
// Why: on 4x4 and 2x2 planes (VGG-CIFAR conv4_x / conv5_x) a 3x3 / pad 1 tap
// lands in the zero padding for 31 % / 56 % of the outputs the reference
// iterates over (_kernels.py:73-84 runs `o = o + v * x` for every tap and every
// output, x = 0 in the padding).  The direct kernels (direct.cuh, dimg.cuh)
// spend a shared-memory load and an FMUL+FADD on each of those.  Here the
// padding taps are dropped at upload time, so the kernel executes only the
// MACs whose input is inside the image, in the reference's order:
//
//  * the outputs of a plane fall into position classes (rows {0}, {1..H-2},
//    {H-1} x the same for columns): all positions of a class see the same set of
//    in-image taps (r, s), at the same relative input offset.  For every output
//    channel, input-channel stage and class the host writes the class's tap list
//    -- the CSR row in colidx order with the padding taps removed -- as
//    {v, byte offset of the input row of the class's first position};
//  * lane = image (NB consecutive images per lane, 32*NB per CTA), the whole plane
//    of accumulators in registers, the class's positions a compile-time set of
//    immediate row offsets: per tap one broadcast descriptor, then per position
//    one conflict-free vector load of the lane's NB images and NB MACs -- no
//    data-dependent control flow, no padding MACs;
//  * class split (CS): CS warps share an output channel, each owning a fixed set of
//    classes (lane_class_group; 8x8 planes by quadrant) -- shorter per-warp chains
//    for small batches, more warps per SM; pooled windows that straddle two warps'
//    positions are exchanged through the drained ring;
//  * activations are IMAGE-MINOR: x[(c*H + y)*W + x][n] with a row stride ldx
//    (>= n): a stage (cc channels of a block's images) is one 2D TMA box
//    {32*NB images, cc*H*W rows} (cp.async.bulk.tensor, out-of-bounds images /
//    channels zero-filled) plus one 1D bulk copy of the CTA's descriptor slots,
//    issued by a producer warp into an NBUF-deep mbarrier ring (1D bulk copies
//    per row were measured at ~70 clk each per SM -- far too slow);
//    consumer warps release a slot with one mbarrier arrive (no CTA barrier,
//    warps drift up to NBUF-1 stages apart);
//  * the epilogue writes image-minor rows too (coalesced 128-byte stores), or NCHW
//    for the last layer of an image-minor run (SCB_FLAG_Y_NCHW), with bias / ReLU /
//    2x2 max-pool / activation fake-quant fused as in direct.cuh;
//  * f16 storage (F16): two images per 32-bit load, FHFMA (exact against the
//    reference's f16 profile), weight formats decoded in registers; MODE_HALF2 is the
//    opt-in fast mode (HFMA2 within a stage, f32 across stages, tolerance 1e-2).
//
// Exactness.  Dropping `o = o + v*(+0)` is exact when v is finite and o is not
// -0.0: v*(+0) is +-0 and o + (+-0) = o.  o can only be -0.0 while every term so
// far (bias included) was -0.0; then a dropped padding tap with a non-negative v
// (v*(+0) = +0) would have turned it into +0 for good, and a later -0.0 product
// keeps +0.  So the only possible difference is a final -0.0 where the reference
// has +0.0, exactly when some dropped tap of that class has a sign-clear v: the
// per-(channel, class) bit in `zmask` restores it in the epilogue.  Layers with a
// non-finite weight are not eligible (the host checks; v*0 would be NaN).
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <type_traits>
#include <vector>

#include "direct.cuh"
#include "kernels.cuh"
#include "sparseconv_b200.h"
#include "ws.cuh"

namespace scb {

// Position classes along one axis of an H-long output axis (3-tap kernel, pad 1):
// class i covers positions lo(i)..hi(i), which all see the same in-image taps.
template <int H>
struct LaneAxis {
    static constexpr int N = H == 1 ? 1 : (H == 2 ? 2 : 3);
    __host__ __device__ static constexpr int lo(int i) { return H <= 2 ? i : (i == 0 ? 0 : (i == 1 ? 1 : H - 1)); }
    __host__ __device__ static constexpr int hi(int i) { return H <= 2 ? i : (i == 0 ? 0 : (i == 1 ? H - 2 : H - 1)); }
};

struct __align__(8) LaneTap {
    float v;
    int32_t off;  // byte offset of the input row (c_local*H*W + first position's input) * RB
};

constexpr int LANE_HDR = 32;  // chunk header: uint16 cumulative class ends (<= 16 classes)

struct alignas(64) LaneParams {
    CUtensorMap tmap;         // x as {images (dim 0), C*H*W rows}, box {32*NB, boxrows}
    const float* bias;        // f32, may be null
    void* y;                  // image-minor output (f32 or f16), row stride ldy elements
    const uint4* desc;        // [nst][K][cap] 16-byte units: per (k, stage) slot = header + LaneTaps
    const uint32_t* zmask;    // [K] classes whose dropped taps include a sign-clear v
    int n, c, k;              // batch (images of this call), input / output channels
    int ldx, ldy;             // image-minor row strides (elements)
    int cc, nst;              // input channels per stage, stages
    int warps, kw;            // consumer warps, channels per warp (= template KW)
    int kgroups;              // channel groups (CTA = image block x channel group)
    int cap;                  // 16-byte units per (channel, stage) descriptor slot
    int boxrows;              // rows per TMA box (cc*H*W = boxrows * copies)
    int nbuf;                 // ring depth
    int slot_bytes;           // bytes of one ring slot (inputs + descriptors)
    ActQuant aq;
    QuantAux q;               // f16 kernels: codebook / scales of the in-register weight decode
    uint32_t flags;
    int h, w;                 // plane (k_tile: the 4x4 tile grid)
};

// U > 1: every class segment is padded by the host to a multiple of U taps with
// no-op taps {v = -0.0, input = a zero row} (-0 * +0 = -0 and o + (-0) = o for
// every o, so exact), and the tap loop runs U taps per iteration with no remainder.
// NB consecutive floats (a lane's images) from shared memory in one vector load
template <int NB>
__device__ __forceinline__ void lds_nb(const unsigned char* p, float (&v)[NB]) {
    if constexpr (NB == 1) {
        v[0] = *reinterpret_cast<const float*>(p);
    } else if constexpr (NB == 2) {
        const float2 t = *reinterpret_cast<const float2*>(p);
        v[0] = t.x; v[1] = t.y;
    } else {
        static_assert(NB == 4, "images per lane");
        const float4 t = *reinterpret_cast<const float4*>(p);
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    }
}

// NB consecutive halves (a lane's images, f16 storage) in one vector load
template <int NB>
__device__ __forceinline__ void lds_nb(const unsigned char* p, unsigned short (&v)[NB]) {
    if constexpr (NB == 2) {
        const unsigned t = *reinterpret_cast<const unsigned*>(p);
        v[0] = (unsigned short)(t & 0xffffu); v[1] = (unsigned short)(t >> 16);
    } else {
        static_assert(NB == 4, "f16 images per lane");
        const uint2 t = *reinterpret_cast<const uint2*>(p);
        v[0] = (unsigned short)(t.x & 0xffffu); v[1] = (unsigned short)(t.x >> 16);
        v[2] = (unsigned short)(t.y & 0xffffu); v[3] = (unsigned short)(t.y >> 16);
    }
}

// f16 store of NB images (rounded to nearest even, like astype(f16))
template <int NB>
__device__ __forceinline__ void store_nb(__half* y, const float (&o)[NB], int nvalid, bool vec) {
    if constexpr (NB == 2) {
        if (vec && nvalid >= 2) { *reinterpret_cast<__half2*>(y) = __floats2half2_rn(o[0], o[1]); return; }
    } else if constexpr (NB == 4) {
        if (vec && nvalid >= 4) {
            const __half2 a = __floats2half2_rn(o[0], o[1]), b = __floats2half2_rn(o[2], o[3]);
            uint2 t;
            t.x = *reinterpret_cast<const unsigned*>(&a);
            t.y = *reinterpret_cast<const unsigned*>(&b);
            *reinterpret_cast<uint2*>(y) = t;
            return;
        }
    }
#pragma unroll
    for (int j = 0; j < NB; ++j)
        if (j < nvalid) y[j] = __float2half_rn(o[j]);
}

// NCHW store of a lane's NB images of output (k, position q): y[(n*K + k)*PLANE + q]
template <int NB, typename T>
__device__ __forceinline__ void store_nchw(T* y, int K, int plane, int k, int q, int nfirst, int n, const float (&o)[NB]) {
#pragma unroll
    for (int j = 0; j < NB; ++j)
        if (nfirst + j < n) y[((size_t)(nfirst + j) * K + k) * plane + q] = T(o[j]);
}

// store a lane's NB consecutive images (nvalid of them exist), one vector store when allowed
template <int NB>
__device__ __forceinline__ void store_nb(float* y, const float (&o)[NB], int nvalid, bool vec) {
    if constexpr (NB == 2) {
        if (vec && nvalid >= 2) { *reinterpret_cast<float2*>(y) = make_float2(o[0], o[1]); return; }
    } else if constexpr (NB == 4) {
        if (vec && nvalid >= 4) { *reinterpret_cast<float4*>(y) = make_float4(o[0], o[1], o[2], o[3]); return; }
    }
#pragma unroll
    for (int j = 0; j < NB; ++j)
        if (j < nvalid) y[j] = o[j];
}

// thread limit: 16 consumer warps + the producer; 8 + 1 for 8x8 planes (64 accumulators per lane)
template <int H, int W, int CS = 1>
constexpr int lane_max_threads() { return CS == 3 ? 768 : (CS > 1 ? 1024 : (H * W >= 64 ? 288 : 544)); }

// class index (cy * AX::N + cx) of output position q of an H x W plane
template <int H, int W>
__host__ __device__ constexpr int lane_class_of(int q) {
    return (q / W == 0 ? 0 : (q / W == H - 1 && H > 1 ? LaneAxis<H>::N - 1 : (H <= 2 ? q / W : 1))) * LaneAxis<W>::N +
           (q % W == 0 ? 0 : (q % W == W - 1 && W > 1 ? LaneAxis<W>::N - 1 : (W <= 2 ? q % W : 1)));
}
// class split: group of class ci when CS warps share an output channel (balanced MACs):
// 4x4 (CS = 2) -- {interior, top edge, top-left corner} | {other edges and corners};
// 2x2 -- CS = 2: rows, CS = 4: one position each
// 4x4 (CS = 3) -- {interior} | {top, bottom edges, TL, BR corners} | {left, right edges, TR, BL}
template <int H, int W, int CS>
__host__ __device__ constexpr int lane_class_group(int ci) {
    static_assert(CS == 1 || CS == 2 || (CS == 3 && H == 4 && W == 4) ||
                      (CS == 4 && ((H == 2 && W == 2) || (H == 8 && W == 8))),
                  "class split");
    return CS == 1 || H == 8 ? 0
           : H == 2          ? ci * CS / 4
           : CS == 3         ? (ci == 4 ? 0 : ((ci == 1 || ci == 7 || ci == 0 || ci == 8) ? 1 : 2))
                             : ((ci == 4 || ci == 1 || ci == 0) ? 0 : 1);
}
// 8x8 planes split by QUADRANT instead (CS = 4): group G owns rows / columns [lo, hi] of
// its 4x4 quadrant (every class list is shared; a warp covers class positions in its window)
// TQ = 1: the CTA owns one quadrant (a 4x4 output tile) of an 8x8 plane and stages only its
// 5x5 input window (4D TMA box), one warp per output channel -- group G = the CTA's quadrant
template <int H, int W, int CS, int TQ = 0>
__host__ __device__ constexpr bool lane_quadrants() { return H == 8 && W == 8 && (CS == 4 || TQ); }
template <int H, int W, int CS, int TQ = 0>
__host__ __device__ constexpr int lane_win_y0(int g) { return lane_quadrants<H, W, CS, TQ>() ? 4 * (g / 2) : 0; }
template <int H, int W, int CS, int TQ = 0>
__host__ __device__ constexpr int lane_win_x0(int g) { return lane_quadrants<H, W, CS, TQ>() ? 4 * (g % 2) : 0; }
template <int H, int W, int CS, int TQ = 0>
__host__ __device__ constexpr int lane_win_y1(int g) { return lane_quadrants<H, W, CS, TQ>() ? 4 * (g / 2) + 3 : H - 1; }
template <int H, int W, int CS, int TQ = 0>
__host__ __device__ constexpr int lane_win_x1(int g) { return lane_quadrants<H, W, CS, TQ>() ? 4 * (g % 2) + 3 : W - 1; }
// group owning output position (y, x)
template <int H, int W, int CS, int TQ = 0>
__host__ __device__ constexpr int lane_pos_group(int y, int x) {
    return lane_quadrants<H, W, CS, TQ>() ? 2 * (y / 4) + x / 4
                                           : lane_class_group<H, W, CS>(lane_class_of<H, W>(y * W + x));
}
// largest position set a tap's loads cover at once (bigger classes run in row chunks)
constexpr int LANE_PMAX = 16;
#ifndef LANE_UNROLL
#define LANE_UNROLL 4
#endif
constexpr int kLaneUnroll = LANE_UNROLL;  // tap-loop unroll of the U = 1 kernels
#ifndef TILE_UNROLL
#define TILE_UNROLL 2
#endif
constexpr int kTileUnroll = TILE_UNROLL;  // tap-loop unroll of k_tile (~7-12 taps per stage)

// F16: f16 storage (x, y, weights; f32 accumulation by FHFMA -- f16 x f16 is exact in f32, so
// one fma.rn.f32.f16 per MAC equals the reference's f32 mul + add); WF = the weight format
// decoded in registers from the descriptor's 32-bit payload (kernels.cuh tap_f16).
template <int H, int W, int NB, int KW, int MODE, int U = 1, bool F16 = false, int WF = WF_F32, int CS = 1,
          int TQ = 0>
__global__ void __launch_bounds__(TQ ? 544 : lane_max_threads<H, W, CS>(), 1) k_lane(const __grid_constant__ LaneParams p) {
    static_assert(!TQ || (H == 8 && W == 8 && CS == 1 && U == 1), "quadrant tiles: 8x8 planes");
    static_assert(!F16 || U == 1, "f16: no padded no-op taps (a quantized payload has no -0.0)");
    using XT = typename std::conditional<F16, unsigned short, float>::type;  // staged operand
    using TIO = typename std::conditional<F16, __half, float>::type;         // stored output
    constexpr int HW = H * W;
    constexpr int BI = 32 * NB;   // images per CTA
    constexpr int ES = F16 ? 2 : 4;
    constexpr int RB = BI * ES;   // bytes of one (channel, position) row in shared memory
    using AY = LaneAxis<H>;
    using AX = LaneAxis<W>;
    extern __shared__ __align__(128) unsigned char smem[];

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int WK = p.warps, NBUF = p.nbuf;
    const int kg = blockIdx.x % p.kgroups;
    const int quad = TQ ? (blockIdx.x / p.kgroups) % 4 : 0;  // TQ: the CTA's output quadrant
    const int n0 = (blockIdx.x / p.kgroups / (TQ ? 4 : 1)) * BI;
    constexpr int SP = TQ ? 25 : H * W;  // staged input positions per channel (TQ: 5x5 window)
    const int KC = WK / CS * KW;  // output channels per CTA
    const int kbase = kg * KC;
    const int in_bytes = p.cc * SP * RB;
    __shared__ unsigned short cbt[16];  // WF_CB4 table (f16 bits), published by the barrier below
    if (F16 && tid < 16) cbt[tid] = p.q.cb16[tid];
    const float qscale = p.q.scale;
    const double qstep = p.q.step;
    const int d_bytes = in_bytes + (U > 1 ? HW * RB : 0);  // descriptors after inputs (+ zero rows)

    unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + (size_t)NBUF * p.slot_bytes);
    const unsigned full0 = smem_u32(bars), empty0 = smem_u32(bars + NBUF);
    if constexpr (U > 1) {  // zero rows read by the no-op taps (never written by the TMA)
        for (int b = 0; b < NBUF; ++b)
            for (int i = tid; i < HW * RB / 16; i += blockDim.x)
                reinterpret_cast<uint4*>(smem + (size_t)b * p.slot_bytes + in_bytes)[i] = make_uint4(0, 0, 0, 0);
    }
    if (tid == 0) {
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(full0 + 8 * b, 1);
            mbar_init(empty0 + 8 * b, WK);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == WK) {
        // ------------------------------------------------------------ producer
        asm volatile("griddepcontrol.wait;" ::: "memory");  // x is the previous kernel's output
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&p.tmap) : "memory");
            const int kn = min(KC, p.k - kbase);
            const unsigned dbytes = (unsigned)(kn * p.cap * 16);
            const int copies = p.cc * HW / p.boxrows;
            const unsigned tx = (unsigned)in_bytes + dbytes;
            for (int st = 0; st < p.nst; ++st) {
                const int buf = st % NBUF;
                if (st >= NBUF) mbar_wait(empty0 + 8 * buf, ((st / NBUF) - 1) & 1);
                const unsigned fb = full0 + 8 * buf;
                mbar_arrive_tx(fb, tx);
                const unsigned dst = smem_u32(smem + (size_t)buf * p.slot_bytes);
                if constexpr (TQ) {  // the quadrant's 5x5 input window of cc channels: one 4D box
                    asm volatile(
                        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
                        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst), "l"(&p.tmap), "r"(n0),
                        "r"((quad % 2) ? 3 : 0), "r"((quad / 2) ? 3 : 0), "r"(st * p.cc), "r"(fb)
                        : "memory");
                } else {
                for (int i = 0; i < copies; ++i)
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                        " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst + (unsigned)(i * p.boxrows * RB)),
                        "l"(&p.tmap), "r"(n0), "r"(st * p.cc * HW + i * p.boxrows), "r"(fb)
                        : "memory");
                }
                bulk_g2s(dst + (unsigned)d_bytes, p.desc + (((size_t)quad * p.nst + st) * p.k + kbase) * p.cap, dbytes, fb);
            }
        }
        return;
    }

    // -------------------------------------------------------------- consumers
    // CS = 2: two warps per output channel, each owning a fixed set of position classes
    // (lane_class_group) -- twice the warps for latency hiding, the same shared-memory traffic
    const int cq = warp / CS, cgrp = warp % CS;
    const int k0 = kbase + cq * KW;
    auto consume = [&](auto GC) {
    constexpr int G = decltype(GC)::value;
    float acc[KW][HW][NB];
    // MODE_HALF2 (f16 opt-in fast mode, the north star's "half2 FMA"): within a stage the lane's
    // image pairs accumulate in __half2 with one HFMA2 per two MACs; each stage's partial sums
    // are folded into the f32 accumulators (a whole 461-tap sum in f16 measured 0.043 off)
    constexpr bool H2 = F16 && MODE == MODE_HALF2;
    static_assert(!H2 || NB % 2 == 0, "half2 accumulators pair a lane's images");
    __half2 acc2[KW][HW][H2 ? NB / 2 : 1];
#pragma unroll
    for (int kk = 0; kk < KW; ++kk) {
        const int k = k0 + kk;
        const float b = (p.bias != nullptr && k < p.k) ? p.bias[k] : 0.f;
#pragma unroll
        for (int q = 0; q < HW; ++q)
#pragma unroll
            for (int j = 0; j < NB; ++j) acc[kk][q][j] = b;
        if constexpr (H2) {
#pragma unroll
            for (int q = 0; q < HW; ++q)
#pragma unroll
                for (int j = 0; j < NB / 2; ++j) acc2[kk][q][j] = __float2half2_rn(0.f);
        }
    }
    for (int st = 0; st < p.nst; ++st) {
        const int buf = st % NBUF;
        mbar_wait(full0 + 8 * buf, (st / NBUF) & 1);
        const unsigned char* slot = smem + (size_t)buf * p.slot_bytes;
        const unsigned char* xin = slot + lane * ES * NB;  // lane's images n0 + NB*lane + j
#pragma unroll
        for (int kk = 0; kk < KW; ++kk) {
            if (k0 + kk >= p.k) break;
            const unsigned char* ch = slot + d_bytes + (size_t)(cq * KW + kk) * p.cap * 16;
            unsigned short hd[LANE_HDR / 2];  // cumulative class ends, two 16-byte loads
            *reinterpret_cast<uint4*>(hd) = *reinterpret_cast<const uint4*>(ch);
            *reinterpret_cast<uint4*>(hd + 8) = *reinterpret_cast<const uint4*>(ch + 16);
            const LaneTap* tp = reinterpret_cast<const LaneTap*>(ch + LANE_HDR);
            LaneTap dn = tp[0];  // running prefetch over the slot's contiguous class lists
            int beg = 0;
#pragma unroll
            for (int cy = 0; cy < AY::N; ++cy) {
#pragma unroll
                for (int cx = 0; cx < AX::N; ++cx) {
                    const int y0 = AY::lo(cy), y1 = AY::hi(cy), x0 = AX::lo(cx), x1 = AX::hi(cx);
                    const int end = hd[cy * AX::N + cx];
                    // this warp's positions of the class: the class range inside the group window
                    const int ey0 = y0 > lane_win_y0<H, W, CS, TQ>(G) ? y0 : lane_win_y0<H, W, CS, TQ>(G);
                    const int ey1 = y1 < lane_win_y1<H, W, CS, TQ>(G) ? y1 : lane_win_y1<H, W, CS, TQ>(G);
                    const int ex0 = x0 > lane_win_x0<H, W, CS, TQ>(G) ? x0 : lane_win_x0<H, W, CS, TQ>(G);
                    const int ex1 = x1 < lane_win_x1<H, W, CS, TQ>(G) ? x1 : lane_win_x1<H, W, CS, TQ>(G);
                    const bool mine = lane_quadrants<H, W, CS, TQ>() || lane_class_group<H, W, CS>(cy * AX::N + cx) == G;
                    if (!mine || ey0 > ey1 || ex0 > ex1) {  // another warp's class / no position in the window
                        beg = end;
                        continue;
                    }
                    if constexpr (U == 1) {
                        const int rc = LANE_PMAX / (ex1 - ex0 + 1) > 0 ? LANE_PMAX / (ex1 - ex0 + 1) : 1;  // rows per chunk
#pragma unroll
                        for (int ya = ey0; ya <= ey1; ya += rc) {
                            const int yb = ya + rc - 1 < ey1 ? ya + rc - 1 : ey1;
                            // one tap: vector loads of the class positions' inputs, then the MACs
                            auto tap = [&](const LaneTap& d) {
                                const unsigned char* xa = xin + d.off;
                                if constexpr (H2) {  // one HFMA2 per image pair and position
                                    const unsigned short vh = tap_f16<WF>(__float_as_uint(d.v), cbt, qscale, qstep);
                                    const __half2 v2 = __half2half2(__ushort_as_half(vh));
#pragma unroll
                                    for (int yy = ya; yy <= yb; ++yy)
#pragma unroll
                                        for (int xx = ex0; xx <= ex1; ++xx) {
                                            __half2 xh[NB / 2];
                                            if constexpr (NB == 2) {
                                                xh[0] = *reinterpret_cast<const __half2*>(xa + ((yy - y0) * W + (xx - x0)) * RB);
                                            } else {
                                                const uint2 t = *reinterpret_cast<const uint2*>(xa + ((yy - y0) * W + (xx - x0)) * RB);
                                                xh[0] = *reinterpret_cast<const __half2*>(&t.x);
                                                xh[1] = *reinterpret_cast<const __half2*>(&t.y);
                                            }
#pragma unroll
                                            for (int j = 0; j < NB / 2; ++j)
                                                acc2[kk][yy * W + xx][j] = __hfma2(v2, xh[j], acc2[kk][yy * W + xx][j]);
                                        }
                                    return;
                                }
                                XT xv[HW][NB];
                                unsigned short vh = 0;
                                if constexpr (F16) vh = tap_f16<WF>(__float_as_uint(d.v), cbt, qscale, qstep);
#pragma unroll
                                for (int yy = ya; yy <= yb; ++yy)
#pragma unroll
                                    for (int xx = ex0; xx <= ex1; ++xx)
                                        lds_nb<NB>(xa + (TQ ? (yy - ey0) * 5 + (xx - ex0) : (yy - y0) * W + (xx - x0)) * RB,
                                                   xv[(yy - y0) * W + xx - x0]);
#pragma unroll
                                for (int yy = ya; yy <= yb; ++yy)
#pragma unroll
                                    for (int xx = ex0; xx <= ex1; ++xx)
#pragma unroll
                                        for (int j = 0; j < NB; ++j) {
                                            if constexpr (F16)
                                                acc[kk][yy * W + xx][j] =
                                                    fhfma(acc[kk][yy * W + xx][j], vh, xv[(yy - y0) * W + xx - x0][j]);
                                            else
                                                acc[kk][yy * W + xx][j] =
                                                    mac1<MODE>(acc[kk][yy * W + xx][j], d.v, xv[(yy - y0) * W + xx - x0][j]);
                                        }
                            };
                            LaneTap dq = (ya == ey0 && CS == 1) ? dn : tp[beg];
#pragma unroll kLaneUnroll
                            for (int t = beg; t < end; ++t) {
                                const LaneTap d = dq;
                                dq = tp[t + 1];  // (one past the slot's last tap: slack, never used)
                                tap(d);
                            }
                            if (ya + rc > ey1) dn = dq;  // = tp[end]: the next class's first tap
                        }
                    } else {
                        for (int t = beg; t < end; t += U) {
                            LaneTap d[U];
#pragma unroll
                            for (int u = 0; u < U; u += 2) {
                                const float4 q = *reinterpret_cast<const float4*>(tp + t + u);
                                d[u].v = q.x;
                                d[u].off = __float_as_int(q.y);
                                d[u + 1].v = q.z;
                                d[u + 1].off = __float_as_int(q.w);
                            }
                            XT xv[U][HW][NB];
#pragma unroll
                            for (int u = 0; u < U; ++u)
#pragma unroll
                                for (int yy = y0; yy <= y1; ++yy)
#pragma unroll
                                    for (int xx = x0; xx <= x1; ++xx)
                                        lds_nb<NB>(xin + d[u].off + ((yy - y0) * W + (xx - x0)) * RB,
                                                   xv[u][(yy - y0) * W + xx - x0]);
#pragma unroll
                            for (int u = 0; u < U; ++u)
#pragma unroll
                                for (int yy = y0; yy <= y1; ++yy)
#pragma unroll
                                    for (int xx = x0; xx <= x1; ++xx)
#pragma unroll
                                        for (int j = 0; j < NB; ++j)
                                            if constexpr (!F16)
                                                acc[kk][yy * W + xx][j] = mac1<MODE>(
                                                    acc[kk][yy * W + xx][j], d[u].v, xv[u][(yy - y0) * W + xx - x0][j]);
                        }
                    }
                    beg = end;
                }
            }
        }
        if constexpr (H2) {  // fold the stage's half2 partial sums into the f32 accumulators
#pragma unroll
            for (int kk = 0; kk < KW; ++kk)
#pragma unroll
                for (int q = 0; q < HW; ++q) {
                    if (lane_pos_group<H, W, CS, TQ>(q / W, q % W) != G) continue;
#pragma unroll
                    for (int j = 0; j < NB / 2; ++j) {
                        const float2 f = __half22float2(acc2[kk][q][j]);
                        acc[kk][q][2 * j] += f.x;
                        acc[kk][q][2 * j + 1] += f.y;
                        acc2[kk][q][j] = __float2half2_rn(0.f);
                    }
                }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8 * buf);
    }

    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // ---- epilogue: lane holds the whole plane (its class group's positions) of images n0 + NB*lane + j
    const bool aq = p.flags & SCB_FLAG_ACT_QUANT;
    const bool relu = (p.flags & SCB_FLAG_RELU) && !aq;
    const bool pool = p.flags & SCB_FLAG_POOL2;
    // vector stores when every row start is NB-element aligned (row stride and base)
    const bool vec = (p.ldy % NB) == 0 && (reinterpret_cast<uintptr_t>(p.y) % (ES * NB)) == 0;
    const bool ynchw = p.flags & SCB_FLAG_Y_NCHW;  // NCHW output (the last layer of an image-minor run)
#pragma unroll
    for (int kk = 0; kk < KW; ++kk) {
        const int k = k0 + kk;
        const uint32_t zm = k < p.k ? p.zmask[k] : 0u;
#pragma unroll
        for (int cy = 0; cy < AY::N; ++cy)
#pragma unroll
            for (int cx = 0; cx < AX::N; ++cx) {
#pragma unroll
                for (int yy = AY::lo(cy); yy <= AY::hi(cy); ++yy)
#pragma unroll
                    for (int xx = AX::lo(cx); xx <= AX::hi(cx); ++xx)
#pragma unroll
                        for (int j = 0; j < NB; ++j) {
                            if (lane_pos_group<H, W, CS, TQ>(yy, xx) != G) continue;
                            float& o = acc[kk][yy * W + xx][j];
                            if (__float_as_uint(o) == 0x80000000u && ((zm >> (cy * AX::N + cx)) & 1u)) o = 0.f;
                            if (aq) o = fq_store<TIO>((p.flags & SCB_FLAG_RELU) ? relu_io<TIO>(o) : o, p.aq);
                            if (relu && !pool) o = relu_io<TIO>(o);
                        }
            }
        if (!pool) {
            if (k >= p.k) continue;
            TIO* yp = static_cast<TIO*>(p.y) + (size_t)k * HW * p.ldy + n0 + NB * lane;
#pragma unroll
            for (int q = 0; q < HW; ++q) {
                if (lane_pos_group<H, W, CS, TQ>(q / W, q % W) != G) continue;
                float o[NB];
#pragma unroll
                for (int j = 0; j < NB; ++j) o[j] = acc[kk][q][j];
                if (ynchw) store_nchw<NB>(static_cast<TIO*>(p.y), p.k, HW, k, q, n0 + NB * lane, p.n, o);
                else store_nb<NB>(yp + (size_t)q * p.ldy, o, p.n - (n0 + NB * lane), vec);
            }
        }
    }
    if (pool) {
        constexpr int PW = W / 2, PHW = (H / 2) * (W / 2);
        float* ex = reinterpret_cast<float*>(smem);  // CS = 2: [channel][position][image] exchange
        if constexpr (CS > 1) {
            asm volatile("bar.sync 1, %0;" ::"r"(WK * 32) : "memory");  // every warp is past the ring
#pragma unroll
            for (int q = 0; q < HW; ++q) {
                if (lane_pos_group<H, W, CS, TQ>(q / W, q % W) != G) continue;
#pragma unroll
                for (int j = 0; j < NB; ++j) ex[((size_t)cq * HW + q) * BI + NB * lane + j] = acc[0][q][j];
            }
            asm volatile("bar.sync 1, %0;" ::"r"(WK * 32) : "memory");
        }
#pragma unroll
        for (int kk = 0; kk < KW; ++kk) {
            const int k = k0 + kk;
            if (k >= p.k) break;
            TIO* yp = static_cast<TIO*>(p.y) + (size_t)k * PHW * p.ldy + n0 + NB * lane;
#pragma unroll
            for (int py = 0; py < H / 2; ++py)
#pragma unroll
                for (int px = 0; px < PW; ++px) {
                    if (CS > 1 && (py * PW + px) % CS != G) continue;  // pooled outputs dealt over the group
                    if (TQ && lane_pos_group<H, W, CS, TQ>(2 * py, 2 * px) != G) continue;  // other quadrants
                    float o[NB];
#pragma unroll
                    for (int j = 0; j < NB; ++j) {
                        const int a = (2 * py) * W + 2 * px;
                        float v[4];
                        if constexpr (CS > 1) {
                            const float* e = ex + (size_t)cq * HW * BI + NB * lane + j;
                            v[0] = e[(size_t)a * BI]; v[1] = e[(size_t)(a + 1) * BI];
                            v[2] = e[(size_t)(a + W) * BI]; v[3] = e[(size_t)(a + W + 1) * BI];
                        } else {
                            v[0] = acc[kk][a][j]; v[1] = acc[kk][a + 1][j];
                            v[2] = acc[kk][a + W][j]; v[3] = acc[kk][a + W + 1][j];
                        }
                        o[j] = fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3]));
                        if (relu) o[j] = relu_io<TIO>(o[j]);
                    }
                    if (ynchw) store_nchw<NB>(static_cast<TIO*>(p.y), p.k, PHW, k, py * PW + px, n0 + NB * lane, p.n, o);
                    else store_nb<NB>(yp + (size_t)(py * PW + px) * p.ldy, o, p.n - (n0 + NB * lane), vec);
                }
        }
    }
    };  // consume
    const int grp = TQ ? quad : cgrp;
    if (grp == 0) consume(std::integral_constant<int, 0>{});
    else if constexpr (TQ) {
        if (grp == 1) consume(std::integral_constant<int, 1>{});
        else if (grp == 2) consume(std::integral_constant<int, 2>{});
        else consume(std::integral_constant<int, 3>{});
    }
    else if constexpr (CS == 2) consume(std::integral_constant<int, 1>{});
    else if constexpr (CS == 3) {
        if (cgrp == 1) consume(std::integral_constant<int, 1>{});
        else consume(std::integral_constant<int, 2>{});
    }
    else if constexpr (CS == 4) {
        if (cgrp == 1) consume(std::integral_constant<int, 1>{});
        else if (cgrp == 2) consume(std::integral_constant<int, 2>{});
        else consume(std::integral_constant<int, 3>{});
    }
}

template <int H, int W, int NB, int KW, int MODE, int U = 1, bool F16 = false, int WF = WF_F32, int CS = 1,
          int TQ = 0>
cudaError_t launch_lane_t(const LaneParams& p, unsigned grid, unsigned threads, size_t smem, cudaStream_t st) {
    auto kern = k_lane<H, W, NB, KW, MODE, U, F16, WF, CS, TQ>;
    static int lim[64];  // per device
    const cudaError_t e = dyn_smem_ok(kern, smem, lim);
    if (e != cudaSuccess) return e;
    return launch_pdl(kern, p, grid, threads, smem, st);
}

// ---------------------------------------------------- 4x4 output tiles of larger planes
// Dispatch 4 (16x16 / 32x32 planes: VGG conv1_x / conv2_x): a CTA owns one 4x4 output tile
// of 32*NB images and stages, per channel, the tile's 6x6 input window -- one 4D TMA box
// {images, 6, 6, cc} whose rows / columns outside the plane the TMA zero-fills, i.e. the
// reference's zero padding (shapes.py:98-105).  Every tile position sees every tap inside
// its window, so one tap list per (stage, channel) serves all tiles: the CSR row in colidx
// order with the padding taps KEPT -- the MACs are exactly the reference's
// (_kernels.py:73-84, o = o + v*x with x = +0 in the padding), no zmask fix-up, and the
// ~8 % (16x16) / ~4 % (32x32) padding MACs are the price of a class-free tile.  Lane =
// image, 16*NB accumulators per lane, per tap one broadcast descriptor then 16
// conflict-free vector loads and 16*NB MACs; the ring / producer are k_lane's.
// thread limit (consumer warps + the producer): room for 16*NB accumulators + 16*NB operands
constexpr int tile_max_threads(int nb) { return nb == 1 ? 544 : (nb == 2 ? 416 : 288); }
template <int NB, int MODE, bool F16 = false, int WF = WF_F32>
__global__ void __launch_bounds__(tile_max_threads(NB), 1) k_tile(const __grid_constant__ LaneParams p) {
    static_assert(!F16 || NB >= 2, "f16: two images per 32-bit load");
    static_assert(MODE != MODE_HALF2, "tiles: exact / FMA accumulation only");
    using XT = typename std::conditional<F16, unsigned short, float>::type;
    using TIO = typename std::conditional<F16, __half, float>::type;
    constexpr int BI = 32 * NB, ES = F16 ? 2 : 4, RB = BI * ES, SP = 36;
    extern __shared__ __align__(128) unsigned char smem[];

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int WK = p.warps, NBUF = p.nbuf;
    const int ntx = p.w / 4, ntiles = (p.h / 4) * ntx;
    const int kg = blockIdx.x % p.kgroups;
    const int tile = (blockIdx.x / p.kgroups) % ntiles;
    const int n0 = (blockIdx.x / p.kgroups / ntiles) * BI;
    const int ty0 = 4 * (tile / ntx), tx0 = 4 * (tile % ntx);
    const int kbase = kg * WK;
    const int in_bytes = p.cc * SP * RB;
    __shared__ unsigned short cbt[16];
    if (F16 && tid < 16) cbt[tid] = p.q.cb16[tid];
    const float qscale = p.q.scale;
    const double qstep = p.q.step;

    unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + (size_t)NBUF * p.slot_bytes);
    const unsigned full0 = smem_u32(bars), empty0 = smem_u32(bars + NBUF);
    if (tid == 0) {
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(full0 + 8 * b, 1);
            mbar_init(empty0 + 8 * b, WK);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == WK) {  // producer: the 6x6 window of cc channels + the CTA's descriptor slots
        asm volatile("griddepcontrol.wait;" ::: "memory");
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&p.tmap) : "memory");
            const int kn = min(WK, p.k - kbase);
            const unsigned dbytes = (unsigned)(kn * p.cap * 16);
            for (int st = 0; st < p.nst; ++st) {
                const int buf = st % NBUF;
                if (st >= NBUF) mbar_wait(empty0 + 8 * buf, ((st / NBUF) - 1) & 1);
                const unsigned fb = full0 + 8 * buf;
                mbar_arrive_tx(fb, (unsigned)in_bytes + dbytes);
                const unsigned dst = smem_u32(smem + (size_t)buf * p.slot_bytes);
                asm volatile(
                    "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst), "l"(&p.tmap), "r"(n0), "r"(tx0 - 1),
                    "r"(ty0 - 1), "r"(st * p.cc), "r"(fb)
                    : "memory");
                bulk_g2s(dst + (unsigned)in_bytes, p.desc + ((size_t)st * p.k + kbase) * p.cap, dbytes, fb);
            }
        }
        return;
    }

    const int k = kbase + warp;
    float acc[16][NB];
    {
        const float b = (p.bias != nullptr && k < p.k) ? p.bias[k] : 0.f;
#pragma unroll
        for (int q = 0; q < 16; ++q)
#pragma unroll
            for (int j = 0; j < NB; ++j) acc[q][j] = b;
    }
    for (int st = 0; st < p.nst; ++st) {
        const int buf = st % NBUF;
        mbar_wait(full0 + 8 * buf, (st / NBUF) & 1);
        const unsigned char* slot = smem + (size_t)buf * p.slot_bytes;
        const unsigned char* xin = slot + lane * ES * NB;
        if (k < p.k) {
            const unsigned char* ch = slot + in_bytes + (size_t)warp * p.cap * 16;
            const int cnt = *reinterpret_cast<const int*>(ch);
            const LaneTap* tp = reinterpret_cast<const LaneTap*>(ch + LANE_HDR);
            LaneTap dq = tp[0];
#pragma unroll kTileUnroll
            for (int t = 0; t < cnt; ++t) {
                const LaneTap d = dq;
                dq = tp[t + 1];  // (one past the slot's last tap: slack, never used)
                const unsigned char* xa = xin + d.off;
                XT xv[16][NB];
#pragma unroll
                for (int q = 0; q < 16; ++q) lds_nb<NB>(xa + ((q / 4) * 6 + q % 4) * RB, xv[q]);
                if constexpr (F16) {
                    const unsigned short vh = tap_f16<WF>(__float_as_uint(d.v), cbt, qscale, qstep);
#pragma unroll
                    for (int q = 0; q < 16; ++q)
#pragma unroll
                        for (int j = 0; j < NB; ++j) acc[q][j] = fhfma(acc[q][j], vh, xv[q][j]);
                } else {
#pragma unroll
                    for (int q = 0; q < 16; ++q)
#pragma unroll
                        for (int j = 0; j < NB; ++j) acc[q][j] = mac1<MODE>(acc[q][j], d.v, xv[q][j]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8 * buf);
    }

    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (k >= p.k) return;
    const bool aq = p.flags & SCB_FLAG_ACT_QUANT;
    const bool relu = (p.flags & SCB_FLAG_RELU) && !aq;
    const bool pool = p.flags & SCB_FLAG_POOL2;
    const bool vec = (p.ldy % NB) == 0 && (reinterpret_cast<uintptr_t>(p.y) % (ES * NB)) == 0;
    const bool ynchw = p.flags & SCB_FLAG_Y_NCHW;
#pragma unroll
    for (int q = 0; q < 16; ++q)
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            float& o = acc[q][j];
            if (aq) o = fq_store<TIO>((p.flags & SCB_FLAG_RELU) ? relu_io<TIO>(o) : o, p.aq);
            if (relu && !pool) o = relu_io<TIO>(o);
        }
    const int nf = n0 + NB * lane;
    if (!pool) {
        const int HW = p.h * p.w;
        TIO* yp = static_cast<TIO*>(p.y) + (size_t)k * HW * p.ldy + nf;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const int pos = (ty0 + q / 4) * p.w + tx0 + q % 4;
            if (ynchw) store_nchw<NB>(static_cast<TIO*>(p.y), p.k, HW, k, pos, nf, p.n, acc[q]);
            else store_nb<NB>(yp + (size_t)pos * p.ldy, acc[q], p.n - nf, vec);
        }
    } else {
        const int PW = p.w / 2, PHW = (p.h / 2) * PW;
        TIO* yp = static_cast<TIO*>(p.y) + (size_t)k * PHW * p.ldy + nf;
#pragma unroll
        for (int py = 0; py < 2; ++py)
#pragma unroll
            for (int px = 0; px < 2; ++px) {
                const int a = 2 * py * 4 + 2 * px;
                float o[NB];
#pragma unroll
                for (int j = 0; j < NB; ++j) {
                    o[j] = fmaxf(fmaxf(acc[a][j], acc[a + 1][j]), fmaxf(acc[a + 4][j], acc[a + 5][j]));
                    if (relu) o[j] = relu_io<TIO>(o[j]);
                }
                const int pos = (ty0 / 2 + py) * PW + tx0 / 2 + px;
                if (ynchw) store_nchw<NB>(static_cast<TIO*>(p.y), p.k, PHW, k, pos, nf, p.n, o);
                else store_nb<NB>(yp + (size_t)pos * p.ldy, o, p.n - nf, vec);
            }
    }
}

template <int NB, int MODE, bool F16 = false, int WF = WF_F32>
cudaError_t launch_tile_t(const LaneParams& p, unsigned grid, unsigned threads, size_t smem, cudaStream_t st) {
    auto kern = k_tile<NB, MODE, F16, WF>;
    static int lim[64];  // per device
    const cudaError_t e = dyn_smem_ok(kern, smem, lim);
    if (e != cudaSuccess) return e;
    return launch_pdl(kern, p, grid, threads, smem, st);
}

// ---------------------------------------------------------------- host side
// Tap program of a kind-7 launch: per (stage st, output channel k) one slot of
// `cap` 16-byte units = LANE_HDR bytes of cumulative class ends + the class tap
// lists, each in the CSR row's colidx order with the taps that fall into the
// zero padding for that class removed.  Slots are laid out [st][k] so a CTA's
// consecutive channels of a stage are one contiguous bulk copy.  R = S = 3,
// pad 1, stride 1 (H x W output = input plane).
struct LaneProgram {
    std::vector<uint4> desc;     // [nst][K][cap]
    std::vector<uint32_t> zmask; // [K]
    int cap = 0;                 // units per slot
    int nst = 0;
    int64_t macs = 0;            // executed MACs per image (in-image taps x class positions)
};

inline int lane_axis_n(int h) { return h == 1 ? 1 : (h == 2 ? 2 : 3); }
inline int lane_axis_lo(int h, int i) { return h <= 2 ? i : (i == 0 ? 0 : (i == 1 ? 1 : h - 1)); }
inline int lane_axis_hi(int h, int i) { return h <= 2 ? i : (i == 0 ? 0 : (i == 1 ? h - 2 : h - 1)); }

// vbits: f32 bit patterns of the CSR values; colidx = c*pp + r*wp + s, the reference's
// column index into the padded input plane (csr.py:143-160; pp = Hp*Wp, wp = Wp).
// u > 1: pad every class segment to a multiple of u with no-op taps {-0.0, zero row}.
// count_only: cap / zmask / macs only (no descriptor array; the launch-shape check).
// es: bytes per staged element (4 f32, 2 f16); vbits then holds the f16 kernels' 32-bit
// payloads (f16 bits / quantized code), whose sign for the -0.0 mask is `sign`.
inline bool build_lane_program(const uint32_t* vbits, const int32_t* colidx, const int32_t* rowptr, int C, int K,
                               int64_t pp, int wp, int H, int W, int cc, int nb, LaneProgram* out, int u = 1,
                               bool count_only = false, int es = 4, const uint8_t* sign = nullptr) {
    const int HW = H * W, RB = 32 * nb * es;
    const int nst = (C + cc - 1) / cc;
    const int ny = lane_axis_n(H), nx = lane_axis_n(W), ncls = ny * nx;
    if (ncls > LANE_HDR / 2 || cc < 1) return false;
    LaneProgram& P = *out;
    P.zmask.assign(K, 0u);
    P.nst = nst;
    P.macs = 0;
    P.desc.clear();
    uint32_t mz = 0x80000000u;
    float negzero;
    std::memcpy(&negzero, &mz, 4);
    // walk the (k, st) slot: fn(class, tap) for every kept tap (and padding no-ops), returns count
    std::vector<LaneTap> taps;
    uint16_t ends[LANE_HDR / 2];
    auto slot = [&](int k, int st, int t0, int t1, bool account) {
        taps.clear();
        std::fill(ends, ends + LANE_HDR / 2, (uint16_t)0);
        for (int cy = 0; cy < ny; ++cy)
            for (int cx = 0; cx < nx; ++cx) {
                const int y0 = lane_axis_lo(H, cy), x0 = lane_axis_lo(W, cx);
                const int npos = (lane_axis_hi(H, cy) - y0 + 1) * (lane_axis_hi(W, cx) - x0 + 1);
                const size_t seg0 = taps.size();
                for (int i = t0; i < t1; ++i) {
                    const int64_t ci = colidx[i] / pp, rem = colidx[i] % pp;
                    const int r = (int)(rem / wp), s = (int)(rem % wp);
                    const int iy = y0 + r - 1, ix = x0 + s - 1;
                    if (iy < 0 || iy >= H || ix < 0 || ix >= W) {  // padding tap of this class
                        const bool neg = sign ? sign[i] != 0 : (vbits[i] & 0x80000000u) != 0;
                        if (account && !neg) P.zmask[k] |= 1u << (cy * nx + cx);
                        continue;
                    }
                    LaneTap d;
                    std::memcpy(&d.v, &vbits[i], 4);
                    d.off = (int32_t)((((ci - (int64_t)st * cc) * HW) + iy * W + ix) * RB);
                    taps.push_back(d);
                    if (account) P.macs += npos;
                }
                while (u > 1 && (taps.size() - seg0) % u) taps.push_back(LaneTap{negzero, cc * HW * RB});
                ends[cy * nx + cx] = (uint16_t)taps.size();
            }
    };
    // pass 1: the largest slot; pass 2: the padded [st][k][cap] layout
    std::vector<int32_t> tstart((size_t)K * (nst + 1));
    int maxt = 0;
    for (int k = 0; k < K; ++k) {
        int t = rowptr[k];
        for (int st = 0; st < nst; ++st) {
            tstart[(size_t)k * (nst + 1) + st] = t;
            const int64_t cend = std::min<int64_t>(C, (int64_t)(st + 1) * cc);
            while (t < rowptr[k + 1] && colidx[t] / pp < cend) ++t;
        }
        tstart[(size_t)k * (nst + 1) + nst] = t;
        for (int st = 0; st < nst; ++st) {
            slot(k, st, tstart[(size_t)k * (nst + 1) + st], tstart[(size_t)k * (nst + 1) + st + 1], true);
            maxt = std::max(maxt, (int)taps.size());
        }
    }
    if (maxt > 0xffff) return false;
    P.cap = (LANE_HDR + maxt * 8 + 15) / 16;
    if (count_only) return true;
    P.desc.assign((size_t)nst * K * P.cap, make_uint4(0, 0, 0, 0));
    for (int k = 0; k < K; ++k)
        for (int st = 0; st < nst; ++st) {
            slot(k, st, tstart[(size_t)k * (nst + 1) + st], tstart[(size_t)k * (nst + 1) + st + 1], false);
            unsigned char* b = reinterpret_cast<unsigned char*>(P.desc.data() + ((size_t)st * K + k) * P.cap);
            std::memcpy(b, ends, LANE_HDR);
            if (!taps.empty()) std::memcpy(b + LANE_HDR, taps.data(), taps.size() * 8);
        }
    return true;
}

// Tap program of the quadrant-tile mode (TQ): per quadrant q, stage st and channel k one slot
// ([q][st][k][cap]): the plane's class lists restricted to classes with positions in q, offsets
// of the input row of the class's first position IN q within q's 5x5 staged window.
inline bool build_lane_program_tq(const uint32_t* vbits, const int32_t* colidx, const int32_t* rowptr, int C,
                                  int K, int64_t pp, int wp, int cc, int nb, LaneProgram* out, bool count_only = false,
                                  int es = 4, const uint8_t* sign = nullptr) {
    const int H = 8, W = 8, RB = 32 * nb * es;
    const int nst = (C + cc - 1) / cc;
    LaneProgram& P = *out;
    P.zmask.assign(K, 0u);
    P.nst = nst;
    P.macs = 0;
    P.desc.clear();
    std::vector<int32_t> tstart((size_t)K * (nst + 1));
    for (int k = 0; k < K; ++k) {
        int t = rowptr[k];
        for (int st = 0; st < nst; ++st) {
            tstart[(size_t)k * (nst + 1) + st] = t;
            while (t < rowptr[k + 1] && colidx[t] / pp < std::min<int64_t>(C, (int64_t)(st + 1) * cc)) ++t;
        }
        tstart[(size_t)k * (nst + 1) + nst] = t;
    }
    std::vector<LaneTap> taps;
    uint16_t ends[LANE_HDR / 2];
    auto slot = [&](int q, int k, int st, bool account) {
        taps.clear();
        std::fill(ends, ends + LANE_HDR / 2, (uint16_t)0);
        const int qy0 = 4 * (q / 2), qx0 = 4 * (q % 2), wy0 = q / 2 ? 3 : 0, wx0 = q % 2 ? 3 : 0;
        for (int cy = 0; cy < 3; ++cy)
            for (int cx = 0; cx < 3; ++cx) {
                const int y0 = lane_axis_lo(H, cy), y1 = lane_axis_hi(H, cy);
                const int x0 = lane_axis_lo(W, cx), x1 = lane_axis_hi(W, cx);
                const int ey0 = std::max(y0, qy0), ey1 = std::min(y1, qy0 + 3);
                const int ex0 = std::max(x0, qx0), ex1 = std::min(x1, qx0 + 3);
                if (ey0 <= ey1 && ex0 <= ex1) {
                    for (int i = tstart[(size_t)k * (nst + 1) + st]; i < tstart[(size_t)k * (nst + 1) + st + 1]; ++i) {
                        const int64_t ci = colidx[i] / pp, rem = colidx[i] % pp;
                        const int r = (int)(rem / wp), s = (int)(rem % wp);
                        const int iy = y0 + r - 1, ix = x0 + s - 1;  // validity is a class property
                        if (iy < 0 || iy >= H || ix < 0 || ix >= W) {
                            const bool neg = sign ? sign[i] != 0 : (vbits[i] & 0x80000000u) != 0;
                            if (account && q == 0 && !neg) P.zmask[k] |= 1u << (cy * 3 + cx);
                            continue;
                        }
                        LaneTap d;
                        std::memcpy(&d.v, &vbits[i], 4);
                        d.off = (int32_t)((((ci - (int64_t)st * cc) * 25) + (ey0 + r - 1 - wy0) * 5 + (ex0 + s - 1 - wx0)) * RB);
                        taps.push_back(d);
                        if (account) P.macs += (ey1 - ey0 + 1) * (ex1 - ex0 + 1);
                    }
                } else if (account && q == 0) {  // zmask must still see every class's padding taps
                    for (int i = tstart[(size_t)k * (nst + 1) + st]; i < tstart[(size_t)k * (nst + 1) + st + 1]; ++i) {
                        const int64_t rem = colidx[i] % pp;
                        const int iy = y0 + (int)(rem / wp) - 1, ix = x0 + (int)(rem % wp) - 1;
                        const bool neg = sign ? sign[i] != 0 : (vbits[i] & 0x80000000u) != 0;
                        if ((iy < 0 || iy >= H || ix < 0 || ix >= W) && !neg) P.zmask[k] |= 1u << (cy * 3 + cx);
                    }
                }
                ends[cy * 3 + cx] = (uint16_t)taps.size();
            }
    };
    int maxt = 0;
    for (int q = 0; q < 4; ++q)
        for (int k = 0; k < K; ++k)
            for (int st = 0; st < nst; ++st) {
                slot(q, k, st, true);
                maxt = std::max(maxt, (int)taps.size());
            }
    if (maxt > 0xffff) return false;
    P.cap = (LANE_HDR + maxt * 8 + 15) / 16;
    if (count_only) return true;
    P.desc.assign((size_t)4 * nst * K * P.cap, make_uint4(0, 0, 0, 0));
    for (int q = 0; q < 4; ++q)
        for (int st = 0; st < nst; ++st)
            for (int k = 0; k < K; ++k) {
                slot(q, k, st, false);
                unsigned char* b = reinterpret_cast<unsigned char*>(P.desc.data() + (((size_t)q * nst + st) * K + k) * P.cap);
                std::memcpy(b, ends, LANE_HDR);
                if (!taps.empty()) std::memcpy(b + LANE_HDR, taps.data(), taps.size() * 8);
            }
    return true;
}

// Tap program of the 4x4-tile kernel (k_tile, dispatch 4): per (stage st, channel k) one slot
// ([st][k][cap]) = LANE_HDR bytes (int32 tap count first) + the CSR row's taps of the stage in
// colidx order, padding taps included, offsets into the 6x6 window: (c_local*36 + r*6 + s)*RB.
// R = S = 3, pad 1, stride 1 (wp = W + 2).
inline bool build_lane_program_tiles(const uint32_t* vbits, const int32_t* colidx, const int32_t* rowptr, int C,
                                     int K, int64_t pp, int wp, int H, int W, int cc, int nb, LaneProgram* out,
                                     bool count_only = false, int es = 4) {
    const int RB = 32 * nb * es;
    const int nst = (C + cc - 1) / cc;
    if (cc < 1 || H % 4 || W % 4) return false;
    LaneProgram& P = *out;
    P.zmask.assign(K, 0u);  // padding MACs executed: nothing to restore
    P.nst = nst;
    P.macs = (int64_t)(rowptr[K] - rowptr[0]) * H * W;
    P.desc.clear();
    std::vector<int32_t> tstart((size_t)K * (nst + 1));
    int maxt = 0;
    for (int k = 0; k < K; ++k) {
        int t = rowptr[k];
        for (int st = 0; st < nst; ++st) {
            tstart[(size_t)k * (nst + 1) + st] = t;
            while (t < rowptr[k + 1] && colidx[t] / pp < std::min<int64_t>(C, (int64_t)(st + 1) * cc)) ++t;
            maxt = std::max(maxt, t - tstart[(size_t)k * (nst + 1) + st]);
        }
        tstart[(size_t)k * (nst + 1) + nst] = t;
    }
    P.cap = (LANE_HDR + maxt * 8 + 15) / 16;
    if (count_only) return true;
    P.desc.assign((size_t)nst * K * P.cap, make_uint4(0, 0, 0, 0));
    for (int k = 0; k < K; ++k)
        for (int st = 0; st < nst; ++st) {
            const int t0 = tstart[(size_t)k * (nst + 1) + st], t1 = tstart[(size_t)k * (nst + 1) + st + 1];
            unsigned char* b = reinterpret_cast<unsigned char*>(P.desc.data() + ((size_t)st * K + k) * P.cap);
            const int32_t cnt = t1 - t0;
            std::memcpy(b, &cnt, 4);
            for (int i = t0; i < t1; ++i) {
                const int64_t ci = colidx[i] / pp, rem = colidx[i] % pp;
                const int r = (int)(rem / wp), s = (int)(rem % wp);
                LaneTap d;
                std::memcpy(&d.v, &vbits[i], 4);
                d.off = (int32_t)(((ci - (int64_t)st * cc) * 36 + r * 6 + s) * RB);
                std::memcpy(b + LANE_HDR + (size_t)(i - t0) * 8, &d, 8);
            }
        }
    return true;
}

}  // namespace scb
