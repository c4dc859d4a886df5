// Image-lane direct kernel for small planes (sm_100a): VGG-CIFAR conv4_x
// (4x4) and conv5_x (2x2), 3x3 taps, padding 1.
//
// Lane = image (32 images per CTA); a lane owns the whole H x H output plane
// of its image for the KW output channels of its warp (compile-time unrolled,
// as in direct.cuh -- no data-dependent control flow).  Taps are warp-uniform
// and walked in the reference's colidx order per output channel
// (_kernels.py:73-84), so exact mode is bit-identical to the reference.
//
// Shared layout per (image, channel): 3H+4 rows of H floats holding the three
// column-shifted copies of the H input rows, copy_s = padded_row[s .. s+H), with
// the four zero padding rows shared between neighbouring copies:
//   pos 0: 0 | 1..H: copy_1 (the input plane itself) | H+1: 0 | H+2..2H+1: copy_0 |
//   2H+2: 0 | 2H+3..3H+2: copy_2 | 3H+3: 0
// so padded row r (0..H+1) of copy s sits at pos START_s + r, START = {H+1, 0, 2H+2}.
// A tap (c, r, s) then reads output row y's inputs as ONE aligned vector load
// (ld.shared.v4 for H=4, .v2 for H=2) at c*BLK + BASE + (START_s + y + r)*H:
// 4 B per MAC but one instruction per H MACs.  copy_1 is the image plane
// contiguous, so a stage lands with one 16-byte cp.async per thread per chunk;
// copy_0 / copy_2 are built from it in shared memory.  Images sit at a pitch whose
// vector index is odd, so the 8 (v4) / 16 (v2) lanes of a wavefront hit distinct banks.
#pragma once

#include <cuda_runtime.h>

#include "direct.cuh"
#include "kernels.cuh"
#include "sparseconv_b200.h"
#include "tiled.cuh"

namespace scb {

// element type traits: f32 storage (V = H floats) or f16 storage (V = H halves;
// FHFMA accumulation in f32, one final round -- the reference's f16 profile)
template <int H, bool F16>
struct DimgT;
template <> struct DimgT<4, false> { using E = float; using V = float4; };
template <> struct DimgT<2, false> { using E = float; using V = float2; };
template <> struct DimgT<4, true> { using E = __half; using V = uint2; };
template <> struct DimgT<2, true> { using E = __half; using V = unsigned; };

template <int H, bool F16>
__device__ __forceinline__ float dimg_elem(const typename DimgT<H, F16>::V& v, int x) {
    if constexpr (!F16) return reinterpret_cast<const float*>(&v)[x];
    else return 0.f;  // (f16 reads go through dimg_half)
}
template <int H>
__device__ __forceinline__ unsigned short dimg_half(const typename DimgT<H, true>::V& v, int x) {
    const unsigned w = reinterpret_cast<const unsigned*>(&v)[x >> 1];
    return (unsigned short)((x & 1) ? (w >> 16) : (w & 0xffffu));
}

template <int H, int KW, int MODE, bool F16 = false, int WF = (F16 ? WF_F16 : WF_F32)>
__global__ void __launch_bounds__(512, 1) k_dimg(const __grid_constant__ DirectParams p) {
    static_assert(F16 == (WF != WF_F32), "f16 storage <=> compact f16 taps (kernels.cuh tap_f16)");
    using E = typename DimgT<H, F16>::E;
    using V = typename DimgT<H, F16>::V;
    constexpr int ES = (int)sizeof(E);
    constexpr int RW = H;                    // row stride inside a copy (elements)
    // elements per (image, channel); 4x4 planes add 32 bytes so consecutive planes land on
    // different bank groups in the per-(plane, row) copy pass (= layer.cu dimg_blk)
    constexpr int BLK = (3 * H + 4) * H + (H == 4 ? 32 / ES : 0);
    // BASE puts copy_1's plane on its copy alignment: f32 16 B, f16 8 B (H=2) / 16 B (H=4)
    constexpr int BASE = F16 ? (H == 2 ? 2 : 4) : (H == 2 ? 2 : 0);
    constexpr int HW = H * H;
    constexpr int C1 = BASE + H;                  // copy_1 rows 1..H (the plane)
    constexpr int C0 = BASE + (H + 2) * H;        // copy_0 rows 1..H
    constexpr int C2 = BASE + (2 * H + 3) * H;    // copy_2 rows 1..H
    extern __shared__ __align__(128) unsigned char smem[];

    const int tid = threadIdx.x, nthreads = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int kb = blockIdx.x % p.kblocks;
    const int n0 = (blockIdx.x / p.kblocks) * 32;
    const int k0 = (kb * p.wk + warp) * KW;
    const int C = p.c;
    E* xs = reinterpret_cast<E*>(smem);
    const int planes = 32 * p.cc;  // (image, channel) planes per stage
    // tap blocks after the stages: [buf][warp] slots of segcap 16-byte chunks (direct.cuh layout)
    int4* tsm = reinterpret_cast<int4*>(smem + (size_t)p.nbuf * p.stage_el * ES);
    constexpr int HDR = (KW * 4 + 15) / 16;
    const int grp = kb * p.wk + warp;
    const int groups = (p.k + KW - 1) / KW;

    {  // zero both stages: padding rows and the halo ends of copies 0 / 2 stay zero
        float4* z = reinterpret_cast<float4*>(smem);
        const int n16 = (p.nbuf * p.stage_el * ES) / 16;
        for (int i = tid; i < n16; i += nthreads) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();

    // plane t of a stage: image t / cc, channel slot t % cc; chunks of CH bytes, chunk fastest.
    // Odd images sit at half the copy alignment (odd vector image pitch): two half copies.
    constexpr int PB = HW * ES;               // plane bytes
    constexpr int CH = PB >= 16 ? 16 : PB;    // copy chunk
    constexpr int PQ = PB / CH, QE = CH / ES;
    const E* xg = static_cast<const E*>(p.x) + (size_t)n0 * C * HW;
    auto stage = [&](int st, int buf) {
        const int c0 = st * p.cc;
        const int ncl = min(p.cc, C - c0);
        E* dst = xs + (size_t)buf * p.stage_el;
        for (int it = tid; it < planes * PQ; it += nthreads) {
            const int q = it % PQ, t = it / PQ;
            const int cl = t % p.cc, img = t / p.cc;
            if (cl < ncl && n0 + img < p.n) {
                const int off = img * p.ip + cl * BLK + C1 + QE * q;
                E* d = dst + off;
                const E* g = xg + ((size_t)img * C + c0 + cl) * HW + QE * q;
                if ((off * ES) % CH == 0) {
                    cp_async<CH>(d, g);
                } else {
                    cp_async<CH / 2>(d, g);
                    cp_async<CH / 2>(d + QE / 2, g + QE / 2);
                }
            }
        }
        if (grp < groups) {  // this warp's contiguous tap block of the stage
            const int o0 = __ldg(p.blkoff + (size_t)grp * p.nst + st);
            const int o1 = __ldg(p.blkoff + (size_t)grp * p.nst + st + 1);
            const int4* src = reinterpret_cast<const int4*>(p.taps) + o0;
            int4* tb = tsm + ((size_t)buf * p.wk + warp) * p.segcap;
            const int nch = min(o1 - o0, p.segcap);
            for (int i = lane; i < nch; i += 32) cp_async<16>(tb + i, src + i);
        }
    };
    // copy_0 row = (0, x0 .. x_{H-2}), copy_2 row = (x1 .. x_{H-1}, 0), from copy_1
    auto shift = [&](int st, int buf) {
        const int ncl = min(p.cc, C - st * p.cc);
        E* base = xs + (size_t)buf * p.stage_el;
        if constexpr (F16) {  // thread = (plane, row); 32-bit words of halves
            for (int it = tid; it < planes * H; it += nthreads) {
                const int y = it % H, t = it / H;
                const int cl = t % p.cc, img = t / p.cc;
                if (cl >= ncl) continue;
                E* b = base + img * p.ip + cl * BLK + y * H;
                if constexpr (H == 2) {
                    const unsigned w = *reinterpret_cast<const unsigned*>(b + C1);
                    *reinterpret_cast<unsigned*>(b + C0) = w << 16;   // (0, x0)
                    *reinterpret_cast<unsigned*>(b + C2) = w >> 16;   // (x1, 0)
                } else {
                    const uint2 w = *reinterpret_cast<const uint2*>(b + C1);
                    *reinterpret_cast<uint2*>(b + C0) = make_uint2(w.x << 16, __funnelshift_l(w.x, w.y, 16));
                    *reinterpret_cast<uint2*>(b + C2) = make_uint2(__funnelshift_r(w.x, w.y, 16), w.y >> 16);
                }
            }
        } else if constexpr (H == 2) {  // thread = plane (8-byte accesses: odd images are 8-byte aligned)
            for (int t = tid; t < planes; t += nthreads) {
                const int cl = t % p.cc, img = t / p.cc;
                if (cl >= ncl) continue;
                float* b = base + img * p.ip + cl * BLK;
                const float2 r0 = *reinterpret_cast<const float2*>(b + C1);
                const float2 r1 = *reinterpret_cast<const float2*>(b + C1 + 2);
                *reinterpret_cast<float2*>(b + C0) = make_float2(0.f, r0.x);
                *reinterpret_cast<float2*>(b + C0 + 2) = make_float2(0.f, r1.x);
                *reinterpret_cast<float2*>(b + C2) = make_float2(r0.y, 0.f);
                *reinterpret_cast<float2*>(b + C2 + 2) = make_float2(r1.y, 0.f);
            }
        } else {  // thread = (plane, row)
            for (int it = tid; it < planes * H; it += nthreads) {
                const int y = it % H, t = it / H;
                const int cl = t % p.cc, img = t / p.cc;
                if (cl >= ncl) continue;
                float* b = base + img * p.ip + cl * BLK + y * H;
                const float4 m = *reinterpret_cast<const float4*>(b + C1);
                *reinterpret_cast<float4*>(b + C0) = make_float4(0.f, m.x, m.y, m.z);
                *reinterpret_cast<float4*>(b + C2) = make_float4(m.y, m.z, m.w, 0.f);
            }
        }
    };

    __shared__ unsigned short cbt[16];  // WF_CB4: f16 codebook (published by the first stage barrier)
    if constexpr (WF == WF_CB4) {
        if (tid < 16) cbt[tid] = p.q.cb16[tid];
    }
    const float qscale = p.q.scale;
    const double qstep = p.q.step;
    float acc[KW][HW];
#pragma unroll
    for (int kk = 0; kk < KW; ++kk) {
        const int k = k0 + kk;
        const float b = (p.bias != nullptr && k < p.k) ? p.bias[k] : 0.f;
#pragma unroll
        for (int j = 0; j < HW; ++j) acc[kk][j] = b;
    }

    // programmatic dependent launch: everything above overlapped the previous layer's tail;
    // its output (our input) is visible after this wait
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int s0 = 0; s0 < p.nbuf - 1; ++s0) {  // prologue: nbuf-1 stages in flight
        if (s0 < p.nst) stage(s0, s0);
        cp_async_commit();
    }
    for (int st = 0; st < p.nst; ++st) {
        const int buf = st % p.nbuf;
        cp_async_wait_nb2(p.nbuf);
        __syncthreads();  // stage st landed; every warp has left stage st-1
        shift(st, buf);
        __syncthreads();
        if (st + p.nbuf - 1 < p.nst) stage(st + p.nbuf - 1, (st + p.nbuf - 1) % p.nbuf);
        cp_async_commit();  // possibly empty: keeps one group per iteration
        // lane's image block, minus the stage's first channel (tap offsets are absolute)
        const char* xl = reinterpret_cast<const char*>(xs + (size_t)buf * p.stage_el + lane * p.ip) -
                         (size_t)st * p.cc * BLK * ES;
        const int4* tb = tsm + ((size_t)buf * p.wk + warp) * p.segcap;
        const int* cnt = reinterpret_cast<const int*>(tb);
        const DirectTap* seg = reinterpret_cast<const DirectTap*>(tb + HDR);
        const unsigned* segc = reinterpret_cast<const unsigned*>(tb + HDR);  // f16: compact taps
        // compact f16 taps hold STAGE-relative element offsets
        const E* xlc = reinterpret_cast<const E*>(xs + (size_t)buf * p.stage_el + lane * p.ip);
#pragma unroll
        for (int kk = 0; kk < KW; ++kk) {
            const int k = k0 + kk;
            if (k >= p.k) break;
            const int nt = cnt[kk];
#pragma unroll 4
            for (int t = 0; t < nt; ++t) {
                DirectTap tp;
                const E* xp;
                unsigned short vh = 0;
                if constexpr (F16) {
                    const unsigned tw = segc[t];
                    xp = xlc + (tw & 0xffffu);
                    vh = tap_f16<WF>(tw >> 16, cbt, qscale, qstep);
                } else {
                    tp = seg[t];
                    xp = reinterpret_cast<const E*>(xl + tp.off);
                }
#pragma unroll
                for (int y = 0; y < H; ++y) {
                    const V v = *reinterpret_cast<const V*>(xp + y * RW);
                    if constexpr (F16) {
#pragma unroll
                        for (int x = 0; x < H; ++x) acc[kk][y * H + x] = fhfma(acc[kk][y * H + x], vh, dimg_half<H>(v, x));
                    } else {
#pragma unroll
                        for (int x = 0; x < H; ++x)
                            acc[kk][y * H + x] = mac1<MODE>(acc[kk][y * H + x], tp.v, dimg_elem<H, F16>(v, x));
                    }
                }
            }
            seg += nt;
            segc += nt;
        }
    }

    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // next layer may start its prologue
    // ---- epilogue: lane's image plane per output channel is contiguous
    const int n = n0 + lane;
    if (n >= p.n) return;
    const bool aq = p.flags & SCB_FLAG_ACT_QUANT;
    if (aq) {  // ReLU + fake-quant in place (monotone: commutes with the max-pool)
        const bool r0 = p.flags & SCB_FLAG_RELU;
#pragma unroll
        for (int kk = 0; kk < KW; ++kk)
#pragma unroll
            for (int j = 0; j < HW; ++j) acc[kk][j] = fq_store<E>(r0 ? relu_io<E>(acc[kk][j]) : acc[kk][j], p.aq);
    }
    const bool relu = (p.flags & SCB_FLAG_RELU) && !aq;
    const bool pool = p.flags & SCB_FLAG_POOL2;
#pragma unroll
    for (int kk = 0; kk < KW; ++kk) {
        const int k = k0 + kk;
        if (k >= p.k) break;
        float o[HW];
#pragma unroll
        for (int j = 0; j < HW; ++j) o[j] = relu ? relu_io<E>(acc[kk][j]) : acc[kk][j];
        if (!pool) {
            E* yp = static_cast<E*>(p.y) + ((int64_t)n * p.k + k) * HW;
            if constexpr (F16) {
#pragma unroll
                for (int j = 0; j < HW; j += 2)
                    *reinterpret_cast<__half2*>(yp + j) = __floats2half2_rn(o[j], o[j + 1]);
            } else {
#pragma unroll
                for (int j = 0; j < HW; j += H) *reinterpret_cast<V*>(yp + j) = *reinterpret_cast<const V*>(&o[j]);
            }
        } else {
            constexpr int PH = H / 2;
            E* yp = static_cast<E*>(p.y) + ((int64_t)n * p.k + k) * PH * PH;
#pragma unroll
            for (int yy = 0; yy < PH; ++yy)
#pragma unroll
                for (int xx = 0; xx < PH; ++xx)
                    yp[yy * PH + xx] = (E)fmaxf(fmaxf(o[(2 * yy) * H + 2 * xx], o[(2 * yy) * H + 2 * xx + 1]),
                                                fmaxf(o[(2 * yy + 1) * H + 2 * xx], o[(2 * yy + 1) * H + 2 * xx + 1]));
        }
    }
}

template <int H, int KW, int MODE, bool F16 = false, int WF = (F16 ? WF_F16 : WF_F32)>
cudaError_t launch_dimg_t(const DirectParams& p, unsigned grid, unsigned threads, size_t smem, cudaStream_t st) {
    auto kern = k_dimg<H, KW, MODE, F16, WF>;
    static int lim[64];  // per device (the attribute is per device)
    const cudaError_t e = dyn_smem_ok(kern, smem, lim);
    if (e != cudaSuccess) return e;
    return launch_pdl(kern, p, grid, threads, smem, st);
}

}  // namespace scb
