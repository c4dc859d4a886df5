// Whole-plane direct sparse convolution kernel for small spatial extents
// (sm_100a): VGG-CIFAR conv4_x (4x4) and conv5_x (2x2), where the tiled
// kernel's halo patches, per-row staging and tiny per-tap MAC blocks waste
// most of the issue slots (profiles/r01_*).
//
// A lane owns the WHOLE E x F output plane of NBT images for the KT output
// channels of one tap group.  Its input patch is the whole H x W plane of
// each image: the zero padding around it (shapes.py:98-105) is a
// compile-time zero operand in the generated MAC blocks, so only the H*W
// real values are loaded (H*W/4 128-bit shared loads per image and
// channel) and nothing is staged for the halo.
//
// Staging: `cc` input channels per stage, two stages in flight, copied with
// 16-byte cp.async straight from NCHW -- image n's channels [c0, c0+cc) are
// one contiguous run of cc*H*W elements.  Shared layout [image][channel][H*W]
// with an image pitch of (multiple of 128 B) + 16 B so the 8 lanes of a
// quarter-warp (consecutive images) hit distinct 16-byte bank groups.
//
// Taps: the same sentinel-delimited (c, kk, r, s) stream and brx.idx jump
// table as the tiled kernel (gen_taploop.py gen_plane), so exact mode keeps
// the reference's per-output colidx accumulation order bit for bit.
#pragma once

#include <cuda_runtime.h>

#include <type_traits>

#include "kernels.cuh"
#include "sparseconv_b200.h"
#include "tiled.cuh"

namespace scb {

template <int H, int W, int R, int S, int PAD, int KT, int NBT, int WF, int MODE, bool F16IO>
struct PlaneLoop;

template <int H, int W, int R, int S, int PAD, int KT, int NBT, bool F16IO, int WF, int MODE, int MINB>
__global__ void __launch_bounds__(256, MINB) k_plane(const __grid_constant__ TiledParams p) {
    using TIO = typename std::conditional<F16IO, __half, float>::type;
    constexpr int ES = (int)sizeof(TIO);
    constexpr int E = H + 2 * PAD - R + 1, F = W + 2 * PAD - S + 1;
    constexpr int HW = H * W, EF = E * F;
    constexpr int P = NBT * EF;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ QuantAux qs;

    const int tid = threadIdx.x;
    const int nthreads = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int wg = warp / p.wp;               // warp group (tap group) of this warp
    const int pw = warp - wg * p.wp;          // pixel warp inside the group
    const int kb = blockIdx.x % p.kblocks;
    const int nb = blockIdx.x / p.kblocks;
    const int g = kb * p.wk + wg;
    const int k0 = g * KT;
    const int n0 = nb * p.imgs;
    const int C = p.c, cp1 = C + 1;
    const int ipitch = p.row;                 // image pitch in elements
    const int stage_el = p.stage_el;
    const int lanes_img = p.wp * 32;          // images per NBT slot
    const int img0 = pw * 32 + lane;          // lane's first image (CTA-local); then + j*lanes_img
    Tap* tsm = reinterpret_cast<Tap*>(smem + (size_t)2 * stage_el * ES);

    if (tid < 16) qs.cb[tid] = p.q.cb[tid];
    if (tid == 0) qs.scale = p.q.scale;

    float acc[KT * P];
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) {
        const int k = k0 + kk;
        const float b = (p.bias != nullptr && k < p.k) ? p.bias[k] : 0.f;
#pragma unroll
        for (int i = 0; i < P; ++i) acc[kk * P + i] = b;
    }

    // ---- producer: 16-byte chunks of each image's contiguous channel run
    const int run_el = p.cc * HW;             // elements per image per full stage
    const int cpi = run_el * ES / 16;         // chunks per image
    const int total = p.imgs * cpi;
    auto stage = [&](int ch, int buf) {
        const int c0 = ch * p.cc;
        const int valid = (min(C - c0, p.cc) * HW * ES) / 16;  // chunks of real channels
        unsigned char* dst = smem + (size_t)buf * stage_el * ES;
        const unsigned char* src = static_cast<const unsigned char*>(p.x) + ((size_t)c0 * HW) * ES;
        for (int q = tid; q < total; q += nthreads) {
            const int img = q / cpi, off = q - img * cpi;
            const int n = n0 + img;
            if (n < p.n && off < valid)
                cp_async<16>(dst + ((size_t)img * ipitch) * ES + off * 16,
                             src + ((size_t)n * C * HW) * ES + off * 16);
        }
        const int c1 = min(c0 + p.cc, C);
        for (int w = 0; w < p.wk; ++w) {
            const int gg = kb * p.wk + w;
            if (gg >= p.groups) break;
            const int a0 = __ldg(p.tap_ptr + gg * cp1 + c0) & ~1;
            const int a1 = __ldg(p.tap_ptr + gg * cp1 + c1) + 2;
            Tap* d = tsm + ((size_t)buf * p.wk + w) * p.tap_cap;
            for (int i = 2 * tid; i < a1 - a0; i += 2 * nthreads) cp_async<16>(d + i, p.taps + a0 + i);
        }
    };

    const int nch = (C + p.cc - 1) / p.cc;
    stage(0, 0);
    cp_async_commit();
    __syncthreads();  // qs visible
    const unsigned cb_addr = smem_u32(&qs.cb[0]);
    const float lin_scale = qs.scale;
    float pt[NBT * HW];
#pragma unroll
    for (int i = 0; i < NBT * HW; ++i) pt[i] = 0.f;

    for (int ch = 0; ch < nch; ++ch) {
        const int buf = ch & 1;
        if (ch + 1 < nch) {
            stage(ch + 1, buf ^ 1);
            cp_async_commit();
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        if (g < p.groups) {
            const int c0 = ch * p.cc;
            const int ncl = min(p.cc, C - c0);
            const TIO* xb = reinterpret_cast<const TIO*>(smem) + (size_t)buf * stage_el + (size_t)img0 * ipitch;
            const int t0 = __ldg(p.tap_ptr + g * cp1 + c0);
            const Tap* seg = tsm + ((size_t)buf * p.wk + wg) * p.tap_cap + (t0 & 1);
            PlaneLoop<H, W, R, S, PAD, KT, NBT, WF, MODE, F16IO>::run(
                acc, pt, smem_u32(seg), (unsigned)c0, (unsigned)ncl, smem_u32(xb), (unsigned)(HW * ES),
                (unsigned)(lanes_img * ipitch * ES), cb_addr, lin_scale);
        }
        __syncthreads();
    }

    // ---- epilogue: optional ReLU / 2x2 max-pool; a lane's (kk, image) plane is contiguous
    if (g >= p.groups) return;
    const bool relu = p.flags & SCB_FLAG_RELU;
    const bool pool = p.flags & SCB_FLAG_POOL2;
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) {
        const int k = k0 + kk;
        if (k >= p.k) break;
#pragma unroll
        for (int j = 0; j < NBT; ++j) {
            const int n = n0 + img0 + j * lanes_img;
            if (n >= p.n) continue;
            const float* a = &acc[kk * P + j * EF];
            if (!pool) {
                TIO* yp = static_cast<TIO*>(p.y) + ((int64_t)n * p.k + k) * EF;
                float o[EF];
#pragma unroll
                for (int i = 0; i < EF; ++i) o[i] = relu ? relu_io<TIO>(a[i]) : a[i];
                if constexpr (!F16IO && EF % 4 == 0) {
#pragma unroll
                    for (int i = 0; i < EF; i += 4)
                        *reinterpret_cast<float4*>(yp + i) = make_float4(o[i], o[i + 1], o[i + 2], o[i + 3]);
                } else {
#pragma unroll
                    for (int i = 0; i < EF; ++i) {
                        if constexpr (F16IO) yp[i] = __float2half_rn(o[i]);
                        else yp[i] = o[i];
                    }
                }
            } else {
                constexpr int PE = E / 2, PF = F / 2;
                TIO* yp = static_cast<TIO*>(p.y) + ((int64_t)n * p.k + k) * PE * PF;
#pragma unroll
                for (int yy = 0; yy < PE; ++yy)
#pragma unroll
                    for (int xx = 0; xx < PF; ++xx) {
                        float o = fmaxf(fmaxf(a[(2 * yy) * F + 2 * xx], a[(2 * yy) * F + 2 * xx + 1]),
                                        fmaxf(a[(2 * yy + 1) * F + 2 * xx], a[(2 * yy + 1) * F + 2 * xx + 1]));
                        if (relu) o = relu_io<TIO>(o);
                        if constexpr (F16IO) yp[yy * PF + xx] = __float2half_rn(o);
                        else yp[yy * PF + xx] = o;
                    }
            }
        }
    }
}

template <int H, int W, int R, int S, int PAD, int KT, int NBT, bool F16IO, int WF, int MODE, int MINB>
cudaError_t launch_plane_t(const TiledParams& p, unsigned grid, unsigned threads, size_t smem, cudaStream_t st) {
    auto kern = k_plane<H, W, R, S, PAD, KT, NBT, F16IO, WF, MODE, MINB>;
    static int lim[64];  // per device (the attribute is per device)
    const cudaError_t e = dyn_smem_ok(kern, smem, lim);
    if (e != cudaSuccess) return e;
    kern<<<grid, threads, smem, st>>>(p);
    return cudaGetLastError();
}

}  // namespace scb
