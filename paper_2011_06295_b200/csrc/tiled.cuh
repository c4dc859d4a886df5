// Register-tiled direct sparse convolution kernel (sm_100a).
//
// CTA = `wk` warp groups x `wp` pixel warps.  A warp group owns KT output
// channels (one tap group of the device program); every lane owns an
// NBT x TH x TW output tile (NBT images) and keeps KT x NBT x TH x TW f32
// accumulators in registers.
//
// Input staging: `cc` input channels per stage, two stages in flight.  Each
// (image, channel) window of the CTA's output block lives in shared memory in
// a zero-halo layout: row pitch ROW, input column gx at XOFF + gx - ox0 with
// XOFF = 16 bytes, so the tile-aligned middle of every lane's patch row is one
// aligned vector load.  Rows and columns outside the image are zeroed once at
// kernel start and never written again -- that IS the reference's zero
// padding (shapes.py:98-105), never materialised in HBM.  In-image row
// segments are copied with 16/8/4-byte cp.async.  (TMA would be the natural
// tool, but a tile box with negative start coordinates traps on B200 --
// tools/tma_test.cu.)
//
// Per input channel a lane loads its (TH+R-1) x (TW+S-1) patch per image into
// registers once, then applies the warp group's taps of that channel through
// generated inline PTX (gen_taploop.py), either a brx.idx jump table per tap
// or an in-order mask walk; every MAC reads registers only.  Taps are ordered
// (c, kk, r, s), i.e. colidx order per accumulator (csr.py:143-160), so exact
// mode reproduces the reference bit for bit.
#pragma once

#include <cuda_runtime.h>

#include <type_traits>

#include "kernels.cuh"
#include "sparseconv_b200.h"

namespace scb {

template <int R, int S, int PAD, int KT, int NBT, int TH, int TW, int WF, int MODE, int DISPATCH, bool F16IO>
struct TapLoop;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem) {
    if constexpr (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem));
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(smem_u32(smem)), "l"(gmem), "n"(BYTES));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <typename T>
__device__ __forceinline__ float to_f32(T v) {
    if constexpr (std::is_same<T, __half>::value) return __half2float(v);
    else return v;
}

// Load N consecutive elements starting at an address aligned to ALIGN bytes
// into dst[0..N), converting to f32, with the widest shared loads allowed.
template <int N, int ALIGN, typename T>
__device__ __forceinline__ void load_row(float* dst, const T* src) {
    constexpr int ES = (int)sizeof(T);
    constexpr int A = ALIGN >= 16 ? 16 : ALIGN;
    int j = 0;
#pragma unroll
    for (int step = 0; step < 16; ++step) {
        if (j >= N) break;
        const int rem = (N - j) * ES;
        const int vb = (A >= 16 && rem >= 16) ? 16 : ((A >= 8 && rem >= 8) ? 8 : ((rem >= 4 && A >= 4) ? 4 : ES));
        if (vb == 16) {
            float4 t = *reinterpret_cast<const float4*>(src + j);
            const T* tv = reinterpret_cast<const T*>(&t);
#pragma unroll
            for (int u = 0; u < 16 / ES; ++u) dst[j + u] = to_f32(tv[u]);
            j += 16 / ES;
        } else if (vb == 8) {
            float2 t = *reinterpret_cast<const float2*>(src + j);
            const T* tv = reinterpret_cast<const T*>(&t);
#pragma unroll
            for (int u = 0; u < 8 / ES; ++u) dst[j + u] = to_f32(tv[u]);
            j += 8 / ES;
        } else if (vb == 4) {
            float t = *reinterpret_cast<const float*>(src + j);
            const T* tv = reinterpret_cast<const T*>(&t);
#pragma unroll
            for (int u = 0; u < 4 / ES; ++u) dst[j + u] = to_f32(tv[u]);
            j += 4 / ES;
        } else {
            dst[j] = to_f32(src[j]);
            j += 1;
        }
    }
}

template <int R, int S, int PAD, int KT, int NBT, int TH, int TW, bool F16IO, int WF, int MODE, int DISPATCH,
          int MINB>
__global__ void __launch_bounds__(256, MINB) k_tiled(const __grid_constant__ TiledParams p) {
    using TIO = typename std::conditional<F16IO, __half, float>::type;
    constexpr int ES = (int)sizeof(TIO);
    constexpr int XOFF = 16 / ES;  // column of the block's first input column
    constexpr int PH = TH + R - 1, PW = TW + S - 1;
    constexpr int P = NBT * TH * TW;
    constexpr int RIGHT = S - 1 - PAD;
    constexpr int MID_ALIGN = (TW * ES) >= 16 ? 16 : (TW * ES);
    constexpr int NW = (KT + 1) / 2;  // mask words per (group, channel)
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ QuantAux qs;

    const int tid = threadIdx.x;
    const int nthreads = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int wg = warp / p.wp;
    const int ptid = (warp - wg * p.wp) * 32 + lane;
    const int TX = p.bw / TW, TY = p.bh / TH;
    const int tx = ptid % TX, ty = (ptid / TX) % TY, ti = ptid / (TX * TY);

    int bid = blockIdx.x;
    const int kb = bid % p.kblocks;
    bid /= p.kblocks;
    const int fx = bid % p.n_fx;
    bid /= p.n_fx;
    const int ey = bid % p.n_ey;
    const int nb = bid / p.n_ey;
    const int g = kb * p.wk + wg;
    const int k0 = g * KT;
    const int n0 = nb * p.imgs, oy0 = ey * p.bh, ox0 = fx * p.bw;
    const int C = p.c, cp1 = C + 1;
    const int RT = p.bh + R - 1;     // window rows
    const int ROW = p.row;           // smem row pitch (elements)
    const int plane_s = RT * ROW;    // elements per (image, channel)
    const int stage_el = p.stage_el; // elements per stage (128-byte multiple)
    TIO* xs = reinterpret_cast<TIO*>(smem);
    // tap segments of the stage: [buf][warp group][tap_cap] entries after the x stages
    Tap* tsm = reinterpret_cast<Tap*>(smem + (size_t)2 * stage_el * ES);

    // zero both stages once: positions outside the image are never written again
    {
        float4* z = reinterpret_cast<float4*>(smem);
        const int n16 = (2 * stage_el * ES) / 16;
        for (int i = tid; i < n16; i += nthreads) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (tid < 16) qs.cb[tid] = p.q.cb[tid];
    if (tid == 0) qs.scale = p.q.scale;
    __syncthreads();

    // accumulators start at the bias (reference: o[:] = b, _kernels.py:71-72)
    float acc[KT * P];
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) {
        const int k = k0 + kk;
        const float b = (p.bias != nullptr && k < p.k) ? p.bias[k] : 0.f;
#pragma unroll
        for (int i = 0; i < P; ++i) acc[kk * P + i] = b;
    }

    // ---- producer: copy the in-image part of every window row of a stage.
    // Row assignments (image, channel slot, window row) are the same for every
    // stage, so each thread decodes its rows once: a 32-bit source offset from
    // the CTA's first image (channel 0) and a shared-memory byte offset.
    const int ce = p.chunk / ES;  // elements per copy chunk
    const int gx_lo = max(0, ox0 - PAD) / ce * ce;
    const int gx_hi = (min(p.w, ox0 + p.bw + S - 1 - PAD) + ce - 1) / ce * ce;
    const int nchunk = (gx_hi - gx_lo) / ce;
    const int dcol = XOFF + gx_lo - ox0;  // smem column of gx_lo
    const int rows = p.imgs * p.cc * RT;
    const int hw = p.h * p.w;
    const unsigned char* xcta = static_cast<const unsigned char*>(p.x) + (size_t)n0 * C * hw * ES;
    // row descriptors after the tap segments: {source element offset from the
    // CTA's first image at channel 0, smem byte offset | channel slot << 24}
    uint2* rdesc = reinterpret_cast<uint2*>(smem + (size_t)2 * stage_el * ES +
                                            (size_t)2 * p.wk * p.tap_cap * sizeof(Tap));
    for (int rr = tid; rr < rows; rr += nthreads) {
        const int yy = rr % RT, pc = rr / RT;
        const int cl = pc % p.cc, img = pc / p.cc;
        const int gy = oy0 - PAD + yy;
        const bool ok = n0 + img < p.n && (unsigned)gy < (unsigned)p.h;
        const unsigned dst = (unsigned)(((size_t)pc * plane_s + yy * ROW + dcol) * ES);
        rdesc[rr] = make_uint2((unsigned)(((img * C + cl) * p.h + gy) * p.w + gx_lo),
                               dst | ((unsigned)(ok ? cl : 255) << 24));
    }
    __syncthreads();
    auto stage = [&](int ch, int buf) {
        const int c0 = ch * p.cc;
        const unsigned ncl = (unsigned)min(p.cc, C - c0);
        unsigned char* dst = smem + (size_t)buf * stage_el * ES;
        const unsigned char* src = xcta + (size_t)c0 * hw * ES;
        for (int rr = tid; rr < rows; rr += nthreads) {
            const uint2 rd = rdesc[rr];
            if ((rd.y >> 24) < ncl) {
                const unsigned char* s = src + (size_t)rd.x * ES;
                unsigned char* d = dst + (rd.y & 0xffffffu);
                if (p.chunk == 16) {
                    for (int q = 0; q < nchunk; ++q) cp_async<16>(d + q * 16, s + q * 16);
                } else if (p.chunk == 8) {
                    for (int q = 0; q < nchunk; ++q) cp_async<8>(d + q * 8, s + q * 8);
                } else {
                    for (int q = 0; q < nchunk; ++q) cp_async<4>(d + q * 4, s + q * 4);
                }
            }
        }
        if constexpr (DISPATCH == DISPATCH_JUMP) {
            // each warp group's stream segment for channels [c0, c0+cc) plus the exit
            // sentinel and one prefetch slot, copied from its 16-byte-aligned floor
            const int c1 = min(c0 + p.cc, C);
            for (int w = 0; w < p.wk; ++w) {
                const int gg = kb * p.wk + w;
                if (gg >= p.groups) break;
                const int a0 = __ldg(p.tap_ptr + gg * cp1 + c0) & ~1;
                const int a1 = __ldg(p.tap_ptr + gg * cp1 + c1) + 2;
                Tap* d = tsm + ((size_t)buf * p.wk + w) * p.tap_cap;
                for (int i = 2 * tid; i < a1 - a0; i += 2 * nthreads) cp_async<16>(d + i, p.taps + a0 + i);
            }
        }
    };

    const int nch = (C + p.cc - 1) / p.cc;
    stage(0, 0);
    cp_async_commit();
    const unsigned cb_addr = smem_u32(&qs.cb[0]);
    const float lin_scale = qs.scale;
    // lane's patch origin inside a window plane
    const int patch_off = (ty * TH) * ROW + XOFF - PAD + tx * TW;
    float pt[NBT * PH * PW];
#pragma unroll
    for (int i = 0; i < NBT * PH * PW; ++i) pt[i] = 0.f;

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
            const TIO* xb = xs + (size_t)buf * stage_el + (size_t)ti * NBT * p.cc * plane_s + patch_off;
            if constexpr (DISPATCH == DISPATCH_JUMP) {
                // sentinel-driven stream: the PTX loop loads patches and exits at the
                // first sentinel of a channel beyond this stage
                const int t0 = __ldg(p.tap_ptr + g * cp1 + c0);
                const Tap* seg = tsm + ((size_t)buf * p.wk + wg) * p.tap_cap + (t0 & 1);
                TapLoop<R, S, PAD, KT, NBT, TH, TW, WF, MODE, DISPATCH, F16IO>::run(
                    acc, pt, smem_u32(seg), (unsigned)c0, (unsigned)ncl, smem_u32(xb), (unsigned)(plane_s * ES),
                    (unsigned)(p.cc * plane_s * ES), (unsigned)(ROW * ES), cb_addr, lin_scale);
            } else {
                const Tap* vp = p.taps + __ldg(p.tap_ptr + g * cp1 + c0);
                unsigned pc = __ldg(&vp->payload);
                for (int cl = 0; cl < ncl; ++cl) {
                    const int c = c0 + cl;
                    unsigned mk[NW];
                    const unsigned* mp = p.masks + ((size_t)g * C + c) * NW;
                    unsigned any = 0;
#pragma unroll
                    for (int i = 0; i < NW; ++i) { mk[i] = __ldg(mp + i); any |= mk[i]; }
                    if (any == 0) continue;
#pragma unroll
                    for (int j = 0; j < NBT; ++j) {
                        const TIO* pl = xb + (size_t)(j * p.cc + cl) * plane_s;
#pragma unroll
                        for (int yy = 0; yy < PH; ++yy) {
                            float* d = &pt[(j * PH + yy) * PW];
                            const TIO* rp = pl + yy * ROW;
                            if constexpr (PAD > 0) load_row<PAD, ES, TIO>(d, rp);
                            load_row<TW, MID_ALIGN, TIO>(d + PAD, rp + PAD);
                            if constexpr (RIGHT > 0) load_row<RIGHT, MID_ALIGN, TIO>(d + PAD + TW, rp + PAD + TW);
                        }
                    }
                    TapLoop<R, S, PAD, KT, NBT, TH, TW, WF, MODE, DISPATCH, F16IO>::run(acc, pt, vp, pc, mk, cb_addr,
                                                                                       lin_scale);
                }
            }
        }
        __syncthreads();
    }

    // ---- epilogue: optional ReLU / 2x2 max-pool, store in the IO dtype
    if (g >= p.groups) return;
    const bool relu = p.flags & SCB_FLAG_RELU;
    const bool pool = p.flags & SCB_FLAG_POOL2;
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) {
        const int k = k0 + kk;
        if (k >= p.k) break;
#pragma unroll
        for (int j = 0; j < NBT; ++j) {
            const int n = n0 + ti * NBT + j;
            if (n >= p.n) continue;
            const float* a = &acc[kk * P + j * TH * TW];
            if (!pool) {
                const int64_t pbase = ((int64_t)n * p.k + k) * p.e * p.f;
#pragma unroll
                for (int yy = 0; yy < TH; ++yy) {
                    const int oy = oy0 + ty * TH + yy;
                    if (oy >= p.e) continue;
                    const int ox0t = ox0 + tx * TW;
                    TIO* yrow = static_cast<TIO*>(p.y) + pbase + (int64_t)oy * p.f + ox0t;
                    if constexpr (!F16IO && TW == 4) {
                        if (ox0t + 4 <= p.f && ((reinterpret_cast<uintptr_t>(yrow) & 15) == 0)) {
                            float4 v = make_float4(a[yy * TW], a[yy * TW + 1], a[yy * TW + 2], a[yy * TW + 3]);
                            if (relu) {
                                v.x = v.x < 0.f ? 0.f : v.x; v.y = v.y < 0.f ? 0.f : v.y;
                                v.z = v.z < 0.f ? 0.f : v.z; v.w = v.w < 0.f ? 0.f : v.w;
                            }
                            *reinterpret_cast<float4*>(yrow) = v;
                            continue;
                        }
                    }
#pragma unroll
                    for (int xx = 0; xx < TW; ++xx) {
                        if (ox0t + xx >= p.f) continue;
                        float o = a[yy * TW + xx];
                        if (relu) o = relu_io<TIO>(o);
                        if constexpr (F16IO) yrow[xx] = __float2half_rn(o);
                        else yrow[xx] = o;
                    }
                }
            } else {
                const int pe = p.e >> 1, pf = p.f >> 1;
                const int64_t pbase = ((int64_t)n * p.k + k) * pe * pf;
#pragma unroll
                for (int yy = 0; yy < TH; yy += 2) {
                    const int oy = (oy0 + ty * TH + yy) >> 1;
                    if (oy >= pe) continue;
#pragma unroll
                    for (int xx = 0; xx < TW; xx += 2) {
                        const int ox = (ox0 + tx * TW + xx) >> 1;
                        if (ox >= pf) continue;
                        float o = fmaxf(fmaxf(a[yy * TW + xx], a[yy * TW + xx + 1]),
                                        fmaxf(a[(yy + 1) * TW + xx], a[(yy + 1) * TW + xx + 1]));
                        if (relu) o = relu_io<TIO>(o);
                        TIO* yp = static_cast<TIO*>(p.y) + pbase + (int64_t)oy * pf + ox;
                        if constexpr (F16IO) *yp = __float2half_rn(o);
                        else *yp = o;
                    }
                }
            }
        }
    }
}

template <int R, int S, int PAD, int KT, int NBT, int TH, int TW, bool F16IO, int WF, int MODE, int DISPATCH,
          int MINB>
cudaError_t launch_tiled_t(const TiledParams& p, unsigned grid, unsigned threads, size_t smem, cudaStream_t st) {
    auto kern = k_tiled<R, S, PAD, KT, NBT, TH, TW, F16IO, WF, MODE, DISPATCH, MINB>;
    static int lim[64];  // per device (the attribute is per device)
    const cudaError_t e = dyn_smem_ok(kern, smem, lim);
    if (e != cudaSuccess) return e;
    kern<<<grid, threads, smem, st>>>(p);
    return cudaGetLastError();
}

}  // namespace scb
