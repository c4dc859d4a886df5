// Register-tiled direct sparse convolution kernel (sm_100a).
//
// CTA = `wk` warp groups x `wp` pixel warps.  A warp group owns KT output
// channels (one tap group of the device program); every lane owns an
// NBT x TH x TW output tile (NBT images) and keeps KT x NBT x TH x TW f32
// accumulators in registers.  Input channels stream through a two-stage
// shared-memory pipeline, `cc` channels per stage:
//   STAGE_PLANE   whole input planes via cp.async.bulk (one bulk copy of cc
//                 contiguous planes per image, completion on an mbarrier).
//                 The zero padding of the reference (shapes.py:98-105) is
//                 never materialised: halo elements are predicated to 0.0 when
//                 the register patch is loaded.  (TMA tile loads would give the
//                 halo for free, but a box with negative start coordinates
//                 traps on B200 -- tools/tma_test.cu.)
//   STAGE_CPASYNC per-element cp.async with zero fill (any geometry).
// Per input channel a lane loads its (TH+R-1) x (TW+S-1) patch per image into
// registers once, then runs the warp group's taps of that channel through a
// generated PTX jump table (gen_taploop.py): each tap selects a fully unrolled
// block of MACs whose operands are registers at compile-time offsets.  Taps
// are ordered (c, kk, r, s), i.e. colidx order per accumulator
// (csr.py:143-160), so exact mode reproduces the reference bit for bit.
#pragma once

#include <cuda_runtime.h>

#include <type_traits>

#include "kernels.cuh"
#include "sparseconv_b200.h"

namespace scb {

template <int R, int S, int KT, int NBT, int TH, int TW, int WF, int MODE>
struct TapLoop;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    asm volatile(
        "{\n .reg .pred P1;\n WAIT:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        " @!P1 bra WAIT;\n}\n" ::"r"(smem_u32(b)), "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
                 "r"(valid ? 4 : 0));
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
// into dst[0..N), converting to f32.  Uses the widest shared loads allowed.
template <int N, int ALIGN, typename T>
__device__ __forceinline__ void load_row(float* dst, const T* src) {
    constexpr int ES = (int)sizeof(T);
    constexpr int A = ALIGN >= 16 ? 16 : ALIGN;
    int j = 0;
#pragma unroll
    for (int step = 0; step < 8; ++step) {
        // widest chunk size (bytes) usable at element j
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

// Patch of a lane from a dense H x W plane in shared memory, "same" padding
// (pad = (R-1)/2 = (S-1)/2): rows/cols outside the plane read as 0.0 -- the
// reference's materialised zero padding.  The TW middle columns start at the
// lane's tile origin and use one aligned vector load when W % TW == 0.
template <int R, int S, int TH, int TW, typename TIO>
__device__ __forceinline__ void load_patch_plane(float* pt, const TIO* plane, int py0, int px0, int H, int W,
                                                 bool vec_ok) {
    constexpr int PH = TH + R - 1, PW = TW + S - 1, PADS = (S - 1) / 2;
    constexpr int ES = (int)sizeof(TIO);
    const int ox = px0 + PADS;  // first output column of the tile
#pragma unroll
    for (int yy = 0; yy < PH; ++yy) {
        const int gy = py0 + yy;
        const bool row_ok = (unsigned)gy < (unsigned)H;
        const TIO* rp = plane + (row_ok ? gy : 0) * W;
        float* d = pt + yy * PW;
        if (vec_ok && row_ok && ox + TW <= W) {
            load_row<TW, TW * ES, TIO>(d + PADS, rp + ox);
#pragma unroll
            for (int xx = 0; xx < PADS; ++xx) {
                const int gx = px0 + xx;
                d[xx] = gx >= 0 ? to_f32(rp[gx]) : 0.f;
            }
#pragma unroll
            for (int xx = PADS + TW; xx < PW; ++xx) {
                const int gx = px0 + xx;
                d[xx] = gx < W ? to_f32(rp[gx]) : 0.f;
            }
        } else {
#pragma unroll
            for (int xx = 0; xx < PW; ++xx) {
                const int gx = px0 + xx;
                d[xx] = (row_ok && (unsigned)gx < (unsigned)W) ? to_f32(rp[gx]) : 0.f;
            }
        }
    }
}

template <int R, int S, int KT, int NBT, int TH, int TW, bool F16IO, int WF, int MODE, int STAGE>
__global__ void __launch_bounds__(256, 1) k_tiled(const __grid_constant__ TiledParams p) {
    using TIO = typename std::conditional<F16IO, __half, float>::type;
    constexpr int ES = (int)sizeof(TIO);
    constexpr int PH = TH + R - 1, PW = TW + S - 1;
    constexpr int P = NBT * TH * TW;
    constexpr int PADR = (R - 1) / 2, PADS = (S - 1) / 2;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bars[2];
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
    const int BHP = (STAGE == STAGE_PLANE) ? p.h : p.bh + R - 1;
    const int ROW = (STAGE == STAGE_PLANE) ? p.w : p.row;
    const int plane_s = BHP * ROW;  // elements per (image, channel)
    const int stage_el = ((p.imgs * p.cc * plane_s * ES + 127) & ~127) / ES;
    // bulk-copy destinations need 16-byte alignment; align the dynamic window
    // explicitly (the host adds 128 bytes of slack to the allocation)
    TIO* xs = reinterpret_cast<TIO*>(smem + ((128u - (smem_u32(smem) & 127u)) & 127u));

    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
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

    // ---- producer side -------------------------------------------------
    auto issue = [&](int ch, int buf) {  // STAGE_PLANE: executed by warp 0
        const int c0 = ch * p.cc;
        TIO* dst = xs + (size_t)buf * stage_el;
        {
            const int nc = min(p.cc, C - c0);
            const int ni = min(p.imgs, p.n - n0);
            const unsigned bytes = (unsigned)(nc * p.h * p.w * ES);
            if (lane == 0) mbar_expect_tx(&bars[buf], bytes * (unsigned)ni);
            __syncwarp();
            const TIO* src = static_cast<const TIO*>(p.x);
            for (int i = lane; i < ni; i += 32)
                bulk_load(dst + (size_t)i * p.cc * plane_s, src + ((size_t)(n0 + i) * C + c0) * p.h * p.w, bytes,
                          &bars[buf]);
        }
    };
    auto stage_cpasync = [&](int ch, int buf) {  // all threads
        const int c0 = ch * p.cc;
        TIO* dst = xs + (size_t)buf * stage_el;
        const int bwp = p.bw + S - 1;
        const int total = p.imgs * p.cc * BHP * bwp;
        // incremental mixed-radix walk (xx, yy, cl, img) with stride nthreads
        int i = tid;
        int xx = i % bwp, rowi = i / bwp;
        const int dxx = nthreads % bwp, drow = nthreads / bwp;
        int yy = rowi % BHP, pc = rowi / BHP;
        const int dyy = drow % BHP, dpc = drow / BHP;
        for (; i < total; i += nthreads) {
            const int cl = pc % p.cc, img = pc / p.cc;
            const int n = n0 + img, c = c0 + cl, gy = oy0 + yy - p.pad, gx = ox0 + xx - p.pad;
            const bool ok = n < p.n && c < C && gy >= 0 && gy < p.h && gx >= 0 && gx < p.w;
            TIO* d = dst + (size_t)pc * plane_s + yy * ROW + xx;
            const TIO* s = static_cast<const TIO*>(p.x);
            if constexpr (F16IO) {
                *d = ok ? s[(((size_t)n * C + c) * p.h + gy) * p.w + gx] : __float2half_rn(0.f);
            } else {
                cp_async4(d, ok ? s + (((size_t)n * C + c) * p.h + gy) * p.w + gx : s, ok);
            }
            xx += dxx;
            int carry = 0;
            if (xx >= bwp) { xx -= bwp; carry = 1; }
            yy += dyy + carry;
            pc += dpc;
            while (yy >= BHP) { yy -= BHP; ++pc; }
        }
    };

    // STAGE_PLANE: top-left input coordinate of this lane's patch ("same" padding)
    const int py0 = oy0 + ty * TH - p.pad, px0 = ox0 + tx * TW - p.pad;
    const bool vec_ok = (p.w % TW) == 0 && ((TW * ES) % 4) == 0 && p.pad == (S - 1) / 2;
    const int nch = (C + p.cc - 1) / p.cc;
    if constexpr (STAGE == STAGE_CPASYNC) {
        stage_cpasync(0, 0);
        cp_async_commit();
    } else {
        if (warp == 0) issue(0, 0);
    }
    const unsigned cb_addr = smem_u32(&qs.cb[0]);
    for (int ch = 0; ch < nch; ++ch) {
        const int buf = ch & 1;
        if constexpr (STAGE == STAGE_CPASYNC) {
            if (ch + 1 < nch) {
                stage_cpasync(ch + 1, buf ^ 1);
                cp_async_commit();
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncthreads();
        } else {
            if (ch + 1 < nch && warp == 0) issue(ch + 1, buf ^ 1);
            mbar_wait(&bars[buf], (unsigned)((ch >> 1) & 1));
        }
        if (g < p.groups) {
            const int c0 = ch * p.cc;
            const TIO* xb = xs + (size_t)buf * stage_el;
            int tb = __ldg(p.tap_ptr + g * cp1 + c0);
            for (int cl = 0; cl < p.cc; ++cl) {
                const int c = c0 + cl;
                if (c >= C) break;
                const int te = __ldg(p.tap_ptr + g * cp1 + c + 1);
                if (te == tb) continue;
                float pt[NBT * PH * PW];
#pragma unroll
                for (int j = 0; j < NBT; ++j) {
                    const TIO* pl = xb + (size_t)((ti * NBT + j) * p.cc + cl) * plane_s;
                    if constexpr (STAGE == STAGE_PLANE) {
                        load_patch_plane<R, S, TH, TW, TIO>(&pt[j * PH * PW], pl, py0, px0, p.h, p.w, vec_ok);
                    } else {
                        const TIO* rb = pl + (ty * TH) * ROW + tx * TW;
#pragma unroll
                        for (int yy = 0; yy < PH; ++yy)
                            load_row<PW, (TW * ES) & -(TW * ES), TIO>(&pt[(j * PH + yy) * PW], rb + yy * ROW);
                    }
                }
                TapLoop<R, S, KT, NBT, TH, TW, WF, MODE>::run(acc, pt, p.taps + tb, p.taps + te, cb_addr,
                                                              qs.scale);
                tb = te;
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
                            if (relu) { v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f); v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f); }
                            *reinterpret_cast<float4*>(yrow) = v;
                            continue;
                        }
                    }
#pragma unroll
                    for (int xx = 0; xx < TW; ++xx) {
                        if (ox0t + xx >= p.f) continue;
                        float o = a[yy * TW + xx];
                        if (relu && o < 0.f) o = 0.f;
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
                        if (relu && o < 0.f) o = 0.f;
                        TIO* yp = static_cast<TIO*>(p.y) + pbase + (int64_t)oy * pf + ox;
                        if constexpr (F16IO) *yp = __float2half_rn(o);
                        else *yp = o;
                    }
                }
            }
        }
    }
}

template <int R, int S, int KT, int NBT, int TH, int TW, bool F16IO, int WF, int MODE, int STAGE>
cudaError_t launch_tiled_t(const TiledParams& p, unsigned grid, unsigned threads, size_t smem, cudaStream_t st) {
    auto kern = k_tiled<R, S, KT, NBT, TH, TW, F16IO, WF, MODE, STAGE>;
    static int max_dyn = -1;  // benign race: idempotent
    if (max_dyn < 0) {
        cudaFuncAttributes fa;
        cudaError_t e = cudaFuncGetAttributes(&fa, kern);
        if (e != cudaSuccess) return e;
        const int lim = 227 * 1024 - (int)fa.sharedSizeBytes;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
        if (e != cudaSuccess) return e;
        max_dyn = lim;
    }
    if ((int)smem > max_dyn) return cudaErrorInvalidValue;
    kern<<<grid, threads, smem, st>>>(p);
    return cudaGetLastError();
}

}  // namespace scb
