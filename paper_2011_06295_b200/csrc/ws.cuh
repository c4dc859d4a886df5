// Warp-specialised direct kernel (sm_100a): the direct kernel's tap loop
// (direct.cuh) fed by a producer warp through an mbarrier ring instead of
// CTA-wide __syncthreads.
//
// The isolated tap loop of direct.cuh runs at ~8 TMAC/s on B200 (one shared
// load per MAC: the 128 B/clk/SM shared-memory pipe is the ceiling;
// tools/mb_direct.cu); inside the kernel it reached ~60 % of that, the rest
// lost to per-stage barriers (every warp waits for the slowest warp of the
// stage) and to staging issued by the compute warps.  Here:
//
//  * warp WK (the last warp) is the producer: for every stage it waits on the
//    buffer's `empty` barrier, announces the stage's bytes on its `full`
//    barrier (mbarrier expect_tx) and issues 1D bulk copies
//    (cp.async.bulk ... mbarrier::complete_tx) of every in-image input row and
//    of each consumer warp's tap segments;
//  * consumer warps wait on `full`, run the tap loop, and release the buffer
//    with one arrive on `empty` -- no CTA barrier inside the channel loop, so
//    warps drift up to NB-1 stages apart and absorb the per-stage tap-count
//    imbalance;
//  * arithmetic, tap order and the zero-halo layout are those of direct.cuh,
//    so exact mode stays bit-identical to the reference (_kernels.py:73-84).
#pragma once

#include <cuda_runtime.h>

#include "direct.cuh"
#include "kernels.cuh"
#include "sparseconv_b200.h"
#include "tiled.cuh"

namespace scb {

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred P;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        " @!P bra WAIT_%=;\n}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

template <int R, int S, int PAD, int TH, int LW, int KW, int MODE>
__global__ void __launch_bounds__(288, 2) k_dws(const __grid_constant__ DirectParams p) {
    using RG = DirectRow<S, PAD, LW, 1, 4>;
    constexpr int XO = RG::XO, ROW = RG::ROW;
    constexpr int RT = TH + R - 1;
    constexpr int PLANE = RT * ROW;
    constexpr int G = 32 / LW;  // images per CTA
    extern __shared__ __align__(128) unsigned char smem[];

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int WK = p.wk, NB = p.nbuf;
    const int lx = lane % LW, lg = lane / LW;
    int bid = blockIdx.x;
    const int kb = bid % p.kblocks;
    bid /= p.kblocks;
    const int ey = bid % p.n_ey;
    const int nbk = bid / p.n_ey;
    const int n0 = nbk * G, oy0 = ey * TH;
    const int C = p.c, np1 = p.nst + 1;
    const int slot = (p.segcap + 3) & ~1;  // tap slot: segment copied from its 16-byte-aligned floor

    float* xs = reinterpret_cast<float*>(smem);
    DirectTap* tsm = reinterpret_cast<DirectTap*>(smem + (size_t)NB * p.stage_el * 4);
    int* sps = reinterpret_cast<int*>(tsm + (size_t)NB * WK * KW * slot);
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(
        (reinterpret_cast<uintptr_t>(sps + WK * KW * np1) + 7) & ~(uintptr_t)7);
    const unsigned full0 = smem_u32(bars), empty0 = smem_u32(bars + NB);

    {  // zero all stage buffers (the halo is never written again); stage pointers; barriers
        float4* z = reinterpret_cast<float4*>(smem);
        const int n16 = (NB * p.stage_el * 4) / 16;
        for (int i = tid; i < n16; i += blockDim.x) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        const int kc0 = kb * WK * KW;
        for (int i = tid; i < WK * KW * np1; i += blockDim.x) {
            const int k = kc0 + i / np1;
            sps[i] = k < p.k ? __ldg(p.sptr + (size_t)k * np1 + i % np1) : 0;
        }
        if (tid == 0) {
            for (int b = 0; b < NB; ++b) {
                mbar_init(full0 + 8 * b, 1);
                mbar_init(empty0 + 8 * b, WK);
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
    }

    if (warp == WK) {
        // ------------------------------------------------------------ producer
        const float* xg = static_cast<const float*>(p.x) + (size_t)n0 * C * p.h * p.w;
        const unsigned rowb = (unsigned)p.w * 4;
        const int gy0 = oy0 - PAD;
        const int y_lo = max(0, -gy0), y_hi = min(RT, p.h - gy0);  // in-image window rows
        const int ng = min(G, p.n - n0);
        for (int st = 0; st < p.nst; ++st) {
            const int buf = st % NB;
            if (st >= NB) mbar_wait(empty0 + 8 * buf, ((st / NB) - 1) & 1);
            const int c0 = st * p.cc;
            const int ncl = min(p.cc, C - c0);
            // bytes of the stage: input rows + tap segments (16-byte floors/ceilings)
            unsigned bytes = (unsigned)(ng * ncl * max(0, y_hi - y_lo)) * rowb;
            for (int q = 0; q < WK * KW; ++q) {
                const int t0 = sps[q * np1 + st], t1 = sps[q * np1 + st + 1];
                bytes += (unsigned)(((t1 + 1) & ~1) - (t0 & ~1)) * 8u;
            }
            if (lane == 0) mbar_arrive_tx(full0 + 8 * buf, bytes);
            __syncwarp();
            const unsigned fb = full0 + 8 * buf;
            const unsigned dst0 = smem_u32(xs + (size_t)buf * p.stage_el);
            const int nrows = ng * ncl * (y_hi - y_lo);
            for (int rr = lane; rr < nrows; rr += 32) {
                const int yy = y_lo + rr % (y_hi - y_lo), q = rr / (y_hi - y_lo);
                const int cl = q % ncl, g = q / ncl;
                const float* src = xg + (((size_t)g * C + c0 + cl) * p.h + gy0 + yy) * p.w;
                bulk_g2s(dst0 + 4u * (unsigned)(g * p.ip + cl * PLANE + yy * ROW + XO), src, rowb, fb);
            }
            for (int q = lane; q < WK * KW; q += 32) {
                const int t0 = sps[q * np1 + st], t1 = sps[q * np1 + st + 1];
                const int a0 = t0 & ~1, a1 = (t1 + 1) & ~1;
                if (a1 > a0)
                    bulk_g2s(smem_u32(tsm + ((size_t)buf * WK * KW + q) * slot), p.taps + a0, 8u * (a1 - a0), fb);
            }
        }
        return;
    }

    // -------------------------------------------------------------- consumers
    const int k0 = (kb * WK + warp) * KW;
    float acc[KW][TH];
#pragma unroll
    for (int kk = 0; kk < KW; ++kk) {
        const int k = k0 + kk;
        const float b = (p.bias != nullptr && k < p.k) ? p.bias[k] : 0.f;
#pragma unroll
        for (int j = 0; j < TH; ++j) acc[kk][j] = b;
    }
    const int lane_off = lg * p.ip + lx;
    for (int st = 0; st < p.nst; ++st) {
        const int buf = st % NB;
        mbar_wait(full0 + 8 * buf, (st / NB) & 1);
        const float* xl = xs + (size_t)buf * p.stage_el + lane_off - st * p.cc * PLANE;
#pragma unroll
        for (int kk = 0; kk < KW; ++kk) {
            const int k = k0 + kk;
            if (k >= p.k) break;
            const int* sp = sps + (warp * KW + kk) * np1 + st;
            const int t0 = sp[0], nt = sp[1] - t0;
            const DirectTap* seg = tsm + ((size_t)buf * WK * KW + warp * KW + kk) * slot + (t0 & 1);
#pragma unroll 4
            for (int t = 0; t < nt; ++t) {
                const DirectTap tp = seg[t];
                const float* xp = reinterpret_cast<const float*>(reinterpret_cast<const char*>(xl) + tp.off);
#pragma unroll
                for (int j = 0; j < TH; ++j) acc[kk][j] = mac1<MODE>(acc[kk][j], tp.v, xp[j * ROW]);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8 * buf);
    }

    // ---- epilogue (as direct.cuh, VX = 1)
    const int n = n0 + lg;
    const bool relu = p.flags & SCB_FLAG_RELU;
    const bool pool = p.flags & SCB_FLAG_POOL2;
#pragma unroll
    for (int kk = 0; kk < KW; ++kk) {
        const int k = k0 + kk;
        if (k >= p.k) break;
        if (!pool) {
            if (n < p.n && lx < p.f) {
                float* yp = static_cast<float*>(p.y) + (((int64_t)n * p.k + k) * p.e + oy0) * p.f + lx;
#pragma unroll
                for (int j = 0; j < TH; ++j) {
                    if (oy0 + j >= p.e) break;
                    float o = acc[kk][j];
                    if (relu && o < 0.f) o = 0.f;
                    yp[(int64_t)j * p.f] = o;
                }
            }
        } else {
            const int pe = p.e >> 1, pf = p.f >> 1;
#pragma unroll
            for (int j = 0; j < TH; j += 2) {
                float o = fmaxf(acc[kk][j], acc[kk][j + 1]);
                o = fmaxf(o, __shfl_xor_sync(0xffffffffu, o, 1));
                if (relu && o < 0.f) o = 0.f;
                const int py = (oy0 + j) >> 1;
                if (n < p.n && !(lx & 1) && lx < p.f && py < pe)
                    static_cast<float*>(p.y)[(((int64_t)n * p.k + k) * pe + py) * pf + (lx >> 1)] = o;
            }
        }
    }
}

template <int R, int S, int PAD, int TH, int LW, int KW, int MODE>
cudaError_t launch_dws_t(const DirectParams& p, unsigned grid, unsigned threads, size_t smem, cudaStream_t st) {
    auto kern = k_dws<R, S, PAD, TH, LW, KW, MODE>;
    static int lim[64];  // per device (the attribute is per device)
    const cudaError_t e = dyn_smem_ok(kern, smem, lim);
    if (e != cudaSuccess) return e;
    kern<<<grid, threads, smem, st>>>(p);
    return cudaGetLastError();
}

}  // namespace scb
