// TMEM-operand direct kernel (sm_100a, kind 5).
//
// The direct kernel (direct.cuh) streams one 4-byte input per MAC from shared
// memory and is bound by the 128 B/clk/SM shared-memory pipe.  Tensor memory
// reads (tcgen05.ld) run at ~260 B/clk/SM on B200 (tools/mb_tmem.cu), and a
// tcgen05.ld takes a WARP-UNIFORM column address while each lane reads its own
// TMEM lane -- exactly the access a warp-uniform tap needs: one instruction
// delivers a lane's TH inputs of tap (c, r, s).
//
// Layout: 4 subpartitions x M warps.  TMEM lane quarter p (warps w with
// w % 4 == p) holds the input strips of pixel set p: lane = (column x, image),
// and per staged input channel a 32-column slot
//     [s = 0: rows 0..TH+1][s = 1: rows 0..TH+1][s = 2: rows 0..TH+1][pad]
// holding column x+s-PAD of window rows oy0-PAD .. oy0+TH+R-2.  Tap (c, r, s)
// is then `tcgen05.ld.32x32b.x{TH}` at column slot(c) + s*(TH+R-1) + r.  Two
// 256-column buffers (8 channels each) double-buffer the stages; strips are
// filled from the zero-halo shared-memory window of direct.cuh (cp.async
// staging) with one tcgen05.st.32x32b.x32 per channel and lane.
//
// Warps of the same quarter share the strips and own different output
// channels (KW each, compile-time unrolled accumulators, tap blocks as in
// direct.cuh), so the accumulation order per output is the reference's
// colidx order and exact mode stays bit-identical (_kernels.py:73-84).
//
// Measured (profiles/r01_tmem_*): correct, but 4.1-4.4 TMAC/s vs 5.3-5.6 for
// direct.cuh on the VGG-CIFAR mid layers -- issue-bound: each tap pays
// R2UR (the TMEM address must be uniform), WARPSYNC and NOPs around the
// .sync.aligned tcgen05.ld besides the FMUL/FADD block, and the staging adds a
// shared->TMEM fill; the tuner keeps it as a candidate.
#pragma once

#include <cuda_runtime.h>

#include "direct.cuh"
#include "kernels.cuh"
#include "sparseconv_b200.h"
#include "tiled.cuh"

namespace scb {

template <int N>
struct TmLd;
template <>
struct TmLd<8> {
    static __device__ __forceinline__ void ld(float (&x)[8], unsigned a) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]), "=f"(x[4]), "=f"(x[5]), "=f"(x[6]), "=f"(x[7])
                     : "r"(a));
    }
};
template <>
struct TmLd<4> {
    static __device__ __forceinline__ void ld(float (&x)[4], unsigned a) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3])
                     : "r"(a));
    }
};
template <>
struct TmLd<2> {
    static __device__ __forceinline__ void ld(float (&x)[2], unsigned a) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=f"(x[0]), "=f"(x[1]) : "r"(a));
    }
};

__device__ __forceinline__ void tm_st32(unsigned a, const float (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(a),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
        "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
        "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
        "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
        : "memory");
}

__device__ __forceinline__ void tm_sync() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// TH: output rows per lane (<= 8), LW: output columns per lane group (= F),
// KW: output channels per warp, M: warps per TMEM lane quarter.
template <int R, int S, int PAD, int TH, int LW, int KW, int M, int MODE>
__global__ void __launch_bounds__(128 * M, 1) k_dtm(const __grid_constant__ DirectParams p) {
    using RG = DirectRow<S, PAD, LW, 1, 4>;
    constexpr int XO = RG::XO, ROW = RG::ROW;
    constexpr int RT = TH + R - 1;           // window rows (<= 10)
    constexpr int PLANE = RT * ROW;
    constexpr int GL = 32 / LW;              // images per lane set (one TMEM quarter)
    constexpr int G = 4 * GL;                // images per CTA
    constexpr int CC = 8;                    // channels per stage (8 x 32 columns per buffer)
    constexpr int SLOT = 32;
    static_assert(S * RT <= SLOT, "strips of one channel must fit a 32-column slot");
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ unsigned taddr_s;

    const int tid = threadIdx.x, nthreads = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int q4 = warp & 3, mw = warp >> 2;  // TMEM lane quarter, warp within the quarter
    const int lx = lane % LW, lg = lane / LW;
    int bid = blockIdx.x;
    const int kb = bid % p.kblocks;
    bid /= p.kblocks;
    const int ey = bid % p.n_ey;
    const int nbk = bid / p.n_ey;
    const int n0 = nbk * G, oy0 = ey * TH;
    const int C = p.c;
    float* xs = reinterpret_cast<float*>(smem);

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    {
        float4* z = reinterpret_cast<float4*>(smem);
        const int n16 = (2 * p.stage_el * 4) / 16;
        for (int i = tid; i < n16; i += nthreads) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const int rows = G * CC * RT;
    uint2* rdesc = reinterpret_cast<uint2*>(smem + (size_t)2 * p.stage_el * 4);
    const int hw = p.h * p.w;
    for (int rr = tid; rr < rows; rr += nthreads) {
        const int yy = rr % RT, q = rr / RT;
        const int cl = q % CC, g = q / CC;
        const int gy = oy0 - PAD + yy;
        const bool ok = n0 + g < p.n && (unsigned)gy < (unsigned)p.h;
        rdesc[rr] = make_uint2((unsigned)((g * C + cl) * hw + gy * p.w),
                               (unsigned)(g * p.ip + cl * PLANE + yy * ROW + XO) | ((unsigned)(ok ? cl : 255) << 24));
    }
    int4* tsm = reinterpret_cast<int4*>(smem + (size_t)2 * p.stage_el * 4 + (((size_t)rows * 8 + 15) & ~(size_t)15));
    constexpr int HDR = (KW * 4 + 15) / 16;
    const int groups = (p.k + KW - 1) / KW;
    tm_sync();
    const unsigned tbase = taddr_s + ((unsigned)(32 * q4) << 16);

    const float* xg = static_cast<const float*>(p.x) + (size_t)n0 * C * hw;
    const int nchunk = p.w / 4;
    auto stage = [&](int st, int buf) {  // global -> shared window (+ the M tap blocks)
        const int c0 = st * CC;
        const unsigned ncl = (unsigned)min(CC, C - c0);
        float* dst = xs + (size_t)buf * p.stage_el;
        const float* src = xg + (size_t)c0 * hw;
        for (int rr = tid; rr < rows; rr += nthreads) {
            const uint2 rd = rdesc[rr];
            if ((rd.y >> 24) < ncl) {
                const float* s = src + rd.x;
                float* d = dst + (rd.y & 0xffffffu);
                for (int q = 0; q < nchunk; ++q) cp_async<16>(d + 4 * q, s + 4 * q);
            }
        }
        if (q4 == 0) {  // one copy of each channel group's tap block per CTA
            const int grp = kb * M + mw;
            if (grp < groups) {
                const int o0 = __ldg(p.blkoff + (size_t)grp * p.nst + st);
                const int o1 = __ldg(p.blkoff + (size_t)grp * p.nst + st + 1);
                const int4* srcb = reinterpret_cast<const int4*>(p.taps) + o0;
                int4* tb = tsm + ((size_t)buf * M + mw) * p.segcap;
                const int nch = min(o1 - o0, p.segcap);
                for (int i = lane; i < nch; i += 32) cp_async<16>(tb + i, srcb + i);
            }
        }
    };
    // shared window -> TMEM strips of buffer tb (each warp of a quarter fills CC/M channels)
    const int lane_off = (q4 * GL + lg) * p.ip + XO - PAD + lx;
    auto fill = [&](int buf, int tb) {
        const float* w = xs + (size_t)buf * p.stage_el + lane_off;
        for (int cl = mw; cl < CC; cl += M) {
            float v[32];
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
                for (int y = 0; y < RT; ++y) v[s * RT + y] = w[cl * PLANE + y * ROW + s];
#pragma unroll
            for (int i = S * RT; i < 32; ++i) v[i] = 0.f;
            tm_st32(tbase + (unsigned)(tb * 256 + cl * SLOT), v);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    };

    float acc[KW][TH];
    const int k0 = (kb * M + mw) * KW;
#pragma unroll
    for (int kk = 0; kk < KW; ++kk) {
        const int k = k0 + kk;
        const float b = (p.bias != nullptr && k < p.k) ? p.bias[k] : 0.f;
#pragma unroll
        for (int j = 0; j < TH; ++j) acc[kk][j] = b;
    }

    asm volatile("griddepcontrol.wait;" ::: "memory");
    stage(0, 0);
    cp_async_commit();
    if (p.nst > 1) stage(1, 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    fill(0, 0);
    tm_sync();
    for (int st = 0; st < p.nst; ++st) {
        const int buf = st & 1;
        // ---- compute stage st from TMEM buffer `buf`
        const int4* tbk = tsm + ((size_t)buf * M + mw) * p.segcap;
        const int* cnt = reinterpret_cast<const int*>(tbk);
        const DirectTap* seg = reinterpret_cast<const DirectTap*>(tbk + HDR);
        const unsigned tb0 = tbase + (unsigned)(buf * 256) - (unsigned)(st * CC * SLOT);
#pragma unroll
        for (int kk = 0; kk < KW; ++kk) {
            const int k = k0 + kk;
            if (k >= p.k) break;
            const int nt = cnt[kk];
#pragma unroll 2
            for (int t = 0; t < nt; ++t) {
                const DirectTap tp = seg[t];
                float x[TH];
                TmLd<TH>::ld(x, tb0 + (unsigned)tp.off);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int j = 0; j < TH; ++j) acc[kk][j] = mac1<MODE>(acc[kk][j], tp.v, x[j]);
            }
            seg += nt;
        }
        // ---- next stage: shared window landed -> TMEM; refill the shared buffer just drained
        if (st + 1 < p.nst) {
            cp_async_wait<0>();
            __syncthreads();  // stage st+1's window visible to every warp
            fill(buf ^ 1, buf ^ 1);
            __syncthreads();  // every warp read shared buffer buf^1 ... and buffer buf's taps
            if (st + 2 < p.nst) stage(st + 2, buf);
            cp_async_commit();
        }
        tm_sync();  // TMEM buffer buf^1 complete; nobody still reads buffer buf
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    // ---- epilogue (direct.cuh, VX = 1): lane holds rows oy0.. of column lx of image n
    const int n = n0 + q4 * GL + lg;
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
    tm_sync();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
}

template <int R, int S, int PAD, int TH, int LW, int KW, int M, int MODE>
cudaError_t launch_dtm_t(const DirectParams& p, unsigned grid, unsigned threads, size_t smem, cudaStream_t st) {
    auto kern = k_dtm<R, S, PAD, TH, LW, KW, M, MODE>;
    static int lim[64];  // per device (the attribute is per device)
    const cudaError_t e = dyn_smem_ok(kern, smem, lim);
    if (e != cudaSuccess) return e;
    return launch_pdl(kern, p, grid, threads, smem, st);
}

}  // namespace scb
