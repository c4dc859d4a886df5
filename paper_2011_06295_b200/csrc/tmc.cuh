// Tensor-memory image-lane kernel with a TMA -> tcgen05.cp fill (sm_100a,
// kind 7): the tmi.cuh tap loop, fed without any per-lane fill work.
//
// tmi.cuh fills TMEM from registers (shared -> registers -> tcgen05.st), one
// filler warp per lane quarter; measured with tools/tmi_harness.cu that filler
// is the critical path (~1800 cycles per stage on conv4_2, the consumers wait
// half of it).  Here ONE thread moves the data, entirely asynchronously:
//
//  * TMA (cp.async.bulk.tensor.4d) loads, per stage and 16-byte column chunk,
//    the box {4 columns, 32 images, H rows, CS channels} of x viewed as
//    (w, n, h, c): shared [c][h][n][16 bytes].  (A TMA box may not start at a
//    negative or unaligned innermost coordinate -- measured: "illegal
//    instruction", tools/tma_test.cu -- so the zero padding cannot come from
//    the out-of-bounds fill on the column axis.)
//  * For every (channel, row, chunk) one tcgen05.cp.32x128b.warpx4 moves the
//    32 images x 16 bytes into TMEM of all four lane quarters at once
//    (lane = image), and tcgen05.commit signals the stage's mbarrier.
//  * TMEM row layout: [4 zero columns][W data columns], RP = W + 4 columns per
//    input row, H rows per channel slot with one all-zero row between slots.
//    The zero columns / rows are written once at kernel start and never
//    touched again: they ARE the zero padding of shapes.py:98-105.  The window
//    of tap (r, s) for output row e is the W contiguous columns starting at
//    row (e + r - 1), column 3 + s: one tcgen05.ld.32x32b.x{W} per output row.
//
// Consumers (warps 1..4*WQ, KW output channels each) accumulate exactly like
// tmi.cuh -- bias, then FMUL+FADD per tap in colidx order, bit-identical to
// _kernels.py:73-84.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "tmi.cuh"

namespace scb {

struct TmcParams {
    CUtensorMap tmap;       // x as (w, n, h, c), box {4, 32, H, CS}, out-of-bounds zero fill
    const float* bias;
    float* y;
    const TmiTap* taps;     // col = (c % CS)*SLOTC + (r-1)*RP + 3 + s (mod 2^32), relative to the stage set
    const int32_t* tbase;
    const int32_t* soff;
    int n, c, k;
    int nst, nblk;
    int depth;              // TMA ring depth (stages of shared memory, <= 8)
    int tcap;
    int items;
    ActQuant aq;
    uint32_t flags;
};

// Geometry (host and device agree: layer.cu TmcG)
template <int W>
struct TmcGeom {
    static constexpr int H = W;
    static constexpr int RP = W + 4;                       // TMEM columns per input row (4 zero + W data)
    static constexpr int SLOTC = (H + 1) * RP;             // per channel: H data rows + one zero row
    static constexpr int Z0 = RP;                          // leading zero row
    static constexpr int NSLOT = (512 - RP) / SLOTC;
    static constexpr int CS = NSLOT >= 8 ? NSLOT / 4 : 1;  // channels per stage
    static constexpr int NSET = NSLOT / CS > 8 ? 8 : NSLOT / CS;
    static constexpr int CH = W / 4;                       // 16-byte column chunks per row
    static constexpr int IMGS = 128;                       // images per lane block (lane quarter q: 32q..32q+31)
    static constexpr int BOX = 16 * IMGS * H * CS;         // bytes of one TMA box (one column chunk)
    static constexpr int SLOT = CH * BOX;                  // bytes of one stage in the ring
    static_assert(W % 4 == 0 && NSET >= 2, "TMA fill: 16-byte rows; two stage sets");
};

// shared-memory matrix descriptor (tcgen05, SWIZZLE_NONE, K-major): 8-row core
// matrices of 16 bytes per row, core matrices SBO bytes apart
__device__ __forceinline__ uint64_t tmc_desc(uint32_t saddr, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3fff);
    d |= (uint64_t)((sbo >> 4) & 0x3fff) << 16;  // leading byte offset (one 16-byte column: unused)
    d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;  // stride byte offset
    d |= (uint64_t)1 << 46;                      // descriptor version (sm_100)
    return d;
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}

template <int W, int KW, int WQ, int MODE>
__global__ void __launch_bounds__(32 * (1 + 4 * WQ), 1) k_tmc(const __grid_constant__ TmcParams p) {
    using G = TmcGeom<W>;
    constexpr int H = G::H, RP = G::RP, SLOTC = G::SLOTC, Z0 = G::Z0, CS = G::CS, NSET = G::NSET, CH = G::CH;
    constexpr int BOX = G::BOX, SLOT = G::SLOT;
    constexpr int WIN = H * W;
    constexpr int NCW = 4 * WQ;
    constexpr int CAP = WQ * KW;   // channels per chunk: every channel is computed by one warp per quarter
    constexpr int IMGS = G::IMGS;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ unsigned taddr_s;
    __shared__ uint64_t full_b[NSET], empty_b[NSET];
    __shared__ uint64_t tma_b[8], sfree_b[8];

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int q4 = warp & 3;
    const int C = p.c, K = p.k;
    const int depth = p.depth;

    unsigned char* ring = smem;  // [depth][SLOT], 128-byte aligned boxes
    TmiTap* tsm = reinterpret_cast<TmiTap*>(smem + (size_t)depth * SLOT);
    int32_t* ssm = reinterpret_cast<int32_t*>(tsm + (size_t)CAP * p.tcap);

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 32) {
        for (int i = 0; i < NSET; ++i) {
            mbar_init(&full_b[i], 1);
            mbar_init(&empty_b[i], NCW);
        }
        for (int i = 0; i < depth; ++i) {
            mbar_init(&tma_b[i], 1);
            mbar_init(&sfree_b[i], 1);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tmem0 = taddr_s;
    // zero all 512 columns once (warps 1..4 = quarters 1,2,3,0): the never-rewritten zero
    // columns and rows are the convolution's zero padding
    if (warp >= 1 && warp <= 4) {
        const unsigned qb = tmem0 + ((unsigned)(32 * q4) << 16);
        float z[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) z[i] = 0.f;
        for (int c0 = 0; c0 < 512; c0 += 16) tmi_st16(qb + c0, z);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    asm volatile("griddepcontrol.wait;" ::: "memory");

    const int64_t T = p.items;
    const int64_t a_beg = T * blockIdx.x / gridDim.x, a_end = T * (blockIdx.x + 1) / gridDim.x;
    // chunks of at most CAP channels of one lane block, equal sizes
    auto next_chunk = [&](int64_t& a, int& blk, int& k0, int& nch) -> bool {
        if (a >= a_end) return false;
        blk = (int)(a / K);
        k0 = (int)(a % K);
        const int64_t left = min(a_end, (int64_t)(blk + 1) * K) - a;
        const int nchunks = (int)((left + CAP - 1) / CAP);
        nch = (int)((left + nchunks - 1) / nchunks);
        a += nch;
        return true;
    };
    if (warp == 0) {
        // ================= producer: one thread =================
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&p.tmap) : "memory");
            unsigned gt = 0, gc = 0;  // stages loaded by TMA / copied into TMEM (running counters)
            int64_t at = a_beg;
            int blk_t = 0, k0_t, nch_t, st_t = 0;
            bool t_live = next_chunk(at, blk_t, k0_t, nch_t);
            int64_t ac = a_beg;
            int blk_c, k0_c, nch_c;
            while (next_chunk(ac, blk_c, k0_c, nch_c)) {
                for (int s = 0; s < p.nst; ++s, ++gc) {
                    TMI_STAMP(0, s, 0);
                    // keep up to depth stages of TMA loads in flight
                    while (t_live && gt + 1 < gc + depth) {
                        const int slot = (int)(gt % depth);
                        if (gt >= (unsigned)depth) mbar_wait(&sfree_b[slot], ((gt / depth) - 1) & 1);
                        mbar_arrive_tx(&tma_b[slot], SLOT);
                        unsigned char* dst = ring + (size_t)slot * SLOT;
#pragma unroll
                        for (int chk = 0; chk < CH; ++chk)
                            asm volatile(
                                "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
                                " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst + chk * BOX)),
                                "l"(&p.tmap), "r"(4 * chk), "r"(blk_t * IMGS), "r"(0), "r"(st_t * CS),
                                "r"(smem_u32(&tma_b[slot]))
                                : "memory");
                        ++gt;
                        if (++st_t == p.nst) {
                            st_t = 0;
                            t_live = next_chunk(at, blk_t, k0_t, nch_t);
                        }
                    }
                    TMI_STAMP(0, s, 1);
                    const int slot = (int)(gc % depth);
                    mbar_wait(&tma_b[slot], (gc / depth) & 1);
                    TMI_STAMP(0, s, 2);
                    const int set = (int)(gc % NSET);
                    if (gc >= NSET) mbar_wait(&empty_b[set], ((gc / NSET) - 1) & 1);
                    TMI_STAMP(0, s, 3);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t sb = smem_u32(ring + (size_t)slot * SLOT);
                    const unsigned tset = tmem0 + (unsigned)(Z0 + set * CS * SLOTC);
                    const int ncl = min(CS, C - s * CS);
                    for (int cl = 0; cl < ncl; ++cl)
#pragma unroll
                        for (int h = 0; h < H; ++h)
#pragma unroll
                            for (int chk = 0; chk < CH; ++chk) {
                                // box [c][h][n][16 B]: (cl, h) = 128 images x 16 bytes -> lanes 0..127
                                const uint32_t src = sb + chk * BOX + ((cl * H + h) * IMGS) * 16;
                                const unsigned dcol = tset + (unsigned)(cl * SLOTC + h * RP + 4 + 4 * chk);
                                asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(dcol),
                                             "l"(tmc_desc(src, 128))
                                             : "memory");
                            }
                    TMI_STAMP(0, s, 4);
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                     smem_u32(&full_b[set]))
                                 : "memory");
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                     smem_u32(&sfree_b[slot]))
                                 : "memory");
                    TMI_STAMP(0, s, 5);
                }
            }
        }
        __syncwarp();
    } else {
        // ================= consumers =================
        const int cw = (warp - 1) >> 2;  // warp within its lane quarter (quarter = warp % 4 = image group)
        const unsigned tbase = tmem0 + ((unsigned)(32 * q4) << 16);
        unsigned g = 0;
        int64_t a = a_beg;
        int blk, k0, nch;
        while (next_chunk(a, blk, k0, nch)) {
            const int n0 = blk * IMGS + 32 * q4;  // this quarter's 32 images
            const int nimg = min(32, p.n - n0);
            // channel slot taps: loaded by the quarter-0 warp of each slot, published by a
            // consumer-only named barrier (the producer thread never joins it)
#pragma unroll
            for (int kk = 0; kk < KW; ++kk) {
                const int slot = cw + WQ * kk;
                if (q4 == 1 && slot < nch) {
                    const int k = k0 + slot;
                    const int t0 = __ldg(p.tbase + k), t1 = __ldg(p.tbase + k + 1);
                    const int4* src = reinterpret_cast<const int4*>(p.taps + t0);
                    int4* dst = reinterpret_cast<int4*>(tsm + (size_t)slot * p.tcap);
                    for (int i = lane; i < (t1 - t0) / 2; i += 32) cp_async<16>(dst + i, src + i);
                    const int32_t* so = p.soff + (size_t)k * (p.nst + 1);
                    int32_t* sd = ssm + (size_t)slot * (p.nst + 1);
                    for (int i = lane; i <= p.nst; i += 32) sd[i] = __ldg(so + i);
                }
            }
            cp_async_commit();
            float acc[KW][WIN];
#pragma unroll
            for (int kk = 0; kk < KW; ++kk) {
                const int slot = cw + WQ * kk;
                const float b = (p.bias != nullptr && slot < nch) ? __ldg(p.bias + k0 + slot) : 0.f;
#pragma unroll
                for (int j = 0; j < WIN; ++j) acc[kk][j] = b;
            }
            cp_async_wait<0>();
            asm volatile("bar.sync 1, %0;" ::"n"(NCW * 32) : "memory");
            for (int s = 0; s < p.nst; ++s, ++g) {
                const int set = (int)(g % NSET);
                if (cw == 0) TMI_STAMP(1, s, 0);
                mbar_wait(&full_b[set], (g / NSET) & 1);
                if (cw == 0) TMI_STAMP(1, s, 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const unsigned tset = tbase + (unsigned)(Z0 + set * CS * SLOTC);
#pragma unroll
                for (int kk = 0; kk < KW; ++kk) {
                    const int slot = cw + WQ * kk;
                    if (slot >= nch) break;
                    const int32_t* so = ssm + (size_t)slot * (p.nst + 1);
                    const int t0 = so[s];
#ifdef TMC_DEBUG
                    const int t1 = (p.flags & 0x1000u) ? t0 : so[s + 1];
#else
                    const int t1 = so[s + 1];
#endif
                    const TmiTap* tl = tsm + (size_t)slot * p.tcap;
#pragma unroll 2
                    for (int t = t0; t < t1; ++t) {
                        const TmiTap tp = tl[t];
                        const unsigned a0 = tset + tp.col;
                        float xv[H][W];
#pragma unroll
                        for (int e = 0; e < H; ++e) tmi_ld<W>(xv[e], a0 + e * RP);
#pragma unroll
                        for (int e = 0; e < H; ++e) tmi_wait<W>(xv[e]);
#pragma unroll
                        for (int e = 0; e < H; ++e)
#pragma unroll
                            for (int f = 0; f < W; ++f)
                                acc[kk][e * W + f] = mac1<MODE>(acc[kk][e * W + f], tp.v, xv[e][f]);
                    }
                }
                if (cw == 0) TMI_STAMP(1, s, 2);
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty_b[set]);
                if (cw == 0) { TMI_STAMP(1, s, 3); TMI_STAMP(1, s, 4); TMI_STAMP(1, s, 5); }
            }
            // ---- epilogue: lane = image, window index = e*W + f
            const bool aq = p.flags & SCB_FLAG_ACT_QUANT;
            const bool relu = p.flags & SCB_FLAG_RELU;
            const bool pool = p.flags & SCB_FLAG_POOL2;
            if (lane < nimg) {
                const int n = n0 + lane;
#pragma unroll
                for (int kk = 0; kk < KW; ++kk) {
                    const int slot = cw + WQ * kk;
                    if (slot >= nch) break;
                    const int k = k0 + slot;
                    if (aq) {
#pragma unroll
                        for (int j = 0; j < WIN; ++j)
                            acc[kk][j] = fq_store<float>(relu && acc[kk][j] < 0.f ? 0.f : acc[kk][j], p.aq);
                    }
                    if (!pool) {
                        float4* yp = reinterpret_cast<float4*>(p.y + ((int64_t)n * K + k) * WIN);
#pragma unroll
                        for (int j = 0; j < WIN; j += 4) {
                            float4 o = make_float4(acc[kk][j], acc[kk][j + 1], acc[kk][j + 2], acc[kk][j + 3]);
                            if (relu && !aq) {
                                if (o.x < 0.f) o.x = 0.f;
                                if (o.y < 0.f) o.y = 0.f;
                                if (o.z < 0.f) o.z = 0.f;
                                if (o.w < 0.f) o.w = 0.f;
                            }
                            yp[j / 4] = o;
                        }
                    } else {
                        constexpr int PW = W / 2;
                        float* yp = p.y + ((int64_t)n * K + k) * PW * PW;
#pragma unroll
                        for (int ro = 0; ro < H; ro += 2)
#pragma unroll
                            for (int f = 0; f < W; f += 2) {
                                const int b0 = ro * W + f;
                                float o = fmaxf(fmaxf(acc[kk][b0], acc[kk][b0 + 1]),
                                                fmaxf(acc[kk][b0 + W], acc[kk][b0 + W + 1]));
                                if (relu && !aq && o < 0.f) o = 0.f;
                                yp[(ro / 2) * PW + f / 2] = o;
                            }
                    }
                }
            }
            asm volatile("bar.sync 1, %0;" ::"n"(NCW * 32) : "memory");  // taps of this chunk no longer read
        }
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
}

template <int W, int KW, int WQ, int MODE>
cudaError_t launch_tmc_t(const TmcParams& p, unsigned grid, size_t smem, cudaStream_t st) {
    auto kern = k_tmc<W, KW, WQ, MODE>;
    static int lim[64];  // per device (the attribute is per device)
    const cudaError_t e = dyn_smem_ok(kern, smem, lim);
    if (e != cudaSuccess) return e;
    return launch_pdl(kern, p, grid, 32 * (1 + 4 * WQ), smem, st);
}

}  // namespace scb
