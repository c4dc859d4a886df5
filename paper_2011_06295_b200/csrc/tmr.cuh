// Tensor-memory image-lane kernel, compact planes (sm_100a, kind 7) -- the
// VGG-CIFAR 4x4 layers (conv4_x).
//
// Lane = image.  Each input channel occupies W*W contiguous TMEM columns of
// its lane -- the NCHW plane itself -- with four zero columns between
// channel slots (the zero rows above / below the plane).  The window of tap
// (r, s) is the W*W contiguous columns starting at (r-1)*W + (s-1) relative
// to the plane: rows are exact, and the only wrong entries are column f = 0
// (s = 0) or f = W-1 (s = 2), which read the neighbouring row's edge instead
// of the zero padding.  For those outputs the kernel adds v (x) (+0) -- one
// FMUL per tap, then the FADDs -- exactly the reference's MAC with the padded
// zero (xpad = 0, shapes.py:98-105), so accumulation stays bit-identical to
// _kernels.py:73-84 (bias, then per tap in colidx order, mul and add rounded
// separately).  One tcgen05.ld.32x32b.x16 per tap; 20 TMEM columns per
// channel, 24 channel slots in the 512 columns.
//
// Why compact: the fill, not the MAC loop, bounds a TMEM kernel on these
// layers (tools/tmi_harness.cu traces: shifted copies -- 4x the data -- made
// the filler the critical path; tcgen05.cp moved ~10 B/clk).  Here:
//   TMA (cp.async.bulk.tensor.4d, box {4 columns, 32 images, W rows, CS
//   channels} of x viewed as (w, n, h, c), all coordinates >= 0) -> shared
//   ring -> one filler warp per TMEM lane quarter: W LDS.128 + one
//   tcgen05.st.32x32b.x16 per (lane, channel).
// All four quarters hold the same 32 images (each warp reads only its own
// quarter of TMEM), so a CTA computes 4*WQ*KW output channels from one
// staged input stream: L2 reads are a quarter of a 128-image lane block's.
//
// Synchronisation is by mbarriers only (no CTA barrier in the stage loop):
// tma[slot] (TMA -> fillers), sfree[slot] (4 fillers -> TMA issuer),
// full[q][set] (filler q -> consumers of quarter q), empty[q][set]
// (consumers -> filler).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "tmc.cuh"
#include "tmi.cuh"

namespace scb {

// Geometry (host and device agree: layer.cu TmrG)
template <int W>
struct TmrGeom {
    static constexpr int HW = W * W;                // window = plane
    static constexpr int PITCH = HW + W;            // plane + one zero row between channel slots
    static constexpr int BASE = 8;                  // first data column (windows reach W+1 columns left)
    static constexpr int NSLOT = (512 - BASE - W - 1) / PITCH;
    static constexpr int CS = NSLOT / 4;            // channels per stage
    static constexpr int NSET = 4;
    static constexpr int IMGS = 32;
    // TMA box {2 planes = 128 bytes, 32 images, CS/2 plane pairs} of x viewed as (2*HW, n, c/2),
    // 128-byte swizzle: shared row (pair, image) holds 8 16-byte chunks at chunk ^ (image & 7)
    static constexpr int SLOT = (CS / 2) * IMGS * 128;
    static_assert(HW == 16 && CS % 2 == 0 && SLOT % 1024 == 0, "4x4 planes, plane pairs");
};

// empty volatile asm "redefining" the accumulators: orders the MACs after the preceding
// (volatile) tcgen05.ld, so that load is in flight while they run
template <int N>
__device__ __forceinline__ void tmr_pin(float (&a)[N]) {
#pragma unroll
    for (int j = 0; j < N; j += 8)
        asm volatile("" : "+f"(a[j]), "+f"(a[j + 1]), "+f"(a[j + 2]), "+f"(a[j + 3]), "+f"(a[j + 4]), "+f"(a[j + 5]),
                     "+f"(a[j + 6]), "+f"(a[j + 7]));
}
// tcgen05.wait::ld for window x, after the accumulators' MACs (they flow through the asm)
template <int N>
__device__ __forceinline__ void tmr_wait2(float (&x)[N], float (&a)[N]) {
    tmr_pin<N>(a);
    tmi_wait<N>(x);
}
// one tap: acc (+)= v (x) window, with the wrapped edge column (s = 0: f = 0, s = 2: f = W-1)
// replaced by the reference's padded zero: acc (+) v (x) (+0)
template <int W, int MODE, int FZ>
__device__ __forceinline__ void tmr_mac_v(float (&acc)[W * W], float v, const float (&x)[W * W]) {
    float z = 0.f;
    if constexpr (FZ >= 0 && MODE == MODE_EXACT) z = __fmul_rn(v, 0.f);
#pragma unroll
    for (int e = 0; e < W; ++e)
#pragma unroll
        for (int f = 0; f < W; ++f) {
            const int j = e * W + f;
            if (f == FZ) {
                if constexpr (MODE == MODE_EXACT) acc[j] = __fadd_rn(acc[j], z);
                else acc[j] = __fmaf_rn(v, 0.f, acc[j]);
            } else {
                acc[j] = mac1<MODE>(acc[j], v, x[j]);
            }
        }
}
template <int W, int MODE>
__device__ __forceinline__ void tmr_mac(float (&acc)[W * W], const TmiTap& tp, const float (&x)[W * W]) {
    const unsigned sc = tp.col >> 16;
    if (sc == 1) tmr_mac_v<W, MODE, -1>(acc, tp.v, x);
    else if (sc == 0) tmr_mac_v<W, MODE, 0>(acc, tp.v, x);
    else tmr_mac_v<W, MODE, W - 1>(acc, tp.v, x);
}

// tap meta: bits 0..15 = window column + 8 relative to the stage set, bits 16..17 = s
template <int W, int KW, int WQ, int MODE>
__global__ void __launch_bounds__(32 * (4 + 4 * WQ), 1) k_tmr(const __grid_constant__ TmcParams p) {
    using G = TmrGeom<W>;
    constexpr int HW = G::HW, PITCH = G::PITCH, BASE = G::BASE, CS = G::CS, NSET = G::NSET, IMGS = G::IMGS;
    constexpr int SLOT = G::SLOT;
    constexpr int NCW = 4 * WQ;
    constexpr int CAP = NCW * KW;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ unsigned taddr_s;
    __shared__ uint64_t full_b[4][NSET], empty_b[4][NSET];
    __shared__ uint64_t tma_b[8], sfree_b[8];

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int q4 = warp & 3;
    const int C = p.c, K = p.k;
    const int depth = p.depth;

    // [depth][SLOT] ring, 1024-byte aligned (128-byte swizzle atoms); the host adds 1 KB of slack
    unsigned char* ring = smem + ((1024u - (smem_u32(smem) & 1023u)) & 1023u);
    TmiTap* tsm = reinterpret_cast<TmiTap*>(ring + (size_t)depth * SLOT);
    int32_t* ssm = reinterpret_cast<int32_t*>(tsm + (size_t)CAP * p.tcap);

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 32) {
        for (int q = 0; q < 4; ++q)
            for (int i = 0; i < NSET; ++i) {
                mbar_init(&full_b[q][i], 1);
                mbar_init(&empty_b[q][i], WQ);
            }
        for (int i = 0; i < depth; ++i) {
            mbar_init(&tma_b[i], 1);
            mbar_init(&sfree_b[i], 4);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tbase = taddr_s + ((unsigned)(32 * q4) << 16);
    if (warp < 4) {  // zero the quarter's 512 columns once: the zero rows are never rewritten
        float z[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) z[i] = 0.f;
        for (int c0 = 0; c0 < 512; c0 += 16) tmi_st16(tbase + c0, z);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    asm volatile("griddepcontrol.wait;" ::: "memory");

    const int64_t T = p.items;
    const int64_t a_beg = T * blockIdx.x / gridDim.x, a_end = T * (blockIdx.x + 1) / gridDim.x;
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

    if (warp < 4) {
        // ================= filler of lane quarter q4 (warp 0 lane 0 also issues the TMA) =================
        unsigned gt = 0, g = 0;
        int64_t at = a_beg;
        int blk_t = 0, k0_t, nch_t, st_t = 0;
        bool t_live = (warp == 0) && next_chunk(at, blk_t, k0_t, nch_t);
        if (warp == 0 && lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(&p.tmap) : "memory");
        int64_t a = a_beg;
        int blk, k0, nch;
        while (next_chunk(a, blk, k0, nch)) {
            for (int s = 0; s < p.nst; ++s, ++g) {
                if (warp == 0) TMI_STAMP(0, s, 0);
                if (warp == 0) {  // TMA issue: keep depth-1 stages in flight
                    while (t_live && gt + 1 < g + depth) {
                        const int slot = (int)(gt % depth);
                        if (gt >= (unsigned)depth) mbar_wait(&sfree_b[slot], ((gt / depth) - 1) & 1);
                        if (lane == 0) {
                            mbar_arrive_tx(&tma_b[slot], SLOT);
                            asm volatile(
                                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
                                " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(ring + (size_t)slot * SLOT)),
                                "l"(&p.tmap), "r"(0), "r"(blk_t * IMGS), "r"(st_t * (CS / 2)),
                                "r"(smem_u32(&tma_b[slot]))
                                : "memory");
                        }
                        __syncwarp();
                        ++gt;
                        if (++st_t == p.nst) {
                            st_t = 0;
                            t_live = next_chunk(at, blk_t, k0_t, nch_t);
                        }
                    }
                }
                if (warp == 0) TMI_STAMP(0, s, 1);
                const int slot = (int)(g % depth);
                mbar_wait(&tma_b[slot], (g / depth) & 1);
                if (warp == 0) TMI_STAMP(0, s, 2);
                const int set = (int)(g % NSET);
                if (g >= NSET) mbar_wait(&empty_b[q4][set], ((g / NSET) - 1) & 1);
                if (warp == 0) TMI_STAMP(0, s, 3);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const unsigned char* sb = ring + (size_t)slot * SLOT;
                const unsigned tset = tbase + (unsigned)(BASE + set * CS * PITCH);
#ifdef TMC_DEBUG
                const int ncl = (p.flags & 0x2000u) ? 0 : min(CS, C - s * CS);
#else
                const int ncl = min(CS, C - s * CS);
#endif
#pragma unroll 2
                for (int cl = 0; cl < CS; ++cl) {
                    if (cl >= ncl) break;
                    float v[16];
                    const unsigned char* row = sb + ((cl >> 1) * IMGS + lane) * 128;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int phys = ((cl & 1) * 4 + q) ^ (lane & 7);  // 128-byte swizzle
                        const float4 r4 = *reinterpret_cast<const float4*>(row + phys * 16);
                        v[4 * q] = r4.x;
                        v[4 * q + 1] = r4.y;
                        v[4 * q + 2] = r4.z;
                        v[4 * q + 3] = r4.w;
                    }
                    tmi_st16(tset + (unsigned)(cl * PITCH), v);
                }
                if (warp == 0) TMI_STAMP(0, s, 4);
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&full_b[q4][set]);
                    mbar_arrive(&sfree_b[slot]);
                }
                if (warp == 0) TMI_STAMP(0, s, 5);
            }
        }
    } else {
        // ================= consumers =================
        const int cw = warp - 4;  // quarter = warp % 4
        unsigned g = 0;
        int64_t a = a_beg;
        int blk, k0, nch;
        while (next_chunk(a, blk, k0, nch)) {
            const int n0 = blk * IMGS;
            const int nimg = min(IMGS, p.n - n0);
#pragma unroll
            for (int kk = 0; kk < KW; ++kk) {
                const int slot = cw + NCW * kk;
                if (slot < nch) {
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
            float acc[KW][HW];
#pragma unroll
            for (int kk = 0; kk < KW; ++kk) {
                const int slot = cw + NCW * kk;
                const float b = (p.bias != nullptr && slot < nch) ? __ldg(p.bias + k0 + slot) : 0.f;
#pragma unroll
                for (int j = 0; j < HW; ++j) acc[kk][j] = b;
            }
            cp_async_wait<0>();
            __syncwarp();
            for (int s = 0; s < p.nst; ++s, ++g) {
                const int set = (int)(g % NSET);
                if (cw == 0) TMI_STAMP(1, s, 0);
                mbar_wait(&full_b[q4][set], (g / NSET) & 1);
                if (cw == 0) TMI_STAMP(1, s, 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const unsigned tset = tbase + (unsigned)(BASE - 8 + set * CS * PITCH);
#pragma unroll
                for (int kk = 0; kk < KW; ++kk) {
                    const int slot = cw + NCW * kk;
                    if (slot >= nch) break;
                    const int32_t* so = ssm + (size_t)slot * (p.nst + 1);
                    const int t0 = so[s];
#ifdef TMC_DEBUG
                    const int t1 = (p.flags & 0x1000u) ? t0 : so[s + 1];
#else
                    const int t1 = so[s + 1];
#endif
                    const TmiTap* tl = tsm + (size_t)slot * p.tcap;
                    if (t0 < t1) {
                        // ping-pong windows: the tcgen05.ld of tap t+1 is in flight during tap t's MACs
                        TmiTap ta = tl[t0], tb;
                        float xa[HW], xb[HW];
                        tmi_ld<HW>(xa, tset + (ta.col & 0xffffu));
                        tmi_wait<HW>(xa);
                        int t = t0;
                        for (; t + 2 <= t1; t += 2) {
                            tb = tl[t + 1];
                            tmi_ld<HW>(xb, tset + (tb.col & 0xffffu));
                            tmr_pin<HW>(acc[kk]);
                            tmr_mac<W, MODE>(acc[kk], ta, xa);
                            tmr_wait2<HW>(xb, acc[kk]);
                            const bool more = t + 2 < t1;
                            if (more) {
                                ta = tl[t + 2];
                                tmi_ld<HW>(xa, tset + (ta.col & 0xffffu));
                                tmr_pin<HW>(acc[kk]);
                            }
                            tmr_mac<W, MODE>(acc[kk], tb, xb);
                            if (more) tmr_wait2<HW>(xa, acc[kk]);
                        }
                        if (t < t1) tmr_mac<W, MODE>(acc[kk], ta, xa);
                    }
                }
                if (cw == 0) TMI_STAMP(1, s, 2);
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty_b[q4][set]);
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
                    const int slot = cw + NCW * kk;
                    if (slot >= nch) break;
                    const int k = k0 + slot;
                    if (aq) {
#pragma unroll
                        for (int j = 0; j < HW; ++j)
                            acc[kk][j] = fq_store<float>(relu && acc[kk][j] < 0.f ? 0.f : acc[kk][j], p.aq);
                    }
                    if (!pool) {
                        float4* yp = reinterpret_cast<float4*>(p.y + ((int64_t)n * K + k) * HW);
#pragma unroll
                        for (int j = 0; j < HW; j += 4) {
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
                        for (int ro = 0; ro < W; ro += 2)
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
        }
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
}

template <int W, int KW, int WQ, int MODE>
cudaError_t launch_tmr_t(const TmcParams& p, unsigned grid, size_t smem, cudaStream_t st) {
    auto kern = k_tmr<W, KW, WQ, MODE>;
    static int lim[64];  // per device (the attribute is per device)
    const cudaError_t e = dyn_smem_ok(kern, smem, lim);
    if (e != cudaSuccess) return e;
    return launch_pdl(kern, p, grid, 32 * (4 + 4 * WQ), smem, st);
}

}  // namespace scb
