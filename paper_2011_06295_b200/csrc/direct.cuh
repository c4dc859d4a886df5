// Dispatch-free direct sparse convolution kernel (sm_100a).
//
// The tiled/plane kernels keep an input patch in registers and jump to a
// per-(channel, r, s) MAC block for every tap (PTX brx.idx).  ncu shows that
// indirect branch -- LDC of the jump table, branch resolution, instruction
// fetch -- dominating their stalls (profiles/r01_*).  This kernel has no
// data-dependent control flow at all:
//
//  * a warp owns KW output channels (an unrolled, compile-time loop: the
//    accumulator index is never dynamic) and TH output rows of LW columns of
//    32/LW images -- lane = (column, image);
//  * taps are warp-uniform: for output channel k and the stage's input
//    channels the warp walks the reference's CSR row in colidx order
//    (csr.py:143-160), so every output accumulates exactly like
//    _kernels.py:73-84 (bias first, then v*x per nonzero, mul and add rounded
//    separately in exact mode);
//  * a tap is {v, off} with off = c*PLANE + r*ROW + s precomputed on upload;
//    a lane's input is xs[lane_base - c0*PLANE + off + j*ROW] -- one shared
//    load per MAC with an immediate row offset, lanes of a warp on 32
//    distinct banks (consecutive columns; images at a pitch = LW mod 32);
//  * input channels are staged `cc` at a time (two stages in flight,
//    16-byte cp.async) into zero-halo windows: the zero padding
//    (shapes.py:98-105) is the never-written halo of shared memory.
//
// Shared-memory bandwidth (4 B per MAC in fp32) bounds this kernel at about
// half of the FMUL+FADD issue rate; it trades the dispatch stalls for that
// predictable ceiling.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <type_traits>

#include "kernels.cuh"
#include "sparseconv_b200.h"
#include "tiled.cuh"

namespace scb {

struct __align__(8) DirectTap {
    float v;
    int32_t off;  // byte offset (c*PLANE + r*ROW + s) * 4
};

struct DirectParams {
    const void* x;
    const float* bias;        // f32, may be null
    void* y;
    const DirectTap* taps;    // reference CSR order (rowptr[k] .. rowptr[k+1])
    const int32_t* sptr;      // [K][nst+1]: first tap of channel k with c >= st*cc
    int n, c, h, w, k, e, f;
    int cc, nst, wk;          // channels per stage, stages, warps per CTA
    int ip;                   // image pitch in shared memory (elements)
    int stage_el;             // elements per stage (128-byte multiple)
    int kblocks, n_ey, nb;
    int segcap;               // taps per (output channel, stage) segment slot in shared memory
    int nbuf;                 // stage buffers in flight (2 or 3)
    int nfx;                  // k_direct WIDE: column tiles of LW per output row
    ActQuant aq;              // activation fake-quant (flags & SCB_FLAG_ACT_QUANT)
    QuantAux q;               // f16 kernels: in-register weight decode (codebook / scales)
    const int32_t* blkoff;    // k_direct: [group*nst + st] 16-byte-chunk offset of each tap block (+ end)
    uint32_t flags;
    int64_t ldy;              // SCB_FLAG_Y_IMAGE_MINOR: row stride of the image-minor output
};

// wait until at most NB-1 committed cp.async groups are pending
__device__ __forceinline__ void cp_async_wait_nb(int nbuf) {
    if (nbuf >= 3) cp_async_wait<2>();
    else cp_async_wait<1>();
}
// wait until at most NB-2 committed cp.async groups are pending (the stage
// about to be consumed has landed; the next one may still be in flight)
__device__ __forceinline__ void cp_async_wait_nb2(int nbuf) {
    if (nbuf >= 3) cp_async_wait<1>();
    else cp_async_wait<0>();
}

// Launch with programmatic stream serialization (PDL): the kernel's prologue
// (shared-memory zeroing, descriptors) overlaps the previous kernel's tail and
// `griddepcontrol.wait` orders the first read of its input.
template <typename K, typename P>
cudaError_t launch_pdl(K kern, const P& p, unsigned grid, unsigned threads, size_t smem, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (p.flags & SCB_FLAG_NO_PDL) ? 0 : 1;  // without it griddepcontrol.* are no-ops
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p);
    return e != cudaSuccess ? e : cudaGetLastError();
}

// Shared row geometry of a direct variant (host and device agree on it).
template <int S, int PAD, int LW, int VX, int ES = 4, bool WIDE = false>
struct DirectRow {
    static constexpr int Q16 = 16 / ES;  // elements per 16 bytes
    static constexpr int XO = Q16;       // shared column of input column 0 (16-byte aligned)
    // one copy of a row: left padding (XO >= the right halo), LW columns, rounded to 16 bytes.
    // VX = 1: the right halo reads the NEXT row's never-written left padding (zero), so
    // no right-halo columns are stored (the host leaves 16 zero bytes after each stage).
    // WIDE (column tiles of a wider row): the row also holds a real right halo.
    static constexpr int QW0 = WIDE ? XO + LW + Q16
                                    : (VX == 1 ? ((XO + LW) + Q16 - 1) / Q16 * Q16
                                               : ((XO + LW + S) + Q16 - 1) / Q16 * Q16);
    // VX = 2: rows (two copies) a multiple of 128 bytes apart would put every row's chunk i in
    // the same bank group during the shifted-copy pass; one more 16-byte chunk staggers them
    static constexpr int QW = (VX == 2 && !WIDE && (2 * QW0 * ES) % 128 == 0) ? QW0 + Q16 : QW0;
    static_assert(XO >= S - 1 - PAD, "right halo must fit in the next row's left padding");
    static constexpr int ROW = VX * QW;
    // shared column (relative to the lane's first output column) of tap column s
    static constexpr int col(int s) {
        return VX == 1 ? XO - PAD + s : (((s - PAD) % 2 == 0) ? XO + (s - PAD) : QW + XO + (s - PAD) + 1);
    }
};

// f16 storage: acc += v * x with one FHFMA (fma.rn.f32.f16, f16 x f16 + f32):
// the product of two f16 values is exact in f32, so this equals the
// reference's f32 multiply then add (shapes.py:93-95, engine.py:62-64).
__device__ __forceinline__ float fhfma(float acc, unsigned short v, unsigned short x) {
    asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(acc) : "h"(v), "h"(x));
    return acc;
}

// LW: output columns per lane group (= F when F <= 32), TH: output rows per
// lane, VX: adjacent output columns per lane (1 or 2; f16 storage needs 2).
// WIDE: output rows wider than LW are cut into column tiles (grid dimension
// nfx); each staged row then carries its real left/right halo columns.
// ONED (1D convolution, H = R = 1): a lane's TH outputs are columns lx + j*LW of
// one tile of TH*LW columns, staged as one contiguous row per (image, channel).
// WF (f16 storage only): weight format of the compact 4-byte taps (kernels.cuh tap_f16).
template <int R, int S, int PAD, int TH, int LW, int KW, int MODE, int VX, int MINB, bool F16IO = false,
          bool WIDE = false, bool ONED = false, int WF = WF_F32>
// (MINB = 2 variants may run 16 warps per CTA: 512 threads, one CTA per SM, same 128 registers)
__global__ void __launch_bounds__(MINB == 2 ? 512 : 256, MINB == 2 ? 1 : MINB) k_direct(const __grid_constant__ DirectParams p) {
    static_assert(F16IO == (WF != WF_F32), "f16 storage <=> compact f16 taps");
    static_assert(!F16IO || !WIDE, "f16 storage: narrow rows");
    static_assert(!WIDE || (VX == 1 && !F16IO), "wide tiles: f32, one column per lane");
    static_assert(!ONED || (WIDE && R == 1), "1D tiles are wide tiles of one input row");
    using TIO = typename std::conditional<F16IO, __half, float>::type;
    constexpr int ES = (int)sizeof(TIO);
    using RG = DirectRow<S, PAD, LW, VX, ES, WIDE>;
    constexpr int XO = RG::XO, QW = RG::QW, ROW = RG::ROW;
    constexpr int RT = ONED ? 1 : TH + R - 1;                        // staged rows per channel
    constexpr int PLANE = ONED ? XO + TH * LW + RG::Q16 : RT * ROW;  // elements per channel
    constexpr int JS = ONED ? LW : ROW;                              // smem stride of a lane's outputs
    constexpr int TC = ONED ? TH * LW : LW;                          // output columns per CTA tile
    constexpr int LPI = LW / VX;   // lanes per image row
    constexpr int G = 32 / LPI;    // images per CTA
    extern __shared__ __align__(128) unsigned char smem[];

    const int tid = threadIdx.x, nthreads = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int lx = (lane % LPI) * VX, lg = lane / LPI;
    int bid = blockIdx.x;
    const int kb = bid % p.kblocks;
    bid /= p.kblocks;
    const int ey = bid % p.n_ey;
    bid /= p.n_ey;
    const int fx = WIDE ? bid % p.nfx : 0;
    const int nbk = WIDE ? bid / p.nfx : bid;
    const int n0 = nbk * G, oy0 = ONED ? 0 : ey * TH, ox0 = fx * TC;
    const int k0 = (kb * p.wk + warp) * KW;
    const int C = p.c;
    TIO* xs = reinterpret_cast<TIO*>(smem);

    // zero both stages once: halo positions are never written again
    {
        float4* z = reinterpret_cast<float4*>(smem);
        const int n16 = (p.nbuf * p.stage_el * ES) / 16;
        for (int i = tid; i < n16; i += nthreads) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    // row descriptors after the stages: {src element offset from (n0, channel 0), dst | cl << 24}
    const int rows = G * p.cc * RT;
    uint2* rdesc = reinterpret_cast<uint2*>(smem + (size_t)p.nbuf * p.stage_el * ES);
    const int hw = p.h * p.w;
    for (int rr = tid; rr < rows; rr += nthreads) {
        const int yy = rr % RT, q = rr / RT;
        const int cl = q % p.cc, g = q / p.cc;
        const int gy = oy0 - PAD + yy;
        const bool ok = n0 + g < p.n && (unsigned)gy < (unsigned)p.h;
        rdesc[rr] = make_uint2((unsigned)((g * C + cl) * hw + gy * p.w),
                               (unsigned)(g * p.ip + cl * PLANE + yy * ROW + (WIDE ? 0 : XO)) |
                                   ((unsigned)(ok ? cl : 255) << 24));
    }
    __syncthreads();

    // tap blocks after the row descriptors: [buf][warp] slots of segcap 16-byte chunks; a
    // block is [KW int32 counts, padded to 16 B][taps of the KW channels, kk-major]
    int4* tsm = reinterpret_cast<int4*>(
        smem + (size_t)p.nbuf * p.stage_el * ES + (((size_t)rows * 8 + 15) & ~(size_t)15));
    constexpr int HDR = (KW * 4 + 15) / 16;  // header chunks
    const int grp = kb * p.wk + warp;        // this warp's channel group
    const int groups = (p.k + KW - 1) / KW;

    constexpr int Q16 = 16 / ES;
    // WIDE: a staged row is global columns ox0-XO .. ox0+ROW-XO-1, elements e_lo..e_hi of it
    // (in copies of ce elements: 16, 8 or 4 bytes as the row width's alignment allows)
    const TIO* xg = static_cast<const TIO*>(p.x) + (size_t)n0 * C * hw + (WIDE ? ox0 - XO : 0);
    const int e_lo = WIDE ? max(0, XO - ox0) : 0;  // first element at global column >= 0
    const int e_hi = WIDE ? min(ONED ? PLANE : ROW, p.w - (ox0 - XO)) : 0;
    // = layer.cu direct_copy_elems: the widest copy both the global and the shared row allow
    const int ce = (p.w % Q16 == 0 && ROW % Q16 == 0) ? Q16 : ((p.w % 2 == 0 && ROW % 2 == 0) ? 2 : 1);
    // narrow: 16-byte chunks per input row (rows have W == F == LW; derive() requires 16-byte rows)
    constexpr int CB = LW * ES >= 16 ? 16 : LW * ES;  // bytes per staged chunk (rows under 16 B: one)
    constexpr int QC = CB / ES;                        // elements per chunk
    constexpr int NCH = (LW * ES) / CB;
    auto stage = [&](int st, int buf) {
        const int c0 = st * p.cc;
        const unsigned ncl = (unsigned)min(p.cc, C - c0);
        TIO* dst = xs + (size_t)buf * p.stage_el;
        const TIO* src = xg + (size_t)c0 * hw;
        if constexpr (WIDE) {
            for (int rr = tid; rr < rows; rr += nthreads) {
                const uint2 rd = rdesc[rr];
                if ((rd.y >> 24) < ncl) {
                    const TIO* s = src + rd.x;
                    TIO* d = dst + (rd.y & 0xffffffu);
                    if (ce == Q16)
                        for (int q = e_lo; q < e_hi; q += Q16) cp_async<16>(d + q, s + q);
                    else if (ce == 2)
                        for (int q = e_lo; q < e_hi; q += 2) cp_async<8>(d + q, s + q);
                    else
                        for (int q = e_lo; q < e_hi; ++q) cp_async<4>(d + q, s + q);
                }
            }
        } else {
            // thread = (row, 16-byte chunk), chunk fastest: a warp's copies land in a few
            // contiguous shared-memory runs (one thread per row costs ~1 wavefront per thread)
            for (int it = tid; it < rows * NCH; it += nthreads) {
                const int rr = it / NCH, q = it % NCH;
                const uint2 rd = rdesc[rr];
                if ((rd.y >> 24) < ncl) cp_async<CB>(dst + (rd.y & 0xffffffu) + QC * q, src + rd.x + QC * q);
            }
        }
        // this warp's contiguous tap block of the stage: 16-byte chunks, one per lane
        if (grp < groups) {
            const int o0 = __ldg(p.blkoff + (size_t)grp * p.nst + st);
            const int o1 = __ldg(p.blkoff + (size_t)grp * p.nst + st + 1);  // blocks are consecutive
            const int4* src = reinterpret_cast<const int4*>(p.taps) + o0;
            int4* tb = tsm + ((size_t)buf * p.wk + warp) * p.segcap;
            const int nch = min(o1 - o0, p.segcap);
            for (int i = lane; i < nch; i += 32) cp_async<16>(tb + i, src + i);
        }
    };

    // VX = 2: P copy of every staged row = Q shifted right by one element
    auto shift = [&](int st, int buf) {
        const unsigned ncl = (unsigned)min(p.cc, C - st * p.cc);
        TIO* base = xs + (size_t)buf * p.stage_el;
        // thread = (row, chunk i of CB bytes), chunk fastest (conflict-free accesses); the
        // chunks cover the columns the odd taps read, XO .. XO+LW+S-1
        constexpr int NSH = (LW + S + QC - 1) / QC;
        for (int it = tid; it < rows * NSH; it += nthreads) {
            const int rr = it / NSH, i = it % NSH;
            const uint2 rd = rdesc[rr];
            if ((rd.y >> 24) >= ncl) continue;
            const TIO* q = base + (rd.y & 0xffffffu);  // Q[XO]
            TIO* pr = const_cast<TIO*>(q) + QW;         // P[XO]
            // last 32-bit word of the previous chunk (chunk -1 = the zero left padding)
            const unsigned prevw = *reinterpret_cast<const unsigned*>(q + QC * i - 4 / ES);
            if constexpr (CB == 16) {
                const uint4 cur = *reinterpret_cast<const uint4*>(q + QC * i);
                uint4 o;
                if constexpr (ES == 4) {
                    o = make_uint4(prevw, cur.x, cur.y, cur.z);
                } else {  // shift by one half: word w = (cur[w] << 16) | (prev word >> 16)
                    o = make_uint4(__funnelshift_l(prevw, cur.x, 16), __funnelshift_l(cur.x, cur.y, 16),
                                   __funnelshift_l(cur.y, cur.z, 16), __funnelshift_l(cur.z, cur.w, 16));
                }
                *reinterpret_cast<uint4*>(pr + QC * i) = o;
            } else if constexpr (CB == 8 && ES == 2) {  // f16 rows of 4: only 8-byte aligned
                const uint2 cur = *reinterpret_cast<const uint2*>(q + QC * i);
                *reinterpret_cast<uint2*>(pr + QC * i) =
                    make_uint2(__funnelshift_l(prevw, cur.x, 16), __funnelshift_l(cur.x, cur.y, 16));
            }
        }
    };

    __shared__ unsigned short cbt[16];  // WF_CB4: f16 codebook (published by the first stage barrier)
    if constexpr (WF == WF_CB4) {
        if (tid < 16) cbt[tid] = p.q.cb16[tid];
    }
    const float qscale = p.q.scale;
    const double qstep = p.q.step;

    float acc[KW][TH * VX];
#pragma unroll
    for (int kk = 0; kk < KW; ++kk) {
        const int k = k0 + kk;
        const float b = (p.bias != nullptr && k < p.k) ? p.bias[k] : 0.f;
#pragma unroll
        for (int j = 0; j < TH * VX; ++j) acc[kk][j] = b;
    }

    // programmatic dependent launch: everything above overlapped the previous layer's tail;
    // its output (our input) is visible after this wait
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int s0 = 0; s0 < p.nbuf - 1; ++s0) {  // prologue: nbuf-1 stages in flight
        if (s0 < p.nst) stage(s0, s0);
        cp_async_commit();
    }
    const int lane_off = lg * p.ip + lx;  // + tap off - c0*PLANE
    for (int st = 0; st < p.nst; ++st) {
        const int buf = st % p.nbuf;
        // one barrier per stage: it publishes stage st AND proves every warp has left
        // stage st-1, whose buffer the refill below then overwrites
        cp_async_wait_nb2(p.nbuf);
        __syncthreads();
        if constexpr (VX == 2) {
            shift(st, buf);
            __syncthreads();
        }
        if (st + p.nbuf - 1 < p.nst) stage(st + p.nbuf - 1, (st + p.nbuf - 1) % p.nbuf);
        cp_async_commit();  // possibly empty: keeps one group per iteration
        const TIO* xl = xs + (size_t)buf * p.stage_el + lane_off - st * p.cc * PLANE;
        const int4* tb = tsm + ((size_t)buf * p.wk + warp) * p.segcap;
        const int* cnt = reinterpret_cast<const int*>(tb);
        const DirectTap* seg = reinterpret_cast<const DirectTap*>(tb + HDR);
        const unsigned* segc = reinterpret_cast<const unsigned*>(tb + HDR);  // f16: compact taps
#pragma unroll
        for (int kk = 0; kk < KW; ++kk) {
            const int k = k0 + kk;
            if (k >= p.k) break;
            const int nt = cnt[kk];
#pragma unroll 4
            for (int t = 0; t < nt; ++t) {
                if constexpr (F16IO) {
                    const unsigned tw = segc[t];
                    const TIO* xp = xl + (tw & 0xffffu) + st * p.cc * PLANE;  // offsets are stage-relative
                    const unsigned short vh = tap_f16<WF>(tw >> 16, cbt, qscale, qstep);
                    if constexpr (VX == 1) {  // one half per MAC: no shifted copy needed
#pragma unroll
                        for (int j = 0; j < TH; ++j)
                            acc[kk][j] = fhfma(acc[kk][j], vh, *reinterpret_cast<const unsigned short*>(xp + j * JS));
                    } else {
#pragma unroll
                        for (int j = 0; j < TH; ++j) {
                            const unsigned w2 = *reinterpret_cast<const unsigned*>(xp + j * ROW);
                            acc[kk][2 * j] = fhfma(acc[kk][2 * j], vh, (unsigned short)(w2 & 0xffffu));
                            acc[kk][2 * j + 1] = fhfma(acc[kk][2 * j + 1], vh, (unsigned short)(w2 >> 16));
                        }
                    }
                    continue;
                }
                const DirectTap tp = seg[t];
                const TIO* xp = reinterpret_cast<const TIO*>(reinterpret_cast<const char*>(xl) + tp.off);
                if constexpr (F16IO) {
                } else if constexpr (VX == 1) {
#pragma unroll
                    for (int j = 0; j < TH; ++j) acc[kk][j] = mac1<MODE>(acc[kk][j], tp.v, xp[j * JS]);
                } else {
#pragma unroll
                    for (int j = 0; j < TH; ++j) {
                        const float2 v2 = *reinterpret_cast<const float2*>(xp + j * ROW);
                        acc[kk][2 * j] = mac1<MODE>(acc[kk][2 * j], tp.v, v2.x);
                        acc[kk][2 * j + 1] = mac1<MODE>(acc[kk][2 * j + 1], tp.v, v2.y);
                    }
                }
            }
            seg += nt;
            segc += nt;
        }
    }

    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // next layer may start its prologue
    // ---- epilogue: lane holds rows oy0..oy0+TH-1 of columns lx..lx+VX-1 of image n0+lg
    const int n = n0 + lg;
    const bool aq = p.flags & SCB_FLAG_ACT_QUANT;
    // activation fake-quant in place, ahead of the stores: ReLU then the quantizer (store.py:
    // 284-286); the quantizer is monotone, so it commutes with the 2x2 max-pool below
    if (aq) {
        const bool r0 = p.flags & SCB_FLAG_RELU;
#pragma unroll
        for (int kk = 0; kk < KW; ++kk)
#pragma unroll
            for (int j = 0; j < TH * VX; ++j) acc[kk][j] = fq_store<TIO>(r0 ? relu_io<TIO>(acc[kk][j]) : acc[kk][j], p.aq);
    }
    const bool relu = (p.flags & SCB_FLAG_RELU) && !aq;  // (already applied with the quantizer)
    const bool pool = p.flags & SCB_FLAG_POOL2;
    const bool ymin = !WIDE && !ONED && (p.flags & SCB_FLAG_Y_IMAGE_MINOR);
#pragma unroll
    for (int kk = 0; kk < KW; ++kk) {
        const int k = k0 + kk;
        if (k >= p.k) break;
        if constexpr (ONED) {  // E = 1: outputs (n, k, 0, ox0 + lx + j*LW)
            if (n < p.n) {
                TIO* yp = static_cast<TIO*>(p.y) + ((int64_t)n * p.k + k) * p.f + ox0 + lx;
#pragma unroll
                for (int j = 0; j < TH; ++j) {
                    float o0 = acc[kk][j];
                    if (relu) o0 = relu_io<TIO>(o0);
                    if (ox0 + lx + j * LW < p.f) yp[j * LW] = o0;
                }
            }
        } else if (!pool && ymin) {  // image-minor output: element (n, k, y, x) at ((k*E + y)*F + x)*ldy + n
            if (n < p.n && ox0 + lx < p.f) {
                const int jmax = min(TH, p.e - oy0);
#pragma unroll
                for (int j = 0; j < TH; ++j) {
                    if (j >= jmax) break;
#pragma unroll
                    for (int v = 0; v < VX; ++v) {
                        float o0 = acc[kk][j * VX + v];
                        if (relu) o0 = relu_io<TIO>(o0);
                        static_cast<TIO*>(p.y)[(((int64_t)k * p.e + oy0 + j) * p.f + ox0 + lx + v) * p.ldy + n] = (TIO)o0;
                    }
                }
            }
        } else if (!pool) {
            if (n < p.n && ox0 + lx < p.f) {
                // narrow variants have F == LW (derive), so row offsets are immediates
                constexpr int FP = WIDE ? 1 : LW;
                const int fpitch = WIDE ? p.f : 1;
                TIO* yp = static_cast<TIO*>(p.y) + (((int64_t)n * p.k + k) * p.e + oy0) * (WIDE ? p.f : LW) + ox0 + lx;
                const int jmax = min(TH, p.e - oy0);
#pragma unroll
                for (int j = 0; j < TH; ++j) {
                    if (j >= jmax) break;
                    float o0 = acc[kk][j * VX];
                    if (relu) o0 = relu_io<TIO>(o0);
                    if constexpr (VX == 1) {
                        yp[j * FP * fpitch] = (TIO)o0;
                    } else {
                        float o1 = acc[kk][j * VX + 1];
                        if (relu) o1 = relu_io<TIO>(o1);
                        if constexpr (F16IO)
                            *reinterpret_cast<__half2*>(yp + j * LW) = __floats2half2_rn(o0, o1);
                        else
                            *reinterpret_cast<float2*>(yp + j * LW) = make_float2(o0, o1);
                    }
                }
            }
        } else {
            const int pe = p.e >> 1, pf = p.f >> 1;
#pragma unroll
            for (int j = 0; j < TH; j += 2) {
                float o;
                if constexpr (VX == 1) {
                    o = fmaxf(acc[kk][j], acc[kk][j + 1]);
                    o = fmaxf(o, __shfl_xor_sync(0xffffffffu, o, 1));
                } else {
                    o = fmaxf(fmaxf(acc[kk][2 * j], acc[kk][2 * j + 1]), fmaxf(acc[kk][2 * j + 2], acc[kk][2 * j + 3]));
                }
                if (relu) o = relu_io<TIO>(o);
                const int py = (oy0 + j) >> 1;
                if (n < p.n && !(lx & 1) && ox0 + lx < p.f && py < pe) {
                    const int64_t pq = (int64_t)py * pf + ((ox0 + lx) >> 1);  // pooled position
                    const int64_t plane = (int64_t)pe * pf;
                    static_cast<TIO*>(p.y)[ymin ? ((int64_t)k * plane + pq) * p.ldy + n
                                                : ((int64_t)n * p.k + k) * plane + pq] = (TIO)o;
                }
            }
        }
    }
}

template <int R, int S, int PAD, int TH, int LW, int KW, int MODE, int VX, int MINB, bool F16IO = false,
          bool WIDE = false, bool ONED = false, int WF = (F16IO ? WF_F16 : WF_F32)>
cudaError_t launch_direct_t(const DirectParams& p, unsigned grid, unsigned threads, size_t smem, cudaStream_t st) {
    auto kern = k_direct<R, S, PAD, TH, LW, KW, MODE, VX, MINB, F16IO, WIDE, ONED, WF>;
    static int lim[64];  // per device (the attribute is per device)
    const cudaError_t e = dyn_smem_ok(kern, smem, lim);
    if (e != cudaSuccess) return e;
    return launch_pdl(kern, p, grid, threads, smem, st);
}

}  // namespace scb
