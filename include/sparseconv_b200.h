/*
 * sparseconv_b200.h -- C ABI of the B200 (sm_100a) direct sparse convolution
 * engine.  Plain pointers and sizes only: no torch, no C++ types.
 *
 * Each entry point names the reference interface it replaces (paths relative
 * to /root/reference/pkg/src/sparseconv).  The Python drop-in
 * (paper_2011_06295_b200/) binds these with ctypes; INTEGRATION.md shows the
 * binding a maintainer of the reference would add.
 *
 * Conventions
 *  - Every function returns an scb_status; on failure scb_last_error() returns
 *    a thread-local message.  SCB_ERR_SHAPE maps to the reference ShapeError
 *    (errors.py:8), SCB_ERR_FORMAT to FormatError (errors.py:12),
 *    SCB_ERR_CUDA / SCB_ERR_UNSUPPORTED to SparseConvError (errors.py:4).
 *  - Host arrays are C-contiguous.  Device arrays are device pointers in the
 *    current CUDA context of `device`.  `stream` is a cudaStream_t (NULL =
 *    legacy default stream).  scb_conv_sparse never allocates or synchronises:
 *    the device tables of a tiled launch are built by scb_layer_prepare (an
 *    unprepared launch fails with SCB_ERR_ARG), so a prepared launch can be
 *    captured into a CUDA graph.
 *  - dtype codes: the element type of activations/bias/values.
 */
#ifndef SPARSECONV_B200_H
#define SPARSECONV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SCB_API __attribute__((visibility("default")))
#else
#define SCB_API
#endif

typedef enum {
    SCB_OK = 0,
    SCB_ERR_SHAPE = 1,       /* -> ShapeError   (errors.py:8)  */
    SCB_ERR_FORMAT = 2,      /* -> FormatError  (errors.py:12) */
    SCB_ERR_INTEGRITY = 3,   /* -> IntegrityError (errors.py:16) */
    SCB_ERR_CUDA = 4,        /* -> SparseConvError */
    SCB_ERR_ARG = 5,         /* -> SparseConvError (bad pointer / size) */
    SCB_ERR_UNSUPPORTED = 6  /* -> SparseConvError */
} scb_status;

typedef enum { SCB_F32 = 0, SCB_F64 = 1, SCB_F16 = 2 } scb_dtype;

/* Weight payload formats of the device tap program.
 *  NATIVE : values stored in the activation dtype (f32 / f16 / f64)
 *  CB4    : 4-bit codebook index + a 16-entry table (the paper's "4b/16b",
 *           quantize.py:194-246; table = the layer's distinct values)
 *  LIN16  : int16 fixed-point code * 2^-frac (quantize.py:28-71)          */
typedef enum { SCB_W_NATIVE = 0, SCB_W_CB4 = 1, SCB_W_LIN16 = 2, SCB_W_AFF16 = 3 } scb_wfmt;

/* Geometry of one layer: ConvShape (shapes.py:17-77).  n is ignored by the
 * layer object (the batch comes from each call, engine.py:52-54). */
typedef struct {
    int32_t n, c, h, w, k, r, s, stride, padding;
} scb_shape;

/* Arithmetic modes (flags for scb_conv_sparse). */
#define SCB_FLAG_RELU      0x1u   /* fused max(.,0) epilogue (store.py:284)          */
#define SCB_FLAG_FAST      0x2u   /* f32: single-rounding FFMA instead of mul+add   */
#define SCB_FLAG_POOL2     0x4u   /* fused 2x2/2 max-pool epilogue (VGG stage glue) */
#define SCB_FLAG_GENERIC   0x8u   /* force the generic (any-geometry) kernel        */
#define SCB_FLAG_NO_PDL    0x10u  /* launch without programmatic dependent launch   */
#define SCB_FLAG_ACT_QUANT 0x20u  /* fused activation fake-quant epilogue with the
                                     layer's scb_act_quant (store.py:285-286)      */
#define SCB_FLAG_IMAGE_MINOR 0x40u /* x and y are IMAGE-MINOR: element (n, c, h, w) at
                                     ((c*H + h)*W + w)*ld + n (ld = the row stride of
                                     scb_conv_sparse_ld, = n for scb_conv_sparse); the
                                     layout of the kind-7 image-lane kernels, which only
                                     accept it (scb_to_image_minor converts NCHW)  */
#define SCB_FLAG_Y_IMAGE_MINOR 0x80u /* NCHW x, image-minor y (row stride ldy): the
                                     narrow direct kernels (kind 2, dispatch 0) write the
                                     next kind-7 layer's input layout directly       */
#define SCB_FLAG_Y_NCHW    0x100u /* with SCB_FLAG_IMAGE_MINOR: kind-7 kernels write an
                                     NCHW y (the last layer of an image-minor run)  */

/* Launch configuration: replaces EnginePlan.sub_batch_size (engine.py:28-39)
 * and the timed tune_sub_batch (engine.py:143-166). variant < 0 = generic. */
typedef struct {
    int32_t variant;   /* index into the compiled tiled-kernel table, -1 = generic */
    int32_t warps_k;   /* warp groups per CTA along output channels               */
    int32_t imgs;      /* images per CTA                                          */
    int32_t bh, bw;    /* output block per CTA                                    */
    int32_t cc;        /* input channels staged per pipeline stage                */
    int32_t stages;    /* shared-memory stage buffers in flight (direct kinds 2/3: 2 or 3,
                          kind 4: 2..4; 0 = default; ignored by tiled / plane)    */
} scb_launch;

/* Static description of a compiled tiled variant (for the tuner). */
typedef struct {
    int32_t r, s;        /* kernel extent it is specialised for */
    int32_t kt;          /* output channels per warp group (accumulator rows) */
    int32_t nbt, th, tw; /* images x rows x cols per thread */
    int32_t io;          /* scb_dtype of activations */
    int32_t wf;          /* payload: 0 f32, 1 f16, 2 codebook-4bit, 3 int16 fixed-point */
    int32_t mode;        /* 0 exact mul+add, 1 fma */
    int32_t dispatch;    /* tap dispatch: 0 brx.idx jump table, 1 per-channel mask walk;
                            direct kind: 2 = column tiles of tw for any output row width,
                            3 = 1D rows (H = R = 1) in tiles of th*tw columns;
                            kind 7: 1 / 2 = tap unroll of the whole-plane kernel, 3 = 4x4
                            quadrants of an 8x8 plane (5x5 windows), 4 = 4x4 output tiles of
                            a plane of 4-multiples >= 8x8 (6x6 zero-filled TMA windows,
                            padding taps executed; th = tw = 4) */
    int32_t pad;         /* padding the variant is specialised for */
    int32_t kind;        /* 0 tiled (output blocks, halo patches); 1 whole plane (th x tw = the
                            input plane a lane holds; small spatial extents); 2 direct
                            (dispatch-free: th rows x tw columns per lane group, kt = output
                            channels per warp); 3 image-lane direct (lane = image, whole
                            th x tw plane, shifted-copy vector loads); 4 warp-specialised
                            direct (producer warp + mbarrier ring, bulk copies); 5 direct with
                            tensor-memory operands (tcgen05.ld of a lane's tap inputs; nbt =
                            warps per TMEM lane quarter) */
} scb_variant_info;

/* ---------------------------------------------------------------------- */
/* host-side weight-format builder (csr.py)                               */
/* ---------------------------------------------------------------------- */

/* analyze_sparsity (csr.py:80-91): per-channel nonzero counts of a KCRS
 * tensor viewed as k rows of vol elements. */
SCB_API scb_status scb_channel_nnz(const void* w, scb_dtype dt, int32_t k, int64_t vol,
                                   int64_t* nnz_out);

/* select_padding_zeros (csr.py:94-117). out has room for `deficit`. */
SCB_API scb_status scb_select_padding_zeros(const void* flat, scb_dtype dt, int64_t len,
                                            int64_t deficit, int64_t* out);

/* build_csr (csr.py:120-165), two phases: count, then fill.  values are
 * raw element copies (sign of promoted -0.0 preserved). */
SCB_API scb_status scb_csr_count(const void* w, scb_dtype dt, const scb_shape* shape,
                                 int32_t unify, int64_t* nnz_out, int32_t* level_out);
SCB_API scb_status scb_build_csr(const void* w, scb_dtype dt, const scb_shape* shape,
                                 int32_t unify, int64_t nnz_cap, void* values,
                                 int32_t* colidx, int32_t* rowptr);

/* CsrKernel.validate (csr.py:50-73). */
SCB_API scb_status scb_validate_csr(const scb_shape* shape, const int32_t* colidx,
                                    const int32_t* rowptr, int64_t nnz,
                                    int32_t unified, int32_t level);

/* decompress (csr.py:168-178) into a zeroed dense KCRS buffer. */
SCB_API scb_status scb_decompress(const scb_shape* shape, scb_dtype dt, const void* values,
                                  const int32_t* colidx, const int32_t* rowptr,
                                  int64_t nnz, void* dense_out);

/* 64-bit FNV-1a of a byte range: the model-store blob checksum
 * (store.py:46-51 fnv1a64, pkg/docs/format.md "checksum"). */
SCB_API scb_status scb_fnv1a64(const void* data, int64_t size, uint64_t* out);

/* ---------------------------------------------------------------------- */
/* device layer: the uploaded, kernel-ready weights of one CsrKernel      */
/* ---------------------------------------------------------------------- */

typedef struct scb_layer scb_layer;

/* Upload a validated CSR (values in `dt`) as a device tap program.
 *  wfmt = CB4  : values must hold <= 16 distinct bit patterns
 *  wfmt = LIN16: values must be exactly code * 2^-frac with |code| < 2^15
 * (SCB_ERR_UNSUPPORTED otherwise). Allocates device memory on `device`. */
SCB_API scb_status scb_layer_create(const scb_shape* shape, scb_dtype dt, scb_wfmt wfmt,
                                    const void* values, const int32_t* colidx,
                                    const int32_t* rowptr, int64_t nnz, int32_t unified,
                                    int32_t device, scb_layer** out);
/* scb_layer_create with a quantizer parameter: for wfmt = AFF16 (symmetric affine
 * int16, quantize.py:99-138) `qstep` is the layer's step and every value must equal
 * the storage-dtype rounding of float64(code) * qstep for an int16 code -- the
 * reference's quantize_weights_array(.., "affine", 16) output (quantize.py:279-283);
 * the f16 kernels decode codes in registers.  qstep is ignored by other formats. */
SCB_API scb_status scb_layer_create_q(const scb_shape* shape, scb_dtype dt, scb_wfmt wfmt,
                                      const void* values, const int32_t* colidx,
                                      const int32_t* rowptr, int64_t nnz, int32_t unified,
                                      int32_t device, double qstep, scb_layer** out);
SCB_API scb_status scb_layer_destroy(scb_layer* layer);
/* device bytes of the tap program used by `variant` (-1 = generic arrays). */
SCB_API scb_status scb_layer_weight_bytes(const scb_layer* layer, int32_t variant,
                                          int64_t* bytes);

/* conv_sparse (engine.py:68-87) on device buffers.
 *  x: (n, C, H, W) in the layer dtype; bias: (K,) in the COMPUTE dtype
 *  (f32 for f16/f32 layers, f64 for f64; engine.py:55-60) or NULL (zeros);
 *  y: (n, K, E, F), or (n, K, E/2, F/2) with SCB_FLAG_POOL2.
 *  cfg NULL = the heuristic default launch for this shape.
 * Replaces _kernels.conv_sparse_kernel (_kernels.py:53-85) and
 * conv_sparse1d_kernel (_kernels.py:88-114). Asynchronous on `stream`. */
SCB_API scb_status scb_conv_sparse(const scb_layer* layer, const void* x, const void* bias,
                                   void* y, int32_t n, uint32_t flags,
                                   const scb_launch* cfg, void* stream);

/* scb_conv_sparse with explicit row strides of IMAGE-MINOR activations
 * (SCB_FLAG_IMAGE_MINOR): x rows (c, h, w) hold images at x[row*ldx + i], i < n, and
 * y rows likewise with ldy -- a sub-batch of a larger image-minor buffer is a pointer
 * offset by its first image with ld = the full batch.  Kind-7 launches need
 * ldx % 4 == 0 and a 16-byte aligned x (TMA).  With SCB_FLAG_Y_IMAGE_MINOR (NCHW x)
 * only ldy is used; with SCB_FLAG_Y_NCHW (image-minor x) y is NCHW and ldy is ignored.
 * Without any layout flag, ldx / ldy are ignored and this is scb_conv_sparse. */
SCB_API scb_status scb_conv_sparse_ld(const scb_layer* layer, const void* x, int64_t ldx,
                                      const void* bias, void* y, int64_t ldy, int32_t n,
                                      uint32_t flags, const scb_launch* cfg, void* stream);

/* Layout conversion for the image-minor kernels: x (n, chw) NCHW -> y[j*ldy + i]
 * (scb_to_image_minor) and back (scb_from_image_minor: x[j*ldx + i] -> y (n, chw)),
 * i < n, j < chw.  Asynchronous on `stream`. */
SCB_API scb_status scb_to_image_minor(scb_dtype dt, const void* x, void* y, int32_t n, int64_t chw,
                                      int64_t ldy, void* stream);
SCB_API scb_status scb_from_image_minor(scb_dtype dt, const void* x, int64_t ldx, void* y, int32_t n,
                                        int64_t chw, void* stream);

/* Build (allocate + upload, synchronously) the device tables launch `cfg`
 * (NULL = the default launch) reads for batch n and `flags`; idempotent.  The
 * reference rebuilds nothing per call either -- its CSR arrays are passed
 * straight to _kernels.conv_sparse_kernel (engine.py:83-84); this is the
 * one-time upload of their per-launch device layout. */
SCB_API scb_status scb_layer_prepare(scb_layer* layer, int32_t n, uint32_t flags, const scb_launch* cfg);
/* SCB_OK iff `cfg` is a valid launch of this layer for batch n and `flags`
 * (shape, shared-memory and grid rules); no device work. */
SCB_API scb_status scb_launch_check(const scb_layer* layer, int32_t n, uint32_t flags, const scb_launch* cfg);

/* Launch candidates for the tuner (replaces SUB_BATCH_CANDIDATES,
 * engine.py:25): writes up to `cap` configs valid for batch n. */
SCB_API scb_status scb_launch_candidates(const scb_layer* layer, int32_t n, uint32_t flags,
                                         scb_launch* out, int32_t cap, int32_t* count);
/* Heuristic default launch; prefer_imgs > 1 restricts it to configs with that
 * many images per CTA when one exists (EnginePlan.sub_batch_size: the
 * paper's images-per-block). */
SCB_API scb_status scb_default_launch(const scb_layer* layer, int32_t n, uint32_t flags,
                                      int32_t prefer_imgs, scb_launch* out);

SCB_API int32_t scb_variant_count(void);
SCB_API scb_status scb_variant_get(int32_t idx, scb_variant_info* out);

/* ---------------------------------------------------------------------- */
/* glue for network runners (Model.forward, store.py:263-292)             */
/* ---------------------------------------------------------------------- */

/* 2x2 stride-2 max pool over (n*c) planes of h x w (h, w even). */
SCB_API scb_status scb_maxpool2(scb_dtype dt, const void* x, void* y, int64_t planes,
                                int32_t h, int32_t w, void* stream);

/* Activation fake-quant parameters (the reference's layer.act_quant dict,
 * quantize.py:324-326; applied by fake_quant_activation, quantize.py:332-338):
 * a -> clip(a, clip_lo, clip_hi) in the activation dtype, code = clamp(rint((c - mu) / step))
 * in f64 over [0, 2^bits-1] (asymmetric) or [-(2^(bits-1)-1), 2^(bits-1)-1] (symmetric),
 * a' = (dtype)(mu + code * step).  Bit-identical to the reference. */
typedef struct {
    int32_t bits;
    int32_t symmetric;   /* 0: "asymmetric", 1: "symmetric" */
    double clip_lo, clip_hi, mu, step;
} scb_act_quant;

/* In-place fake-quant of `count` activations of dtype dt on `stream`
 * (replaces fake_quant_activation, quantize.py:332-338). */
SCB_API scb_status scb_fake_quant(scb_dtype dt, void* y, int64_t count, const scb_act_quant* q,
                                  void* stream);

/* Attach (q != NULL) or clear (NULL) a layer's activation quantizer; conv calls with
 * SCB_FLAG_ACT_QUANT apply it to the layer output (fused into the direct and
 * image-lane epilogues, a following scb_fake_quant pass for the other kernels). */
SCB_API scb_status scb_layer_set_act_quant(scb_layer* layer, const scb_act_quant* q);

/* ---------------------------------------------------------------------- */
/* measurement                                                            */
/* ---------------------------------------------------------------------- */

/* CUDA-core arithmetic peak microbenchmark on `device`.  For each probe i
 * writes name (<=15 chars) and MAC/s (multiply-accumulates per second) into
 * names[i*16] and macs_per_s[i].  Probes: ffma, ffma2, fmul_fadd,
 * fmul2_fadd, fmul_fadd2, fhfma, hfma2. Synchronous. */
SCB_API scb_status scb_fma_peaks(int32_t device, char* names, double* macs_per_s,
                                 int32_t cap, int32_t* count);

SCB_API const char* scb_last_error(void);
SCB_API const char* scb_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SPARSECONV_B200_H */
