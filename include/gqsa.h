/*
 * gqsa.h -- C ABI of libgqsa.so, the B200 (sm_100a) decode hot path of GQSA
 * (arXiv 2412.17560): a group-sparse, weight-only-quantized GEMV / small-batch
 * GEMM over the paper's Block-Sparse-Row (BSR) layout.
 *
 * Citations: PAPER.md:L = /root/reference/PAPER.md line (the paper's LaTeX),
 * SPEC.md:L likewise; DESIGN.md Rn = the readings listed in DESIGN.md §3.
 *
 * Operation (PAPER.md:64-69 [Eq. 3], 95-101 [§3.2 BSR listing], 134 [§3.5
 * "GEMV task of shape 1xNxK", "accessed according to the real group index"]):
 *
 *   y[b][r] = sum_{g in [row_index[r], row_index[r+1])} s_g *
 *             sum_{t < G} (q_{g,t} - z_g) * x[b][group_cols[g]*G + t]  (+ bias[r])
 *
 * accumulated in fp32 (no tensor cores at batch 1, PAPER.md:9, 134 step 4
 * "CudaCores (FMA)").  Results are deterministic: bit-identical reruns for a
 * fixed blob, batch, grid and device.
 *
 * Ownership: the caller owns every buffer, host and device.  The library
 * never allocates or frees device memory and keeps no pointer past a call.
 * A packed blob is immutable and may be shared by concurrent calls on
 * different streams, each with its OWN workspace.  A workspace
 * must be zero-filled once when allocated; every call leaves it zero again
 * (fix-up counters and record flags; the partial-sum words are scratch).
 * Forward progress never depends on CTA co-residency: the stream kernel's
 * fix-up (look-back) only waits for LOWER-indexed warps / CTAs of the same
 * launch, which never wait for a higher one, and CTAs are dispatched in index
 * order; the LAYOUT-TC kernel's fix-up only waits for records whose writers
 * have already arrived.
 *
 * Errors: every int-returning function returns GQSA_OK (0) or a negative
 * gqsa_status_t.  Errors raised during asynchronous device execution surface
 * at the next stream synchronisation (CUDA convention).
 *
 * Byte layout of the packed blob: DESIGN.md §5 ("LAYOUT v3").
 */
#ifndef GQSA_H_
#define GQSA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GQSA_MAGIC 0x41535147u   /* bytes "GQSA" little-endian */
#define GQSA_VERSION 3
#define GQSA_TILE_GROUPS 128     /* kept groups per tile record */
#define GQSA_MAX_COLS 32736      /* K limit: the u16 column field addresses 2K + 64 bytes */
#define GQSA_MAX_BATCH 8

typedef enum {
  GQSA_OK = 0,
  GQSA_ERR_SHAPE = -1,       /* dims mismatch, cols % G != 0, B not in [1,8], bad row range */
  GQSA_ERR_VALIDATION = -2,  /* BSR invariant violated (see gqsa_pack) or inconsistent blob */
  GQSA_ERR_UNSUPPORTED = -3, /* (bits, G) not in {2,4,8} x {16} or {4} x {8,32}; cols > GQSA_MAX_COLS */
  GQSA_ERR_BUFFER = -4,      /* null pointer, blob/workspace too small, misaligned device pointer */
  GQSA_ERR_CUDA = -5         /* CUDA launch / copy failure */
} gqsa_status_t;

/*
 * Plain host BSR.
 *   rows, cols    : N (out_features) and K (in_features) of W[N][K].
 *   group_size    : G, the sparse AND quantization group: 16 (the
 *                   paper's default) for every width; 8 or 32 for
 *                   W4 only (the group-size sweep).
 *   bits          : n, code width: 4 or 2 (the paper's W4/W2), or 8 (W8, the
 *                   paper's other deployed setting).
 *   nnzg          : number of kept groups = row_index[rows].
 *   row_index     : int32[rows+1] row offsets into the kept-group list (rowIndex).
 *   group_cols    : uint16[nnzg] column of each kept group IN GROUP UNITS (groups[]).
 *   codes         : ceil(nnzg*G*n/8) bytes, the kept groups' codes (values[]),
 *                   group-major in CSR order; element e at bits [e*n, e*n+n),
 *                   least-significant bits first (n=4: low nibble first,
 *                   SPEC.md:146).
 *   scales_f16    : uint16[nnzg] IEEE binary16 bit patterns of s_g.
 *   zeros_f16     : uint16[nnzg] binary16 bit patterns of z_g (any finite value,
 *                   not necessarily an integer: E2E-OQP tunes z).
 * For gqsa_unpack the caller allocates the arrays (sizes from gqsa_read_desc)
 * and the function fills them and the scalar fields.
 */
typedef struct {
  int32_t rows, cols, group_size, bits;
  int64_t nnzg;
  const int32_t* row_index;
  const uint16_t* group_cols;
  const uint8_t* codes;
  const uint16_t* scales_f16;
  const uint16_t* zeros_f16;
} gqsa_bsr_t;

/*
 * Offline compression front-end (host; PAPER.md:74-93 [Eq. 4, §3.2, Fig. 3],
 * 50-63 [Eq. 1-2]): dense W -> plain BSR of the kept, quantized groups.
 *   W          : host fp32 [rows][cols] (row-major, nn.Linear layout), finite.
 *   hinv_diag  : host fp64 [cols], diag(H^-1) of the layer's Hessian estimate
 *                (finite, > 0); Eq. 4 saliency s = W^2 / hinv_diag^2.
 *   sparsity   : S in [0, 1): exactly floor(S * rows*cols/G) groups (the
 *                lowest mean saliency of the layer; ties -> lower (row, group)
 *                index) are pruned.
 *   bits       : 2, 4 or 8;  group_size: G (any divisor of cols; the packer
 *                and kernels take G = 16 for every width, G = 8 / 32 for W4).
 *   out        : caller-allocated arrays: row_index int32[rows+1];
 *                group_cols/scales_f16/zeros_f16 [nnzg]; codes
 *                ceil(nnzg*G*bits/8) bytes, where nnzg = gqsa_compress_nnzg();
 *                scalar fields are filled in.  Quantization per kept group by
 *                Eq. 1-2 in fp64 (ties away from zero), s and z stored as
 *                fp16 (round to nearest even); constant groups: DESIGN.md R9.
 *   group_saliency : optional host fp64 [rows][cols/G] out (the group scores), or NULL.
 * Deterministic (fixed fp64 evaluation order).  Errors: GQSA_ERR_SHAPE (dims,
 * cols % G, S outside [0,1)), GQSA_ERR_UNSUPPORTED (bits, cols/G > 65536),
 * GQSA_ERR_VALIDATION (non-finite W, hinv_diag <= 0 or non-finite, s or z
 * not representable in fp16), GQSA_ERR_BUFFER (null pointers).
 */
int gqsa_compress_nnzg(int32_t rows, int32_t cols, int32_t group_size, double sparsity, int64_t* nnzg);
int gqsa_compress(const float* W, int32_t rows, int32_t cols, int32_t group_size, int32_t bits,
                  const double* hinv_diag, double sparsity, gqsa_bsr_t* out, double* group_saliency);

/* Host copy of a packed blob's header (filled by gqsa_pack / gqsa_read_desc). */
typedef struct {
  uint32_t magic, version;
  int32_t rows, cols, group_size, bits;
  int64_t nnzg;
  int32_t tile_groups, num_tiles;
  int32_t n_nzrows, n_empty;
  int32_t tile_bytes, flags;
  int32_t row_begin, row_end;     /* source row range this blob was packed from */
  int32_t num_slices, reserved0;
  uint64_t off_row_index, off_perm, off_empty, off_slice_tile0, off_tile_slice, off_tiles, blob_bytes;
} gqsa_desc_t;

/*
 * gqsa_pack_size: bytes needed to pack rows [row_begin, row_end) of `bsr`.
 * gqsa_pack: validate, then lay rows [row_begin, row_end) of `bsr` out as a
 *   device blob (offline pre-processing, "grouped by size G and
 *   saved ... along with scaling factors and zero points").  The row range
 *   lets each rank pack its output-row shard; row offsets are rebased.
 *   Validation: row_index[0] == 0, non-decreasing,
 *   row_index[rows] == nnzg; group_cols strictly increasing within a row and
 *   < cols/G; scales finite and > 0; zeros finite -> GQSA_ERR_VALIDATION.
 *   `blob` is host memory of at least gqsa_pack_size bytes; `desc` may be NULL.
 */
int gqsa_pack_size(const gqsa_bsr_t* bsr, int32_t row_begin, int32_t row_end, size_t* blob_bytes);
int gqsa_pack(const gqsa_bsr_t* bsr, int32_t row_begin, int32_t row_end,
              void* blob, size_t blob_bytes, gqsa_desc_t* desc);

/*
 * gqsa_pack_size_ex / gqsa_pack_ex: as gqsa_pack_size / gqsa_pack with a
 * choice of device layout:
 *   GQSA_LAYOUT_STREAM (gqsa_pack's): the sliced-ELL tile stream for the
 *     CUDA-core kernel -- the fastest at batch 1-2, every bit width and G.
 *   GQSA_LAYOUT_TC: W4, G = 16 only: rows in blocks of 16, each block's kept
 *     group columns stored as 16 x 16 code matrices (rows that do not keep a
 *     column: zero codes, s = z = 0) in tensor-core fragment order, for the
 *     batch 2-8 GEMM on mma.sync ("TensorCores (MMA) or
 *     CudaCores (FMA)").  It reads ~2x the bytes of the BSR at 50 % group
 *     sparsity but replaces 16 FMA per weight and batch column by one MMA per
 *     16 x 16 x 8 block.  gqsa_gemv / gqsa_gemm_* accept either blob.
 * GQSA_ERR_SHAPE for another layout value, GQSA_ERR_UNSUPPORTED for a TC
 * layout of bits != 4 or G != 16.
 */
#define GQSA_LAYOUT_STREAM 0
#define GQSA_LAYOUT_TC 1
int gqsa_pack_size_ex(const gqsa_bsr_t* bsr, int32_t row_begin, int32_t row_end, int32_t layout,
                      size_t* blob_bytes);
int gqsa_pack_ex(const gqsa_bsr_t* bsr, int32_t row_begin, int32_t row_end, int32_t layout,
                 void* blob, size_t blob_bytes, gqsa_desc_t* desc);

/* Parse and bounds-check a (host) blob header: magic, version, section
 * offsets, sizes.  GQSA_ERR_VALIDATION on any inconsistency. */
int gqsa_read_desc(const void* blob, size_t blob_bytes, gqsa_desc_t* desc);

/* Inverse of gqsa_pack (bit-exact): rebuild the plain BSR of the packed rows
 * from the tile stream, checking it against the stored row offsets.  `out`'s
 * array pointers must point to caller memory of the sizes given by the desc:
 * row_index int32[rows+1], group_cols/scales/zeros [nnzg], codes
 * ceil(nnzg*G*n/8) bytes. */
int gqsa_unpack(const void* blob, size_t blob_bytes, gqsa_bsr_t* out);

/* Workspace bytes a gemv/gemm (or grouped) call needs for `batch` columns on
 * the current device: per-warp fix-up partial-sum records and (LAYOUT-TC)
 * arrival counters.  It depends on the batch and the device's SM count, not on
 * the layer.  Zero-fill once; every call leaves it zero. */
int gqsa_workspace_size(const gqsa_desc_t* desc, int32_t batch, size_t* bytes);

/*
 * gqsa_gemv: y = W_hat x (+ bias), batch 1.
 *   d_blob : device copy of the packed blob (256-B aligned).
 *   d_x    : device fp16 bit patterns [cols] (16-B aligned).
 *   d_y    : device fp32 [rows] (written in full, empty rows = bias or 0).
 *   d_bias : device fp32 [rows] or NULL.
 *   d_ws / ws_bytes : workspace (see gqsa_workspace_size).
 *   stream : cudaStream_t (NULL = legacy default stream).
 * Asynchronous; graph-capturable.  Uses Programmatic Dependent Launch so that
 * weight fetch overlaps the previous kernel on the stream; activations are
 * read only after the previous kernel completes (unless the caller declares
 * them ready, gqsa_options_t.x_ready).
 */
int gqsa_gemv(const gqsa_desc_t* desc, const void* d_blob, const uint16_t* d_x, float* d_y,
              const float* d_bias, void* d_ws, size_t ws_bytes, void* stream);

/*
 * gqsa_gemm_smallbatch: Y[b] = W_hat X[b] (+ bias) for b < B, 1 <= B <= 8.
 *   d_X : device fp16 [B][ldx] (ldx >= cols, ldx % 8 == 0), d_Y : fp32 [B][ldy]
 *   (ldy >= rows).  B == 1 is the GEMV.
 */
int gqsa_gemm_smallbatch(const gqsa_desc_t* desc, const void* d_blob, const uint16_t* d_X,
                         int32_t B, int64_t ldx, float* d_Y, int64_t ldy, const float* d_bias,
                         void* d_ws, size_t ws_bytes, void* stream);

/*
 * gqsa_gemm_ex: gqsa_gemm_smallbatch with options (NULL = defaults).
 *   opts->partition (PAPER.md:161 and App. J):
 *     GQSA_PARTITION_STREAM_K (task-centric, the default): equal (+-1 tile)
 *       contiguous tile ranges per warp regardless of row boundaries; rows
 *       split across warps are finished by the cross-warp fix-up.
 *     GQSA_PARTITION_SLICE_K (data-centric, the paper's baseline): a warp owns
 *       whole 32-lane slices (rows) -- those whose first tile falls in its
 *       Stream-K range -- so there is no fix-up, and work per warp varies with
 *       the row lengths.
 *     Results agree within the parity gates (the fp32 summation order
 *     differs); each mode is bit-identical across reruns.
 *   opts->out_f16: 0 = fp32 Y (default), 1 = fp16 Y (round-to-nearest-even
 *     of the fp32 result (+ bias)); d_Y then points to uint16 [B][ldy]
 *     (2-B aligned).
 *   opts->x_ready: 0 (default) = X may be written by the previous kernel on
 *     the stream, so it is read after that kernel completes; 1 = the caller
 *     guarantees X is NOT written by the previous kernel (e.g. several
 *     GEMVs of one input, or inputs copied before an earlier launch), so the
 *     kernel stages X while the previous kernel drains.  At B <= 2 such a
 *     launch is PIPELINED: it takes half of every SM, so it
 *     streams its weights and computes beside the previous launch, and
 *     defers all its global writes until that launch has completed.  Y, bias
 *     and the workspace are always touched only after the previous kernel
 *     completes, so consecutive launches may share one workspace.  The
 *     pipelined launch uses another grid, hence another fp32 summation order
 *     than x_ready = 0 (both within the parity gates, each deterministic).
 * Other option values return GQSA_ERR_SHAPE.
 */
#define GQSA_PARTITION_STREAM_K 0
#define GQSA_PARTITION_SLICE_K 1
typedef struct {
  int32_t partition;  /* GQSA_PARTITION_* */
  int32_t out_f16;    /* 0: fp32 output, 1: fp16 output */
  int32_t x_ready;    /* 1: X is not produced by the previous kernel on the stream */
  int32_t reserved;   /* 0 */
} gqsa_options_t;
int gqsa_gemm_ex(const gqsa_desc_t* desc, const void* d_blob, const uint16_t* d_X, int32_t B,
                 int64_t ldx, void* d_Y, int64_t ldy, const float* d_bias, void* d_ws,
                 size_t ws_bytes, const gqsa_options_t* opts, void* stream);

/*
 * gqsa_gemm_allgather: the row-sharded GEMM of one rank with the all-gather
 * FUSED into its epilogue: every output element
 * of this rank's shard (global rows [row_offset, row_offset + desc->rows)) is
 * stored directly into each of the n_peers full-length outputs d_peer_Y[k]
 * ([B][ldy], fp32 or fp16 when out_f16) -- the ranks' y buffers mapped into
 * this device's address space (NVLink P2P / symmetric memory; on one GPU
 * they may simply be local buffers).  No NCCL call: the transfer overlaps
 * the GEMV tile by tile.  The kernel ends with a system-scope fence; the
 * caller orders consumers after ALL ranks' launches (e.g. a symmetric-memory
 * barrier on each rank's stream) before reading the gathered y.
 *   desc/d_blob : this rank's shard (gqsa_pack(row_begin, row_end)).
 *   d_bias      : this shard's bias [desc->rows] or NULL.
 * Errors: GQSA_ERR_SHAPE (n_peers not in [1, 8], B, ldy < row_offset + rows,
 * ldx), GQSA_ERR_BUFFER (null / misaligned pointers, small workspace).
 */
int gqsa_gemm_allgather(const gqsa_desc_t* desc, const void* d_blob, const uint16_t* d_X, int32_t B, int64_t ldx,
                        void* const* d_peer_Y, int32_t n_peers, int64_t ldy, int32_t row_offset, int32_t out_f16,
                        const float* d_bias, void* d_ws, size_t ws_bytes, void* stream);

/*
 * gqsa_gemm_allgather_multicast: gqsa_gemm_allgather over NVLink SHARP
 * (NVLS): d_mc_Y is the MULTICAST address of the
 * ranks' full-length outputs [B][ldy] (a CUDA multicast object every rank's y
 * is bound to, e.g. torch symmetric memory's multicast_ptr); every output
 * element of this shard is written ONCE with multimem.st and the NVSwitch
 * replicates it into every rank's y.  Same ordering contract as
 * gqsa_gemm_allgather (system-scope fence at the end; the caller orders the
 * consumers after all ranks' launches).  Needs a multicast-capable device and
 * a multicast object of >= 2 devices: not exercised on a one-GPU box
 * (DESIGN.md §9).  fp32 output only (out_f16 = 1: GQSA_ERR_UNSUPPORTED,
 * multimem.st has no 16-bit scalar form).  Other errors as gqsa_gemm_allgather.
 */
int gqsa_gemm_allgather_multicast(const gqsa_desc_t* desc, const void* d_blob, const uint16_t* d_X, int32_t B,
                                  int64_t ldx, void* d_mc_Y, int64_t ldy, int32_t row_offset, int32_t out_f16,
                                  const float* d_bias, void* d_ws, size_t ws_bytes, void* stream);

/*
 * gqsa_gemm_grouped: n INDEPENDENT GEMMs (e.g. the q/k/v or gate/up
 * projections of a decoder step, or the step's layers when their inputs are
 * ready) in ONE launch: Y_j[b] = W_hat_j X_j[b] (+ bias_j), j < n.  The tile
 * streams of all items are concatenated and cut into equal (+-1 tile) ranges
 * per warp (PAPER.md:161 Stream-K over the total work), so the step pays one
 * launch, one activation staging and one tail instead of n.
 *   items[j].desc / d_blob : packed layer j (all items: the same bits and G)
 *   items[j].d_X           : device fp16 [B][ldx], ldx >= cols, ldx % 8 == 0, 16-B aligned
 *   items[j].d_Y           : device fp32 [B][ldy] (fp16 when opts->out_f16), ldy >= rows
 *   items[j].d_bias        : device fp32 [rows] or NULL
 *   n in [1, GQSA_MAX_ITEMS], 1 <= B <= 8; opts as gqsa_gemm_ex (NULL = defaults).
 * No item may read another item's output (they run concurrently).  Each
 * item's result equals gqsa_gemm_ex on it alone up to the fp32 summation
 * order (bit-identical reruns for a fixed item list and device).  Items whose
 * activations do not fit in shared memory together run as several launches.
 * Workspace: gqsa_workspace_size(items[0].desc, B) bytes.
 * Errors: GQSA_ERR_SHAPE (n, B, ld*, options), GQSA_ERR_UNSUPPORTED (mixed
 * bits / G), GQSA_ERR_BUFFER (null / misaligned pointers, small workspace),
 * GQSA_ERR_VALIDATION (desc).
 */
#define GQSA_MAX_ITEMS 8
typedef struct {
  const gqsa_desc_t* desc;
  const void* d_blob;
  const uint16_t* d_X;
  int64_t ldx;
  void* d_Y;
  int64_t ldy;
  const float* d_bias;
} gqsa_gemm_item_t;
int gqsa_gemm_grouped(const gqsa_gemm_item_t* items, int32_t n, int32_t B, const gqsa_options_t* opts,
                      void* d_ws, size_t ws_bytes, void* stream);

/*
 * gqsa_gemm_hostio: the end-to-end call with HOST activations and outputs.
 * Copies h_X (pinned or pageable host fp16 [B][cols], dense) into the
 * device staging area d_stage, runs gqsa_gemm_smallbatch, and copies Y back
 * into h_Y (host fp32 [B][rows], dense), all on `stream`; returns after
 * enqueueing (synchronize the stream before reading h_Y).  d_stage needs
 * gqsa_hostio_stage_size bytes.
 */
int gqsa_hostio_stage_size(const gqsa_desc_t* desc, int32_t B, size_t* bytes);
int gqsa_gemm_hostio(const gqsa_desc_t* desc, const void* d_blob, const uint16_t* h_X, int32_t B,
                     float* h_Y, const float* d_bias, void* d_stage, size_t stage_bytes,
                     void* d_ws, size_t ws_bytes, void* stream);

/*
 * gqsa_gemm_multi_hostio: n INDEPENDENT layers with host I/O in one call --
 * the end-to-end path of a decode step whose activations live on the host:
 * ONE host->device copy of all inputs, the layers as gqsa_gemm_grouped
 * launches (one per GQSA_MAX_ITEMS layers), ONE device->host copy of all
 * outputs.
 *   descs[j], d_blobs[j] : layer j; d_ws[0] / ws_bytes[0]: the workspace
 *   (gqsa_workspace_size; the other entries are ignored)
 *   h_X : host fp16, the concatenation of the n inputs [B][cols_j] (dense,
 *         layer 0 first); pinned memory makes the copy asynchronous
 *   h_Y : host fp32, the concatenation of the n outputs [B][rows_j]
 *   d_stage : device buffer of gqsa_multi_hostio_stage_size bytes (256-B aligned)
 * Returns after enqueueing; synchronize `stream` before reading h_Y.  Each
 * layer reads only its own input segment (no dependency between layers).
 * Errors as gqsa_gemm_smallbatch, plus GQSA_ERR_SHAPE for n < 1.
 */
int gqsa_multi_hostio_stage_size(const gqsa_desc_t* const* descs, int32_t n, int32_t B, size_t* bytes);
int gqsa_gemm_multi_hostio(const gqsa_desc_t* const* descs, const void* const* d_blobs, int32_t n, int32_t B,
                           const uint16_t* h_X, float* h_Y, void* d_stage, size_t stage_bytes,
                           void* const* d_ws, const size_t* ws_bytes, void* stream);

/* Launch plan the next gemv/gemm call will use on the current device (for
 * a split batch: the plan of its first launch):
 * CTAs, warps per CTA, active warps (Stream-K units), tiles.  For tooling.
 * gqsa_launch_plan_ex takes the call's options (NULL = defaults): with
 * x_ready at B <= 2 the launch is the pipelined one. */
typedef struct {
  int32_t grid, warps_per_cta, active_warps, num_tiles, smem_bytes, x_in_smem;
  int32_t stages, ctas_per_sm, ring_bytes;  /* tiles in flight per warp (register buffers); CTAs
                                               per SM the kernel is compiled for; 0 */
  int32_t batch_per_launch, launches;  /* x of batch_per_launch columns fits in shared memory;
                                          larger batches run as `launches` launches */
  int32_t coresident;                  /* 1: pipelined -- the launch takes part of every SM and the
                                          next launch on the stream may run beside it */
} gqsa_plan_t;
int gqsa_launch_plan(const gqsa_desc_t* desc, int32_t B, gqsa_plan_t* plan);
int gqsa_launch_plan_ex(const gqsa_desc_t* desc, int32_t B, const gqsa_options_t* opts, gqsa_plan_t* plan);

/* Number of GQSA kernels launched by this process so far (all entry points). */
uint64_t gqsa_launch_count(void);

/* Profiling hook: while set, every launch writes, per active warp w, eight
 * uint64 %globaltimer stamps at d_buf[8w .. 8w+7] (0 start, 1 after the PDL
 * wait, 2 activations staged, 3 tile loop start, 4 tile loop done, 5 exit)
 * when bytes >= 64 * active_warps.  d_buf = NULL turns it off (default).
 * The buffer is caller-owned device memory; not for production use. */
int gqsa_debug_trace(void* d_buf, size_t bytes);

const char* gqsa_status_string(int status);
int gqsa_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GQSA_H_ */
