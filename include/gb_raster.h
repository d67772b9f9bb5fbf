/*
 * gb_raster.h -- C-ABI of the B200-native Gaussian Billboards rasterizer.
 *
 * This is the drop-in boundary for the reference's rasterizer API
 * (/root/reference/proj/include/gbil).  The reference has no FFI: its
 * boundary is the C++ header API listed below, and each entry point here
 * replaces one of those functions (file:line cited at each declaration).
 * Plain pointers and sizes only; every device pointer is fp32/int32 CUDA
 * global memory owned by the caller unless stated.  All calls are
 * stream-ordered on the context's stream and asynchronous unless stated.
 * A context is not thread-safe: use one per host thread / GPU.
 *
 * Error model: every reference throw site maps to a status code
 * (std::invalid_argument -> GB_INVALID_ARGUMENT / GB_MISMATCH,
 * adam's std::runtime_error -> GB_NONFINITE); the message of the last failure
 * on the calling thread is returned by gb_last_error_string().  NaNs in the
 * inputs propagate silently, as in the reference.
 */
#ifndef GB_RASTER_H
#define GB_RASTER_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GB_ABI_VERSION 1

#if defined(__GNUC__)
#define GB_API __attribute__((visibility("default")))
#else
#define GB_API
#endif

typedef enum {
    GB_OK = 0,
    GB_INVALID_ARGUMENT = 1, /* validate() throws: core.hpp:36-41, 109-115; raster.hpp:28-31 */
    GB_MISMATCH = 2,         /* fingerprint / size guards: raster.hpp:204-205, 280-287 */
    GB_CUDA_ERROR = 3,
    GB_OOM = 4,
    GB_NONFINITE = 5, /* adam_step non-finite gradient: optim.hpp:81-83 */
    GB_NOT_SUPPORTED = 6,
    GB_IO_ERROR = 7, /* SplatIoError (serialize.hpp:23-25) */
    GB_NCCL_ERROR = 8 /* a collective failed or the communicator reported an asynchronous error */
} gb_status;

#define GB_MODE_ORTHO 0   /* the reference's ImagePlaneCamera (core.hpp:102-116) */
#define GB_MODE_PINHOLE 1 /* perspective 2DGS extension (no reference) */

typedef struct gb_context gb_context;
typedef struct gb_binning gb_binning;
typedef struct gb_graph gb_graph;

/* ColorGridConfig (core.hpp:29-42) */
typedef struct {
    int32_t n;
    int32_t _pad;
    double sigma;
} gb_grid_config;

/* SplatSet (core.hpp:53-87), structure-of-arrays, fp32 device pointers.
 * ortho  : position 2K (x,y), depth_key K, theta K
 * pinhole: position 3K world mean (x,y,z), quat 4K (w,x,y,z), unnormalised
 * both   : log_scale 2K (u,v), opacity_logit K, grid K*n*n*3 in
 *          (i_u, i_v, channel) order (core.hpp:44-48).
 * Alignment: quat 16 B, log_scale 8 B, grid_values 16 B for even n (any
 * device allocation is; K1/K3/K4 read them as vectors). */
typedef struct {
    int64_t count;
    gb_grid_config grid;
    const float *position;
    const float *depth_key;
    const float *theta;
    const float *quat;
    const float *log_scale;
    const float *opacity_logit;
    const float *grid_values;
} gb_splats;

/* GradientBuffer (core.hpp:140-178) with the same layout as gb_splats.
 * Backward ACCUMULATES into it (caller zeroes), so several views can sum
 * into one buffer with atomic adds, so backwards on different streams may
 * target the same buffer concurrently.  depth_key never receives a gradient.
 * Alignment (vector atomics): log_scale and the ortho position 8 B, quat and
 * grid_values (even n) 16 B, else GB_INVALID_ARGUMENT. */
typedef struct {
    float *position;
    float *depth_key;
    float *theta;
    float *quat;
    float *log_scale;
    float *opacity_logit;
    float *grid_values;
} gb_grads;

/* ImagePlaneCamera (core.hpp:104-116) plus the pinhole extension:
 * OpenCV convention, x_pix = fx*X/Z + cx with pixel centres at i + 0.5,
 * world->camera [rot | trans].  width, height <= 65520 (GB_NOT_SUPPORTED past it:
 * the compositors pack a pixel's coordinates into 16 + 16 bits). */
typedef struct {
    int32_t mode;
    int32_t width;
    int32_t height;
    int32_t _pad;
    double background[3];
    double fx, fy, cx, cy;
    double rot[9];
    double trans[3];
    double near_plane;
} gb_camera;

/* RasterConfig (raster.hpp:21-32).  `threads` is accepted and ignored
 * (the GPU parallelises over tiles).  tile_size must be in [1, 16] on the GPU path. */
typedef struct {
    int32_t tile_size;
    int32_t threads;
    double cutoff_radius;
    double alpha_skip;
    double early_stop_transmittance;
} gb_raster_config;

/* RenderOutput (core.hpp:123-136), caller-owned device buffers; the
 * fingerprint fields are written by gb_render_forward. */
typedef struct {
    int32_t width;
    int32_t height;
    float *color;               /* W*H*3, HWC, unclamped */
    float *final_transmittance; /* W*H */
    int32_t *last_rank;         /* W*H, -1 if nothing composited */
    int64_t splat_count;
    int32_t grid_n;
    int32_t tile_size;
} gb_render_out;

/* LearningRates / AdamConfig / AdamState (optim.hpp:17-72).  The pinhole
 * rotation quaternion uses the `theta` (rotation) rate. */
typedef struct {
    double position, theta, log_scale, opacity_logit, color_grid, position_gamma;
} gb_learning_rates;

typedef struct {
    int64_t t;
    double beta1, beta2, epsilon;
    gb_grads m; /* first moments, same layout as the gradients, zero-initialised */
    gb_grads v; /* second moments */
} gb_adam_state;

/* ---- context ------------------------------------------------------------ */
GB_API int gb_abi_version(void);
GB_API const char *gb_last_error_string(void);
GB_API gb_status gb_context_create(int device, gb_context **out);
GB_API gb_status gb_context_destroy(gb_context *ctx);
/* Run all subsequent work on `stream` (a cudaStream_t; NULL = the legacy default stream).
 * A fresh context uses its own non-blocking stream. */
GB_API gb_status gb_context_set_stream(gb_context *ctx, void *stream);
GB_API void *gb_context_stream(gb_context *ctx);
GB_API gb_status gb_sync(gb_context *ctx);
/* Number of kernels this context has launched (for the bench's gpu_launches claim). */
GB_API int64_t gb_context_launch_count(const gb_context *ctx);

/* Per-kernel CUDA-event timing on the context's stream (bench roofline).  While
 * enabled, every launch site is bracketed by two events; _read synchronises,
 * returns total milliseconds and launch counts per kernel id, and resets. */
#define GB_K_PROJECT 0   /* K1  per-primitive projection + cull + tile rect */
#define GB_K_SCAN 1      /* K2a per-tile pair counts + their scan (CUB) */
#define GB_K_DUPLICATE 2 /* K2b scatter of the (depth, id) keys into the tile buckets */
#define GB_K_SORT 3      /* K2c per-tile bucket sort -> lists and ranges */
#define GB_K_RANGES 4    /* (no separate pass since the tile-bucket build: ranges come with K2c) */
#define GB_K_FORWARD 5   /* K3  forward compositor */
#define GB_K_BACKWARD 6  /* K4  backward compositor */
#define GB_K_CHAIN 7     /* K5  per-primitive gradient chain */
#define GB_K_LOSS 8      /* K6  photometric loss */
#define GB_K_ADAM 9      /* K7  Adam */
#define GB_K_FUSED 10    /* K3+K6+K4 in one kernel (gb_render_loss_backward) */
#define GB_K_COLLECTIVE 11 /* NCCL collectives of the view-sharded step (gb_allreduce_grads, ...) */
#define GB_NUM_KERNEL_IDS 12
GB_API gb_status gb_context_profile(gb_context *ctx, int enable);
GB_API gb_status gb_context_profile_read(gb_context *ctx, double *total_ms, int64_t *counts, int n);
/* The recorded launches of kernel `id` as (start, stop) in ms after `ref_event` (a cudaEvent_t recorded
 * earlier on any stream of the device): overlapping launches from several contexts can then be merged
 * into busy time.  Synchronous; leaves the records for gb_context_profile_read.  *n = all matches. */
GB_API gb_status gb_context_profile_intervals(gb_context *ctx, void *ref_event, int32_t id, double *start_ms,
                                              double *stop_ms, int64_t cap, int64_t *n);

/* ---- CUDA graphs ------------------------------------------------------------
 * Capture the work a host thread issues on ctxs[0]'s stream -- and on streams that fork from it and join
 * back, e.g. other contexts' streams -- into one CUDA graph (stream capture, thread-local mode), so a
 * training step's views replay with one launch.  Every launch site keeps its gb_context_profile timing:
 * the capture turns its events into event-record nodes, and each profiled gb_graph_launch points them at
 * fresh events of the context that issued the site.  Kernel counts (gb_context_launch_count) move from the
 * capture to every launch.  Between begin and end the calls must not allocate or block (binnings in
 * capacity mode; buffers already sized by an eager run).  No reference counterpart (the reference is a
 * synchronous CPU library). */
GB_API gb_status gb_graph_begin(gb_context *const *ctxs, int32_t n);
GB_API gb_status gb_graph_end(gb_context *const *ctxs, int32_t n, gb_graph **out);
/* Launch on the origin context's stream (asynchronous). */
GB_API gb_status gb_graph_launch(gb_graph *g);
GB_API gb_status gb_graph_destroy(gb_graph *g);
/* The context's stream waits for `event` (a cudaEvent_t).  external = 1: inside a gb_graph capture the
 * graph then waits for the event's record made outside it, at every launch (ignored outside a capture). */
GB_API gb_status gb_stream_wait_event(gb_context *ctx, void *event, int32_t external);

/* Events for a host without CUDA headers (fork/join of several contexts' streams, e.g. view lanes inside
 * a gb_graph capture): a timing-disabled cudaEvent_t recorded on / waited for by a context's stream
 * (gb_stream_wait_event). */
GB_API gb_status gb_event_create(gb_context *ctx, void **event);
GB_API gb_status gb_event_record(gb_context *ctx, void *event);
GB_API gb_status gb_event_destroy(gb_context *ctx, void *event);

/* ---- device memory helpers (so a C/C++ host needs no CUDA headers) -------- */
GB_API gb_status gb_device_alloc(gb_context *ctx, uint64_t bytes, void **out);
GB_API gb_status gb_device_free(gb_context *ctx, void *ptr);
/* Stream-ordered copies on the context stream; pass sync = 1 to block until done. */
GB_API gb_status gb_copy_h2d(gb_context *ctx, void *dst_device, const void *src_host, uint64_t bytes, int sync);
GB_API gb_status gb_copy_d2h(gb_context *ctx, void *dst_host, const void *src_device, uint64_t bytes, int sync);
GB_API gb_status gb_memset_device(gb_context *ctx, void *dst_device, int value, uint64_t bytes);

/* ---- binning: TileBinning + build_binning (raster.hpp:105-147) ------------ */
GB_API gb_status gb_binning_create(gb_context *ctx, gb_binning **out);
GB_API gb_status gb_binning_destroy(gb_binning *b);
/* Replaces build_binning(const SplatSet&, const ImagePlaneCamera&, const RasterConfig&)
 * (raster.hpp:116-117).  Device-resident result, reused by forward and
 * backward; also caches the per-primitive screen headers (K1).  Blocks once
 * on the stream to learn the pair count P. */
GB_API gb_status gb_build_binning(gb_context *ctx, const gb_splats *s, const gb_camera *cam, const gb_raster_config *cfg,
                           gb_binning *b);
/* Capacity mode (capacity > 0): gb_build_binning stops reading the pair count P back to the host.  Its
 * pair buffers hold `capacity` slots and the tile sort runs over all of them (unused slots carry a pad key
 * that lands in no tile), so the tile lists are identical and the build never blocks -- it can run ahead
 * of the GPU and be captured into a CUDA graph.  If a view has P > capacity, only the first `capacity`
 * pairs in (depth, index) order are binned and *overflow (a device int32 the caller zeroes) is set to 1:
 * grow the capacity and rebuild.  capacity = 0 restores the exactly-sized, blocking build.  No reference
 * counterpart (build_binning sizes its lists on the host, raster.hpp:128-146). */
GB_API gb_status gb_binning_set_capacity(gb_binning *b, int64_t capacity, int32_t *overflow);
/* Stream-ordered copy of the last build's pair count P (uint32, before any capacity clamp) to device memory. */
GB_API gb_status gb_binning_store_total(gb_context *ctx, const gb_binning *b, uint32_t *dst_device);
/* total = P (in capacity mode this reads P back synchronously, clamped to the capacity). */
GB_API gb_status gb_binning_info(const gb_binning *b, int32_t *tiles_x, int32_t *tiles_y, int64_t *total);
/* Synchronous test hook: per-tile lists as CSR on the host
 * (offsets[tiles+1], values[total]) -- TileBinning::tiles. */
GB_API gb_status gb_binning_copy_to_host(gb_context *ctx, const gb_binning *b, int64_t *offsets, int32_t *values);

/* ---- render ---------------------------------------------------------------- */
/* Replaces render_forward(const SplatSet&, const ImagePlaneCamera&, const TileBinning&)
 * (raster.hpp:201-202). */
GB_API gb_status gb_render_forward(gb_context *ctx, const gb_splats *s, const gb_camera *cam, const gb_binning *b,
                            gb_render_out *out);
/* Replaces render_backward(..., const RenderOutput&, const std::vector<double>& image_grad)
 * (raster.hpp:277-279).  image_grad is W*H*3 on the device; gradients are
 * accumulated into *g. */
GB_API gb_status gb_render_backward(gb_context *ctx, const gb_splats *s, const gb_camera *cam, const gb_binning *b,
                             const gb_render_out *out, const float *image_grad, gb_grads *g);
/* Replaces render(const SplatSet&, const ImagePlaneCamera&, const RasterConfig&)
 * (raster.hpp:389-392); `scratch` receives the binning. */
GB_API gb_status gb_render(gb_context *ctx, const gb_splats *s, const gb_camera *cam, const gb_raster_config *cfg,
                    gb_binning *scratch, gb_render_out *out);

/* Texel-gradient layout of this context's backwards (no reference counterpart; the default is the
 * reference's).  stride 3: gb_grads.grid_values is K x n x n x 3 in (i_u, i_v, channel) order
 * (core.hpp:44-48).  stride 4: K x n x n x 4, RGBA-padded (the 4th float of each texel is never written and
 * stays as the caller left it; 16-B aligned), so K4 adds each texel's three channels with one 16-byte
 * vector red instead of an 8-byte and a 4-byte one.  A training loop accumulating many views keeps a
 * padded buffer and converts it once per step with gb_texel_grads_unpad. */
GB_API gb_status gb_context_set_texel_grad_stride(gb_context *ctx, int32_t stride);
/* Texel layout the compositors read (no reference counterpart).  rgba == NULL (the default): the splats'
 * grid_values, K x n x n x 3 (core.hpp:44-48).  Otherwise an RGBA-padded copy of them, K x n x n x 4 floats,
 * 16-B aligned (gb_texels_pad writes one): K3/K4 fetch a texel with one 16-byte load -- the same values, so
 * the same results.  The caller keeps the copy in step with grid_values; the backwards then need texel
 * gradient stride 4 (gb_context_set_texel_grad_stride).  A training loop pads once per step, after the
 * optimizer's texel update. */
GB_API gb_status gb_context_set_texel_rgba(gb_context *ctx, const float *rgba);
/* dst[4t + c] = src[3t + c], dst[4t + 3] = 0 for t < texels (dst 16-B aligned). */
GB_API gb_status gb_texels_pad(gb_context *ctx, const float *src, float *dst, int64_t texels);
/* dst[3t + c] (+)= padded[4t + c] for t < texels, c < 3 (accumulate = 0: overwrite). */
GB_API gb_status gb_texel_grads_unpad(gb_context *ctx, const float *padded, float *dst, int64_t texels,
                                      int32_t accumulate);

/* ---- losses (train.hpp:120-133; L1 is the BASELINE configs' loss) --------- */
/* grad[i] = scale*sign(color-target) (sign(0) = 0); *loss += scale*sum|color-target|. */
GB_API gb_status gb_l1_loss(gb_context *ctx, const float *color, const float *target, int64_t n, float scale, float *grad,
                     float *loss);
/* grad[i] = 2*scale*(color-target); *loss += scale*sum (color-target)^2. */
GB_API gb_status gb_mse_loss(gb_context *ctx, const float *color, const float *target, int64_t n, float scale, float *grad,
                      float *loss);

/* One view of a training step (train.hpp:120-133 around raster.hpp:201-371):
 *   gb_render_forward + gb_l1_loss (loss_kind GB_LOSS_L1) or gb_mse_loss (GB_LOSS_MSE) + gb_render_backward,
 * as the forward compositor with the loss in its epilogue (the image never round-trips through memory)
 * followed by the backward compositor.  target: HWC fp32 (device).  out: NULL, or forward buffers filled as gb_render_forward
 * would; image_grad: NULL, or receives the cotangent; *loss (device float) += as the loss entry points
 * (summation order differs); g receives the gradients as gb_render_backward.  Per-pixel arithmetic is the
 * separate calls'. */
#define GB_LOSS_L1 0
#define GB_LOSS_MSE 1
GB_API gb_status gb_render_loss_backward(gb_context *ctx, const gb_splats *s, const gb_camera *cam, const gb_binning *b,
                                         const float *target, int32_t loss_kind, float scale, gb_render_out *out,
                                         float *image_grad, float *loss, gb_grads *g);

/* ---- image metrics (metrics.hpp) ------------------------------------------- */
/* ssim (metrics.hpp:183-185) with clamp01 = 1, ssim_with_gradient (metrics.hpp:189-191) with clamp01 = 0:
 * Wang 2004 SSIM, 11-tap Gaussian window (std 1.5), K1 = 0.01, K2 = 0.03, valid windows, channels averaged,
 * on HWC fp32 images.  *mean_ssim (a DEVICE double) += the mean SSIM; when grad != NULL (clamp01 = 0 only),
 * grad += grad_scale * d(mean SSIM)/d(a).  Asynchronous.  W, H >= 11 (else GB_INVALID_ARGUMENT, as the reference). */
GB_API gb_status gb_ssim(gb_context *ctx, const float *a, const float *b, int32_t width, int32_t height,
                         int32_t clamp01, double *mean_ssim, float *grad, float grad_scale);
/* psnr (metrics.hpp:169-179): both images clamped to [0,1], capped at 99 dB.  Synchronous; *out on the host. */
GB_API gb_status gb_psnr(gb_context *ctx, const float *a, const float *b, int64_t n, double *out);

/* ---- texture diagnostics (texture.hpp:128-197) ------------------------------ */
/* Output size of downsample_grid(n, levels) (texture.hpp:132-166), or GB_INVALID_ARGUMENT with its message. */
GB_API gb_status gb_downsample_size(int32_t n, int32_t levels, int32_t *n_out);
/* downsample_set's grids (texture.hpp:169-188): count grids of n x n x 3 -> n_out x n_out x 3 (device). */
GB_API gb_status gb_downsample_grids(gb_context *ctx, const float *grid, int64_t count, int32_t n, int32_t levels,
                                     float *out);

/* ---- optimiser: adam_step (optim.hpp:96-117) ------------------------------ */
/* params uses the gb_grads layout (mutable parameter arrays).  Increments
 * state->t.  Non-finite gradients are detected on the device first; if any is
 * found no parameter is updated and gb_adam_check() reports GB_NONFINITE with
 * the group and index. */
GB_API gb_status gb_adam_step(gb_context *ctx, int32_t mode, int64_t count, int32_t n, gb_grads *params, const gb_grads *g,
                       gb_adam_state *state, const gb_learning_rates *lrs);
/* Synchronous.  group: 0 position, 1 theta/quat, 2 log_scale, 3 opacity, 4 grid. */
GB_API gb_status gb_adam_check(gb_context *ctx, int32_t *group, int64_t *index);

/* Adam over explicit segments: the sharded optimiser of the multi-GPU step, where each rank updates its
 * slice of a flat parameter buffer (optim.hpp:84-88 per element; the group selects the rate and, for
 * group 0, the position_gamma schedule).  Two phases, so that ranks can agree on the non-finite guard
 * (optim.hpp:81-83) before anything is updated:
 *   phase 0: scan the segments' gradients; *flag (a device int64 the caller sets to GB_ADAM_FLAG_CLEAR)
 *            is lowered to (group << 48) | index-in-segment of a non-finite gradient;
 *   (the caller may min-reduce *flag across ranks)
 *   phase 1: state->t += 1 and update every segment, unless *flag shows a non-finite gradient.
 * Asynchronous; the moments in the segments use the gradient layout. */
typedef struct {
    float *param;
    const float *grad;
    float *m, *v;
    int64_t len;
    int32_t group; /* 0 position, 1 theta/quat, 2 log_scale, 3 opacity_logit, 4 grid */
    int32_t _pad;
} gb_adam_segment;
#define GB_ADAM_FLAG_CLEAR 0x7fffffffffffffffLL
#define GB_ADAM_FLAG_VETO (7LL << 48) /* a vetoed step: below every clear value, above every non-finite code */
/* *flag = GB_ADAM_FLAG_VETO if veto != NULL and *veto != 0 (a device int32, e.g. the binning's overflow
 * flag: skip this update on every rank), else GB_ADAM_FLAG_CLEAR -- on the stream, before phase 0. */
GB_API gb_status gb_adam_flag_init(gb_context *ctx, int64_t *flag, const int32_t *veto);
GB_API gb_status gb_adam_segments(gb_context *ctx, int32_t phase, const gb_adam_segment *seg, int32_t nseg,
                                  gb_adam_state *state, const gb_learning_rates *lrs, int64_t *flag);

/* ---- the view-sharded step's gradient exchange ------------------------------------
 * The reference is single-process (fit, train.hpp:174-219); the multi-GPU step generalises its loop
 * (build_binning -> render_forward -> loss -> render_backward -> adam_step, train.hpp:190-217) by view:
 * every GPU renders and backpropagates its own views into one flat fp32 gradient buffer, then the
 * buffers are summed over the GPUs -- one all-reduce, or a reduce-scatter followed by Adam on each
 * rank's slice and an all-gather of the parameters -- over NCCL (NVLink/NVSwitch).  NCCL is loaded at
 * run time (dlopen "libnccl.so.2"; the copy a host process already loaded, e.g. torch's, is reused).
 * Collectives are stream-ordered on the context's stream and timed under GB_K_COLLECTIVE. */
typedef struct gb_comm gb_comm;
#define GB_COMM_ID_BYTES 128
/* ncclGetUniqueId: rank 0 creates the id and ships it to the other ranks (any side channel). */
GB_API gb_status gb_comm_unique_id(uint8_t id[GB_COMM_ID_BYTES]);
/* ncclCommInitRank on ctx's device (one process or thread per GPU). */
GB_API gb_status gb_comm_init_rank(gb_context *ctx, int32_t nranks, const uint8_t id[GB_COMM_ID_BYTES], int32_t rank,
                                   gb_comm **out);
/* ncclCommInitAll: one communicator per context (distinct devices), rank i = ctxs[i]; single host thread. */
GB_API gb_status gb_comm_init_all(gb_context *const *ctxs, int32_t n, gb_comm **out);
GB_API gb_status gb_comm_destroy(gb_comm *c);
GB_API gb_status gb_comm_info(const gb_comm *c, int32_t *nranks, int32_t *rank);
/* ncclCommGetAsyncError: GB_OK, or GB_NCCL_ERROR with the communicator's error string. */
GB_API gb_status gb_comm_check(gb_comm *c);
/* In-place sum of the flat gradient buffer over all ranks (ncclAllReduce, ncclFloat, ncclSum). */
GB_API gb_status gb_allreduce_grads(gb_context *ctx, gb_comm *c, float *grads, int64_t count);
/* recv[recv_count] = this rank's slice of the sum of every rank's send[nranks * recv_count] (ncclReduceScatter). */
GB_API gb_status gb_reduce_scatter_grads(gb_context *ctx, gb_comm *c, const float *send, float *recv, int64_t recv_count);
/* recv[nranks * send_count] = every rank's send[send_count] in rank order (ncclAllGather); in place when
 * send == recv + rank * send_count. */
GB_API gb_status gb_all_gather_params(gb_context *ctx, gb_comm *c, const float *send, float *recv, int64_t send_count);
/* In-place minimum of a device int64 over all ranks: the Adam non-finite/veto flag (gb_adam_segments). */
GB_API gb_status gb_allreduce_flag_min(gb_context *ctx, gb_comm *c, int64_t *flag);

/* ---- GBIL splat files (serialize.hpp:15-124) -------------------------------
 * Header "GBIL", u32 version, u32 K, u32 N, f32 sigma, then K little-endian
 * fp32 records.  Version 1 is the reference's (ortho) record: x, y, depth_key,
 * theta, log_su, log_sv, opacity_logit, N*N*3 grid.  Version 2 is this build's
 * pinhole extension: mean xyz, quat wxyz, log_su, log_sv, opacity_logit, grid.
 * Errors are GB_IO_ERROR with serialize.hpp's messages ("bad splat file: wrong
 * magic", "... truncated header", "unsupported splat file version N",
 * "... invalid grid config", "... truncated at record R", "cannot open splat
 * file: PATH", "cannot open for writing: PATH", "splat write failed: PATH"). */
typedef struct {
    int32_t version;
    int32_t mode; /* GB_MODE_ORTHO for version 1, GB_MODE_PINHOLE for version 2 */
    int64_t count;
    int32_t n;
    float sigma;
} gb_splat_file_info;
/* Header only (host; no device work).  Replaces the header half of load_splats (serialize.hpp:83-101). */
GB_API gb_status gb_splats_file_info(const char *path, gb_splat_file_info *info);
/* Replaces save_splats(path, set) (serialize.hpp:56-90): device SoA -> records on the GPU -> file. */
GB_API gb_status gb_splats_save(gb_context *ctx, const gb_splats *s, int32_t mode, const char *path);
/* Replaces load_splats(path) (serialize.hpp:92-124) into caller-allocated device buffers (gb_grads layout,
 * sized from gb_splats_file_info; count/n must match the file, else GB_MISMATCH).  Synchronous. */
GB_API gb_status gb_splats_load(gb_context *ctx, const char *path, int64_t count, int32_t n, gb_grads *dst);

/* ---- seeded synthetic inputs (rng.hpp:12-46 semantics), host-only ---------- */
typedef struct {
    int32_t mode;
    int32_t n;
    int64_t count;
    uint64_t seed;
    double mean_lo, mean_hi; /* pinhole: uniform means in [lo,hi)^3 when mean_sigma <= 0 */
    double mean_sigma;       /* pinhole: N(0, mean_sigma^2) means when > 0 */
    double log_scale_lo, log_scale_hi;
    int32_t width, height; /* ortho: positions uniform over the image */
} gb_scene_spec;
/* Geometry from Rng(seed), textures from Rng(seed+1).  Host fp32 buffers. */
GB_API gb_status gb_scene_generate(const gb_scene_spec *spec, float *position, float *depth_key, float *theta, float *quat,
                            float *log_scale, float *opacity_logit, float *grid_values);
/* initialize() of the image-fitting loop (train.hpp:80-111), ortho SplatSet, same Rng draws, fp32 host buffers. */
GB_API gb_status gb_fit_initialize(int32_t width, int32_t height, int64_t count, int32_t n, uint64_t seed,
                                   float *position, float *depth_key, float *theta, float *log_scale,
                                   float *opacity_logit, float *grid_values);
/* n uniforms in [0,1) from Rng(seed), rounded to fp32 (targets use seed+2+view). */
GB_API gb_status gb_uniform_fill(uint64_t seed, int64_t n, float *out);
/* Raw Rng streams in fp64, for parity with rng.hpp. */
GB_API gb_status gb_rng_uniform(uint64_t seed, int64_t n, double *out);
GB_API gb_status gb_rng_normal(uint64_t seed, int64_t n, double mean, double stddev, double *out);

#ifdef __cplusplus
}
#endif
#endif
