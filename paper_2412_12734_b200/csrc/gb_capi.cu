// gb_capi.cu -- the extern "C" boundary (include/gb_raster.h) and the host
// orchestration of K1..K7 on the context's CUDA stream.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <algorithm>
#include <memory>
#include <vector>

#include "gb_internal.cuh"
#include "gb_io.cuh"

namespace gb {
size_t scan_temp_bytes(int64_t K);
size_t sort_temp_bytes(int64_t n);
int sort_launches(int bits);
int tile_sort_bits(int n_keys);
cudaError_t launch_depth_sort(void* temp, size_t temp_bytes, const uint32_t* depth_bits, uint32_t* depth_sorted,
                              int32_t* iota, int32_t* perm, int64_t K, cudaStream_t st);
cudaError_t launch_scan(void* temp, size_t temp_bytes, const int32_t* perm, const uint32_t* counts,
                        uint32_t* offsets, int64_t K, cudaStream_t st);
cudaError_t launch_duplicate(int64_t K, int tiles_x, const int32_t* perm, const uint32_t* offsets, const uint2* rects,
                             uint32_t* keys, int32_t* values, uint32_t cap, int32_t* overflow, cudaStream_t st);
cudaError_t launch_pad(uint32_t cap, const uint32_t* total, int n_tiles, uint32_t* keys, int32_t* values,
                       cudaStream_t st);
cudaError_t launch_tile_sort(void* temp, size_t temp_bytes, uint32_t* keys_in, uint32_t* keys_out, int32_t* vals_in,
                             int32_t* vals_out, int64_t P, int n_keys, cudaStream_t st);
cudaError_t launch_ranges(int64_t P, const uint32_t* keys, uint2* ranges, int n_tiles, cudaStream_t st);
int deep_bucket_mean();
size_t tile_scan_temp_bytes(int n_tiles);
size_t tile_scratch_words(int n_tiles);
int tile_offsets_launches(int64_t K, int n_tiles);
cudaError_t launch_tile_offsets(void* temp, size_t temp_bytes, int64_t K, int tiles_x, int n_tiles,
                                const uint32_t* counts, const uint2* rects, uint32_t* hist, uint32_t* tile_off,
                                cudaStream_t st);
cudaError_t launch_scatter(int64_t K, int tiles_x, int n_tiles, const uint32_t* counts, const uint2* rects,
                           const uint32_t* depth_bits, const uint32_t* tile_off, uint32_t* cursor, uint64_t* keys,
                           uint32_t cap, cudaStream_t st);
cudaError_t launch_tile_lists(int n_tiles, const uint32_t* tile_off, uint32_t limit, uint64_t* keys,
                              uint64_t* scratch, int32_t* values, uint2* ranges, int32_t* overflow, cudaStream_t st);
cudaError_t launch_forward(int mode, int n, int tiles, int ts, const uint2* ranges, const int32_t* values,
                           const ScreenHeader* hdr, const CullRec* cull, const float* tex, const CamConst& cc, const RasterConst& rc,
                           float* color, float* trans, int32_t* last, cudaStream_t st);
cudaError_t launch_backward(int mode, int n, int tiles, int ts, const uint2* ranges, const int32_t* values,
                            const ScreenHeader* hdr, const CullRec* cull, const float* tex, const CamConst& cc, const RasterConst& rc,
                            const float* trans, const int32_t* last, const float* image_grad, real* accum,
                            real* grid_grad, cudaStream_t st);
#ifdef GB_PARITY_F64
cudaError_t launch_add_f64(const double* src, float* dst, int64_t n, cudaStream_t st);
#endif
cudaError_t launch_adam_flag_init(int64_t* flag, const int32_t* veto, cudaStream_t st);
cudaError_t launch_texel_unpad(const float* padded, float* dst, int64_t texels, bool accumulate, int sm_count,
                               cudaStream_t st);
cudaError_t launch_texel_pad(const float* src, float* dst, int64_t texels, int sm_count, cudaStream_t st);
cudaError_t launch_loss(int kind, const float* color, const float* target, int64_t n, float scale, float* grad,
                        float* loss, int sm_count, cudaStream_t st);
cudaError_t launch_adam_check(const float* g, int64_t n, int group, unsigned long long* bad, int sm_count,
                              cudaStream_t st);
cudaError_t launch_ssim(const float* a, const float* b, int W, int H, int clamp, double* sum, float* grad,
                        float grad_scale, float* dcoef, cudaStream_t st);
cudaError_t launch_psnr_sum(const float* a, const float* b, int64_t n, double* sum, int sm_count, cudaStream_t st);
bool downsample_plan(int n, int levels, int& halvings, int& collapse, int& n_out);
cudaError_t launch_downsample(int64_t K, int n, int halvings, int collapse, const float* src, float* dst,
                              int sm_count, cudaStream_t st);
cudaError_t launch_adam_update(float* p, const float* g, float* m, float* v, int64_t n, float lr, float b1, float b2,
                               float omb1, float omb2, float eps, float inv_bias1, float inv_bias2,
                               const unsigned long long* bad, int sm_count, cudaStream_t st);
}  // namespace gb

namespace {

thread_local std::string g_last_error;

gb_status fail(gb_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return st;
}

#define GB_CUDA(call)                                                                                   \
    do {                                                                                                \
        cudaError_t e_ = (call);                                                                        \
        if (e_ != cudaSuccess) {                                                                        \
            if (e_ == cudaErrorMemoryAllocation)                                                        \
                return fail(GB_OOM, "%s:%d: %s", __FILE__, __LINE__, cudaGetErrorString(e_));           \
            return fail(GB_CUDA_ERROR, "%s:%d: %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
        }                                                                                               \
    } while (0)

// Grow-only device buffer.
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap && p) return cudaSuccess;
        if (p) {
            cudaError_t e = cudaFree(p);
            if (e != cudaSuccess) return e;
            p = nullptr;
            cap = 0;
        }
        size_t want = bytes < 256 ? 256 : bytes + bytes / 8;
        cudaError_t e = cudaMalloc(&p, want);
        if (e != cudaSuccess) {
            p = nullptr;
            return e;
        }
        cap = want;
        return cudaSuccess;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

}  // namespace

struct ProfRec {
    int id;
    cudaEvent_t start, stop;
};

struct gb_context {
    int device = 0;
    int sm_count = 148;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    int64_t launches = 0;
    int texel_grad_stride = 3;  // gb_context_set_texel_grad_stride
    const float* tex_rgba = nullptr;  // gb_context_set_texel_rgba
    DevBuf grid64;  // parity build: fp64 texel-gradient scratch (added into the caller's fp32 buffer after K4)
    DevBuf tile_hist, keys64_tmp;  // binning scratch (per-tile counts and CTA bases, bucket merge passes)
    DevBuf sort_temp, keys_tmp, vals_tmp, depth_tmp, iota_tmp;  // radix build scratch
    DevBuf scan_temp, accum, adam_bad, ssim_tmp,
        metric_tmp, fuse_color, fuse_trans, fuse_last, fuse_grad;
    uint32_t* pinned_total = nullptr;
    bool prof = false;
    std::vector<ProfRec> prof_recs;
    std::vector<cudaEvent_t> prof_pool;
};

namespace {
cudaEvent_t prof_event(gb_context* ctx) {
    if (!ctx->prof_pool.empty()) {
        cudaEvent_t e = ctx->prof_pool.back();
        ctx->prof_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// Launch sites recorded while gb_graph_begin's capture is open on this thread: each becomes a pair of
// event-record nodes in the graph, re-pointed at fresh timing events on every profiled launch.
struct CaptureSite {
    gb_context* ctx;
    int id;
    cudaEvent_t start, stop;
};
thread_local std::vector<CaptureSite>* t_capture = nullptr;

// Brackets one launch site with CUDA events on the context stream when profiling (or, inside a
// gb_graph capture, always: the graph decides per launch whether the site is timed).
struct ProfScope {
    gb_context* ctx;
    int id;
    cudaEvent_t start = nullptr;
    bool graph = false;
    ProfScope(gb_context* c, int i) : ctx(c), id(i) {
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(ctx->stream, &cap) != cudaSuccess) return;
        if (cap != cudaStreamCaptureStatusNone) {
            if (!t_capture) return;  // somebody else's capture: events would not time anything
            graph = true;
            start = prof_event(ctx);
            cudaEventRecordWithFlags(start, ctx->stream, cudaEventRecordExternal);
        } else if (ctx->prof) {
            start = prof_event(ctx);
            cudaEventRecord(start, ctx->stream);
        }
    }
    ~ProfScope() {
        if (!start) return;
        cudaEvent_t stop = prof_event(ctx);
        if (graph) {
            cudaEventRecordWithFlags(stop, ctx->stream, cudaEventRecordExternal);
            t_capture->push_back({ctx, id, start, stop});
        } else {
            cudaEventRecord(stop, ctx->stream);
            ctx->prof_recs.push_back({id, start, stop});
        }
    }
};
}  // namespace

struct gb_binning {
    gb_context* ctx = nullptr;
    bool built = false;
    int mode = 0;
    int width = 0, height = 0;
    gb_raster_config cfg{};
    int tiles_x = 0, tiles_y = 0;
    int64_t K = 0;
    int n = 0;
    int64_t P = 0;         // pair count; -1 = on the device only (capacity mode, not read back yet)
    int64_t capacity = 0;  // > 0: capacity mode (no host read-back of P; see gb_binning_set_capacity)
    int32_t* overflow = nullptr;
    DevBuf headers, cull, rects, counts, depth, values, ranges;
    DevBuf tile_off, keys64;  // tile-bucket build: tile offsets (n_tiles + 1; [n_tiles] = P), (depth << 32 | id) keys
    DevBuf offsets, perm, keys;  // radix build (deep scenes): per-primitive pair offsets ([K] = P), depth order
    bool radix = false;          // the last build took the radix path
    DevBuf trans64;  // parity build: the forward's fp64 final transmittance, rewound by the backward
};

namespace {

gb_status set_device(gb_context* ctx) {
    GB_CUDA(cudaSetDevice(ctx->device));
    return GB_OK;
}

constexpr int kMaxImageSide = 65536 - 16;

gb_status validate_camera(const gb_camera* cam) {
    if (!cam) return fail(GB_INVALID_ARGUMENT, "camera is null");
    if (cam->width < 1 || cam->height < 1)
        return fail(GB_INVALID_ARGUMENT, "ImagePlaneCamera: width and height must be >= 1");
    for (int i = 0; i < 3; ++i)
        if (!(cam->background[i] >= 0.0 && cam->background[i] <= 1.0))
            return fail(GB_INVALID_ARGUMENT, "ImagePlaneCamera: background must be in [0,1]");
    if (cam->mode != GB_MODE_ORTHO && cam->mode != GB_MODE_PINHOLE)
        return fail(GB_INVALID_ARGUMENT, "camera mode must be GB_MODE_ORTHO or GB_MODE_PINHOLE");
    if (cam->mode == GB_MODE_PINHOLE && !(cam->fx != 0.0 && cam->fy != 0.0 && std::isfinite(cam->fx) &&
                                          std::isfinite(cam->fy)))
        return fail(GB_INVALID_ARGUMENT, "pinhole camera: fx and fy must be finite and non-zero");
    // the compositors pack a pixel's (x, y) into 16 + 16 bits (tiles overhang the image by < 16 px)
    if (cam->width > kMaxImageSide || cam->height > kMaxImageSide)
        return fail(GB_NOT_SUPPORTED, "image too large (at most 65520 pixels per side)");
    return GB_OK;
}

gb_status validate_config(const gb_raster_config* cfg) {
    if (!cfg) return fail(GB_INVALID_ARGUMENT, "config is null");
    if (cfg->tile_size < 1) return fail(GB_INVALID_ARGUMENT, "RasterConfig: tile_size must be >= 1");
    if (cfg->threads < 1) return fail(GB_INVALID_ARGUMENT, "RasterConfig: threads must be >= 1");
    if (cfg->tile_size > 16) return fail(GB_NOT_SUPPORTED, "RasterConfig: tile_size > 16 is not supported on the GPU path");
    return GB_OK;
}

gb_status validate_splats(const gb_splats* s, int mode) {
    if (!s) return fail(GB_INVALID_ARGUMENT, "splats is null");
    if (s->count < 0) return fail(GB_INVALID_ARGUMENT, "splat count must be >= 0");
    if (s->count >= (int64_t)1 << 31) return fail(GB_NOT_SUPPORTED, "splat count must be < 2^31");
    if (s->grid.n < 1) return fail(GB_INVALID_ARGUMENT, "ColorGridConfig: n must be >= 1");
    if (!(s->grid.sigma > 0.0)) return fail(GB_INVALID_ARGUMENT, "ColorGridConfig: sigma must be > 0");
    if (s->grid.n > 64) return fail(GB_NOT_SUPPORTED, "ColorGridConfig: n > 64 is not supported");
    if (s->count == 0) return GB_OK;
    if (!s->position || !s->log_scale || !s->opacity_logit || !s->grid_values)
        return fail(GB_INVALID_ARGUMENT, "splats: position/log_scale/opacity_logit/grid_values must be non-null");
    if (mode == GB_MODE_ORTHO && (!s->depth_key || !s->theta))
        return fail(GB_INVALID_ARGUMENT, "ortho splats need depth_key and theta");
    if (mode == GB_MODE_PINHOLE && !s->quat) return fail(GB_INVALID_ARGUMENT, "pinhole splats need quat");
    if ((s->grid.n % 2) == 0 && (reinterpret_cast<uintptr_t>(s->grid_values) & 15))
        return fail(GB_INVALID_ARGUMENT, "grid_values must be 16-byte aligned");
    if (reinterpret_cast<uintptr_t>(s->log_scale) & 7) return fail(GB_INVALID_ARGUMENT, "log_scale must be 8-byte aligned");
    if (mode == GB_MODE_PINHOLE && (reinterpret_cast<uintptr_t>(s->quat) & 15))
        return fail(GB_INVALID_ARGUMENT, "quat must be 16-byte aligned");
    return GB_OK;
}

// gradient buffers take vector reds (K4/K5): ortho position and log_scale 8-B aligned, quat and even-n grids 16-B
gb_status validate_grads(const gb_grads* g, int mode, int n, const char* where, int texel_stride = 3) {
    if (!g->position || !g->log_scale || !g->opacity_logit || !g->grid_values ||
        (mode == GB_MODE_ORTHO && !g->theta) || (mode == GB_MODE_PINHOLE && !g->quat))
        return fail(GB_INVALID_ARGUMENT, "%s: null gradient buffer", where);
    const bool bad = (reinterpret_cast<uintptr_t>(g->log_scale) & 7) ||
                     (mode == GB_MODE_ORTHO && (reinterpret_cast<uintptr_t>(g->position) & 7)) ||
                     (mode == GB_MODE_PINHOLE && (reinterpret_cast<uintptr_t>(g->quat) & 15)) ||
                     (((n % 2) == 0 || texel_stride == 4) && (reinterpret_cast<uintptr_t>(g->grid_values) & 15));
    if (bad) return fail(GB_INVALID_ARGUMENT, "%s: misaligned gradient buffer", where);
    return GB_OK;
}

#ifdef GB_PARITY_F64
// parity build: K4 accumulates texel gradients into fp64 scratch, added into the caller's buffer after K4
gb_status grid_scratch(gb_context* ctx, int64_t K, int n, gb::real** out) {
    const size_t bytes = sizeof(double) * (size_t)K * 3 * n * n;
    GB_CUDA(ctx->grid64.ensure(bytes > 0 ? bytes : 8));
    GB_CUDA(cudaMemsetAsync(ctx->grid64.p, 0, bytes, ctx->stream));
    *out = ctx->grid64.as<double>();
    return GB_OK;
}
gb_status trans_scratch(gb_context* ctx, const gb_binning* b) {
    GB_CUDA(const_cast<gb_binning*>(b)->trans64.ensure(sizeof(double) * (size_t)b->width * b->height));
    return GB_OK;
}
#endif

gb::CamConst make_cam_const(const gb_camera* cam) {
    gb::CamConst cc;
    cc.width = cam->width;
    cc.height = cam->height;
    cc.inv_fx = cam->mode == GB_MODE_PINHOLE ? (float)(1.0 / cam->fx) : 0.0f;
    cc.inv_fy = cam->mode == GB_MODE_PINHOLE ? (float)(1.0 / cam->fy) : 0.0f;
    for (int i = 0; i < 3; ++i) cc.bg[i] = (gb::real)cam->background[i];
    return cc;
}

gb::RasterConst make_raster_const(const gb_context* ctx, const gb_binning* b, int n, double sigma) {
    gb::RasterConst rc;
    rc.tile_size = b->cfg.tile_size;
    rc.tiles_x = b->tiles_x;
    rc.tiles_y = b->tiles_y;
    rc.alpha_skip = (gb::real)b->cfg.alpha_skip;
    // <= 0 disables the stop (raster.hpp:250); folded here so the compositors compare against a kernel
    // parameter (a constant-bank operand) instead of re-deriving the threshold in registers
    rc.early_stop = b->cfg.early_stop_transmittance > 0.0 ? (gb::real)b->cfg.early_stop_transmittance : (gb::real)-1;
    rc.tex_scale = (gb::real)((double)(n - 1) / (2.0 * sigma));
    rc.tex_offset = (gb::real)((double)(n - 1) * 0.5);
    rc.sigma = (gb::real)sigma;
#ifdef GB_PARITY_F64
    rc.trans64 = b->trans64.as<double>();
    rc.tgs = 3;  // the parity build's fp64 texel scratch keeps the reference layout
    rc.tex4 = nullptr;
#else
    rc.tgs = ctx->texel_grad_stride;
    rc.tex4 = reinterpret_cast<const float4*>(ctx->tex_rgba);
#endif
#ifdef GB_DEBUG_CHECKS
    rc.dbg_K = b->K;
#endif
    return rc;
}

}  // namespace

extern "C" {

int gb_abi_version(void) { return GB_ABI_VERSION; }

const char* gb_last_error_string(void) { return g_last_error.c_str(); }

gb_status gb_context_create(int device, gb_context** out) {
    if (!out) return fail(GB_INVALID_ARGUMENT, "out is null");
    *out = nullptr;
    int count = 0;
    GB_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) return fail(GB_INVALID_ARGUMENT, "device %d out of range (%d)", device, count);
    GB_CUDA(cudaSetDevice(device));
    gb_context* ctx = new gb_context();
    ctx->device = device;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) == cudaSuccess) ctx->sm_count = prop.multiProcessorCount;
    cudaError_t e = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMallocHost(&ctx->pinned_total, sizeof(uint32_t));
    if (e != cudaSuccess) {
        if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
        delete ctx;
        return fail(GB_CUDA_ERROR, "context setup: %s", cudaGetErrorString(e));
    }
    ctx->stream = ctx->own_stream;
    *out = ctx;
    return GB_OK;
}

gb_status gb_context_destroy(gb_context* ctx) {
    if (!ctx) return GB_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    ctx->scan_temp.release();
    ctx->tile_hist.release();
    ctx->sort_temp.release();
    ctx->keys_tmp.release();
    ctx->vals_tmp.release();
    ctx->depth_tmp.release();
    ctx->iota_tmp.release();
    ctx->keys64_tmp.release();
    ctx->accum.release();
    ctx->grid64.release();
    ctx->adam_bad.release();
    ctx->ssim_tmp.release();
    ctx->metric_tmp.release();
    if (ctx->pinned_total) cudaFreeHost(ctx->pinned_total);
    for (const ProfRec& r : ctx->prof_recs) {
        cudaEventDestroy(r.start);
        cudaEventDestroy(r.stop);
    }
    for (cudaEvent_t e : ctx->prof_pool) cudaEventDestroy(e);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
    return GB_OK;
}

gb_status gb_context_set_stream(gb_context* ctx, void* stream) {
    if (!ctx) return fail(GB_INVALID_ARGUMENT, "ctx is null");
    ctx->stream = static_cast<cudaStream_t>(stream);  // NULL = the legacy default stream
    return GB_OK;
}

void* gb_context_stream(gb_context* ctx) { return ctx ? ctx->stream : nullptr; }

gb_status gb_sync(gb_context* ctx) {
    if (!ctx) return fail(GB_INVALID_ARGUMENT, "ctx is null");
    if (gb_status s = set_device(ctx)) return s;
    GB_CUDA(cudaStreamSynchronize(ctx->stream));
    return GB_OK;
}

int64_t gb_context_launch_count(const gb_context* ctx) { return ctx ? ctx->launches : 0; }

gb_status gb_context_profile(gb_context* ctx, int enable) {
    if (!ctx) return fail(GB_INVALID_ARGUMENT, "ctx is null");
    ctx->prof = enable != 0;
    return GB_OK;
}

gb_status gb_context_profile_read(gb_context* ctx, double* total_ms, int64_t* counts, int n) {
    if (!ctx || n < 0) return fail(GB_INVALID_ARGUMENT, "bad argument");
    if (gb_status st = set_device(ctx)) return st;
    GB_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int i = 0; i < n; ++i) {
        if (total_ms) total_ms[i] = 0.0;
        if (counts) counts[i] = 0;
    }
    for (const ProfRec& r : ctx->prof_recs) {
        float ms = 0.0f;
        GB_CUDA(cudaEventElapsedTime(&ms, r.start, r.stop));
        if (r.id < n) {
            if (total_ms) total_ms[r.id] += ms;
            if (counts) counts[r.id] += 1;
        }
        ctx->prof_pool.push_back(r.start);
        ctx->prof_pool.push_back(r.stop);
    }
    ctx->prof_recs.clear();
    return GB_OK;
}

// ---- CUDA graphs of context work (one training step's views) ----------------------------------
struct gb_graph {
    gb_context* origin = nullptr;
    cudaGraph_t graph = nullptr;  // kept: the exec's event-record nodes are addressed through its nodes
    cudaGraphExec_t exec = nullptr;
    cudaEvent_t dummy = nullptr;
    struct Site {
        gb_context* ctx;
        int id;
        cudaGraphNode_t start, stop;
    };
    std::vector<Site> sites;
    std::vector<std::pair<gb_context*, int64_t>> launches;  // kernels per replay, per context
};

namespace {
struct CaptureState {
    std::vector<CaptureSite> sites;
    std::vector<std::pair<gb_context*, int64_t>> launches0;
};
thread_local CaptureState* t_state = nullptr;
}  // namespace

gb_status gb_graph_begin(gb_context* const* ctxs, int32_t n) {
    if (!ctxs || n < 1 || !ctxs[0]) return fail(GB_INVALID_ARGUMENT, "graph_begin: no context");
    if (t_state) return fail(GB_INVALID_ARGUMENT, "graph_begin: a capture is already open on this thread");
    if (gb_status st = set_device(ctxs[0])) return st;
    auto* state = new CaptureState();
    for (int i = 0; i < n; ++i)
        if (ctxs[i]) state->launches0.push_back({ctxs[i], ctxs[i]->launches});
    cudaError_t e = cudaStreamBeginCapture(ctxs[0]->stream, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) {
        delete state;
        return fail(GB_CUDA_ERROR, "graph_begin: %s", cudaGetErrorString(e));
    }
    t_state = state;
    t_capture = &state->sites;
    return GB_OK;
}

gb_status gb_graph_end(gb_context* const* ctxs, int32_t n, gb_graph** out) {
    if (!ctxs || n < 1 || !ctxs[0] || !out) return fail(GB_INVALID_ARGUMENT, "graph_end: bad argument");
    if (!t_state) return fail(GB_INVALID_ARGUMENT, "graph_end: no capture open on this thread");
    std::unique_ptr<CaptureState> state(t_state);
    t_state = nullptr;
    t_capture = nullptr;
    *out = nullptr;
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(ctxs[0]->stream, &graph);
    auto give_back = [&]() {
        for (const CaptureSite& c : state->sites) {
            c.ctx->prof_pool.push_back(c.start);
            c.ctx->prof_pool.push_back(c.stop);
        }
    };
    if (e != cudaSuccess) {
        give_back();
        return fail(GB_CUDA_ERROR, "graph_end: capture failed: %s", cudaGetErrorString(e));
    }
    std::unique_ptr<gb_graph> g(new gb_graph());
    g->origin = ctxs[0];
    // the capture launched nothing: move its launch counts from the contexts to the graph
    for (auto& [c, l0] : state->launches0) {
        g->launches.push_back({c, c->launches - l0});
        c->launches = l0;
    }
    // map every site's events to their event-record nodes
    size_t nn = 0;
    cudaGraphGetNodes(graph, nullptr, &nn);
    std::vector<cudaGraphNode_t> nodes(nn);
    if (nn) cudaGraphGetNodes(graph, nodes.data(), &nn);
    std::vector<std::pair<cudaEvent_t, cudaGraphNode_t>> rec;
    for (cudaGraphNode_t nd : nodes) {
        cudaGraphNodeType t;
        cudaGraphNodeGetType(nd, &t);
        if (t != cudaGraphNodeTypeEventRecord) continue;
        cudaEvent_t ev = nullptr;
        cudaGraphEventRecordNodeGetEvent(nd, &ev);
        rec.push_back({ev, nd});
    }
    auto node_of = [&](cudaEvent_t ev) -> cudaGraphNode_t {
        for (auto& r : rec)
            if (r.first == ev) return r.second;
        return nullptr;
    };
    for (const CaptureSite& c : state->sites) {
        cudaGraphNode_t a = node_of(c.start), b = node_of(c.stop);
        if (a && b) g->sites.push_back({c.ctx, c.id, a, b});
    }
    g->graph = graph;
    e = cudaGraphInstantiate(&g->exec, graph, 0);
    if (e == cudaSuccess) e = cudaEventCreate(&g->dummy);
    for (const auto& st : g->sites) {  // untimed until a profiled launch re-points them
        if (e != cudaSuccess) break;
        e = cudaGraphExecEventRecordNodeSetEvent(g->exec, st.start, g->dummy);
        if (e == cudaSuccess) e = cudaGraphExecEventRecordNodeSetEvent(g->exec, st.stop, g->dummy);
    }
    give_back();
    if (e != cudaSuccess) {
        if (g->exec) cudaGraphExecDestroy(g->exec);
        if (g->dummy) cudaEventDestroy(g->dummy);
        cudaGraphDestroy(graph);
        return fail(GB_CUDA_ERROR, "graph_end: %s", cudaGetErrorString(e));
    }
    *out = g.release();
    return GB_OK;
}

gb_status gb_graph_launch(gb_graph* g) {
    if (!g || !g->exec) return fail(GB_INVALID_ARGUMENT, "graph_launch: null graph");
    if (gb_status st = set_device(g->origin)) return st;
    for (const auto& st : g->sites) {
        cudaEvent_t a = g->dummy, b = g->dummy;
        if (st.ctx->prof) {
            a = prof_event(st.ctx);
            b = prof_event(st.ctx);
            st.ctx->prof_recs.push_back({st.id, a, b});
        }
        GB_CUDA(cudaGraphExecEventRecordNodeSetEvent(g->exec, st.start, a));
        GB_CUDA(cudaGraphExecEventRecordNodeSetEvent(g->exec, st.stop, b));
    }
    GB_CUDA(cudaGraphLaunch(g->exec, g->origin->stream));
    for (auto& [c, l] : g->launches) c->launches += l;
    return GB_OK;
}

gb_status gb_graph_destroy(gb_graph* g) {
    if (!g) return GB_OK;
    cudaSetDevice(g->origin->device);
    cudaStreamSynchronize(g->origin->stream);
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    if (g->dummy) cudaEventDestroy(g->dummy);
    delete g;
    return GB_OK;
}

gb_status gb_context_profile_intervals(gb_context* ctx, void* ref_event, int32_t id, double* start_ms,
                                      double* stop_ms, int64_t cap, int64_t* n) {
    if (!ctx || !ref_event || !n || cap < 0) return fail(GB_INVALID_ARGUMENT, "bad argument");
    if (gb_status st = set_device(ctx)) return st;
    GB_CUDA(cudaStreamSynchronize(ctx->stream));
    cudaEvent_t ref = reinterpret_cast<cudaEvent_t>(ref_event);
    int64_t k = 0;
    for (const ProfRec& r : ctx->prof_recs) {
        if (r.id != id) continue;
        if (k < cap) {
            float a = 0.0f, b = 0.0f;
            GB_CUDA(cudaEventElapsedTime(&a, ref, r.start));
            GB_CUDA(cudaEventElapsedTime(&b, ref, r.stop));
            if (start_ms) start_ms[k] = a;
            if (stop_ms) stop_ms[k] = b;
        }
        ++k;
    }
    *n = k;
    return GB_OK;
}

gb_status gb_stream_wait_event(gb_context* ctx, void* event, int32_t external) {
    if (!ctx || !event) return fail(GB_INVALID_ARGUMENT, "null argument");
    if (gb_status st = set_device(ctx)) return st;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    GB_CUDA(cudaStreamIsCapturing(ctx->stream, &cap));
    // the external flag only means something (and is only accepted) inside a capture
    const bool ext = external && cap == cudaStreamCaptureStatusActive;
    GB_CUDA(cudaStreamWaitEvent(ctx->stream, reinterpret_cast<cudaEvent_t>(event),
                                ext ? cudaEventWaitExternal : cudaEventWaitDefault));
    return GB_OK;
}

gb_status gb_event_create(gb_context* ctx, void** event) {
    if (!ctx || !event) return fail(GB_INVALID_ARGUMENT, "null argument");
    if (gb_status st = set_device(ctx)) return st;
    cudaEvent_t e = nullptr;
    GB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    *event = e;
    return GB_OK;
}

gb_status gb_event_record(gb_context* ctx, void* event) {
    if (!ctx || !event) return fail(GB_INVALID_ARGUMENT, "null argument");
    if (gb_status st = set_device(ctx)) return st;
    GB_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(event), ctx->stream));
    return GB_OK;
}

gb_status gb_event_destroy(gb_context* ctx, void* event) {
    if (!ctx || !event) return GB_OK;
    if (gb_status st = set_device(ctx)) return st;
    GB_CUDA(cudaEventDestroy(static_cast<cudaEvent_t>(event)));
    return GB_OK;
}

gb_status gb_device_alloc(gb_context* ctx, uint64_t bytes, void** out) {
    if (!ctx || !out) return fail(GB_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    if (gb_status st = set_device(ctx)) return st;
    GB_CUDA(cudaMalloc(out, bytes > 0 ? bytes : 1));
    return GB_OK;
}

gb_status gb_device_free(gb_context* ctx, void* ptr) {
    if (!ctx) return fail(GB_INVALID_ARGUMENT, "ctx is null");
    if (!ptr) return GB_OK;
    if (gb_status st = set_device(ctx)) return st;
    GB_CUDA(cudaFree(ptr));
    return GB_OK;
}

gb_status gb_copy_h2d(gb_context* ctx, void* dst, const void* src, uint64_t bytes, int sync) {
    if (!ctx || (bytes && (!dst || !src))) return fail(GB_INVALID_ARGUMENT, "null argument");
    if (gb_status st = set_device(ctx)) return st;
    if (bytes) GB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    if (sync) GB_CUDA(cudaStreamSynchronize(ctx->stream));
    return GB_OK;
}

gb_status gb_copy_d2h(gb_context* ctx, void* dst, const void* src, uint64_t bytes, int sync) {
    if (!ctx || (bytes && (!dst || !src))) return fail(GB_INVALID_ARGUMENT, "null argument");
    if (gb_status st = set_device(ctx)) return st;
    if (bytes) GB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    if (sync) GB_CUDA(cudaStreamSynchronize(ctx->stream));
    return GB_OK;
}

gb_status gb_memset_device(gb_context* ctx, void* dst, int value, uint64_t bytes) {
    if (!ctx || (bytes && !dst)) return fail(GB_INVALID_ARGUMENT, "null argument");
    if (gb_status st = set_device(ctx)) return st;
    if (bytes) GB_CUDA(cudaMemsetAsync(dst, value, bytes, ctx->stream));
    return GB_OK;
}

gb_status gb_binning_create(gb_context* ctx, gb_binning** out) {
    if (!ctx || !out) return fail(GB_INVALID_ARGUMENT, "null argument");
    *out = new gb_binning();
    (*out)->ctx = ctx;
    return GB_OK;
}

gb_status gb_binning_destroy(gb_binning* b) {
    if (!b) return GB_OK;
    cudaSetDevice(b->ctx->device);
    cudaStreamSynchronize(b->ctx->stream);
    b->headers.release();
    b->cull.release();
    b->rects.release();
    b->counts.release();
    b->depth.release();
    b->values.release();
    b->tile_off.release();
    b->offsets.release();
    b->perm.release();
    b->keys.release();
    b->keys64.release();
    b->ranges.release();
    b->trans64.release();
    delete b;
    return GB_OK;
}

gb_status gb_build_binning(gb_context* ctx, const gb_splats* s, const gb_camera* cam, const gb_raster_config* cfg,
                           gb_binning* b) {
    if (!ctx || !b) return fail(GB_INVALID_ARGUMENT, "null context or binning");
    if (gb_status st = validate_camera(cam)) return st;
    if (gb_status st = validate_config(cfg)) return st;
    if (gb_status st = validate_splats(s, cam->mode)) return st;
    if (gb_status st = set_device(ctx)) return st;
    cudaStream_t stream = ctx->stream;
    const int64_t K = s->count;
    b->built = false;
    b->mode = cam->mode;
    b->width = cam->width;
    b->height = cam->height;
    b->cfg = *cfg;
    b->tiles_x = (cam->width + cfg->tile_size - 1) / cfg->tile_size;
    b->tiles_y = (cam->height + cfg->tile_size - 1) / cfg->tile_size;
    b->K = K;
    b->n = s->grid.n;
    const int n_tiles = b->tiles_x * b->tiles_y;
    const int64_t Kc = K > 0 ? K : 1;
    GB_CUDA(b->headers.ensure(sizeof(gb::ScreenHeader) * Kc));
    GB_CUDA(b->cull.ensure(sizeof(gb::CullRec) * Kc));
    GB_CUDA(b->rects.ensure(sizeof(uint2) * Kc));
    GB_CUDA(b->counts.ensure(sizeof(uint32_t) * Kc));
    // K1, then K2 (gb_binning.cu): tile buckets sorted in place, or -- deep scenes, more than
    // deep_bucket_mean() pairs per tile on average -- the two stable radix sorts
    GB_CUDA(b->depth.ensure(sizeof(uint32_t) * Kc));
    GB_CUDA(b->ranges.ensure(sizeof(uint2) * (n_tiles > 0 ? n_tiles : 1)));
    gb::ProjParams pp = gb::make_proj_params(s, cam, cfg, b->tiles_x, b->tiles_y);
    {
        ProfScope ps(ctx, GB_K_PROJECT);
        GB_CUDA(gb::launch_project(pp, b->headers.as<gb::ScreenHeader>(), b->cull.as<gb::CullRec>(), b->rects.as<uint2>(),
                                   b->counts.as<uint32_t>(), b->depth.as<uint32_t>(), stream));
    }
    ctx->launches += K > 0;
    const int64_t deep = (int64_t)gb::deep_bucket_mean() * n_tiles;
    // capacity mode decides by the slots; the blocking mode by the pair count its tile scan reads back
    bool radix = b->capacity > deep;
    int64_t P = 0;  // pair slots the lists are built in: the exact count, or the capacity
    if (!radix) {
        GB_CUDA(b->tile_off.ensure(sizeof(uint32_t) * ((size_t)n_tiles + 1)));
        GB_CUDA(ctx->tile_hist.ensure(sizeof(uint32_t) * gb::tile_scratch_words(n_tiles)));
        GB_CUDA(ctx->scan_temp.ensure(gb::tile_scan_temp_bytes(n_tiles)));
        {
            ProfScope ps(ctx, GB_K_SCAN);
            GB_CUDA(gb::launch_tile_offsets(ctx->scan_temp.p, ctx->scan_temp.cap, K, b->tiles_x, n_tiles,
                                            b->counts.as<uint32_t>(), b->rects.as<uint2>(),
                                            ctx->tile_hist.as<uint32_t>(), b->tile_off.as<uint32_t>(), stream));
        }
        ctx->launches += gb::tile_offsets_launches(K, n_tiles);
        if (b->capacity > 0) {
            P = b->capacity;
            b->P = -1;
        } else {
            GB_CUDA(cudaMemcpyAsync(ctx->pinned_total, b->tile_off.as<uint32_t>() + n_tiles, sizeof(uint32_t),
                                    cudaMemcpyDeviceToHost, stream));
            GB_CUDA(cudaStreamSynchronize(stream));
            P = *ctx->pinned_total;
            if (P >= 0x7fffffffll)
                return fail(GB_NOT_SUPPORTED,
                            "build_binning: %lld+ tile/primitive pairs exceed the 2^31 - 1 the lists index",
                            (long long)P);
            b->P = P;
            radix = P > deep;
        }
    }
    b->radix = radix;
    if (!radix) {
        const int64_t Pc = P > 0 ? P : 1;
        GB_CUDA(b->keys64.ensure(sizeof(uint64_t) * Pc));
        GB_CUDA(b->values.ensure(sizeof(int32_t) * Pc));
        GB_CUDA(ctx->keys64_tmp.ensure(sizeof(uint64_t) * Pc));
        {
            ProfScope ps(ctx, GB_K_DUPLICATE);
            GB_CUDA(gb::launch_scatter(K, b->tiles_x, n_tiles, b->counts.as<uint32_t>(), b->rects.as<uint2>(),
                                       b->depth.as<uint32_t>(), b->tile_off.as<uint32_t>(),
                                       ctx->tile_hist.as<uint32_t>(), b->keys64.as<uint64_t>(), (uint32_t)P, stream));
        }
        {
            ProfScope ps(ctx, GB_K_SORT);
            GB_CUDA(gb::launch_tile_lists(n_tiles, b->tile_off.as<uint32_t>(), (uint32_t)P, b->keys64.as<uint64_t>(),
                                          ctx->keys64_tmp.as<uint64_t>(), b->values.as<int32_t>(),
                                          b->ranges.as<uint2>(), b->capacity > 0 ? b->overflow : nullptr, stream));
        }
        ctx->launches += (K > 0 && n_tiles > 0) + (n_tiles > 0);
        b->built = true;
        return GB_OK;
    }
    // deep scenes: K2a primitives in (depth, index) order
    GB_CUDA(b->offsets.ensure(sizeof(uint32_t) * (Kc + 1)));
    GB_CUDA(b->perm.ensure(sizeof(int32_t) * Kc));
    GB_CUDA(ctx->depth_tmp.ensure(sizeof(uint32_t) * Kc));
    GB_CUDA(ctx->iota_tmp.ensure(sizeof(int32_t) * Kc));
    GB_CUDA(ctx->scan_temp.ensure(gb::scan_temp_bytes(Kc)));
    GB_CUDA(ctx->sort_temp.ensure(gb::sort_temp_bytes(Kc)));
    {
        ProfScope ps(ctx, GB_K_SORT);
        GB_CUDA(gb::launch_depth_sort(ctx->sort_temp.p, ctx->sort_temp.cap, b->depth.as<uint32_t>(),
                                      ctx->depth_tmp.as<uint32_t>(), ctx->iota_tmp.as<int32_t>(),
                                      b->perm.as<int32_t>(), K, stream));
    }
    ctx->launches += K > 0 ? 1 + gb::sort_launches(32) : 0;
    // K2b tile counts in that order, scanned -> P
    {
        ProfScope ps(ctx, GB_K_SCAN);
        GB_CUDA(gb::launch_scan(ctx->scan_temp.p, ctx->scan_temp.cap, b->perm.as<int32_t>(), b->counts.as<uint32_t>(),
                                b->offsets.as<uint32_t>(), K, stream));
    }
    ctx->launches += K > 0 ? 2 : 0;  // CUB scan (init + scan) over the permuted counts
    if (b->capacity > 0) {
        P = b->capacity;
        b->P = -1;
    }  // (blocking: P and b->P from the tile scan above)
    const int64_t Pc = P > 0 ? P : 1;
    const int n_keys = n_tiles + (b->capacity > 0);
    GB_CUDA(b->keys.ensure(sizeof(uint32_t) * Pc));
    GB_CUDA(b->values.ensure(sizeof(int32_t) * Pc));
    GB_CUDA(ctx->keys_tmp.ensure(sizeof(uint32_t) * Pc));
    GB_CUDA(ctx->vals_tmp.ensure(sizeof(int32_t) * Pc));
    GB_CUDA(ctx->sort_temp.ensure(gb::sort_temp_bytes(Pc)));
    // K2c duplicate in depth order, K2d stable sort on the tile id, K2e ranges
    {
        ProfScope ps(ctx, GB_K_DUPLICATE);
        GB_CUDA(gb::launch_duplicate(K, b->tiles_x, b->perm.as<int32_t>(), b->offsets.as<uint32_t>(),
                                     b->rects.as<uint2>(), ctx->keys_tmp.as<uint32_t>(), ctx->vals_tmp.as<int32_t>(),
                                     (uint32_t)P, b->overflow, stream));
        if (b->capacity > 0)
            GB_CUDA(gb::launch_pad((uint32_t)P, b->offsets.as<uint32_t>() + K, n_tiles, ctx->keys_tmp.as<uint32_t>(),
                                   ctx->vals_tmp.as<int32_t>(), stream));
    }
    {
        ProfScope ps(ctx, GB_K_SORT);
        GB_CUDA(gb::launch_tile_sort(ctx->sort_temp.p, ctx->sort_temp.cap, ctx->keys_tmp.as<uint32_t>(),
                                     b->keys.as<uint32_t>(), ctx->vals_tmp.as<int32_t>(), b->values.as<int32_t>(), P,
                                     n_keys, stream));
    }
    {
        ProfScope ps(ctx, GB_K_RANGES);
        GB_CUDA(gb::launch_ranges(P, b->keys.as<uint32_t>(), b->ranges.as<uint2>(), n_tiles, stream));
    }
    ctx->launches += (K > 0) + (b->capacity > 0) + (P > 0 ? 1 + gb::sort_launches(gb::tile_sort_bits(n_keys)) : 0);
    b->built = true;
    return GB_OK;
}

namespace {
// the device word holding the build's pair count P
const uint32_t* total_ptr(const gb_binning* b) {
    return b->radix ? b->offsets.as<uint32_t>() + b->K : b->tile_off.as<uint32_t>() + (size_t)b->tiles_x * b->tiles_y;
}

// capacity mode: read the pair count back (synchronous); clamps to the capacity on overflow
gb_status resolve_total(const gb_binning* b) {
    if (b->P >= 0) return GB_OK;
    gb_binning* m = const_cast<gb_binning*>(b);
    if (gb_status st = set_device(b->ctx)) return st;
    GB_CUDA(cudaMemcpyAsync(b->ctx->pinned_total, total_ptr(b), sizeof(uint32_t), cudaMemcpyDeviceToHost,
                            b->ctx->stream));
    GB_CUDA(cudaStreamSynchronize(b->ctx->stream));
    m->P = std::min<int64_t>(*b->ctx->pinned_total, b->capacity);
    return GB_OK;
}
}  // namespace

gb_status gb_binning_set_capacity(gb_binning* b, int64_t capacity, int32_t* overflow) {
    if (!b) return fail(GB_INVALID_ARGUMENT, "null binning");
    if (capacity < 0 || capacity >= 0x7fffffffll)
        return fail(GB_INVALID_ARGUMENT, "binning capacity out of range [0, 2^31 - 1)");
    b->capacity = capacity;
    b->overflow = capacity > 0 ? overflow : nullptr;
    b->built = false;
    return GB_OK;
}

gb_status gb_binning_store_total(gb_context* ctx, const gb_binning* b, uint32_t* dst) {
    if (!ctx || !b || !dst) return fail(GB_INVALID_ARGUMENT, "null argument");
    if (!b->built) return fail(GB_INVALID_ARGUMENT, "binning not built");
    if (gb_status st = set_device(ctx)) return st;
    GB_CUDA(cudaMemcpyAsync(dst, total_ptr(b), sizeof(uint32_t), cudaMemcpyDeviceToDevice, ctx->stream));
    return GB_OK;
}

gb_status gb_binning_info(const gb_binning* b, int32_t* tiles_x, int32_t* tiles_y, int64_t* total) {
    if (!b || !b->built) return fail(GB_INVALID_ARGUMENT, "binning not built");
    if (total)
        if (gb_status st = resolve_total(b)) return st;
    if (tiles_x) *tiles_x = b->tiles_x;
    if (tiles_y) *tiles_y = b->tiles_y;
    if (total) *total = b->P;
    return GB_OK;
}

gb_status gb_binning_copy_to_host(gb_context* ctx, const gb_binning* b, int64_t* offsets, int32_t* values) {
    if (!ctx || !b || !b->built) return fail(GB_INVALID_ARGUMENT, "binning not built");
    if (gb_status st = resolve_total(b)) return st;
    if (gb_status st = set_device(ctx)) return st;
    const int n_tiles = b->tiles_x * b->tiles_y;
    std::string tmp(sizeof(uint2) * (size_t)n_tiles, '\0');
    uint2* ranges = reinterpret_cast<uint2*>(&tmp[0]);
    GB_CUDA(cudaMemcpyAsync(ranges, b->ranges.p, sizeof(uint2) * n_tiles, cudaMemcpyDeviceToHost, ctx->stream));
    if (b->P > 0 && values)
        GB_CUDA(cudaMemcpyAsync(values, b->values.p, sizeof(int32_t) * b->P, cudaMemcpyDeviceToHost, ctx->stream));
    GB_CUDA(cudaStreamSynchronize(ctx->stream));
    // ranges are contiguous and in tile order; empty tiles have start == end == 0
    int64_t o = 0;
    for (int t = 0; t < n_tiles; ++t) {
        offsets[t] = o;
        if (ranges[t].y > ranges[t].x) {
            if ((int64_t)ranges[t].x != o) return fail(GB_CUDA_ERROR, "binning ranges are not contiguous");
            o = ranges[t].y;
        }
    }
    offsets[n_tiles] = o;
    if (o != b->P) return fail(GB_CUDA_ERROR, "binning ranges do not cover all pairs");
    return GB_OK;
}

gb_status gb_render_forward(gb_context* ctx, const gb_splats* s, const gb_camera* cam, const gb_binning* b,
                            gb_render_out* out) {
    if (!ctx || !b || !out) return fail(GB_INVALID_ARGUMENT, "null argument");
    if (gb_status st = validate_camera(cam)) return st;
    if (gb_status st = validate_splats(s, cam->mode)) return st;
    if (!b->built) return fail(GB_INVALID_ARGUMENT, "binning not built");
    if (b->width != cam->width || b->height != cam->height || b->mode != cam->mode)
        return fail(GB_MISMATCH, "render_forward: binning built for different image size");
    if (b->K != s->count || b->n != s->grid.n)
        return fail(GB_MISMATCH, "render_forward: binning built for a different splat set");
    if (out->width != cam->width || out->height != cam->height)
        return fail(GB_MISMATCH, "render_forward: output buffers sized for a different image");
    if (!out->color || !out->final_transmittance || !out->last_rank)
        return fail(GB_INVALID_ARGUMENT, "render_forward: null output buffer");
    if (gb_status st = set_device(ctx)) return st;
#ifdef GB_PARITY_F64
    if (gb_status st = trans_scratch(ctx, b)) return st;
#endif
    const gb::CamConst cc = make_cam_const(cam);
    const gb::RasterConst rc = make_raster_const(ctx, b, s->grid.n, s->grid.sigma);
    ProfScope ps(ctx, GB_K_FORWARD);
    GB_CUDA(gb::launch_forward(cam->mode, s->grid.n, b->tiles_x * b->tiles_y, b->cfg.tile_size,
                               b->ranges.as<uint2>(), b->values.as<int32_t>(), b->headers.as<gb::ScreenHeader>(),
                               b->cull.as<gb::CullRec>(), s->grid_values, cc, rc, out->color, out->final_transmittance, out->last_rank,
                               ctx->stream));
    ctx->launches += 1;
    out->splat_count = s->count;
    out->grid_n = s->grid.n;
    out->tile_size = b->cfg.tile_size;
    return GB_OK;
}

gb_status gb_render_backward(gb_context* ctx, const gb_splats* s, const gb_camera* cam, const gb_binning* b,
                             const gb_render_out* out, const float* image_grad, gb_grads* g) {
    if (!ctx || !b || !out || !g) return fail(GB_INVALID_ARGUMENT, "null argument");
    if (gb_status st = validate_camera(cam)) return st;
    if (gb_status st = validate_splats(s, cam->mode)) return st;
    if (!b->built) return fail(GB_INVALID_ARGUMENT, "binning not built");
    // raster.hpp:280-287
    if (out->splat_count != s->count || out->grid_n != s->grid.n || out->tile_size != b->cfg.tile_size)
        return fail(GB_MISMATCH, "render_backward: output does not match forward inputs");
    if (out->width != cam->width || out->height != cam->height || b->width != cam->width ||
        b->height != cam->height || b->mode != cam->mode || b->K != s->count)
        return fail(GB_MISMATCH, "render_backward: image size mismatch");
    if (!image_grad) return fail(GB_MISMATCH, "render_backward: image_grad size mismatch");
    if (s->count == 0) return GB_OK;
    if (gb_status st = validate_grads(g, cam->mode, s->grid.n, "render_backward", ctx->texel_grad_stride)) return st;
    if (ctx->tex_rgba && ctx->texel_grad_stride != 4)
        return fail(GB_INVALID_ARGUMENT, "render_backward: RGBA texels need texel gradient stride 4");
    if (gb_status st = set_device(ctx)) return st;
    cudaStream_t stream = ctx->stream;
    const int64_t K = s->count;
    GB_CUDA(ctx->accum.ensure(sizeof(gb::real) * gb::kAccumStride * K));
    GB_CUDA(cudaMemsetAsync(ctx->accum.p, 0, sizeof(gb::real) * gb::kAccumStride * K, stream));
    const gb::CamConst cc = make_cam_const(cam);
    const gb::RasterConst rc = make_raster_const(ctx, b, s->grid.n, s->grid.sigma);
#ifdef GB_PARITY_F64
    gb::real* grid_grad = nullptr;
    if (gb_status st = grid_scratch(ctx, K, s->grid.n, &grid_grad)) return st;
#else
    gb::real* grid_grad = g->grid_values;
#endif
    {
        ProfScope ps(ctx, GB_K_BACKWARD);
        GB_CUDA(gb::launch_backward(cam->mode, s->grid.n, b->tiles_x * b->tiles_y, b->cfg.tile_size,
                                    b->ranges.as<uint2>(), b->values.as<int32_t>(),
                                    b->headers.as<gb::ScreenHeader>(), b->cull.as<gb::CullRec>(), s->grid_values, cc, rc,
                                    out->final_transmittance, out->last_rank, image_grad, ctx->accum.as<gb::real>(),
                                    grid_grad, stream));
    }
#ifdef GB_PARITY_F64
    GB_CUDA(gb::launch_add_f64(ctx->grid64.as<double>(), g->grid_values, K * 3 * s->grid.n * s->grid.n, stream));
#endif
    gb::ProjParams pp = gb::make_proj_params(s, cam, &b->cfg, b->tiles_x, b->tiles_y);
    {
        ProfScope ps(ctx, GB_K_CHAIN);
        GB_CUDA(gb::launch_chain(pp, b->counts.as<uint32_t>(), ctx->accum.as<gb::real>(), *g, stream));
    }
    ctx->launches += 2;
    return GB_OK;
}

gb_status gb_render(gb_context* ctx, const gb_splats* s, const gb_camera* cam, const gb_raster_config* cfg,
                    gb_binning* scratch, gb_render_out* out) {
    if (gb_status st = gb_build_binning(ctx, s, cam, cfg, scratch)) return st;
    return gb_render_forward(ctx, s, cam, scratch, out);
}

gb_status gb_l1_loss(gb_context* ctx, const float* color, const float* target, int64_t n, float scale, float* grad,
                     float* loss) {
    if (!ctx || (n > 0 && (!color || !target || !grad))) return fail(GB_INVALID_ARGUMENT, "null argument");
    if (gb_status st = set_device(ctx)) return st;
    ProfScope ps(ctx, GB_K_LOSS);
    GB_CUDA(gb::launch_loss(0, color, target, n, scale, grad, loss, ctx->sm_count, ctx->stream));
    ctx->launches += n > 0;
    return GB_OK;
}

gb_status gb_mse_loss(gb_context* ctx, const float* color, const float* target, int64_t n, float scale, float* grad,
                      float* loss) {
    if (!ctx || (n > 0 && (!color || !target || !grad))) return fail(GB_INVALID_ARGUMENT, "null argument");
    if (gb_status st = set_device(ctx)) return st;
    ProfScope ps(ctx, GB_K_LOSS);
    GB_CUDA(gb::launch_loss(1, color, target, n, scale, grad, loss, ctx->sm_count, ctx->stream));
    ctx->launches += n > 0;
    return GB_OK;
}

gb_status gb_render_loss_backward(gb_context* ctx, const gb_splats* s, const gb_camera* cam, const gb_binning* b,
                                  const float* target, int32_t loss_kind, float scale, gb_render_out* out,
                                  float* image_grad, float* loss, gb_grads* g) {
    if (!ctx || !b || !g || !target) return fail(GB_INVALID_ARGUMENT, "null argument");
    if (loss_kind != GB_LOSS_L1 && loss_kind != GB_LOSS_MSE)
        return fail(GB_INVALID_ARGUMENT, "render_loss_backward: unknown loss kind");
    if (gb_status st = validate_camera(cam)) return st;
    if (gb_status st = validate_splats(s, cam->mode)) return st;
    if (!b->built) return fail(GB_INVALID_ARGUMENT, "binning not built");
    if (b->width != cam->width || b->height != cam->height || b->mode != cam->mode)
        return fail(GB_MISMATCH, "render_loss_backward: binning built for different image size");
    if (b->K != s->count || b->n != s->grid.n)
        return fail(GB_MISMATCH, "render_loss_backward: binning built for a different splat set");
    if (out) {
        if (out->width != cam->width || out->height != cam->height)
            return fail(GB_MISMATCH, "render_loss_backward: output buffers sized for a different image");
        if (!out->color || !out->final_transmittance || !out->last_rank)
            return fail(GB_INVALID_ARGUMENT, "render_loss_backward: null output buffer");
    }
    if (s->count > 0)
        if (gb_status st = validate_grads(g, cam->mode, s->grid.n, "render_loss_backward", ctx->texel_grad_stride)) return st;
    if (ctx->tex_rgba && ctx->texel_grad_stride != 4)
        return fail(GB_INVALID_ARGUMENT, "render_loss_backward: RGBA texels need texel gradient stride 4");
    if (gb_status st = set_device(ctx)) return st;
    const int64_t npix = (int64_t)cam->width * cam->height;
    cudaStream_t stream = ctx->stream;
    const int64_t K = s->count;
    if (K > 0) {
        GB_CUDA(ctx->accum.ensure(sizeof(gb::real) * gb::kAccumStride * K));
        GB_CUDA(cudaMemsetAsync(ctx->accum.p, 0, sizeof(gb::real) * gb::kAccumStride * K, stream));
    }
#ifdef GB_PARITY_F64
    if (gb_status st = trans_scratch(ctx, b)) return st;
#endif
    const gb::CamConst cc = make_cam_const(cam);
    const gb::RasterConst rc = make_raster_const(ctx, b, s->grid.n, s->grid.sigma);
    const int tiles = b->tiles_x * b->tiles_y;
#ifdef GB_PARITY_F64
    gb::real* grid_grad = nullptr;
    if (gb_status st = grid_scratch(ctx, K, s->grid.n, &grid_grad)) return st;
#else
    gb::real* grid_grad = g->grid_values;
#endif
#ifdef GB_FUSED_SINGLE_KERNEL
    if (true) {  // variant build: K3 + K6 + K4 in one kernel (measured slower)
        ProfScope ps(ctx, GB_K_FUSED);
        GB_CUDA(gb::launch_fused(cam->mode, s->grid.n, tiles, b->cfg.tile_size, b->ranges.as<uint2>(),
                                 b->values.as<int32_t>(), b->headers.as<gb::ScreenHeader>(),
                                 b->cull.as<gb::CullRec>(), s->grid_values, cc, rc, loss_kind, target, scale,
                                 out ? out->color : nullptr, out ? out->final_transmittance : nullptr,
                                 out ? out->last_rank : nullptr, image_grad, loss,
                                 K > 0 ? ctx->accum.as<gb::real>() : nullptr, grid_grad, stream));
        ctx->launches += 1;
    }
#else
    {  // K3 with the loss in its epilogue, then K4: no image round trip, no K6 pass
        float* trans = out ? out->final_transmittance : nullptr;
        int32_t* last = out ? out->last_rank : nullptr;
        if (!out) {
            GB_CUDA(ctx->fuse_trans.ensure(sizeof(float) * npix));
            GB_CUDA(ctx->fuse_last.ensure(sizeof(int32_t) * npix));
            trans = ctx->fuse_trans.as<float>();
            last = ctx->fuse_last.as<int32_t>();
        }
        float* grad = image_grad;
        if (!grad) {
            GB_CUDA(ctx->fuse_grad.ensure(sizeof(float) * 3 * npix));
            grad = ctx->fuse_grad.as<float>();
        }
        {
            ProfScope ps(ctx, GB_K_FORWARD);
            GB_CUDA(gb::launch_forward_loss(cam->mode, s->grid.n, tiles, b->cfg.tile_size, b->ranges.as<uint2>(),
                                            b->values.as<int32_t>(), b->headers.as<gb::ScreenHeader>(),
                                            b->cull.as<gb::CullRec>(), s->grid_values, cc, rc, loss_kind, target,
                                            scale, out ? out->color : nullptr, trans, last, grad, loss, stream));
        }
        {
            ProfScope ps(ctx, GB_K_BACKWARD);
            GB_CUDA(gb::launch_backward(cam->mode, s->grid.n, tiles, b->cfg.tile_size, b->ranges.as<uint2>(),
                                        b->values.as<int32_t>(), b->headers.as<gb::ScreenHeader>(),
                                        b->cull.as<gb::CullRec>(), s->grid_values, cc, rc, trans, last, grad,
                                        K > 0 ? ctx->accum.as<gb::real>() : nullptr, grid_grad, stream));
        }
        ctx->launches += 2;
    }
#endif
    if (out) {
        out->splat_count = s->count;
        out->grid_n = s->grid.n;
        out->tile_size = b->cfg.tile_size;
    }
    if (K == 0) return GB_OK;
#ifdef GB_PARITY_F64
    GB_CUDA(gb::launch_add_f64(ctx->grid64.as<double>(), g->grid_values, K * 3 * s->grid.n * s->grid.n, stream));
#endif
    gb::ProjParams pp = gb::make_proj_params(s, cam, &b->cfg, b->tiles_x, b->tiles_y);
    {
        ProfScope ps(ctx, GB_K_CHAIN);
        GB_CUDA(gb::launch_chain(pp, b->counts.as<uint32_t>(), ctx->accum.as<gb::real>(), *g, stream));
    }
    ctx->launches += 1;
    return GB_OK;
}

gb_status gb_ssim(gb_context* ctx, const float* a, const float* b, int32_t width, int32_t height, int32_t clamp01,
                  double* mean_ssim, float* grad, float grad_scale) {
    if (!ctx || !a || !b || !mean_ssim) return fail(GB_INVALID_ARGUMENT, "null argument");
    if (width < 11 || height < 11)
        return fail(GB_INVALID_ARGUMENT, "ssim: image smaller than the 11x11 window");  // metrics.hpp:103-104
    if (grad && clamp01) return fail(GB_INVALID_ARGUMENT, "ssim: the gradient is taken on unclamped images");
    if (gb_status st = set_device(ctx)) return st;
    if (grad) GB_CUDA(ctx->ssim_tmp.ensure(sizeof(float) * 9 * (size_t)(width - 10) * (height - 10)));
    ProfScope ps(ctx, GB_K_LOSS);
    GB_CUDA(gb::launch_ssim(a, b, width, height, clamp01, mean_ssim, grad, grad_scale, ctx->ssim_tmp.as<float>(),
                            ctx->stream));
    ctx->launches += grad ? 2 : 1;
    return GB_OK;
}

gb_status gb_psnr(gb_context* ctx, const float* a, const float* b, int64_t n, double* out) {
    if (!ctx || !out || (n > 0 && (!a || !b))) return fail(GB_INVALID_ARGUMENT, "null argument");
    if (gb_status st = set_device(ctx)) return st;
    GB_CUDA(ctx->metric_tmp.ensure(sizeof(double)));
    GB_CUDA(cudaMemsetAsync(ctx->metric_tmp.p, 0, sizeof(double), ctx->stream));
    GB_CUDA(gb::launch_psnr_sum(a, b, n, ctx->metric_tmp.as<double>(), ctx->sm_count, ctx->stream));
    ctx->launches += n > 0;
    double sum = 0.0;
    GB_CUDA(cudaMemcpyAsync(&sum, ctx->metric_tmp.p, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    GB_CUDA(cudaStreamSynchronize(ctx->stream));
    // metrics.hpp:176-178
    const double mse = n > 0 ? sum / (double)n : 0.0;
    *out = mse == 0.0 ? 99.0 : std::fmin(99.0, 10.0 * std::log10(1.0 / mse));
    return GB_OK;
}

gb_status gb_downsample_size(int32_t n, int32_t levels, int32_t* n_out) {
    if (!n_out) return fail(GB_INVALID_ARGUMENT, "null argument");
    if (levels < 0) return fail(GB_INVALID_ARGUMENT, "downsample_grid: negative level count");  // texture.hpp:133
    if (n < 1) return fail(GB_INVALID_ARGUMENT, "ColorGridConfig: n must be >= 1");
    int h, c, out;
    if (!gb::downsample_plan(n, levels, h, c, out))
        return fail(GB_INVALID_ARGUMENT, "downsample_grid: grid size not divisible by 2^levels");
    *n_out = out;
    return GB_OK;
}

gb_status gb_downsample_grids(gb_context* ctx, const float* grid, int64_t count, int32_t n, int32_t levels,
                              float* out) {
    if (!ctx || (count > 0 && (!grid || !out))) return fail(GB_INVALID_ARGUMENT, "null argument");
    int32_t n_out;
    if (gb_status st = gb_downsample_size(n, levels, &n_out)) return st;
    int h, c, o;
    gb::downsample_plan(n, levels, h, c, o);
    if (gb_status st = set_device(ctx)) return st;
    GB_CUDA(gb::launch_downsample(count, n, h, c, grid, out, ctx->sm_count, ctx->stream));
    ctx->launches += count > 0;
    return GB_OK;
}

gb_status gb_adam_step(gb_context* ctx, int32_t mode, int64_t count, int32_t n, gb_grads* params, const gb_grads* g,
                       gb_adam_state* state, const gb_learning_rates* lrs) {
    if (!ctx || !params || !g || !state || !lrs) return fail(GB_INVALID_ARGUMENT, "null argument");
    if (mode != GB_MODE_ORTHO && mode != GB_MODE_PINHOLE) return fail(GB_INVALID_ARGUMENT, "bad mode");
    // optim.hpp:33-39
    if (!(lrs->position > 0.0 && lrs->theta > 0.0 && lrs->log_scale > 0.0 && lrs->opacity_logit > 0.0 &&
          lrs->color_grid > 0.0))
        return fail(GB_INVALID_ARGUMENT, "LearningRates: all rates must be positive");
    if (!(lrs->position_gamma > 0.0 && lrs->position_gamma <= 1.0))
        return fail(GB_INVALID_ARGUMENT, "LearningRates: position_gamma must be in (0, 1]");
    if (count < 0 || n < 1) return fail(GB_INVALID_ARGUMENT, "adam_step: gradient shape mismatch");
    if (gb_status st = set_device(ctx)) return st;
    cudaStream_t stream = ctx->stream;
    GB_CUDA(ctx->adam_bad.ensure(sizeof(unsigned long long)));
    GB_CUDA(cudaMemsetAsync(ctx->adam_bad.p, 0xff, sizeof(unsigned long long), stream));
    state->t += 1;
    const double bias1 = 1.0 - std::pow(state->beta1, (double)state->t);
    const double bias2 = 1.0 - std::pow(state->beta2, (double)state->t);
    const double pos_lr = lrs->position * std::pow(lrs->position_gamma, (double)(state->t - 1));
    struct Group {
        float *p, *g, *m, *v;
        int64_t len;
        double lr;
    };
    const bool ortho = mode == GB_MODE_ORTHO;
    const int64_t tex = count * (int64_t)n * n * 3;
    Group groups[5] = {
        {params->position, g->position, state->m.position, state->v.position, count * (ortho ? 2 : 3), pos_lr},
        {ortho ? params->theta : params->quat, ortho ? g->theta : g->quat, ortho ? state->m.theta : state->m.quat,
         ortho ? state->v.theta : state->v.quat, count * (ortho ? 1 : 4), lrs->theta},
        {params->log_scale, g->log_scale, state->m.log_scale, state->v.log_scale, count * 2, lrs->log_scale},
        {params->opacity_logit, g->opacity_logit, state->m.opacity_logit, state->v.opacity_logit, count,
         lrs->opacity_logit},
        {params->grid_values, g->grid_values, state->m.grid_values, state->v.grid_values, tex, lrs->color_grid}};
    auto* bad = ctx->adam_bad.as<unsigned long long>();
    ProfScope ps(ctx, GB_K_ADAM);
    for (int i = 0; i < 5; ++i) {
        if (groups[i].len == 0) continue;
        if (!groups[i].p || !groups[i].g || !groups[i].m || !groups[i].v)
            return fail(GB_INVALID_ARGUMENT, "adam_step: null buffer in group %d", i);
        GB_CUDA(gb::launch_adam_check(groups[i].g, groups[i].len, i, bad, ctx->sm_count, stream));
        ctx->launches++;
    }
    for (int i = 0; i < 5; ++i) {
        if (groups[i].len == 0) continue;
        GB_CUDA(gb::launch_adam_update(groups[i].p, groups[i].g, groups[i].m, groups[i].v, groups[i].len,
                                       (float)groups[i].lr, (float)state->beta1, (float)state->beta2,
                                       (float)(1.0 - state->beta1), (float)(1.0 - state->beta2),
                                       (float)state->epsilon, (float)(1.0 / bias1), (float)(1.0 / bias2), bad,
                                       ctx->sm_count, stream));
        ctx->launches++;
    }
    return GB_OK;
}

gb_status gb_context_set_texel_grad_stride(gb_context* ctx, int32_t stride) {
    if (!ctx) return fail(GB_INVALID_ARGUMENT, "null context");
    if (stride != 3 && stride != 4) return fail(GB_INVALID_ARGUMENT, "texel gradient stride must be 3 or 4");
    ctx->texel_grad_stride = stride;
    return GB_OK;
}

gb_status gb_context_set_texel_rgba(gb_context* ctx, const float* rgba) {
    if (!ctx) return fail(GB_INVALID_ARGUMENT, "null context");
    if (reinterpret_cast<uintptr_t>(rgba) & 15) return fail(GB_INVALID_ARGUMENT, "RGBA texels must be 16-byte aligned");
    ctx->tex_rgba = rgba;
    return GB_OK;
}

gb_status gb_texels_pad(gb_context* ctx, const float* src, float* dst, int64_t texels) {
    if (!ctx || (texels > 0 && (!src || !dst))) return fail(GB_INVALID_ARGUMENT, "null argument");
    if (texels < 0) return fail(GB_INVALID_ARGUMENT, "texel count must be >= 0");
    if (reinterpret_cast<uintptr_t>(dst) & 15) return fail(GB_INVALID_ARGUMENT, "RGBA texels must be 16-byte aligned");
    if (gb_status st = set_device(ctx)) return st;
    ProfScope ps(ctx, GB_K_ADAM);
    GB_CUDA(gb::launch_texel_pad(src, dst, texels, ctx->sm_count, ctx->stream));
    ctx->launches += texels > 0;
    return GB_OK;
}

gb_status gb_texel_grads_unpad(gb_context* ctx, const float* padded, float* dst, int64_t texels, int32_t accumulate) {
    if (!ctx || (texels > 0 && (!padded || !dst))) return fail(GB_INVALID_ARGUMENT, "null argument");
    if (texels < 0) return fail(GB_INVALID_ARGUMENT, "texel count must be >= 0");
    if (reinterpret_cast<uintptr_t>(padded) & 15) return fail(GB_INVALID_ARGUMENT, "padded texel gradients must be 16-byte aligned");
    if (gb_status st = set_device(ctx)) return st;
    ProfScope ps(ctx, GB_K_CHAIN);
    GB_CUDA(gb::launch_texel_unpad(padded, dst, texels, accumulate != 0, ctx->sm_count, ctx->stream));
    ctx->launches += texels > 0;
    return GB_OK;
}

gb_status gb_adam_flag_init(gb_context* ctx, int64_t* flag, const int32_t* veto) {
    if (!ctx || !flag) return fail(GB_INVALID_ARGUMENT, "null argument");
    if (gb_status st = set_device(ctx)) return st;
    ProfScope ps(ctx, GB_K_ADAM);
    GB_CUDA(gb::launch_adam_flag_init(flag, veto, ctx->stream));
    ctx->launches++;
    return GB_OK;
}

gb_status gb_adam_segments(gb_context* ctx, int32_t phase, const gb_adam_segment* seg, int32_t nseg,
                           gb_adam_state* state, const gb_learning_rates* lrs, int64_t* flag) {
    if (!ctx || (nseg > 0 && !seg) || !state || !lrs || !flag) return fail(GB_INVALID_ARGUMENT, "null argument");
    if (phase != 0 && phase != 1) return fail(GB_INVALID_ARGUMENT, "adam_segments: phase must be 0 or 1");
    // optim.hpp:33-39
    if (!(lrs->position > 0.0 && lrs->theta > 0.0 && lrs->log_scale > 0.0 && lrs->opacity_logit > 0.0 &&
          lrs->color_grid > 0.0))
        return fail(GB_INVALID_ARGUMENT, "LearningRates: all rates must be positive");
    if (!(lrs->position_gamma > 0.0 && lrs->position_gamma <= 1.0))
        return fail(GB_INVALID_ARGUMENT, "LearningRates: position_gamma must be in (0, 1]");
    for (int i = 0; i < nseg; ++i) {
        if (seg[i].group < 0 || seg[i].group > 4 || seg[i].len < 0)
            return fail(GB_INVALID_ARGUMENT, "adam_segments: bad segment %d", i);
        if (seg[i].len > 0 && (!seg[i].param || !seg[i].grad || !seg[i].m || !seg[i].v))
            return fail(GB_INVALID_ARGUMENT, "adam_segments: null buffer in segment %d", i);
    }
    if (gb_status st = set_device(ctx)) return st;
    cudaStream_t stream = ctx->stream;
    auto* bad = reinterpret_cast<unsigned long long*>(flag);
    ProfScope ps(ctx, GB_K_ADAM);
    if (phase == 0) {
        for (int i = 0; i < nseg; ++i) {
            if (seg[i].len == 0) continue;
            GB_CUDA(gb::launch_adam_check(seg[i].grad, seg[i].len, seg[i].group, bad, ctx->sm_count, stream));
            ctx->launches++;
        }
        return GB_OK;
    }
    state->t += 1;
    const double bias1 = 1.0 - std::pow(state->beta1, (double)state->t);
    const double bias2 = 1.0 - std::pow(state->beta2, (double)state->t);
    const double rate[5] = {lrs->position * std::pow(lrs->position_gamma, (double)(state->t - 1)), lrs->theta,
                            lrs->log_scale, lrs->opacity_logit, lrs->color_grid};
    for (int i = 0; i < nseg; ++i) {
        if (seg[i].len == 0) continue;
        GB_CUDA(gb::launch_adam_update(seg[i].param, seg[i].grad, seg[i].m, seg[i].v, seg[i].len,
                                       (float)rate[seg[i].group], (float)state->beta1, (float)state->beta2,
                                       (float)(1.0 - state->beta1), (float)(1.0 - state->beta2),
                                       (float)state->epsilon, (float)(1.0 / bias1), (float)(1.0 / bias2), bad,
                                       ctx->sm_count, stream));
        ctx->launches++;
    }
    return GB_OK;
}

gb_status gb_adam_check(gb_context* ctx, int32_t* group, int64_t* index) {
    if (!ctx) return fail(GB_INVALID_ARGUMENT, "ctx is null");
    if (!ctx->adam_bad.p) return GB_OK;
    if (gb_status st = set_device(ctx)) return st;
    unsigned long long v = 0;
    GB_CUDA(cudaMemcpyAsync(&v, ctx->adam_bad.p, sizeof(v), cudaMemcpyDeviceToHost, ctx->stream));
    GB_CUDA(cudaStreamSynchronize(ctx->stream));
    if (v == ~0ull) return GB_OK;
    static const char* names[5] = {"position", "theta", "log_scale", "opacity_logit", "color_grid"};
    const int grp = (int)(v >> 48);
    const int64_t idx = (int64_t)(v & ((1ull << 48) - 1));
    if (group) *group = grp;
    if (index) *index = idx;
    return fail(GB_NONFINITE, "adam_step: non-finite gradient in group '%s' at index %lld", names[grp & 7],
                (long long)idx);
}

// ---- GBIL splat files (serialize.hpp:15-124) --------------------------------------------------
namespace {
constexpr size_t kHeaderBytes = 20;           // "GBIL", u32 version, u32 K, u32 N, f32 sigma
constexpr size_t kChunkBytes = 16u << 20;     // pinned staging half-buffer

struct FileCloser {
    FILE* f;
    ~FileCloser() {
        if (f) std::fclose(f);
    }
};

struct PinnedBuf {
    void* p = nullptr;
    ~PinnedBuf() {
        if (p) cudaFreeHost(p);
    }
};

struct ScopedDev : DevBuf {
    ~ScopedDev() { release(); }
};

struct EventPair {
    cudaEvent_t e[2] = {nullptr, nullptr};
    cudaError_t create() {
        for (auto& x : e) {
            cudaError_t r = cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
            if (r != cudaSuccess) return r;
        }
        return cudaSuccess;
    }
    ~EventPair() {
        for (auto x : e)
            if (x) cudaEventDestroy(x);
    }
};

int record_fields(int version) { return version == 1 ? 7 : 10; }

// serialize.hpp:83-101 (header checks, same messages); fills info, leaves f after the header
gb_status read_header(FILE* f, gb_splat_file_info* info) {
    unsigned char h[kHeaderBytes];
    if (std::fread(h, 1, 4, f) != 4 || std::memcmp(h, "GBIL", 4) != 0)
        return fail(GB_IO_ERROR, "bad splat file: wrong magic");
    if (std::fread(h + 4, 1, 16, f) != 16) return fail(GB_IO_ERROR, "bad splat file: truncated header");
    uint32_t version, k, n;
    float sigma;
    std::memcpy(&version, h + 4, 4);  // little-endian host (x86-64 / aarch64)
    std::memcpy(&k, h + 8, 4);
    std::memcpy(&n, h + 12, 4);
    std::memcpy(&sigma, h + 16, 4);
    if (version != 1 && version != 2) return fail(GB_IO_ERROR, "unsupported splat file version %u", version);
    if (n < 1 || !(sigma > 0.0f)) return fail(GB_IO_ERROR, "bad splat file: invalid grid config");
    info->version = (int32_t)version;
    info->mode = version == 1 ? GB_MODE_ORTHO : GB_MODE_PINHOLE;
    info->count = k;
    info->n = (int32_t)n;
    info->sigma = sigma;
    return GB_OK;
}
// serialize.hpp:104-117: the first record that is not complete names the truncation
gb_status check_records(FILE* f, const gb_splat_file_info& info, const char* path) {
    const size_t rec_bytes = sizeof(float) * ((size_t)record_fields(info.version) + 3u * info.n * info.n);
    if (std::fseek(f, 0, SEEK_END) != 0) return fail(GB_IO_ERROR, "cannot read splat file: %s", path);
    const long long size = std::ftell(f);
    if (size < (long long)kHeaderBytes) return fail(GB_IO_ERROR, "cannot read splat file: %s", path);
    const size_t avail = (size_t)size - kHeaderBytes;
    if (avail / rec_bytes < (size_t)info.count)
        return fail(GB_IO_ERROR, "bad splat file: truncated at record %lld", (long long)(avail / rec_bytes));
    if (std::fseek(f, (long)kHeaderBytes, SEEK_SET) != 0) return fail(GB_IO_ERROR, "cannot read splat file: %s", path);
    return GB_OK;
}
}  // namespace

gb_status gb_splats_file_info(const char* path, gb_splat_file_info* info) {
    if (!path || !info) return fail(GB_INVALID_ARGUMENT, "null argument");
    FileCloser fc{std::fopen(path, "rb")};
    if (!fc.f) return fail(GB_IO_ERROR, "cannot open splat file: %s", path);
    if (gb_status st = read_header(fc.f, info)) return st;
    return check_records(fc.f, *info, path);
}

gb_status gb_splats_save(gb_context* ctx, const gb_splats* s, int32_t mode, const char* path) {
    if (!ctx || !s || !path) return fail(GB_INVALID_ARGUMENT, "null argument");
    if (gb_status st = validate_splats(s, mode)) return st;
    if (gb_status st = set_device(ctx)) return st;
    const int version = mode == GB_MODE_ORTHO ? 1 : 2;
    const gb::RecordMap m = gb::record_map(version, s);
    const size_t rec_bytes = sizeof(float) * (size_t)(gb::record_fields_of(m));
    const size_t total = rec_bytes * (size_t)s->count;
    ScopedDev dev;
    PinnedBuf pin;
    if (total) {
        GB_CUDA(dev.ensure(total));
        GB_CUDA(cudaMallocHost(&pin.p, 2 * kChunkBytes));
        GB_CUDA(gb::launch_pack(s->count, m, s->grid_values, dev.as<float>(), ctx->sm_count, ctx->stream));
        ctx->launches += 1;
    }
    FileCloser fc{std::fopen(path, "wb")};
    if (!fc.f) return fail(GB_IO_ERROR, "cannot open for writing: %s", path);
    unsigned char h[kHeaderBytes];
    const uint32_t v = (uint32_t)version, k = (uint32_t)s->count, n = (uint32_t)s->grid.n;
    const float sigma = (float)s->grid.sigma;
    std::memcpy(h, "GBIL", 4);
    std::memcpy(h + 4, &v, 4);
    std::memcpy(h + 8, &k, 4);
    std::memcpy(h + 12, &n, 4);
    std::memcpy(h + 16, &sigma, 4);
    bool ok = std::fwrite(h, 1, kHeaderBytes, fc.f) == kHeaderBytes;
    // double-buffered: the D2H copy of chunk i+1 overlaps the fwrite of chunk i
    EventPair evp;
    if (total) GB_CUDA(evp.create());
    cudaEvent_t* ev = evp.e;
    char* hp = static_cast<char*>(pin.p);
    size_t off = 0;
    int b = 0;
    if (total) {
        const size_t len0 = total < kChunkBytes ? total : kChunkBytes;
        GB_CUDA(cudaMemcpyAsync(hp, dev.p, len0, cudaMemcpyDeviceToHost, ctx->stream));
        GB_CUDA(cudaEventRecord(ev[0], ctx->stream));
    }
    while (off < total) {
        const size_t len = total - off < kChunkBytes ? total - off : kChunkBytes;
        const size_t nxt = off + len;
        if (nxt < total) {
            const size_t len2 = total - nxt < kChunkBytes ? total - nxt : kChunkBytes;
            GB_CUDA(cudaMemcpyAsync(hp + (size_t)(b ^ 1) * kChunkBytes, static_cast<char*>(dev.p) + nxt, len2,
                                    cudaMemcpyDeviceToHost, ctx->stream));
            GB_CUDA(cudaEventRecord(ev[b ^ 1], ctx->stream));
        }
        GB_CUDA(cudaEventSynchronize(ev[b]));
        ok = ok && std::fwrite(hp + (size_t)b * kChunkBytes, 1, len, fc.f) == len;
        off = nxt;
        b ^= 1;
    }
    GB_CUDA(cudaStreamSynchronize(ctx->stream));
    ok = ok && std::fflush(fc.f) == 0;
    if (!ok) return fail(GB_IO_ERROR, "splat write failed: %s", path);
    return GB_OK;
}

gb_status gb_splats_load(gb_context* ctx, const char* path, int64_t count, int32_t n, gb_grads* dst) {
    if (!ctx || !path || !dst) return fail(GB_INVALID_ARGUMENT, "null argument");
    FileCloser fc{std::fopen(path, "rb")};
    if (!fc.f) return fail(GB_IO_ERROR, "cannot open splat file: %s", path);
    gb_splat_file_info info;
    if (gb_status st = read_header(fc.f, &info)) return st;
    if (info.count != count || info.n != n)
        return fail(GB_MISMATCH, "load_splats: destination sized for K=%lld n=%d, file has K=%lld n=%d",
                    (long long)count, n, (long long)info.count, info.n);
    gb_splats s{};
    s.count = count;
    s.grid.n = n;
    s.grid.sigma = info.sigma;
    s.position = dst->position;
    s.depth_key = dst->depth_key;
    s.theta = dst->theta;
    s.quat = dst->quat;
    s.log_scale = dst->log_scale;
    s.opacity_logit = dst->opacity_logit;
    s.grid_values = dst->grid_values;
    if (gb_status st = validate_splats(&s, info.mode)) return st;
    const gb::RecordMap m = gb::record_map(info.version, &s);
    const size_t rec_bytes = sizeof(float) * (size_t)gb::record_fields_of(m);
    const size_t total = rec_bytes * (size_t)count;
    if (gb_status st = check_records(fc.f, info, path)) return st;
    if (total == 0) return GB_OK;
    if (gb_status st = set_device(ctx)) return st;
    ScopedDev dev;
    PinnedBuf pin;
    GB_CUDA(dev.ensure(total));
    GB_CUDA(cudaMallocHost(&pin.p, 2 * kChunkBytes));
    EventPair evp;
    GB_CUDA(evp.create());
    cudaEvent_t* ev = evp.e;
    char* hp = static_cast<char*>(pin.p);
    size_t off = 0;
    int b = 0;
    bool ok = true, used[2] = {false, false};
    // double-buffered: the fread of chunk i+1 overlaps the H2D copy of chunk i
    while (off < total && ok) {
        const size_t len = total - off < kChunkBytes ? total - off : kChunkBytes;
        if (used[b]) GB_CUDA(cudaEventSynchronize(ev[b]));
        ok = std::fread(hp + (size_t)b * kChunkBytes, 1, len, fc.f) == len;
        if (!ok) break;
        GB_CUDA(cudaMemcpyAsync(static_cast<char*>(dev.p) + off, hp + (size_t)b * kChunkBytes, len,
                                cudaMemcpyHostToDevice, ctx->stream));
        GB_CUDA(cudaEventRecord(ev[b], ctx->stream));
        used[b] = true;
        off += len;
        b ^= 1;
    }
    if (ok) {
        GB_CUDA(gb::launch_unpack(count, m, dst->grid_values, dev.as<float>(), ctx->sm_count, ctx->stream));
        ctx->launches += 1;
    }
    GB_CUDA(cudaStreamSynchronize(ctx->stream));
    if (!ok) return fail(GB_IO_ERROR, "bad splat file: truncated at record %lld", (long long)(off / rec_bytes));
    return GB_OK;
}

}  // extern "C"

// ---- NCCL: the view-sharded step's gradient exchange ------------------------------------------------
// NCCL is resolved with dlopen on first use so that a host process which already loaded a libnccl.so.2
// (torch) shares it instead of mixing two NCCL builds in one process.
namespace {
struct NcclApi {
    bool ok = false;
    std::string why;
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommInitAll) CommInitAll = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclCommCount) CommCount = nullptr;
    decltype(&ncclCommUserRank) CommUserRank = nullptr;
    decltype(&ncclCommGetAsyncError) CommGetAsyncError = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
    decltype(&ncclAllReduce) AllReduce = nullptr;
    decltype(&ncclReduceScatter) ReduceScatter = nullptr;
    decltype(&ncclAllGather) AllGather = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.why = std::string("cannot load libnccl.so.2: ") + dlerror();
            return a;
        }
#define GB_NCCL_SYM(name)                                                         \
    a.name = reinterpret_cast<decltype(a.name)>(dlsym(h, "nccl" #name));          \
    if (!a.name) {                                                                \
        a.why = "libnccl.so.2 lacks nccl" #name;                                  \
        return a;                                                                 \
    }
        GB_NCCL_SYM(GetUniqueId)
        GB_NCCL_SYM(CommInitRank)
        GB_NCCL_SYM(CommInitAll)
        GB_NCCL_SYM(CommDestroy)
        GB_NCCL_SYM(CommCount)
        GB_NCCL_SYM(CommUserRank)
        GB_NCCL_SYM(CommGetAsyncError)
        GB_NCCL_SYM(GetErrorString)
        GB_NCCL_SYM(AllReduce)
        GB_NCCL_SYM(ReduceScatter)
        GB_NCCL_SYM(AllGather)
#undef GB_NCCL_SYM
        a.ok = true;
        return a;
    }();
    return api;
}

#define GB_NCCL(call)                                                                                      \
    do {                                                                                                   \
        ncclResult_t r_ = (call);                                                                          \
        if (r_ != ncclSuccess)                                                                             \
            return fail(GB_NCCL_ERROR, "%s:%d: %s: %s", __FILE__, __LINE__, #call, nccl().GetErrorString(r_)); \
    } while (0)

gb_status need_nccl() {
    if (!nccl().ok) return fail(GB_NCCL_ERROR, "%s", nccl().why.c_str());
    return GB_OK;
}
}  // namespace

struct gb_comm {
    ncclComm_t comm = nullptr;
    int device = 0;
    int nranks = 1, rank = 0;
};

extern "C" {

gb_status gb_comm_unique_id(uint8_t id[GB_COMM_ID_BYTES]) {
    if (!id) return fail(GB_INVALID_ARGUMENT, "null id");
    if (gb_status st = need_nccl()) return st;
    static_assert(sizeof(ncclUniqueId) == GB_COMM_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId u;
    GB_NCCL(nccl().GetUniqueId(&u));
    std::memcpy(id, &u, sizeof(u));
    return GB_OK;
}

gb_status gb_comm_init_rank(gb_context* ctx, int32_t nranks, const uint8_t id[GB_COMM_ID_BYTES], int32_t rank,
                            gb_comm** out) {
    if (!ctx || !id || !out) return fail(GB_INVALID_ARGUMENT, "null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(GB_INVALID_ARGUMENT, "rank %d of %d", rank, nranks);
    if (gb_status st = need_nccl()) return st;
    if (gb_status st = set_device(ctx)) return st;
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    std::unique_ptr<gb_comm> c(new gb_comm());
    GB_NCCL(nccl().CommInitRank(&c->comm, nranks, u, rank));
    c->device = ctx->device;
    c->nranks = nranks;
    c->rank = rank;
    *out = c.release();
    return GB_OK;
}

gb_status gb_comm_init_all(gb_context* const* ctxs, int32_t n, gb_comm** out) {
    if (!ctxs || !out || n < 1) return fail(GB_INVALID_ARGUMENT, "null argument");
    if (gb_status st = need_nccl()) return st;
    std::vector<int> devs(n);
    for (int i = 0; i < n; ++i) {
        if (!ctxs[i]) return fail(GB_INVALID_ARGUMENT, "null context %d", i);
        devs[i] = ctxs[i]->device;
        for (int j = 0; j < i; ++j)
            if (devs[j] == devs[i]) return fail(GB_INVALID_ARGUMENT, "contexts %d and %d share device %d", j, i, devs[i]);
    }
    std::vector<ncclComm_t> comms(n);
    GB_NCCL(nccl().CommInitAll(comms.data(), n, devs.data()));
    for (int i = 0; i < n; ++i) {
        out[i] = new gb_comm();
        out[i]->comm = comms[i];
        out[i]->device = devs[i];
        out[i]->nranks = n;
        out[i]->rank = i;
    }
    return GB_OK;
}

gb_status gb_comm_destroy(gb_comm* c) {
    if (!c) return GB_OK;
    if (c->comm && nccl().ok) {
        cudaSetDevice(c->device);
        nccl().CommDestroy(c->comm);
    }
    delete c;
    return GB_OK;
}

gb_status gb_comm_info(const gb_comm* c, int32_t* nranks, int32_t* rank) {
    if (!c) return fail(GB_INVALID_ARGUMENT, "null communicator");
    if (nranks) *nranks = c->nranks;
    if (rank) *rank = c->rank;
    return GB_OK;
}

gb_status gb_comm_check(gb_comm* c) {
    if (!c) return fail(GB_INVALID_ARGUMENT, "null communicator");
    if (gb_status st = need_nccl()) return st;
    ncclResult_t async = ncclSuccess;
    GB_NCCL(nccl().CommGetAsyncError(c->comm, &async));
    if (async != ncclSuccess && async != ncclInProgress)
        return fail(GB_NCCL_ERROR, "communicator error: %s", nccl().GetErrorString(async));
    return GB_OK;
}

namespace {
gb_status comm_args(gb_context* ctx, gb_comm* c, const void* a, const void* b, int64_t count) {
    if (!ctx || !c) return fail(GB_INVALID_ARGUMENT, "null context or communicator");
    if (count < 0 || (count > 0 && (!a || !b))) return fail(GB_INVALID_ARGUMENT, "null buffer");
    if (c->device != ctx->device) return fail(GB_MISMATCH, "communicator on device %d, context on %d", c->device, ctx->device);
    if (gb_status st = need_nccl()) return st;
    return set_device(ctx);
}
}  // namespace

gb_status gb_allreduce_grads(gb_context* ctx, gb_comm* c, float* grads, int64_t count) {
    if (gb_status st = comm_args(ctx, c, grads, grads, count)) return st;
    ProfScope ps(ctx, GB_K_COLLECTIVE);
    GB_NCCL(nccl().AllReduce(grads, grads, (size_t)count, ncclFloat, ncclSum, c->comm, ctx->stream));
    return GB_OK;
}

gb_status gb_reduce_scatter_grads(gb_context* ctx, gb_comm* c, const float* send, float* recv, int64_t recv_count) {
    if (gb_status st = comm_args(ctx, c, send, recv, recv_count)) return st;
    ProfScope ps(ctx, GB_K_COLLECTIVE);
    GB_NCCL(nccl().ReduceScatter(send, recv, (size_t)recv_count, ncclFloat, ncclSum, c->comm, ctx->stream));
    return GB_OK;
}

gb_status gb_all_gather_params(gb_context* ctx, gb_comm* c, const float* send, float* recv, int64_t send_count) {
    if (gb_status st = comm_args(ctx, c, send, recv, send_count)) return st;
    ProfScope ps(ctx, GB_K_COLLECTIVE);
    GB_NCCL(nccl().AllGather(send, recv, (size_t)send_count, ncclFloat, c->comm, ctx->stream));
    return GB_OK;
}

gb_status gb_allreduce_flag_min(gb_context* ctx, gb_comm* c, int64_t* flag) {
    if (gb_status st = comm_args(ctx, c, flag, flag, 1)) return st;
    ProfScope ps(ctx, GB_K_COLLECTIVE);
    GB_NCCL(nccl().AllReduce(flag, flag, 1, ncclInt64, ncclMin, c->comm, ctx->stream));
    return GB_OK;
}

}  // extern "C"
