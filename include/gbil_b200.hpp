// gbil_b200.hpp -- C++ drop-in for the reference rasterizer API, over the C-ABI.
//
// Mirrors the value types and free functions of the reference's header API
// (/root/reference/proj/include/gbil: core.hpp:28-178, raster.hpp:21-400,
// optim.hpp:17-117) name for name, so a caller of gbil::build_binning /
// render_forward / render_backward / render / adam_step can switch namespace:
//
//     namespace gbil = gbil_b200;      // was: #include "gbil/raster.hpp"
//
// Semantics kept: host-side std::vector<double> SoA inputs and owning outputs,
// std::invalid_argument on the reference's validation and fingerprint throw
// sites, synchronous blocking calls.  Differences: the compute runs on a B200
// through libgb_raster.so in fp32 (values are rounded to fp32 on upload, so
// results match the fp64 reference to the tolerance documented in DESIGN.md);
// TileBinning is device-resident (its `tiles` lists are materialised lazily
// by tiles()); `RasterConfig::threads` is accepted and ignored.
//
// Every call uploads its SplatSet, so this path is the host-buffer (e2e)
// boundary; keep parameters resident with the C-ABI directly for training.
// Header-only; link with -lgb_raster (paper_2412_12734_b200/libgb_raster.so).
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "gb_raster.h"

namespace gbil_b200 {

inline constexpr double kMaxAlpha = 0.999;  // core.hpp:16
inline constexpr double kMinScale = 1e-8;   // core.hpp:19

namespace detail {

[[noreturn]] inline void raise(gb_status st, const char* where) {
    std::string msg = std::string(where) + ": " + gb_last_error_string();
    if (st == GB_INVALID_ARGUMENT || st == GB_MISMATCH) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

inline void check(gb_status st, const char* where) {
    if (st != GB_OK) raise(st, where);
}

// One context per process-thread on device 0 (the reference has no device notion).
inline gb_context* context() {
    thread_local std::unique_ptr<gb_context, gb_status (*)(gb_context*)> ctx(nullptr, gb_context_destroy);
    if (!ctx) {
        gb_context* c = nullptr;
        check(gb_context_create(0, &c), "gb_context_create");
        ctx.reset(c);
    }
    return ctx.get();
}

// Device buffer owned by the C-ABI allocator.
struct DeviceBuffer {
    void* ptr = nullptr;
    std::size_t bytes = 0;
    DeviceBuffer() = default;
    explicit DeviceBuffer(std::size_t n) : bytes(n) { check(gb_device_alloc(context(), n, &ptr), "gb_device_alloc"); }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    ~DeviceBuffer() {
        if (ptr) gb_device_free(context(), ptr);
    }
    float* f() const { return static_cast<float*>(ptr); }
};

inline std::shared_ptr<DeviceBuffer> upload(const std::vector<double>& v) {
    std::vector<float> f(v.begin(), v.end());
    auto d = std::make_shared<DeviceBuffer>(f.size() * sizeof(float) + 16);
    check(gb_copy_h2d(context(), d->ptr, f.data(), f.size() * sizeof(float), 0), "gb_copy_h2d");
    return d;
}

inline std::vector<double> download(const DeviceBuffer& d, std::size_t count) {
    std::vector<float> f(count);
    check(gb_copy_d2h(context(), f.data(), d.ptr, count * sizeof(float), 1), "gb_copy_d2h");
    return std::vector<double>(f.begin(), f.end());
}

}  // namespace detail

// core.hpp:29-42
struct ColorGridConfig {
    int n = 1;
    double sigma = 0.5;
    static constexpr int channels = 3;
    int texels_per_splat() const { return n * n * channels; }
    void validate() const {
        if (n < 1) throw std::invalid_argument("ColorGridConfig: n must be >= 1");
        if (!(sigma > 0.0)) throw std::invalid_argument("ColorGridConfig: sigma must be > 0");
    }
};

inline std::size_t texel_offset(int n, int i_u, int i_v, int c) {  // core.hpp:46-48
    return (static_cast<std::size_t>(i_u) * n + i_v) * ColorGridConfig::channels + c;
}

// core.hpp:53-87 (ortho image-plane splats)
struct SplatSet {
    std::size_t count = 0;
    ColorGridConfig grid_config;
    std::vector<double> position, depth_key, theta, log_scale, opacity_logit, grid;

    SplatSet() = default;
    SplatSet(std::size_t k, const ColorGridConfig& cfg) { resize(k, cfg); }
    void resize(std::size_t k, const ColorGridConfig& cfg) {
        cfg.validate();
        count = k;
        grid_config = cfg;
        position.assign(2 * k, 0.0);
        depth_key.assign(k, 0.0);
        theta.assign(k, 0.0);
        log_scale.assign(2 * k, 0.0);
        opacity_logit.assign(k, 0.0);
        grid.assign(k * cfg.texels_per_splat(), 0.0);
    }
    std::span<double> grid_of(std::size_t k) {
        const std::size_t s = grid_config.texels_per_splat();
        return {grid.data() + k * s, s};
    }
    std::span<const double> grid_of(std::size_t k) const {
        const std::size_t s = grid_config.texels_per_splat();
        return {grid.data() + k * s, s};
    }
};

// core.hpp:104-116
struct ImagePlaneCamera {
    int width = 0;
    int height = 0;
    std::array<double, 3> background = {0.0, 0.0, 0.0};
    void validate() const {
        if (width < 1 || height < 1) throw std::invalid_argument("ImagePlaneCamera: width and height must be >= 1");
        for (double b : background)
            if (!(b >= 0.0 && b <= 1.0)) throw std::invalid_argument("ImagePlaneCamera: background must be in [0,1]");
    }
};

// raster.hpp:21-32
struct RasterConfig {
    int tile_size = 16;
    double cutoff_radius = 3.0;
    double alpha_skip = 1.0 / 255.0;
    double early_stop_transmittance = 1e-4;
    int threads = 1;
    void validate() const {
        if (tile_size < 1) throw std::invalid_argument("RasterConfig: tile_size must be >= 1");
        if (threads < 1) throw std::invalid_argument("RasterConfig: threads must be >= 1");
    }
};

// core.hpp:123-136
struct RenderOutput {
    int width = 0;
    int height = 0;
    std::vector<double> color;
    std::vector<double> final_transmittance;
    std::vector<std::int32_t> last_rank;
    std::size_t splat_count = 0;
    int grid_n = 0;
    int tile_size = 0;
    double color_at(int x, int y, int c) const { return color[(static_cast<std::size_t>(y) * width + x) * 3 + c]; }
};

// core.hpp:140-178
struct GradientBuffer {
    std::size_t count = 0;
    ColorGridConfig grid_config;
    std::vector<double> position, depth_key, theta, log_scale, opacity_logit, grid;
    GradientBuffer() = default;
    explicit GradientBuffer(const SplatSet& like) { reset(like); }
    void reset(const SplatSet& like) {
        count = like.count;
        grid_config = like.grid_config;
        position.assign(2 * count, 0.0);
        depth_key.assign(count, 0.0);
        theta.assign(count, 0.0);
        log_scale.assign(2 * count, 0.0);
        opacity_logit.assign(count, 0.0);
        grid.assign(count * grid_config.texels_per_splat(), 0.0);
    }
};

namespace detail {

// Device mirror of a SplatSet for one call.
struct DeviceSplats {
    std::shared_ptr<DeviceBuffer> position, depth_key, theta, log_scale, opacity, grid;
    gb_splats view{};
    explicit DeviceSplats(const SplatSet& s) {
        position = upload(s.position);
        depth_key = upload(s.depth_key);
        theta = upload(s.theta);
        log_scale = upload(s.log_scale);
        opacity = upload(s.opacity_logit);
        grid = upload(s.grid);
        view.count = static_cast<int64_t>(s.count);
        view.grid.n = s.grid_config.n;
        view.grid.sigma = s.grid_config.sigma;
        view.position = position->f();
        view.depth_key = depth_key->f();
        view.theta = theta->f();
        view.log_scale = log_scale->f();
        view.opacity_logit = opacity->f();
        view.grid_values = grid->f();
    }
};

inline gb_camera to_c(const ImagePlaneCamera& c) {
    gb_camera cam{};
    cam.mode = GB_MODE_ORTHO;
    cam.width = c.width;
    cam.height = c.height;
    for (int i = 0; i < 3; ++i) cam.background[i] = c.background[i];
    cam.fx = cam.fy = 1.0;
    return cam;
}

inline gb_raster_config to_c(const RasterConfig& r) {
    return gb_raster_config{r.tile_size, r.threads, r.cutoff_radius, r.alpha_skip, r.early_stop_transmittance};
}

struct BinningHandle {
    gb_binning* b = nullptr;
    BinningHandle() { check(gb_binning_create(context(), &b), "gb_binning_create"); }
    ~BinningHandle() {
        if (b) gb_binning_destroy(b);
    }
};

}  // namespace detail

// raster.hpp:105-114: per-tile lists, device resident.
struct TileBinning {
    RasterConfig config;
    int width = 0;
    int height = 0;
    int tiles_x = 0;
    int tiles_y = 0;
    std::shared_ptr<detail::BinningHandle> handle;
    int tile_count() const { return tiles_x * tiles_y; }
    // TileBinning::tiles of the reference, copied to the host on demand.
    std::vector<std::vector<std::int32_t>> tiles() const {
        int32_t tx = 0, ty = 0;
        int64_t total = 0;
        detail::check(gb_binning_info(handle->b, &tx, &ty, &total), "gb_binning_info");
        std::vector<int64_t> offsets(static_cast<std::size_t>(tx) * ty + 1);
        std::vector<int32_t> values(static_cast<std::size_t>(total > 0 ? total : 1));
        detail::check(gb_binning_copy_to_host(detail::context(), handle->b, offsets.data(), values.data()),
                      "gb_binning_copy_to_host");
        std::vector<std::vector<std::int32_t>> out(static_cast<std::size_t>(tx) * ty);
        for (std::size_t t = 0; t < out.size(); ++t) out[t].assign(values.begin() + offsets[t], values.begin() + offsets[t + 1]);
        return out;
    }
};

// raster.hpp:116-147
inline TileBinning build_binning(const SplatSet& set, const ImagePlaneCamera& camera, const RasterConfig& config = {}) {
    camera.validate();
    config.validate();
    set.grid_config.validate();
    detail::DeviceSplats d(set);
    TileBinning bin;
    bin.config = config;
    bin.width = camera.width;
    bin.height = camera.height;
    bin.tiles_x = (camera.width + config.tile_size - 1) / config.tile_size;
    bin.tiles_y = (camera.height + config.tile_size - 1) / config.tile_size;
    bin.handle = std::make_shared<detail::BinningHandle>();
    const gb_camera cam = detail::to_c(camera);
    const gb_raster_config cfg = detail::to_c(config);
    detail::check(gb_build_binning(detail::context(), &d.view, &cam, &cfg, bin.handle->b), "build_binning");
    detail::check(gb_sync(detail::context()), "build_binning");
    return bin;
}

// raster.hpp:201-261
inline RenderOutput render_forward(const SplatSet& set, const ImagePlaneCamera& camera, const TileBinning& binning) {
    camera.validate();
    if (binning.width != camera.width || binning.height != camera.height)
        throw std::invalid_argument("render_forward: binning built for different image size");
    detail::DeviceSplats d(set);
    const std::size_t npx = static_cast<std::size_t>(camera.width) * camera.height;
    detail::DeviceBuffer color(npx * 3 * sizeof(float)), trans(npx * sizeof(float)), last(npx * sizeof(int32_t));
    gb_render_out out{camera.width, camera.height, color.f(), trans.f(), static_cast<int32_t*>(last.ptr), 0, 0, 0};
    const gb_camera cam = detail::to_c(camera);
    detail::check(gb_render_forward(detail::context(), &d.view, &cam, binning.handle->b, &out), "render_forward");
    RenderOutput r;
    r.width = camera.width;
    r.height = camera.height;
    r.color = detail::download(color, npx * 3);
    r.final_transmittance = detail::download(trans, npx);
    r.last_rank.resize(npx);
    detail::check(gb_copy_d2h(detail::context(), r.last_rank.data(), last.ptr, npx * sizeof(int32_t), 1),
                  "render_forward");
    r.splat_count = set.count;
    r.grid_n = set.grid_config.n;
    r.tile_size = binning.config.tile_size;
    return r;
}

// raster.hpp:277-387
inline GradientBuffer render_backward(const SplatSet& set, const ImagePlaneCamera& camera, const TileBinning& binning,
                                      const RenderOutput& output, const std::vector<double>& image_grad) {
    if (output.splat_count != set.count || output.grid_n != set.grid_config.n ||
        output.tile_size != binning.config.tile_size)
        throw std::invalid_argument("render_backward: output does not match forward inputs");
    if (output.width != camera.width || output.height != camera.height || binning.width != camera.width ||
        binning.height != camera.height)
        throw std::invalid_argument("render_backward: image size mismatch");
    if (image_grad.size() != output.color.size())
        throw std::invalid_argument("render_backward: image_grad size mismatch");
    detail::DeviceSplats d(set);
    const std::size_t npx = static_cast<std::size_t>(camera.width) * camera.height;
    auto trans = detail::upload(output.final_transmittance);
    auto ig = detail::upload(image_grad);
    detail::DeviceBuffer last(npx * sizeof(int32_t));
    detail::check(gb_copy_h2d(detail::context(), last.ptr, output.last_rank.data(), npx * sizeof(int32_t), 0),
                  "render_backward");
    gb_render_out out{camera.width, camera.height, nullptr, trans->f(), static_cast<int32_t*>(last.ptr),
                      static_cast<int64_t>(output.splat_count), output.grid_n, output.tile_size};
    const std::size_t K = set.count, T = set.grid_config.texels_per_splat();
    detail::DeviceBuffer gpos(2 * K * 4 + 16), gdk(K * 4 + 16), gth(K * 4 + 16), gls(2 * K * 4 + 16),
        gop(K * 4 + 16), ggr(K * T * 4 + 16);
    for (detail::DeviceBuffer* b : {&gpos, &gdk, &gth, &gls, &gop, &ggr})
        detail::check(gb_memset_device(detail::context(), b->ptr, 0, b->bytes), "render_backward");
    gb_grads g{gpos.f(), gdk.f(), gth.f(), nullptr, gls.f(), gop.f(), ggr.f()};
    const gb_camera cam = detail::to_c(camera);
    detail::check(gb_render_backward(detail::context(), &d.view, &cam, binning.handle->b, &out, ig->f(), &g),
                  "render_backward");
    GradientBuffer r(set);
    r.position = detail::download(gpos, 2 * K);
    r.depth_key.assign(K, 0.0);
    r.theta = detail::download(gth, K);
    r.log_scale = detail::download(gls, 2 * K);
    r.opacity_logit = detail::download(gop, K);
    r.grid = detail::download(ggr, K * T);
    return r;
}

// raster.hpp:389-392
inline RenderOutput render(const SplatSet& set, const ImagePlaneCamera& camera, const RasterConfig& config = {}) {
    return render_forward(set, camera, build_binning(set, camera, config));
}

}  // namespace gbil_b200
