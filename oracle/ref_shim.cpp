// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" wrapper that compiles the UNMODIFIED reference headers
// where they lie (/root/reference/proj/include/gbil, passed with -I; nothing
// is copied into this repo) into oracle/_ref/libgbil_ref.so.  It lets the
// Python tests (a) pin the C restatement in oracle/gb_oracle.c bit-exactly
// against the reference and (b) generate tests/golden fixtures.  bench.py
// uses it as the CPU baseline (kind "reference") for the reference's own
// ortho path when it is present.
//
// Only arrays and sizes cross this boundary; the reference's value types are
// rebuilt on each call.
#include <cstdint>
#include <cstdio>
#include <string>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

#include "gbil/core.hpp"
#include "gbil/optim.hpp"
#include "gbil/raster.hpp"
#include "gbil/reference.hpp"
#include "gbil/rng.hpp"
#include "gbil/serialize.hpp"
#include "gbil/train.hpp"  // + metrics.hpp, image.hpp (png.h: oracle/stub, never called)
#include "gbil/texture.hpp"

using namespace gbil;

namespace {

SplatSet make_set(int64_t k, int n, double sigma, const double* position, const double* depth_key,
                  const double* theta, const double* log_scale, const double* opacity, const double* grid) {
    SplatSet s(static_cast<std::size_t>(k), ColorGridConfig{n, sigma});
    std::memcpy(s.position.data(), position, sizeof(double) * 2 * k);
    std::memcpy(s.depth_key.data(), depth_key, sizeof(double) * k);
    std::memcpy(s.theta.data(), theta, sizeof(double) * k);
    std::memcpy(s.log_scale.data(), log_scale, sizeof(double) * 2 * k);
    std::memcpy(s.opacity_logit.data(), opacity, sizeof(double) * k);
    std::memcpy(s.grid.data(), grid, sizeof(double) * k * n * n * 3);
    return s;
}

ImagePlaneCamera make_cam(int w, int h, const double* bg) {
    ImagePlaneCamera c;
    c.width = w;
    c.height = h;
    c.background = {bg[0], bg[1], bg[2]};
    return c;
}

RasterConfig make_cfg(int tile, double cutoff, double skip, double es, int threads) {
    RasterConfig c;
    c.tile_size = tile;
    c.cutoff_radius = cutoff;
    c.alpha_skip = skip;
    c.early_stop_transmittance = es;
    c.threads = threads;
    return c;
}

void export_grads(const GradientBuffer& g, double* position, double* depth_key, double* theta, double* log_scale,
                  double* opacity, double* grid) {
    std::memcpy(position, g.position.data(), sizeof(double) * g.position.size());
    std::memcpy(depth_key, g.depth_key.data(), sizeof(double) * g.depth_key.size());
    std::memcpy(theta, g.theta.data(), sizeof(double) * g.theta.size());
    std::memcpy(log_scale, g.log_scale.data(), sizeof(double) * g.log_scale.size());
    std::memcpy(opacity, g.opacity_logit.data(), sizeof(double) * g.opacity_logit.size());
    std::memcpy(grid, g.grid.data(), sizeof(double) * g.grid.size());
}

}  // namespace

extern "C" {

// build_binning (raster.hpp:116-147) + render_forward (raster.hpp:201-261),
// and, when image_grad != nullptr, render_backward (raster.hpp:277-387).
// The per-tile lists are exported as CSR (offsets[tiles+1], values[total]);
// call once with values == nullptr to learn total via *total.
int ref_render(int64_t k, int n, double sigma, const double* position, const double* depth_key, const double* theta,
               const double* log_scale, const double* opacity, const double* grid, int width, int height,
               const double* bg, int tile, double cutoff, double skip, double es, int threads, int64_t* total,
               int64_t* offsets, int32_t* values, double* color, double* trans, int32_t* last,
               const double* image_grad, double* g_position, double* g_depth, double* g_theta, double* g_log_scale,
               double* g_opacity, double* g_grid) {
    try {
        const SplatSet s = make_set(k, n, sigma, position, depth_key, theta, log_scale, opacity, grid);
        const ImagePlaneCamera cam = make_cam(width, height, bg);
        const TileBinning bin = build_binning(s, cam, make_cfg(tile, cutoff, skip, es, threads));
        int64_t t = 0;
        for (const auto& l : bin.tiles) t += static_cast<int64_t>(l.size());
        *total = t;
        if (values == nullptr) return 0;
        int64_t o = 0;
        for (std::size_t i = 0; i < bin.tiles.size(); ++i) {
            offsets[i] = o;
            for (int32_t v : bin.tiles[i]) values[o++] = v;
        }
        offsets[bin.tiles.size()] = o;
        if (color == nullptr) return 0;
        const RenderOutput out = render_forward(s, cam, bin);
        std::memcpy(color, out.color.data(), sizeof(double) * out.color.size());
        std::memcpy(trans, out.final_transmittance.data(), sizeof(double) * out.final_transmittance.size());
        std::memcpy(last, out.last_rank.data(), sizeof(int32_t) * out.last_rank.size());
        if (image_grad == nullptr) return 0;
        std::vector<double> ig(image_grad, image_grad + static_cast<std::size_t>(width) * height * 3);
        const GradientBuffer g = render_backward(s, cam, bin, out, ig);
        export_grads(g, g_position, g_depth, g_theta, g_log_scale, g_opacity, g_grid);
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (const std::exception&) {
        return 3;
    }
}

// reference.hpp:20-60
int ref_render_naive(int64_t k, int n, double sigma, const double* position, const double* depth_key,
                     const double* theta, const double* log_scale, const double* opacity, const double* grid,
                     int width, int height, const double* bg, double* color, double* trans) {
    try {
        const SplatSet s = make_set(k, n, sigma, position, depth_key, theta, log_scale, opacity, grid);
        const RenderOutput out = render_naive(s, make_cam(width, height, bg));
        std::memcpy(color, out.color.data(), sizeof(double) * out.color.size());
        std::memcpy(trans, out.final_transmittance.data(), sizeof(double) * out.final_transmittance.size());
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    }
}

// reference.hpp:87-105 with the linear loss L = sum(weights * color)
int ref_gradient_fd(int64_t k, int n, double sigma, const double* position, const double* depth_key,
                    const double* theta, const double* log_scale, const double* opacity, const double* grid, int width,
                    int height, const double* bg, const double* weights, double step, double* g_position,
                    double* g_depth, double* g_theta, double* g_log_scale, double* g_opacity, double* g_grid) {
    try {
        const SplatSet s = make_set(k, n, sigma, position, depth_key, theta, log_scale, opacity, grid);
        const std::size_t npx = static_cast<std::size_t>(width) * height * 3;
        std::vector<double> w(weights, weights + npx);
        ImageLoss loss = [w](const RenderOutput& o) {
            double acc = 0.0;
            for (std::size_t i = 0; i < w.size(); ++i) acc += w[i] * o.color[i];
            return acc;
        };
        const GradientBuffer g = gradient_fd(s, make_cam(width, height, bg), loss, step);
        export_grads(g, g_position, g_depth, g_theta, g_log_scale, g_opacity, g_grid);
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    }
}

// texture.hpp:41-47, 49-66, 119-127
void ref_uv_to_grid(double u, double v, int n, double sigma, int32_t* iu, int32_t* iv, double* fu, double* fv) {
    const TexelIndex t = uv_to_grid(u, v, ColorGridConfig{n, sigma});
    *iu = t.i_u;
    *iv = t.i_v;
    *fu = t.f_u;
    *fv = t.f_v;
}

void ref_bilinear(double u, double v, int n, double sigma, const double* grid, double* c) {
    const auto r = bilinear(u, v, ColorGridConfig{n, sigma},
                            std::span<const double>(grid, static_cast<std::size_t>(n) * n * 3));
    c[0] = r[0];
    c[1] = r[1];
    c[2] = r[2];
}

void ref_adj_bilinear(double u, double v, int n, double sigma, const double* grid, const double* c_hat,
                      double* grid_grad, double* u_hat, double* v_hat) {
    const auto r = adj_bilinear(u, v, ColorGridConfig{n, sigma},
                                std::span<const double>(grid, static_cast<std::size_t>(n) * n * 3),
                                {c_hat[0], c_hat[1], c_hat[2]});
    std::memcpy(grid_grad, r.grid_grad.data(), sizeof(double) * r.grid_grad.size());
    *u_hat = r.u_hat;
    *v_hat = r.v_hat;
}

// optim.hpp:96-117 on a single-primitive set is awkward; restate one group
// through the reference's detail::adam_group instead.
int ref_adam_group(double* p, const double* g, double* m, double* v, int64_t n, double lr, double beta1, double beta2,
                   double eps, double bias1, double bias2) {
    try {
        AdamConfig cfg{beta1, beta2, eps};
        detail::adam_group(std::span<double>(p, n), std::span<const double>(g, n), std::span<double>(m, n),
                           std::span<double>(v, n), lr, cfg, bias1, bias2, "group");
        return 0;
    } catch (const std::runtime_error&) {
        return 1;
    }
}

// rng.hpp:12-46
void ref_rng_uniform(uint64_t seed, int64_t n, double* out) {
    Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.uniform();
}

void ref_rng_normal(uint64_t seed, int64_t n, double mean, double stddev, double* out) {
    Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.normal(mean, stddev);
}

// save_splats(path, set) (serialize.hpp:83-90); 0 on success, 1 on SplatIoError (message in msg).
int ref_save_splats(const char* path, int64_t k, int n, double sigma, const double* position,
                    const double* depth_key, const double* theta, const double* log_scale, const double* opacity,
                    const double* grid, char* msg, int cap) {
    try {
        save_splats(std::string(path), make_set(k, n, sigma, position, depth_key, theta, log_scale, opacity, grid));
        return 0;
    } catch (const std::exception& e) {
        std::snprintf(msg, cap, "%s", e.what());
        return 1;
    }
}

// load_splats(path) (serialize.hpp:118-124): on success returns 0 and the header values; on
// SplatIoError returns 1 with its message.  Fields are copied out when the pointers are non-null.
int ref_load_splats(const char* path, int64_t* k, int* n, double* sigma, double* position, double* depth_key,
                    double* theta, double* log_scale, double* opacity, double* grid, char* msg, int cap) {
    try {
        SplatSet s = load_splats(std::string(path));
        *k = (int64_t)s.count;
        *n = s.grid_config.n;
        *sigma = s.grid_config.sigma;
        if (position) {
            std::memcpy(position, s.position.data(), sizeof(double) * s.position.size());
            std::memcpy(depth_key, s.depth_key.data(), sizeof(double) * s.depth_key.size());
            std::memcpy(theta, s.theta.data(), sizeof(double) * s.theta.size());
            std::memcpy(log_scale, s.log_scale.data(), sizeof(double) * s.log_scale.size());
            std::memcpy(opacity, s.opacity_logit.data(), sizeof(double) * s.opacity_logit.size());
            std::memcpy(grid, s.grid.data(), sizeof(double) * s.grid.size());
        }
        return 0;
    } catch (const std::exception& e) {
        std::snprintf(msg, cap, "%s", e.what());
        return 1;
    }
}

// downsample_grid (texture.hpp:132-166) of one grid; 0 ok (n_out set), 1 with the invalid_argument text.
int ref_downsample_grid(const double* grid, int n, int levels, double* out, int* n_out, char* msg, int cap) {
    try {
        int no = 0;
        const std::vector<double> g(grid, grid + 3 * n * n);
        const std::vector<double> r = downsample_grid(g, n, levels, no);
        std::memcpy(out, r.data(), sizeof(double) * r.size());
        *n_out = no;
        return 0;
    } catch (const std::exception& e) {
        std::snprintf(msg, cap, "%s", e.what());
        return 1;
    }
}

// randomize_colors (texture.hpp:192-197): the replacement grid values.
void ref_randomize_colors(int64_t k, int n, uint64_t seed, double* grid) {
    SplatSet s(static_cast<std::size_t>(k), ColorGridConfig{n, 0.5});
    const SplatSet r = randomize_colors(s, seed);
    std::memcpy(grid, r.grid.data(), sizeof(double) * r.grid.size());
}

// ssim / ssim_with_gradient / psnr (metrics.hpp:169-191) on W x H x 3 images; grad may be null.
double ref_ssim(int w, int h, const double* a, const double* b, int with_grad, double* grad) {
    Image ia(w, h), ib(w, h);
    std::memcpy(ia.data.data(), a, sizeof(double) * ia.data.size());
    std::memcpy(ib.data.data(), b, sizeof(double) * ib.data.size());
    if (!with_grad) return ssim(ia, ib);
    const auto r = ssim_with_gradient(ia, ib);
    std::memcpy(grad, r.grad_a.data.data(), sizeof(double) * r.grad_a.data.size());
    return r.value;
}

double ref_psnr(int w, int h, const double* a, const double* b) {
    Image ia(w, h), ib(w, h);
    std::memcpy(ia.data.data(), a, sizeof(double) * ia.data.size());
    std::memcpy(ib.data.data(), b, sizeof(double) * ib.data.size());
    return psnr(ia, ib);
}

// initialize() (train.hpp:80-111) for a W x H target: the fp64 parameters.
void ref_initialize(int w, int h, int64_t k, int n, uint64_t seed, double* position, double* depth_key,
                    double* theta, double* log_scale, double* opacity, double* grid) {
    TrainConfig cfg;
    cfg.splat_count = (std::size_t)k;
    cfg.seed = seed;
    cfg.grid = ColorGridConfig{n, 0.5};
    cfg.allow_any_n = true;
    const SplatSet s = initialize(Image(w, h), cfg);
    std::memcpy(position, s.position.data(), sizeof(double) * s.position.size());
    std::memcpy(depth_key, s.depth_key.data(), sizeof(double) * s.depth_key.size());
    std::memcpy(theta, s.theta.data(), sizeof(double) * s.theta.size());
    std::memcpy(log_scale, s.log_scale.data(), sizeof(double) * s.log_scale.size());
    std::memcpy(opacity, s.opacity_logit.data(), sizeof(double) * s.opacity_logit.size());
    std::memcpy(grid, s.grid.data(), sizeof(double) * s.grid.size());
}

// fit() (train.hpp:174-219) on a W x H x 3 target.  hist receives (iter, loss, psnr, ssim) per logged
// record (up to hist_cap records, count in *n_hist).  Returns 0, or 1 with FitError/invalid_argument text.
int ref_fit(int w, int h, const double* target, int64_t k, int n, double sigma, int64_t iterations, int mse_ssim,
            double ssim_weight, uint64_t seed, int64_t log_every, int tile, double* position, double* depth_key,
            double* theta, double* log_scale, double* opacity, double* grid, double* hist, int64_t hist_cap,
            int64_t* n_hist, char* msg, int cap) {
    try {
        Image t(w, h);
        std::memcpy(t.data.data(), target, sizeof(double) * t.data.size());
        TrainConfig cfg;
        cfg.splat_count = (std::size_t)k;
        cfg.iterations = iterations;
        cfg.loss = mse_ssim ? LossKind::mse_plus_ssim : LossKind::mse;
        cfg.ssim_weight = ssim_weight;
        cfg.seed = seed;
        cfg.grid = ColorGridConfig{n, sigma};
        cfg.allow_any_n = true;
        cfg.log_every = log_every;
        cfg.raster.tile_size = tile;
        cfg.raster.threads = (int)std::max(1u, std::thread::hardware_concurrency());
        const FitResult r = fit(t, cfg);
        const SplatSet& s = r.splats;
        std::memcpy(position, s.position.data(), sizeof(double) * s.position.size());
        std::memcpy(depth_key, s.depth_key.data(), sizeof(double) * s.depth_key.size());
        std::memcpy(theta, s.theta.data(), sizeof(double) * s.theta.size());
        std::memcpy(log_scale, s.log_scale.data(), sizeof(double) * s.log_scale.size());
        std::memcpy(opacity, s.opacity_logit.data(), sizeof(double) * s.opacity_logit.size());
        std::memcpy(grid, s.grid.data(), sizeof(double) * s.grid.size());
        int64_t m = 0;
        for (const MetricRecord& rec : r.history) {
            if (m >= hist_cap) break;
            hist[4 * m + 0] = (double)rec.iter;
            hist[4 * m + 1] = rec.loss;
            hist[4 * m + 2] = rec.psnr;
            hist[4 * m + 3] = rec.ssim;
            ++m;
        }
        *n_hist = m;
        return 0;
    } catch (const std::exception& e) {
        std::snprintf(msg, cap, "%s", e.what());
        return 1;
    }
}

}  // extern "C"
