// gb_scene.cpp -- seeded synthetic inputs (host only).
//
// Rng restates rng.hpp:12-46 exactly: std::mt19937_64 (bit-identical across
// standard libraries), uniform() = (x >> 11) * 2^-53, Box-Muller normal()
// with a cached spare.  Scenes follow SURVEY.md §8(d): geometry from
// Rng(seed), textures from Rng(seed + 1), targets from Rng(seed + 2 + view);
// everything is generated in fp64 and rounded to fp32 once, so the oracle and
// the GPU consume identical bits.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>
#include <unordered_set>

#include "../../include/gb_raster.h"

namespace {

class Rng {
public:
    explicit Rng(uint64_t seed) : engine_(seed) {}
    double uniform() { return static_cast<double>(engine_() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    double normal(double mean, double stddev) {
        if (have_spare_) {
            have_spare_ = false;
            return mean + stddev * spare_;
        }
        const double u1 = 1.0 - uniform();
        const double u2 = uniform();
        const double radius = std::sqrt(-2.0 * std::log(u1));
        const double angle = 2.0 * M_PI * u2;
        spare_ = radius * std::sin(angle);
        have_spare_ = true;
        return mean + stddev * radius * std::cos(angle);
    }

private:
    std::mt19937_64 engine_;
    double spare_ = 0.0;
    bool have_spare_ = false;
};

}  // namespace

extern "C" {

gb_status gb_scene_generate(const gb_scene_spec* spec, float* position, float* depth_key, float* theta, float* quat,
                            float* log_scale, float* opacity_logit, float* grid_values) {
    if (!spec || spec->count < 0 || spec->n < 1) return GB_INVALID_ARGUMENT;
    const int64_t K = spec->count;
    if (K == 0) return GB_OK;
    if (!position || !log_scale || !opacity_logit || !grid_values) return GB_INVALID_ARGUMENT;
    Rng geo(spec->seed);
    if (spec->mode == GB_MODE_PINHOLE) {
        if (!quat) return GB_INVALID_ARGUMENT;
        for (int64_t k = 0; k < K; ++k) {
            for (int i = 0; i < 3; ++i) {
                const double m = spec->mean_sigma > 0.0 ? geo.normal(0.0, spec->mean_sigma)
                                                        : geo.uniform(spec->mean_lo, spec->mean_hi);
                position[3 * k + i] = (float)m;
            }
            for (int i = 0; i < 2; ++i)
                log_scale[2 * k + i] = (float)geo.uniform(spec->log_scale_lo, spec->log_scale_hi);
            double q[4], nn = 0.0;
            for (int i = 0; i < 4; ++i) {
                q[i] = geo.normal(0.0, 1.0);
                nn += q[i] * q[i];
            }
            const double inv = 1.0 / std::sqrt(nn);
            for (int i = 0; i < 4; ++i) quat[4 * k + i] = (float)(q[i] * inv);
            opacity_logit[k] = (float)geo.normal(0.0, 1.0);
        }
    } else if (spec->mode == GB_MODE_ORTHO) {
        if (!depth_key || !theta) return GB_INVALID_ARGUMENT;
        for (int64_t k = 0; k < K; ++k) {
            position[2 * k + 0] = (float)geo.uniform(0.0, (double)spec->width);
            position[2 * k + 1] = (float)geo.uniform(0.0, (double)spec->height);
            depth_key[k] = (float)geo.uniform();
            theta[k] = (float)geo.uniform(0.0, 2.0 * M_PI);
            for (int i = 0; i < 2; ++i)
                log_scale[2 * k + i] = (float)geo.uniform(spec->log_scale_lo, spec->log_scale_hi);
            opacity_logit[k] = (float)geo.normal(0.0, 1.0);
        }
    } else {
        return GB_INVALID_ARGUMENT;
    }
    Rng tex(spec->seed + 1);
    const int64_t nt = K * (int64_t)spec->n * spec->n * 3;
    for (int64_t i = 0; i < nt; ++i) grid_values[i] = (float)tex.uniform();
    return GB_OK;
}

// train.hpp:80-111 initialize(): uniform positions over the image, uniform
// orientation, distinct depth keys, scales sized so a splat's 3-unit footprint
// covers about W*H/K pixels (jittered x[0.5,2] per axis), opacity 0.5, a flat
// base colour with N(0, 0.05) per-texel variation -- the same Rng draws in the
// same order, rounded to fp32 once.
gb_status gb_fit_initialize(int32_t width, int32_t height, int64_t count, int32_t n, uint64_t seed, float* position,
                            float* depth_key, float* theta, float* log_scale, float* opacity_logit,
                            float* grid_values) {
    if (width < 1 || height < 1 || count < 1 || n < 1) return GB_INVALID_ARGUMENT;
    if (!position || !depth_key || !theta || !log_scale || !opacity_logit || !grid_values) return GB_INVALID_ARGUMENT;
    const double w = width, h = height;
    if ((double)count > w * h)
        std::fprintf(stderr, "warning: %lld splats exceed the %d x %d pixel count\n", (long long)count, width, height);
    Rng rng(seed);
    const double s_init = std::sqrt(w * h / (M_PI * (double)count)) / 3.0;
    std::unordered_set<double> used;
    const int64_t F = 3LL * n * n;
    for (int64_t k = 0; k < count; ++k) {
        position[2 * k + 0] = (float)rng.uniform(0.0, w);
        position[2 * k + 1] = (float)rng.uniform(0.0, h);
        theta[k] = (float)rng.uniform(0.0, 2.0 * M_PI);
        double key = rng.uniform();
        while (!used.insert(key).second) key = rng.uniform();
        depth_key[k] = (float)key;
        log_scale[2 * k + 0] = (float)std::log(s_init * rng.uniform(0.5, 2.0));
        log_scale[2 * k + 1] = (float)std::log(s_init * rng.uniform(0.5, 2.0));
        opacity_logit[k] = 0.0f;  // logit(0.5)
        double base[3];
        for (double& b : base) b = rng.uniform(0.2, 0.8);
        for (int64_t i = 0; i < F; ++i) grid_values[k * F + i] = (float)(base[i % 3] + rng.normal(0.0, 0.05));
    }
    return GB_OK;
}

gb_status gb_uniform_fill(uint64_t seed, int64_t n, float* out) {
    if (n < 0 || (n > 0 && !out)) return GB_INVALID_ARGUMENT;
    Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = (float)r.uniform();
    return GB_OK;
}

gb_status gb_rng_uniform(uint64_t seed, int64_t n, double* out) {
    if (n < 0 || (n > 0 && !out)) return GB_INVALID_ARGUMENT;
    Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.uniform();
    return GB_OK;
}

gb_status gb_rng_normal(uint64_t seed, int64_t n, double mean, double stddev, double* out) {
    if (n < 0 || (n > 0 && !out)) return GB_INVALID_ARGUMENT;
    Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.normal(mean, stddev);
    return GB_OK;
}

}  // extern "C"
