/*
 * gb_oracle.h -- TEST INFRASTRUCTURE ONLY (not product code).
 *
 * CPU fp64 restatement of the Gaussian Billboards rasterizer hot path of the
 * reference (/root/reference/proj/include/gbil), used as the parity checker
 * for the CUDA path.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product library
 * (paper_2412_12734_b200/libgb_raster.so) never links or calls it.
 *
 * Two geometry modes:
 *   ORC_MODE_ORTHO   -- the reference's image-plane camera, restated
 *                       operation-for-operation (raster.hpp:36-387,
 *                       texture.hpp:27-111, core.hpp:21-100).  Pinned
 *                       bit-exactly against the compiled reference
 *                       (oracle/_ref/libgbil_ref.so) by tests/test_oracle_ref.py.
 *   ORC_MODE_PINHOLE -- the perspective 2DGS extension the BASELINE configs
 *                       need.  The reference has no perspective path
 *                       (SPEC.md:279), so only the intersection, the cull box
 *                       and the projection Jacobian are new; binning,
 *                       compositing, thresholds, bilinear texture and the
 *                       back-to-front adjoint are the reference's.  Geometry
 *                       parity is pinned by finite differences and
 *                       naive-vs-tiled checks (tests/test_oracle_pinhole.py),
 *                       not by a reference test ("geometry parity unpinned").
 */
#ifndef GB_ORACLE_H
#define GB_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MODE_ORTHO 0
#define ORC_MODE_PINHOLE 1

#define ORC_OK 0
#define ORC_INVALID_ARGUMENT 1
#define ORC_MISMATCH 2
#define ORC_OOM 4

typedef struct {
    int32_t mode;
    int32_t width;
    int32_t height;
    int32_t _pad;
    double background[3];
    /* pinhole only */
    double fx, fy, cx, cy;
    double rot[9];   /* world->camera rotation, row-major */
    double trans[3]; /* world->camera translation */
    double near_plane;
} orc_camera;

typedef struct {
    int32_t tile_size;
    int32_t threads;
    double cutoff_radius;
    double alpha_skip;
    double early_stop;
} orc_config;

typedef struct {
    int64_t count;
    int32_t n;
    int32_t _pad;
    double sigma;
    const double *position;      /* ortho: 2K (x,y); pinhole: 3K world mean */
    const double *depth_key;     /* ortho: K */
    const double *theta;         /* ortho: K */
    const double *quat;          /* pinhole: 4K (w,x,y,z), unnormalised */
    const double *log_scale;     /* 2K */
    const double *opacity_logit; /* K */
    const double *grid;          /* K*n*n*3, (i_u, i_v, ch) order */
} orc_splats;

typedef struct {
    double *position; /* same shapes as orc_splats */
    double *depth_key;
    double *theta;
    double *quat;
    double *log_scale;
    double *opacity_logit;
    double *grid;
} orc_grads;

typedef struct {
    int32_t tiles_x;
    int32_t tiles_y;
    int64_t total;
    int64_t *offsets; /* tiles_x*tiles_y + 1 */
    int32_t *values;  /* total */
} orc_binning;

/* Kink margins for the parity protocol. */
typedef struct {
    double alpha_rel; /* |alpha - alpha_skip| <= alpha_rel*alpha_skip, same vs 0.999 cap */
    double trans_rel; /* |T - early_stop| <= trans_rel*early_stop at any composite */
    double grid_abs;  /* |u' - k| <= grid_abs for an interior texel boundary k; ||u|-sigma| <= grid_abs*2sigma/(n-1) */
    double cond_min;  /* fp32 sensitivity: estimated |error| of (u,v) in texel units above this */
    double uv_rel;    /* > 0: fp32 (u,v) error propagation -- alpha-threshold margins from the evaluation's
                         uncertainty and slack uv_rel * delta * (1/|u| + 1/|v|) * |terms|; 0 for an fp64 GPU build */
} orc_kink;

int orc_build_binning(const orc_splats *s, const orc_camera *cam, const orc_config *cfg, orc_binning *out);
void orc_binning_free(orc_binning *b);

/* Per-primitive binning geometry: depth key (fp32-rounded for pinhole), and
 * the pixel range [x0,x1]x[y0,y1] or x0=-1 when culled. */
int orc_project(const orc_splats *s, const orc_camera *cam, const orc_config *cfg, double *depth, int32_t *rect);

int orc_render_forward(const orc_splats *s, const orc_camera *cam, const orc_config *cfg, const orc_binning *b,
                       double *color, double *trans, int32_t *last, uint8_t *kink_px, const orc_kink *kink);

/* kink_px (nullable): per-pixel flags from orc_render_forward (bit0 decision kink, bit1 early-stop kink,
 * bit2 an fp32-ill-conditioned evaluation).
 * mag / slack (nullable): per-entry sum of |terms| and the kink slack (see gb_oracle.c). */
int orc_render_backward(const orc_splats *s, const orc_camera *cam, const orc_config *cfg, const orc_binning *b,
                        const double *trans, const int32_t *last, const double *image_grad, orc_grads *g,
                        const uint8_t *kink_px, orc_grads *mag, orc_grads *slack, const orc_kink *kink);

/* ... and tmag (nullable): the per-entry sum of |terms| * kappa, kappa = sum over the pixel's composited
 * entries of alpha / (1 - alpha) -- the transmittance-chain term of the fp32 error model. */
int orc_render_backward_tm(const orc_splats *s, const orc_camera *cam, const orc_config *cfg, const orc_binning *b,
                           const double *trans, const int32_t *last, const double *image_grad, orc_grads *g,
                           const uint8_t *kink_px, orc_grads *mag, orc_grads *slack, orc_grads *tmag,
                           const orc_kink *kink);

int orc_render_naive(const orc_splats *s, const orc_camera *cam, double *color, double *trans);

/* Central finite differences of L = sum(weights * render_naive(...).color)
 * over every raw parameter (reference.hpp:66-105). */
int orc_gradient_fd(const orc_splats *s, const orc_camera *cam, const double *weights, double step, orc_grads *g);

/* Unit-level restatements for the SPEC known-answer tests. */
void orc_uv_to_grid(double u, double v, int n, double sigma, int32_t *iu, int32_t *iv, double *fu, double *fv);
void orc_bilinear(double u, double v, int n, double sigma, const double *grid, double *c);
void orc_adj_bilinear(double u, double v, int n, double sigma, const double *grid, const double *c_hat,
                      double *grid_grad, double *u_hat, double *v_hat);
void orc_intersect_ortho(double px, double py, double x, double y, double theta, double log_su, double log_sv,
                         double *u, double *v);
int orc_intersect_pinhole(const orc_camera *cam, const double *mean, const double *quat, const double *log_scale,
                          double px, double py, double *u, double *v);

/* Adam for one parameter group (optim.hpp:76-90); returns index+1 of the first
 * non-finite gradient, 0 if none. */
int64_t orc_adam_group(double *p, const double *g, double *m, double *v, int64_t n, double lr, double beta1,
                       double beta2, double eps, double bias1, double bias2);

/* L1 loss: value = scale*sum|c-t|, grad = scale*sign(c-t) (sign(0)=0). */
double orc_l1_loss(const double *c, const double *t, int64_t n, double scale, double *grad);

/* Seeded synthetic inputs, restated independently of the product library so that bench.py's
 * reference arm never loads it.  Rng (rng.hpp:12-46): std::mt19937_64 (restated from its published
 * definition), uniform() = (x >> 11) * 2^-53, Box-Muller normal() with a cached spare.  Scenes as
 * geometry from Rng(seed), textures from Rng(seed+1); fp64 draws rounded to fp32 once.
 * Bit-identity with the product's gb_scene_generate is a CPU test (tests/test_oracle_scene.py). */
typedef struct {
    uint64_t mt[312];
    int32_t idx;
    int32_t have_spare;
    double spare;
} orc_rng;
void orc_rng_seed(orc_rng *r, uint64_t seed);
uint64_t orc_rng_next(orc_rng *r);
double orc_rng_uniform(orc_rng *r);
double orc_rng_normal(orc_rng *r, double mean, double stddev);
/* pinhole scene: means N(0, mean_sigma^2) when mean_sigma > 0 else U[mean_lo, mean_hi)^3; log-scales
 * U[log_scale_lo, log_scale_hi); quaternion = normalised N(0,1)^4; logit N(0,1); texels U[0,1). */
int orc_scene_generate_pinhole(int64_t count, int32_t n, uint64_t seed, double mean_lo, double mean_hi,
                               double mean_sigma, double log_scale_lo, double log_scale_hi, float *position,
                               float *quat, float *log_scale, float *opacity_logit, float *grid);
/* n uniforms from Rng(seed) rounded to fp32 (the seeded-noise targets use seed + 2 + view). */
void orc_uniform_fill(uint64_t seed, int64_t n, float *out);

#ifdef __cplusplus
}
#endif
#endif
