/*
 * gb_oracle.c -- TEST INFRASTRUCTURE ONLY (parity checker, not product).
 *
 * fp64 CPU restatement of the reference rasterizer hot path.  Every function
 * cites the reference lines it restates.  Build flags mirror the reference's
 * CMake contract (CMakeLists.txt:12-15): -O2 -ffp-contract=off, so the ortho
 * mode reproduces the reference bit-for-bit (verified against the compiled
 * reference by tests/test_oracle_ref.py).
 *
 * Threading mirrors detail::for_each_tile (raster.hpp:177-194): static
 * contiguous tile ranges per thread; the backward keeps per-(tile, rank)
 * partial records and reduces them in tile order (raster.hpp:293-302,
 * 368-385), so results are bit-identical for any thread count.
 */
#include "gb_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

static const double kMaxAlpha = 0.999; /* core.hpp:16 */
static const double kMinScale = 1e-8;  /* core.hpp:19 */

/* core.hpp:21 */
static double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }
/* std::max / std::min / std::clamp semantics (NaN behaviour included) */
static double dmax(double a, double b) { return (a < b) ? b : a; }
static double dmin(double a, double b) { return (b < a) ? b : a; }
static double dclamp(double v, double lo, double hi) { return (v < lo) ? lo : ((hi < v) ? hi : v); }
static int imax(int a, int b) { return (a < b) ? b : a; }
static int imin(int a, int b) { return (b < a) ? b : a; }

/* ------------------------------------------------------------------------- */
/* texture.hpp:27-111 (paper Alg. 2)                                          */
/* ------------------------------------------------------------------------- */

/* texture.hpp:27-30 */
static double uv_to_grid_coord(double u, int n, double sigma) {
    const double scaled = (double)(n - 1) * (u + sigma) / (2.0 * sigma);
    return dclamp(scaled, 0.0, (double)(n - 1));
}

/* texture.hpp:34-37 */
static void split_coord(double coord, int n, int *i, double *f) {
    *i = imin((int)floor(coord), n - 2);
    *f = coord - *i;
}

/* texture.hpp:41-47 */
void orc_uv_to_grid(double u, double v, int n, double sigma, int32_t *iu, int32_t *iv, double *fu, double *fv) {
    if (n == 1) {
        *iu = 0;
        *iv = 0;
        *fu = 0.0;
        *fv = 0.0;
        return;
    }
    int a, b;
    split_coord(uv_to_grid_coord(u, n, sigma), n, &a, fu);
    split_coord(uv_to_grid_coord(v, n, sigma), n, &b, fv);
    *iu = a;
    *iv = b;
}

static size_t texel_offset(int n, int iu, int iv, int c) { return ((size_t)iu * n + iv) * 3 + c; } /* core.hpp:46-48 */

/* texture.hpp:49-66 */
void orc_bilinear(double u, double v, int n, double sigma, const double *grid, double *c) {
    if (n == 1) {
        c[0] = grid[0];
        c[1] = grid[1];
        c[2] = grid[2];
        return;
    }
    int32_t iu, iv;
    double fu, fv;
    orc_uv_to_grid(u, v, n, sigma, &iu, &iv, &fu, &fv);
    const double w00 = (1.0 - fu) * (1.0 - fv);
    const double w10 = fu * (1.0 - fv);
    const double w01 = (1.0 - fu) * fv;
    const double w11 = fu * fv;
    for (int ch = 0; ch < 3; ++ch) {
        c[ch] = grid[texel_offset(n, iu, iv, ch)] * w00 + grid[texel_offset(n, iu + 1, iv, ch)] * w10 +
                grid[texel_offset(n, iu, iv + 1, ch)] * w01 + grid[texel_offset(n, iu + 1, iv + 1, ch)] * w11;
    }
}

/* texture.hpp:77-111: accumulates into grid_grad, returns (u_hat, v_hat) */
static void adj_bilinear_accum(double u, double v, int n, double sigma, const double *grid, const double *c_hat,
                               double *grid_grad, double *u_hat, double *v_hat) {
    if (n == 1) {
        for (int ch = 0; ch < 3; ++ch) grid_grad[ch] += c_hat[ch];
        *u_hat = 0.0;
        *v_hat = 0.0;
        return;
    }
    int32_t iu, iv;
    double fu, fv;
    orc_uv_to_grid(u, v, n, sigma, &iu, &iv, &fu, &fv);
    const double w00 = (1.0 - fu) * (1.0 - fv);
    const double w10 = fu * (1.0 - fv);
    const double w01 = (1.0 - fu) * fv;
    const double w11 = fu * fv;
    double fu_hat = 0.0, fv_hat = 0.0;
    for (int ch = 0; ch < 3; ++ch) {
        const double c00 = grid[texel_offset(n, iu, iv, ch)];
        const double c10 = grid[texel_offset(n, iu + 1, iv, ch)];
        const double c01 = grid[texel_offset(n, iu, iv + 1, ch)];
        const double c11 = grid[texel_offset(n, iu + 1, iv + 1, ch)];
        grid_grad[texel_offset(n, iu, iv, ch)] += c_hat[ch] * w00;
        grid_grad[texel_offset(n, iu + 1, iv, ch)] += c_hat[ch] * w10;
        grid_grad[texel_offset(n, iu, iv + 1, ch)] += c_hat[ch] * w01;
        grid_grad[texel_offset(n, iu + 1, iv + 1, ch)] += c_hat[ch] * w11;
        fu_hat += c_hat[ch] * ((c10 - c00) * (1.0 - fv) + (c11 - c01) * fv);
        fv_hat += c_hat[ch] * ((c01 - c00) * (1.0 - fu) + (c11 - c10) * fu);
    }
    const double scale = (double)(n - 1) / (2.0 * sigma);
    *u_hat = (u > -sigma && u < sigma) ? scale * fu_hat : 0.0;
    *v_hat = (v > -sigma && v < sigma) ? scale * fv_hat : 0.0;
}

/* texture.hpp:119-127 */
void orc_adj_bilinear(double u, double v, int n, double sigma, const double *grid, const double *c_hat,
                      double *grid_grad, double *u_hat, double *v_hat) {
    memset(grid_grad, 0, sizeof(double) * (size_t)n * n * 3);
    adj_bilinear_accum(u, v, n, sigma, grid, c_hat, grid_grad, u_hat, v_hat);
}

/* Is (u, v) within margin of a bilinear kink (interior texel boundary or the
 * |u| = sigma clamp edge)?  Used only for the parity protocol. */
static int grid_kink(double u, int n, double sigma, double margin) {
    if (n < 2) return 0;
    const double scaled = (double)(n - 1) * (u + sigma) / (2.0 * sigma);
    if (fabs(scaled) <= margin || fabs(scaled - (n - 1)) <= margin) return 1;
    if (scaled > 0.0 && scaled < n - 1) {
        const double k = floor(scaled + 0.5);
        if (k >= 1.0 && k <= n - 2 && fabs(scaled - k) <= margin) return 1;
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Per-primitive geometry                                                     */
/* ------------------------------------------------------------------------- */

/* raster.hpp:152-175 (ortho SplatGeom) extended with the pinhole frame. */
typedef struct {
    int valid; /* pinhole validity: finite frame, centre in front of the near plane */
    double alpha_k;
    double s_u, s_v;
    int su_clamped, sv_clamped;
    /* ortho */
    double x, y, cos_t, sin_t, inv_su, inv_sv;
    /* pinhole */
    double qn[4], qnorm;
    double tuc[3], tvc[3], pc[3];
    double M[9]; /* camera-space plane map, row-major: columns (s_u tuc, s_v tvc, pc) */
    double depth;
    /* Parity-protocol only: the linear-fractional form the fp32 compositor
     * evaluates, (u, v, 1) ~ (X.x dx + Y.x dy, X.y dx + Y.y dy, 1 + X.z dx + Y.z dy)
     * with (dx, dy) the pixel offset from the projected centre (cpx, cpy),
     * X = Cx/(E_z fx), Y = Cy/(E_z fy), Cx = M1 x M2, Cy = M2 x M0. Used to
     * estimate the fp32 error of (u, v) and the GPU's accumulation magnitudes. */
    double X[3], Y[3], cpx, cpy, ez, dxc, dyc;
} geom_t;

/* Unit quaternion (w,x,y,z) -> rotation columns t_u, t_v (2DGS convention,
 * tangents are the first two columns of R(q)). */
static void quat_frame(const double *q, double *tu, double *tv) {
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    tu[0] = 1.0 - 2.0 * (y * y + z * z);
    tu[1] = 2.0 * (x * y + w * z);
    tu[2] = 2.0 * (x * z - w * y);
    tv[0] = 2.0 * (x * y - w * z);
    tv[1] = 1.0 - 2.0 * (x * x + z * z);
    tv[2] = 2.0 * (y * z + w * x);
}

static void build_geom(const orc_splats *s, const orc_camera *cam, int64_t k, geom_t *g) {
    memset(g, 0, sizeof(*g));
    /* core.hpp:95-100 activate(); raster.hpp:160-172 */
    g->alpha_k = sigmoid(s->opacity_logit[k]);
    const double eu = exp(s->log_scale[2 * k + 0]);
    const double ev = exp(s->log_scale[2 * k + 1]);
    g->s_u = dmax(eu, kMinScale);
    g->s_v = dmax(ev, kMinScale);
    g->su_clamped = eu < kMinScale;
    g->sv_clamped = ev < kMinScale;
    if (cam->mode == ORC_MODE_ORTHO) {
        g->valid = 1;
        g->x = s->position[2 * k + 0];
        g->y = s->position[2 * k + 1];
        g->cos_t = cos(s->theta[k]);
        g->sin_t = sin(s->theta[k]);
        g->inv_su = 1.0 / g->s_u;
        g->inv_sv = 1.0 / g->s_v;
        g->depth = s->depth_key[k];
        return;
    }
    /* pinhole extension */
    const double *q = s->quat + 4 * k;
    const double nn = q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3];
    g->qnorm = sqrt(nn);
    if (!(g->qnorm > 0.0)) return;
    for (int i = 0; i < 4; ++i) g->qn[i] = q[i] / g->qnorm;
    double tu[3], tv[3];
    quat_frame(g->qn, tu, tv);
    const double *R = cam->rot;
    const double *m = s->position + 3 * k;
    for (int r = 0; r < 3; ++r) {
        g->pc[r] = R[3 * r + 0] * m[0] + R[3 * r + 1] * m[1] + R[3 * r + 2] * m[2] + cam->trans[r];
        g->tuc[r] = R[3 * r + 0] * tu[0] + R[3 * r + 1] * tu[1] + R[3 * r + 2] * tu[2];
        g->tvc[r] = R[3 * r + 0] * tv[0] + R[3 * r + 1] * tv[1] + R[3 * r + 2] * tv[2];
        g->M[3 * r + 0] = g->s_u * g->tuc[r];
        g->M[3 * r + 1] = g->s_v * g->tvc[r];
        g->M[3 * r + 2] = g->pc[r];
    }
    /* depth key: camera-space z of the centre, rounded to fp32 */
    g->depth = (double)(float)g->pc[2];
    g->valid = g->pc[2] > cam->near_plane;
    const double *M0 = g->M, *M1 = g->M + 3, *M2 = g->M + 6;
    const double C0z = M0[0] * M1[1] - M0[1] * M1[0];
    const double Cx[3] = {M1[1] * M2[2] - M1[2] * M2[1], M1[2] * M2[0] - M1[0] * M2[2], M1[0] * M2[1] - M1[1] * M2[0]};
    const double Cy[3] = {M2[1] * M0[2] - M2[2] * M0[1], M2[2] * M0[0] - M2[0] * M0[2], M2[0] * M0[1] - M2[1] * M0[0]};
    g->dxc = g->pc[0] / g->pc[2];
    g->dyc = g->pc[1] / g->pc[2];
    g->cpx = cam->fx * g->dxc + cam->cx;
    g->cpy = cam->fy * g->dyc + cam->cy;
    g->ez = C0z + g->dxc * Cx[2] + g->dyc * Cy[2];
    for (int j = 0; j < 3; ++j) {
        g->X[j] = Cx[j] / (g->ez * cam->fx);
        g->Y[j] = Cy[j] / (g->ez * cam->fy);
    }
}

/* raster.hpp:36-42 */
static void intersect_ortho_g(const geom_t *g, double px, double py, double *u, double *v) {
    const double dx = px - g->x;
    const double dy = py - g->y;
    *u = (g->cos_t * dx + g->sin_t * dy) * g->inv_su;
    *v = (-g->sin_t * dx + g->cos_t * dy) * g->inv_sv;
}

/* Pinhole ray-splat intersection (2DGS).  Pixel ray
 * d = ((px-cx)/fx, (py-cy)/fy, 1); the plane point M (u,v,1)^T = t d gives
 * two homogeneous equations a.(u,v,1)=0, b.(u,v,1)=0 with
 * a = M0 - dxn M2, b = M1 - dyn M2, solved by (u,v,1) ~ a x b.
 * A miss (ray parallel to the plane, or the hit behind the camera: t <= 0)
 * returns 0 and the entry is skipped. */
static int intersect_pinhole_g(const geom_t *g, const orc_camera *cam, double px, double py, double *u, double *v,
                               double *a, double *b, double *cz_out) {
    const double dxn = (px - cam->cx) / cam->fx;
    const double dyn = (py - cam->cy) / cam->fy;
    for (int j = 0; j < 3; ++j) {
        a[j] = g->M[j] - dxn * g->M[6 + j];
        b[j] = g->M[3 + j] - dyn * g->M[6 + j];
    }
    const double c0 = a[1] * b[2] - a[2] * b[1];
    const double c1 = a[2] * b[0] - a[0] * b[2];
    const double cz = a[0] * b[1] - a[1] * b[0];
    *cz_out = cz;
    if (cz == 0.0) return 0;
    *u = c0 / cz;
    *v = c1 / cz;
    const double t = g->M[6] * *u + g->M[7] * *v + g->M[8];
    if (!(t > 0.0)) return 0;
    return 1;
}

static double gaussian_weight(double u, double v) { return exp(-0.5 * (u * u + v * v)); } /* raster.hpp:52 */

void orc_intersect_ortho(double px, double py, double x, double y, double theta, double log_su, double log_sv,
                         double *u, double *v) {
    geom_t g;
    memset(&g, 0, sizeof(g));
    g.x = x;
    g.y = y;
    g.cos_t = cos(theta);
    g.sin_t = sin(theta);
    g.inv_su = 1.0 / dmax(exp(log_su), kMinScale);
    g.inv_sv = 1.0 / dmax(exp(log_sv), kMinScale);
    intersect_ortho_g(&g, px, py, u, v);
}

int orc_intersect_pinhole(const orc_camera *cam, const double *mean, const double *quat, const double *log_scale,
                          double px, double py, double *u, double *v) {
    double zero = 0.0;
    orc_splats s;
    memset(&s, 0, sizeof(s));
    s.count = 1;
    s.position = mean;
    s.quat = quat;
    s.log_scale = log_scale;
    s.opacity_logit = &zero;
    geom_t g;
    build_geom(&s, cam, 0, &g);
    double a[3], b[3], cz;
    return intersect_pinhole_g(&g, cam, px, py, u, v, a, b, &cz);
}

/* ------------------------------------------------------------------------- */
/* Binning: raster.hpp:54-147                                                 */
/* ------------------------------------------------------------------------- */

typedef struct {
    double min_x, max_x, min_y, max_y;
} aabb_t;

/* raster.hpp:61-86 (ortho) / SURVEY Appendix C (pinhole cull box). Returns 0 when culled. */
static int cull(const orc_splats *s, const geom_t *g, int64_t k, const orc_camera *cam, const orc_config *cfg,
                aabb_t *box) {
    if (cfg->alpha_skip > 0.0 && sigmoid(s->opacity_logit[k]) < cfg->alpha_skip) return 0;
    if (cam->mode == ORC_MODE_ORTHO) {
        if (cfg->cutoff_radius > 0.0) {
            const double suc = g->s_u * cos(s->theta[k]);
            const double sus = g->s_u * sin(s->theta[k]);
            const double svc = g->s_v * cos(s->theta[k]);
            const double svs = g->s_v * sin(s->theta[k]);
            const double hx = cfg->cutoff_radius * sqrt(suc * suc + svs * svs);
            const double hy = cfg->cutoff_radius * sqrt(sus * sus + svc * svc);
            const double x = s->position[2 * k];
            const double y = s->position[2 * k + 1];
            box->min_x = x - hx;
            box->max_x = x + hx;
            box->min_y = y - hy;
            box->max_y = y + hy;
        } else {
            box->min_x = 0.0;
            box->max_x = (double)cam->width;
            box->min_y = 0.0;
            box->max_y = (double)cam->height;
        }
    } else {
        if (!g->valid) return 0;
        if (cfg->cutoff_radius > 0.0) {
            const double r = cfg->cutoff_radius;
            const double *M = g->M;
            /* whole cutoff disk strictly in front of the near plane */
            const double lat = sqrt(M[6] * M[6] + M[7] * M[7]);
            if (!(M[8] - r * lat > cam->near_plane)) return 0;
            /* pixel homography H = K M; dual conic C* = H diag(r^2, r^2, -1) H^T */
            double H0[3], H1[3], H2[3];
            for (int j = 0; j < 3; ++j) {
                H0[j] = cam->fx * M[j] + cam->cx * M[6 + j];
                H1[j] = cam->fy * M[3 + j] + cam->cy * M[6 + j];
                H2[j] = M[6 + j];
            }
            const double r2 = r * r;
            const double C00 = r2 * (H0[0] * H0[0] + H0[1] * H0[1]) - H0[2] * H0[2];
            const double C02 = r2 * (H0[0] * H2[0] + H0[1] * H2[1]) - H0[2] * H2[2];
            const double C11 = r2 * (H1[0] * H1[0] + H1[1] * H1[1]) - H1[2] * H1[2];
            const double C12 = r2 * (H1[0] * H2[0] + H1[1] * H2[1]) - H1[2] * H2[2];
            const double C22 = r2 * (H2[0] * H2[0] + H2[1] * H2[1]) - H2[2] * H2[2];
            const double dx = C02 * C02 - C00 * C22;
            const double dy = C12 * C12 - C11 * C22;
            if (!(dx >= 0.0) || !(dy >= 0.0)) return 0;
            const double sx = sqrt(dx), sy = sqrt(dy);
            const double xa = (C02 - sx) / C22, xb = (C02 + sx) / C22;
            const double ya = (C12 - sy) / C22, yb = (C12 + sy) / C22;
            box->min_x = dmin(xa, xb);
            box->max_x = dmax(xa, xb);
            box->min_y = dmin(ya, yb);
            box->max_y = dmax(ya, yb);
        } else {
            box->min_x = 0.0;
            box->max_x = (double)cam->width;
            box->min_y = 0.0;
            box->max_y = (double)cam->height;
        }
    }
    /* raster.hpp:80-85 */
    box->min_x = dmax(box->min_x, 0.0);
    box->min_y = dmax(box->min_y, 0.0);
    box->max_x = dmin(box->max_x, (double)cam->width);
    box->max_y = dmin(box->max_y, (double)cam->height);
    if (!(box->min_x < box->max_x) || !(box->min_y < box->max_y)) return 0;
    return 1;
}

/* raster.hpp:93-101 */
static int box_to_pixels(const aabb_t *box, const orc_camera *cam, int32_t *r) {
    r[0] = imax(0, (int)ceil(box->min_x - 0.5));
    r[2] = imax(0, (int)ceil(box->min_y - 0.5));
    r[1] = imin(cam->width - 1, (int)floor(box->max_x - 0.5));
    r[3] = imin(cam->height - 1, (int)floor(box->max_y - 0.5));
    if (r[0] > r[1] || r[2] > r[3]) return 0;
    return 1;
}

static int validate(const orc_camera *cam, const orc_config *cfg, const orc_splats *s) {
    if (cam->width < 1 || cam->height < 1) return ORC_INVALID_ARGUMENT; /* core.hpp:109-115 */
    for (int i = 0; i < 3; ++i)
        if (!(cam->background[i] >= 0.0 && cam->background[i] <= 1.0)) return ORC_INVALID_ARGUMENT;
    if (cfg && (cfg->tile_size < 1 || cfg->threads < 1)) return ORC_INVALID_ARGUMENT; /* raster.hpp:28-31 */
    if (s && (s->n < 1 || !(s->sigma > 0.0))) return ORC_INVALID_ARGUMENT;          /* core.hpp:36-41 */
    if (cam->mode == ORC_MODE_PINHOLE && !(cam->fx != 0.0 && cam->fy != 0.0)) return ORC_INVALID_ARGUMENT;
    return ORC_OK;
}

int orc_project(const orc_splats *s, const orc_camera *cam, const orc_config *cfg, double *depth, int32_t *rect) {
    int st = validate(cam, cfg, s);
    if (st) return st;
    for (int64_t k = 0; k < s->count; ++k) {
        geom_t g;
        build_geom(s, cam, k, &g);
        depth[k] = g.depth;
        aabb_t box;
        int32_t *r = rect + 4 * k;
        if (!cull(s, &g, k, cam, cfg, &box) || !box_to_pixels(&box, cam, r)) {
            r[0] = r[1] = r[2] = r[3] = -1;
        }
    }
    return ORC_OK;
}

typedef struct {
    const double *depth;
} sort_ctx_t;
static const double *g_sort_depth; /* qsort has no context argument in C11 */
static pthread_mutex_t g_sort_mu = PTHREAD_MUTEX_INITIALIZER;

/* raster.hpp:141-145: ascending depth_key, ties by index */
static int cmp_depth_index(const void *pa, const void *pb) {
    const int32_t a = *(const int32_t *)pa, b = *(const int32_t *)pb;
    const double da = g_sort_depth[a], db = g_sort_depth[b];
    if (da != db) return (da < db) ? -1 : 1;
    return (a < b) ? -1 : (a > b);
}

/* raster.hpp:116-147 */
int orc_build_binning(const orc_splats *s, const orc_camera *cam, const orc_config *cfg, orc_binning *out) {
    memset(out, 0, sizeof(*out));
    int st = validate(cam, cfg, s);
    if (st) return st;
    const int ts = cfg->tile_size;
    out->tiles_x = (cam->width + ts - 1) / ts;
    out->tiles_y = (cam->height + ts - 1) / ts;
    const int64_t nt = (int64_t)out->tiles_x * out->tiles_y;
    int64_t *count = calloc((size_t)nt + 1, sizeof(int64_t));
    int32_t *rect = malloc(sizeof(int32_t) * 4 * (size_t)(s->count > 0 ? s->count : 1));
    double *depth = malloc(sizeof(double) * (size_t)(s->count > 0 ? s->count : 1));
    if (!count || !rect || !depth) {
        free(count);
        free(rect);
        free(depth);
        return ORC_OOM;
    }
    orc_project(s, cam, cfg, depth, rect);
    for (int64_t k = 0; k < s->count; ++k) {
        const int32_t *r = rect + 4 * k;
        if (r[0] < 0) continue;
        for (int ty = r[2] / ts; ty <= r[3] / ts; ++ty)
            for (int tx = r[0] / ts; tx <= r[1] / ts; ++tx) count[(int64_t)ty * out->tiles_x + tx + 1]++;
    }
    for (int64_t t = 0; t < nt; ++t) count[t + 1] += count[t];
    out->total = count[nt];
    out->offsets = count;
    out->values = malloc(sizeof(int32_t) * (size_t)(out->total > 0 ? out->total : 1));
    int64_t *fill = malloc(sizeof(int64_t) * (size_t)(nt > 0 ? nt : 1));
    if (!out->values || !fill) {
        free(fill);
        free(rect);
        free(depth);
        orc_binning_free(out);
        return ORC_OOM;
    }
    memcpy(fill, count, sizeof(int64_t) * (size_t)nt);
    /* push k into every overlapped tile, in index order (raster.hpp:128-140) */
    for (int64_t k = 0; k < s->count; ++k) {
        const int32_t *r = rect + 4 * k;
        if (r[0] < 0) continue;
        for (int ty = r[2] / ts; ty <= r[3] / ts; ++ty)
            for (int tx = r[0] / ts; tx <= r[1] / ts; ++tx)
                out->values[fill[(int64_t)ty * out->tiles_x + tx]++] = (int32_t)k;
    }
    pthread_mutex_lock(&g_sort_mu);
    g_sort_depth = depth;
    for (int64_t t = 0; t < nt; ++t)
        qsort(out->values + count[t], (size_t)(count[t + 1] - count[t]), sizeof(int32_t), cmp_depth_index);
    g_sort_depth = NULL;
    pthread_mutex_unlock(&g_sort_mu);
    free(fill);
    free(rect);
    free(depth);
    return ORC_OK;
}

void orc_binning_free(orc_binning *b) {
    free(b->offsets);
    free(b->values);
    b->offsets = NULL;
    b->values = NULL;
}

/* ------------------------------------------------------------------------- */
/* Tile fan-out: raster.hpp:177-194                                           */
/* ------------------------------------------------------------------------- */

typedef void (*tile_fn)(void *ctx, int tile);
typedef struct {
    tile_fn fn;
    void *ctx;
    int begin, end;
} worker_t;

static void *worker_main(void *arg) {
    worker_t *w = (worker_t *)arg;
    for (int t = w->begin; t < w->end; ++t) w->fn(w->ctx, t);
    return NULL;
}

static void for_each_tile(int tile_count, int threads, tile_fn fn, void *ctx) {
    threads = imax(1, imin(threads, tile_count));
    if (threads <= 1) {
        for (int t = 0; t < tile_count; ++t) fn(ctx, t);
        return;
    }
    pthread_t *th = malloc(sizeof(pthread_t) * (size_t)threads);
    worker_t *ws = malloc(sizeof(worker_t) * (size_t)threads);
    for (int w = 0; w < threads; ++w) {
        ws[w].fn = fn;
        ws[w].ctx = ctx;
        ws[w].begin = (int)((int64_t)tile_count * w / threads);
        ws[w].end = (int)((int64_t)tile_count * (w + 1) / threads);
        pthread_create(&th[w], NULL, worker_main, &ws[w]);
    }
    for (int w = 0; w < threads; ++w) pthread_join(th[w], NULL);
    free(th);
    free(ws);
}

/* ------------------------------------------------------------------------- */
/* Forward: raster.hpp:201-261                                                */
/* ------------------------------------------------------------------------- */

typedef struct {
    const orc_splats *s;
    const orc_camera *cam;
    const orc_config *cfg;
    const orc_binning *b;
    const geom_t *geom;
    const orc_kink *kink;
    double *color, *trans;
    int32_t *last;
    uint8_t *kink_px;
    /* backward */
    const double *image_grad;
    const uint8_t *kink_px_in;
    double **partials, **mags, **slacks, **tmags;
    int want_mag, want_slack, want_tmag;
    size_t stride;
} raster_ctx_t;

/* Evaluate entry g at pixel (px,py).  Returns 0 on a (pinhole) miss. */
static int eval_uv(const raster_ctx_t *c, const geom_t *g, double px, double py, double *u, double *v, double *a,
                   double *b, double *cz) {
    if (c->cam->mode == ORC_MODE_ORTHO) {
        intersect_ortho_g(g, px, py, u, v);
        return 1;
    }
    return intersect_pinhole_g(g, c->cam, px, py, u, v, a, b, cz);
}

/* Estimated absolute fp32 error of (u, v) as the compositor evaluates them
 * (coefficients and products rounded once each), in texel-grid units
 * (x (n-1)/(2 sigma) when n > 1).  An evaluation whose estimate exceeds
 * kink->cond_min is "sensitive": its fp32 result is intrinsically uncertain
 * beyond the tolerance (thin, grazing splats), so it is treated like a kink. */
static const double kEps32 = 5.9604644775390625e-08;

static double uv_error32_raw(const raster_ctx_t *c, const geom_t *g, double px, double py, double u, double v) {
    double eu, ev;
    if (c->cam->mode == ORC_MODE_ORTHO) {
        const double dx = px - g->x, dy = py - g->y;
        eu = 4.0 * kEps32 * (fabs(g->cos_t * dx) + fabs(g->sin_t * dy)) * g->inv_su + 2.0 * kEps32 * fabs(u);
        ev = 4.0 * kEps32 * (fabs(g->sin_t * dx) + fabs(g->cos_t * dy)) * g->inv_sv + 2.0 * kEps32 * fabs(v);
    } else {
        const double dx = px - g->cpx, dy = py - g->cpy;
        const double czt = 1.0 + fabs(g->X[2] * dx) + fabs(g->Y[2] * dy);
        const double cz = fabs(1.0 + g->X[2] * dx + g->Y[2] * dy);
        eu = 4.0 * kEps32 * (fabs(g->X[0] * dx) + fabs(g->Y[0] * dy) + fabs(u) * czt + fabs(g->X[0]) + fabs(g->Y[0])) / cz;
        ev = 4.0 * kEps32 * (fabs(g->X[1] * dx) + fabs(g->Y[1] * dy) + fabs(v) * czt + fabs(g->X[1]) + fabs(g->Y[1])) / cz;
    }
    return eu > ev ? eu : ev;
}

static double uv_error32(const raster_ctx_t *c, const geom_t *g, double px, double py, double u, double v) {
    const int n = c->s->n;
    const double grid = n > 1 ? (double)(n - 1) / (2.0 * c->s->sigma) : 1.0;
    return uv_error32_raw(c, g, px, py, u, v) * (grid > 1.0 ? grid : 1.0);
}

/* Relative margin of an alpha threshold decision (alpha-skip, the 0.999 cap): the fixed kink margin, or
 * the evaluation's own fp32 uncertainty when larger -- dalpha/alpha = |u| du + |v| dv (G = exp(-(u^2+v^2)/2))
 * plus the exponential's and the product's rounding -- which dominates for thin, grazing splats. */
static double alpha_margin(const raster_ctx_t *c, const geom_t *g, double px, double py, double u, double v) {
    if (!(c->kink->uv_rel > 0.0)) return c->kink->alpha_rel;
    const double e = 2.0 * ((fabs(u) + fabs(v)) * uv_error32_raw(c, g, px, py, u, v) + 8.0 * kEps32);
    return e > c->kink->alpha_rel ? e : c->kink->alpha_rel;
}

/* alpha within the relative uncertainty m of threshold t, in log space (|ln(alpha / t)| <= m): for small m
 * the usual |alpha - t| <= m t; for a large m (an fp32-ill-conditioned evaluation) a factor e^m either way,
 * and never an alpha that underflowed far below the threshold. */
static int near_threshold(double alpha, double t, double m) { return alpha > 0.0 && fabs(log(alpha / t)) <= m; }

/* relative fp32 error of the u- and v-proportional terms of an evaluation: uv_rel delta (1/|u| + 1/|v|) with |u|, |v|
 * floored at 0.05 and the result capped at 1; 0 when it is below eps32 (negligible) */
static double uv_rel_error(const raster_ctx_t *c, const geom_t *g, double px, double py, double u, double v) {
    if (!c->kink || !(c->kink->uv_rel > 0.0)) return 0.0;
    const double d = uv_error32_raw(c, g, px, py, u, v);
    const double au = fabs(u) > 0.05 ? fabs(u) : 0.05, av = fabs(v) > 0.05 ? fabs(v) : 0.05;
    double f = c->kink->uv_rel * d * (1.0 / au + 1.0 / av);
    if (f > 1.0) f = 1.0;
    return f > kEps32 ? f : 0.0;
}

static int sensitive(const raster_ctx_t *c, const geom_t *g, double px, double py, double u, double v) {
    return c->kink && c->kink->cond_min > 0.0 && uv_error32(c, g, px, py, u, v) > c->kink->cond_min;
}

static void forward_tile(void *vctx, int tile) {
    raster_ctx_t *c = (raster_ctx_t *)vctx;
    const orc_config *cfg = c->cfg;
    const int ts = cfg->tile_size;
    const int tx = tile % c->b->tiles_x, ty = tile / c->b->tiles_x;
    const int x0 = tx * ts, y0 = ty * ts;
    const int x1 = imin(c->cam->width, x0 + ts), y1 = imin(c->cam->height, y0 + ts);
    const int32_t *list = c->b->values + c->b->offsets[tile];
    const int64_t len = c->b->offsets[tile + 1] - c->b->offsets[tile];
    const int n = c->s->n;
    const size_t tex_stride = (size_t)n * n * 3;
    const orc_kink *kk = c->kink;
    for (int y = y0; y < y1; ++y) {
        for (int x = x0; x < x1; ++x) {
            const double px = x + 0.5, py = y + 0.5;
            double t = 1.0;
            double acc[3] = {0.0, 0.0, 0.0};
            int32_t last = -1;
            int flag = 0;
            for (int64_t rank = 0; rank < len; ++rank) {
                const geom_t *g = &c->geom[list[rank]];
                double u, v, a[3], b[3], cz = 0.0;
                if (!eval_uv(c, g, px, py, &u, &v, a, b, &cz)) continue;
                const double alpha_raw = g->alpha_k * gaussian_weight(u, v);
                const double alpha = dmin(alpha_raw, kMaxAlpha);
                if (kk) {
                    const double am = alpha_margin(c, g, px, py, u, v);
                    if (cfg->alpha_skip > 0.0 && near_threshold(alpha, cfg->alpha_skip, am)) flag |= 1;
                    if (near_threshold(alpha_raw, kMaxAlpha, am)) flag |= 1;
                    if (alpha >= cfg->alpha_skip && sensitive(c, g, px, py, u, v)) flag |= 4;
                }
                if (alpha < cfg->alpha_skip) continue;
                double col[3];
                orc_bilinear(u, v, n, c->s->sigma, c->s->grid + (size_t)list[rank] * tex_stride, col);
                const double w = alpha * t;
                acc[0] += col[0] * w;
                acc[1] += col[1] * w;
                acc[2] += col[2] * w;
                t *= 1.0 - alpha;
                last = (int32_t)rank;
                if (kk && cfg->early_stop > 0.0 && fabs(t - cfg->early_stop) <= kk->trans_rel * cfg->early_stop)
                    flag |= 2;
                if (cfg->early_stop > 0.0 && t < cfg->early_stop) break;
            }
            const size_t p = (size_t)y * c->cam->width + x;
            for (int ch = 0; ch < 3; ++ch) c->color[p * 3 + ch] = acc[ch] + t * c->cam->background[ch];
            c->trans[p] = t;
            c->last[p] = last;
            if (c->kink_px) c->kink_px[p] = (uint8_t)flag;
        }
    }
}

static geom_t *build_all_geom(const orc_splats *s, const orc_camera *cam) {
    geom_t *geom = malloc(sizeof(geom_t) * (size_t)(s->count > 0 ? s->count : 1));
    if (!geom) return NULL;
    for (int64_t k = 0; k < s->count; ++k) build_geom(s, cam, k, &geom[k]);
    return geom;
}

int orc_render_forward(const orc_splats *s, const orc_camera *cam, const orc_config *cfg, const orc_binning *b,
                       double *color, double *trans, int32_t *last, uint8_t *kink_px, const orc_kink *kink) {
    int st = validate(cam, cfg, s);
    if (st) return st;
    if (b->tiles_x != (cam->width + cfg->tile_size - 1) / cfg->tile_size ||
        b->tiles_y != (cam->height + cfg->tile_size - 1) / cfg->tile_size)
        return ORC_INVALID_ARGUMENT; /* raster.hpp:204-205 */
    geom_t *geom = build_all_geom(s, cam);
    if (!geom) return ORC_OOM;
    raster_ctx_t c;
    memset(&c, 0, sizeof(c));
    c.s = s;
    c.cam = cam;
    c.cfg = cfg;
    c.b = b;
    c.geom = geom;
    c.kink = kink;
    c.color = color;
    c.trans = trans;
    c.last = last;
    c.kink_px = kink_px;
    for_each_tile(b->tiles_x * b->tiles_y, cfg->threads, forward_tile, &c);
    free(geom);
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* Backward: raster.hpp:277-387                                               */
/* ------------------------------------------------------------------------- */

/* record layout per (tile, rank):
 *   ortho   [x, y, theta, log_su, log_sv, opacity_logit, grid...]  (raster.hpp:293-295)
 *   pinhole [dM (9, row-major), opacity_logit, grid...]            (chained per primitive afterwards)
 * Parallel records (same layout, parity protocol only):
 *   mag   -- sum of |terms| of every increment, propagated with absolute values
 *            (the scale of the fp32 rounding error of the GPU's sums);
 *   slack -- the same magnitudes restricted to evaluations whose discrete
 *            decisions sit within fp32 error of a kink (alpha-skip, the 0.999
 *            cap, early stop, texel/clamp boundaries, grazing pinhole rays):
 *            those contributions may legitimately differ between fp64 and fp32. */
static size_t geom_slots(const orc_camera *cam) { return cam->mode == ORC_MODE_ORTHO ? 6 : 10; }

/* |d(geometry record)| of one evaluation given |u_hat|, |v_hat|, |opacity term|. */
static void geo_abs(const raster_ctx_t *c, const geom_t *g, double u, double v, double uh, double vh, double op,
                    const double *a, const double *b, double cz, double dxn, double dyn, double *out) {
    if (c->cam->mode == ORC_MODE_ORTHO) {
        out[0] = uh * fabs(g->cos_t * g->inv_su) + vh * fabs(g->sin_t * g->inv_sv);
        out[1] = uh * fabs(g->sin_t * g->inv_su) + vh * fabs(g->cos_t * g->inv_sv);
        out[2] = uh * fabs(v * g->s_v * g->inv_su) + vh * fabs(u * g->s_u * g->inv_sv);
        out[3] = g->su_clamped ? 0.0 : uh * fabs(u);
        out[4] = g->sv_clamped ? 0.0 : vh * fabs(v);
        out[5] = op;
        return;
    }
    /* magnitudes in the compositor's decomposition: c = E + dxn Cx + dyn Cy
     * centred on the projected centre, sums of |gc|, |dxn gc|, |dyn gc| */
    (void)a;
    (void)b;
    const double iz = 1.0 / fabs(cz);
    const double gc[3] = {uh * iz, vh * iz, (uh * fabs(u) + vh * fabs(v)) * iz};
    const double ddx = fabs(dxn - g->dxc), ddy = fabs(dyn - g->dyc);
    for (int j = 0; j < 3; ++j) {
        out[j] = gc[j];
        out[3 + j] = ddx * gc[j];
        out[6 + j] = ddy * gc[j];
    }
    out[9] = op;
}

/* Adds |c_hat * w| to the four touched texels of an abs record (texture.hpp:77-101 pattern). */
static void tex_abs(int n, double sigma, double u, double v, const double *c_hat, double *dst) {
    if (n == 1) {
        for (int ch = 0; ch < 3; ++ch) dst[ch] += fabs(c_hat[ch]);
        return;
    }
    int32_t iu, iv;
    double fu, fv;
    orc_uv_to_grid(u, v, n, sigma, &iu, &iv, &fu, &fv);
    const double w[4] = {(1.0 - fu) * (1.0 - fv), fu * (1.0 - fv), (1.0 - fu) * fv, fu * fv};
    const size_t off[4] = {texel_offset(n, iu, iv, 0), texel_offset(n, iu + 1, iv, 0), texel_offset(n, iu, iv + 1, 0),
                           texel_offset(n, iu + 1, iv + 1, 0)};
    for (int k = 0; k < 4; ++k)
        for (int ch = 0; ch < 3; ++ch) dst[off[k] + ch] += fabs(c_hat[ch]) * w[k];
}

/* |u_hat|, |v_hat| of the texture adjoint alone (texture.hpp:102-109 with absolute values). */
static void uv_hat_tex_abs(int n, double sigma, double u, double v, const double *grid, const double *c_hat,
                           double *uh, double *vh) {
    *uh = *vh = 0.0;
    if (n == 1) return;
    int32_t iu, iv;
    double fu, fv;
    orc_uv_to_grid(u, v, n, sigma, &iu, &iv, &fu, &fv);
    double su = 0.0, sv = 0.0;
    for (int ch = 0; ch < 3; ++ch) {
        const double c00 = grid[texel_offset(n, iu, iv, ch)], c10 = grid[texel_offset(n, iu + 1, iv, ch)];
        const double c01 = grid[texel_offset(n, iu, iv + 1, ch)], c11 = grid[texel_offset(n, iu + 1, iv + 1, ch)];
        su += fabs(c_hat[ch]) * (fabs(c10 - c00) * (1.0 - fv) + fabs(c11 - c01) * fv);
        sv += fabs(c_hat[ch]) * (fabs(c01 - c00) * (1.0 - fu) + fabs(c11 - c10) * fu);
    }
    const double scale = (double)(n - 1) / (2.0 * sigma);
    if (u > -sigma && u < sigma) *uh = scale * su;
    if (v > -sigma && v < sigma) *vh = scale * sv;
}

/* |terms| of one evaluation (composited with transmittance t in front of it)
 * added to an abs record: the geometry slots and the four touched texels. */
static void add_abs_terms(const raster_ctx_t *c, const geom_t *g, double px, double py, double u, double v,
                          double alpha, double weight, double t, const double *gacc, const double *behind,
                          const double *gridk, const double *a, const double *b, double cz, double *dst) {
    const int n = c->s->n;
    const double sigma = c->s->sigma;
    const size_t gs = geom_slots(c->cam);
    const int pin = c->cam->mode == ORC_MODE_PINHOLE;
    double col[3];
    orc_bilinear(u, v, n, sigma, gridk, col);
    const double c_hat[3] = {alpha * t * gacc[0], alpha * t * gacc[1], alpha * t * gacc[2]};
    double uh_t, vh_t;
    uv_hat_tex_abs(n, sigma, u, v, gridk, c_hat, &uh_t, &vh_t);
    double ah = 0.0;
    for (int ch = 0; ch < 3; ++ch) ah += fabs(gacc[ch]) * t * (fabs(col[ch]) + fabs(behind[ch]));
    const int gated = g->alpha_k * weight < kMaxAlpha;
    const double op_abs = gated ? ah * weight * (g->alpha_k * (1.0 - g->alpha_k)) : 0.0;
    const double uh = uh_t + (gated ? ah * alpha * fabs(u) : 0.0);
    const double vh = vh_t + (gated ? ah * alpha * fabs(v) : 0.0);
    const double dxn = pin ? (px - c->cam->cx) / c->cam->fx : 0.0;
    const double dyn = pin ? (py - c->cam->cy) / c->cam->fy : 0.0;
    double d[10];
    geo_abs(c, g, u, v, uh, vh, op_abs, a, b, cz, dxn, dyn, d);
    for (size_t j = 0; j < gs; ++j) dst[j] += d[j];
    tex_abs(n, sigma, u, v, c_hat, dst + gs);
}

static void backward_tile(void *vctx, int tile) {
    raster_ctx_t *c = (raster_ctx_t *)vctx;
    const orc_config *cfg = c->cfg;
    const int32_t *list = c->b->values + c->b->offsets[tile];
    const int64_t len = c->b->offsets[tile + 1] - c->b->offsets[tile];
    if (len == 0) return;
    const size_t stride = c->stride;
    const size_t gs = geom_slots(c->cam);
    double *partial = calloc((size_t)len * stride, sizeof(double));
    double *pmag = c->want_mag ? calloc((size_t)len * stride, sizeof(double)) : NULL;
    double *pslk = c->want_slack ? calloc((size_t)len * stride, sizeof(double)) : NULL;
    c->partials[tile] = partial;
    double *ptm = c->want_tmag ? calloc((size_t)len * stride, sizeof(double)) : NULL;
    if (pmag) c->mags[tile] = pmag;
    if (pslk) c->slacks[tile] = pslk;
    if (ptm) c->tmags[tile] = ptm;
    const int ts = cfg->tile_size;
    const int tx = tile % c->b->tiles_x, ty = tile / c->b->tiles_x;
    const int x0 = tx * ts, y0 = ty * ts;
    const int x1 = imin(c->cam->width, x0 + ts), y1 = imin(c->cam->height, y0 + ts);
    const int n = c->s->n;
    const double sigma = c->s->sigma;
    const size_t tex_stride = (size_t)n * n * 3;
    const orc_kink *kk = c->kink;
    const double grid_margin = kk ? kk->grid_abs : 0.0;
    const int pin = c->cam->mode == ORC_MODE_PINHOLE;

    for (int y = y0; y < y1; ++y) {
        for (int x = x0; x < x1; ++x) {
            const size_t p = (size_t)y * c->cam->width + x;
            const int32_t last = c->last[p];
            if (last < 0) continue;
            const double *gacc = &c->image_grad[p * 3];
            if (gacc[0] == 0.0 && gacc[1] == 0.0 && gacc[2] == 0.0) continue;
            const int px_flag = c->kink_px_in ? c->kink_px_in[p] : 0;
            const double px = x + 0.5, py = y + 0.5;
            double t = c->trans[p];
            const double t_final = t;
            /* tmag: the transmittance-chain term of the fp32 error model.  Every composited entry j scales T by
             * (1 - alpha_j) whose fp32 value carries a relative error ~ eps * alpha_j / (1 - alpha_j) (alpha_j
             * itself is exact to a few eps), so the relative error of any T of this pixel is bounded by
             * O(eps) * kappa, kappa = sum_j alpha_j / (1 - alpha_j), and it is shared -- not averaged out -- by
             * the pixel's terms and by neighbouring pixels that see the same splats in front. */
            double kappa = 0.0;
            if (ptm) {
                for (int32_t rank = 0; rank <= last; ++rank) {
                    const geom_t *g = &c->geom[list[rank]];
                    double u, v, a[3], b[3], cz = 0.0;
                    if (!eval_uv(c, g, px, py, &u, &v, a, b, &cz)) continue;
                    const double alpha = dmin(g->alpha_k * gaussian_weight(u, v), kMaxAlpha);
                    if (alpha < cfg->alpha_skip) continue;
                    kappa += alpha / (1.0 - alpha);
                }
            }
            double behind[3] = {c->cam->background[0], c->cam->background[1], c->cam->background[2]};
            if (pslk && (px_flag & 1) && kk && cfg->alpha_skip > 0.0 && !(cfg->early_stop > 0.0 && t < cfg->early_stop)) {
                /* entries skipped just below the threshold AFTER the last composited one: fp32 may composite
                 * them (then its walk starts there); their own terms are the slack */
                for (int64_t rank = len - 1; rank > last; --rank) {
                    const int32_t id = list[rank];
                    const geom_t *g = &c->geom[id];
                    double u, v, a[3], b[3], cz = 0.0;
                    if (!eval_uv(c, g, px, py, &u, &v, a, b, &cz)) continue;
                    const double weight = gaussian_weight(u, v);
                    const double alpha = dmin(g->alpha_k * weight, kMaxAlpha);
                    if (near_threshold(alpha, cfg->alpha_skip, alpha_margin(c, g, px, py, u, v)))
                        add_abs_terms(c, g, px, py, u, v, alpha, weight, t, gacc, behind,
                                      c->s->grid + (size_t)id * tex_stride, a, b, cz, pslk + (size_t)rank * stride);
                }
            }
            for (int32_t rank = last; rank >= 0; --rank) {
                const int32_t id = list[rank];
                const geom_t *g = &c->geom[id];
                double u, v, a[3], b[3], cz = 0.0;
                if (!eval_uv(c, g, px, py, &u, &v, a, b, &cz)) continue;
                const double weight = gaussian_weight(u, v);
                const double alpha_raw = g->alpha_k * weight;
                const double alpha = dmin(alpha_raw, kMaxAlpha);
                const double *gridk = c->s->grid + (size_t)id * tex_stride;
                if (alpha < cfg->alpha_skip) {
                    /* an entry skipped just below the threshold may be composited in fp32 */
                    if (pslk && (px_flag & 1) && kk &&
                        near_threshold(alpha, cfg->alpha_skip, alpha_margin(c, g, px, py, u, v)))
                        add_abs_terms(c, g, px, py, u, v, alpha, weight, t, gacc, behind, gridk, a, b, cz,
                                      pslk + (size_t)rank * stride);
                    continue;
                }
                t /= 1.0 - alpha;
                double col[3];
                orc_bilinear(u, v, n, sigma, gridk, col);
                double *rec = partial + (size_t)rank * stride;
                const double c_hat[3] = {alpha * t * gacc[0], alpha * t * gacc[1], alpha * t * gacc[2]};
                double u_hat, v_hat;
                adj_bilinear_accum(u, v, n, sigma, gridk, c_hat, rec + gs, &u_hat, &v_hat);
                double alpha_hat = 0.0;
                for (int ch = 0; ch < 3; ++ch) alpha_hat += gacc[ch] * t * (col[ch] - behind[ch]);
                const size_t op = gs - 1; /* opacity slot */
                const int gated = alpha_raw < kMaxAlpha;
                if (gated) {
                    rec[op] += alpha_hat * weight * (g->alpha_k * (1.0 - g->alpha_k));
                    u_hat -= alpha_hat * alpha * u;
                    v_hat -= alpha_hat * alpha * v;
                }
                double dxn = 0.0, dyn = 0.0;
                if (!pin) {
                    /* raster.hpp:356-360 */
                    rec[0] += u_hat * (-g->cos_t * g->inv_su) + v_hat * (g->sin_t * g->inv_sv);
                    rec[1] += u_hat * (-g->sin_t * g->inv_su) + v_hat * (-g->cos_t * g->inv_sv);
                    rec[2] += u_hat * (v * g->s_v * g->inv_su) - v_hat * (u * g->s_u * g->inv_sv);
                    if (!g->su_clamped) rec[3] += u_hat * -u;
                    if (!g->sv_clamped) rec[4] += v_hat * -v;
                } else {
                    /* (u,v) = (c0,c1)/cz with c = a x b; a = M0 - dxn M2, b = M1 - dyn M2 */
                    const double gc0 = u_hat / cz, gc1 = v_hat / cz, gc2 = -(u_hat * u + v_hat * v) / cz;
                    const double ga[3] = {b[1] * gc2 - b[2] * gc1, b[2] * gc0 - b[0] * gc2, b[0] * gc1 - b[1] * gc0};
                    const double gb[3] = {gc1 * a[2] - gc2 * a[1], gc2 * a[0] - gc0 * a[2], gc0 * a[1] - gc1 * a[0]};
                    dxn = (px - c->cam->cx) / c->cam->fx;
                    dyn = (py - c->cam->cy) / c->cam->fy;
                    for (int j = 0; j < 3; ++j) {
                        rec[j] += ga[j];
                        rec[3 + j] += gb[j];
                        rec[6 + j] += -dxn * ga[j] - dyn * gb[j];
                    }
                }
                if (pmag || pslk || ptm) {
                    double uh_t, vh_t;
                    uv_hat_tex_abs(n, sigma, u, v, gridk, c_hat, &uh_t, &vh_t);
                    double ah = 0.0;
                    for (int ch = 0; ch < 3; ++ch) ah += fabs(gacc[ch]) * t * (fabs(col[ch]) + fabs(behind[ch]));
                    const double op_abs = gated ? ah * weight * (g->alpha_k * (1.0 - g->alpha_k)) : 0.0;
                    const double uh = uh_t + (gated ? ah * alpha * fabs(u) : 0.0);
                    const double vh = vh_t + (gated ? ah * alpha * fabs(v) : 0.0);
                    double d[10];
                    geo_abs(c, g, u, v, uh, vh, op_abs, a, b, cz, dxn, dyn, d);
                    if (pmag) {
                        double *rm = pmag + (size_t)rank * stride;
                        for (size_t j = 0; j < gs; ++j) rm[j] += d[j];
                        tex_abs(n, sigma, u, v, c_hat, rm + gs);
                    }
                    if (ptm) {
                        double *rt = ptm + (size_t)rank * stride;
                        for (size_t j = 0; j < gs; ++j) rt[j] += kappa * d[j];
                        const double ck[3] = {kappa * c_hat[0], kappa * c_hat[1], kappa * c_hat[2]};
                        tex_abs(n, sigma, u, v, ck, rt + gs);
                    }
                    if (pslk) {
                        double *rs = pslk + (size_t)rank * stride;
                        const double err = kk ? uv_error32(c, g, px, py, u, v) : 0.0;
                        const double margin = grid_margin > 3.0 * err ? grid_margin : 3.0 * err;
                        if ((px_flag & 3) || sensitive(c, g, px, py, u, v)) {
                            /* decision kink in this pixel, or an fp32-ill-conditioned evaluation */
                            for (size_t j = 0; j < gs; ++j) rs[j] += d[j];
                            tex_abs(n, sigma, u, v, c_hat, rs + gs);
                        } else if (uv_rel_error(c, g, px, py, u, v) > 0.0) {
                            /* the fp32 (u, v) carry the absolute error delta of uv_error32_raw; terms proportional
                             * to u or v then carry delta / |u|, delta / |v| relative -- large where u or v is small
                             * (thin, grazing surfels).  Slack: the evaluation's |terms| times that, floored */
                            const double f = uv_rel_error(c, g, px, py, u, v);
                            for (size_t j = 0; j < gs; ++j) rs[j] += f * d[j];
                            const double cf[3] = {f * c_hat[0], f * c_hat[1], f * c_hat[2]};
                            tex_abs(n, sigma, u, v, cf, rs + gs);
                        }
                        if (!((px_flag & 3) || sensitive(c, g, px, py, u, v)) &&
                            (grid_kink(u, n, sigma, margin) || grid_kink(v, n, sigma, margin))) {
                            /* only the texture part of (u_hat, v_hat) jumps across a texel
                             * boundary: bound the jump by both sides' magnitudes */
                            const double du = 2.0 * margin * (2.0 * sigma) / (n - 1);
                            double uh_s = 0.0, vh_s = 0.0, t1, t2;
                            const double sh[4][2] = {{-du, 0.0}, {du, 0.0}, {0.0, -du}, {0.0, du}};
                            for (int q = 0; q < 4; ++q) {
                                uv_hat_tex_abs(n, sigma, u + sh[q][0], v + sh[q][1], gridk, c_hat, &t1, &t2);
                                uh_s += t1;
                                vh_s += t2;
                            }
                            geo_abs(c, g, u, v, uh_s, vh_s, 0.0, a, b, cz, dxn, dyn, d);
                            for (size_t j = 0; j < gs; ++j) rs[j] += d[j];
                        }
                    }
                }
                for (int ch = 0; ch < 3; ++ch) behind[ch] = alpha * col[ch] + (1.0 - alpha) * behind[ch];
            }
            /* near an early stop the fp32 walk may composite a few entries past `last`:
             * bound their contributions with T = T_final */
            if (pslk && (px_flag & 2)) {
                for (int64_t rank = last + 1; rank < len && rank <= last + 16; ++rank) {
                    const int32_t id = list[rank];
                    const geom_t *g = &c->geom[id];
                    double u, v, a[3], b[3], cz = 0.0;
                    if (!eval_uv(c, g, px, py, &u, &v, a, b, &cz)) continue;
                    const double weight = gaussian_weight(u, v);
                    const double alpha = dmin(g->alpha_k * weight, kMaxAlpha);
                    if (alpha < cfg->alpha_skip) continue;
                    const double *gridk = c->s->grid + (size_t)id * tex_stride;
                    const double c_hat[3] = {alpha * t_final * gacc[0], alpha * t_final * gacc[1],
                                             alpha * t_final * gacc[2]};
                    double uh_t, vh_t;
                    uv_hat_tex_abs(n, sigma, u, v, gridk, c_hat, &uh_t, &vh_t);
                    double ah = 0.0;
                    for (int ch = 0; ch < 3; ++ch) ah += fabs(gacc[ch]) * t_final * 2.0;
                    double d[10];
                    const double dxn = pin ? (px - c->cam->cx) / c->cam->fx : 0.0;
                    const double dyn = pin ? (py - c->cam->cy) / c->cam->fy : 0.0;
                    geo_abs(c, g, u, v, uh_t + ah * alpha * fabs(u), vh_t + ah * alpha * fabs(v),
                            ah * weight * (g->alpha_k * (1.0 - g->alpha_k)), a, b, cz, dxn, dyn, d);
                    double *rs = pslk + (size_t)rank * stride;
                    for (size_t j = 0; j < gs; ++j) rs[j] += d[j];
                    tex_abs(n, sigma, u, v, c_hat, rs + gs);
                }
            }
        }
    }
}

/* Per-primitive chain of the pinhole dL/dM to the raw parameters (mean,
 * log-scales, unnormalised quaternion).  No reference: SURVEY Appendix C.
 * With absolute = 1 every product uses |factor| (magnitude propagation). */
static void pinhole_chain(const orc_camera *cam, const geom_t *g, const double *dM, double *g_mean, double *g_quat,
                          double *g_ls, int absolute) {
    double R[9];
    for (int i = 0; i < 9; ++i) R[i] = absolute ? fabs(cam->rot[i]) : cam->rot[i];
    double g_col0[3], g_col1[3], g_pc[3], tuc[3], tvc[3];
    for (int r = 0; r < 3; ++r) {
        g_col0[r] = dM[3 * r + 0];
        g_col1[r] = dM[3 * r + 1];
        g_pc[r] = dM[3 * r + 2];
        tuc[r] = absolute ? fabs(g->tuc[r]) : g->tuc[r];
        tvc[r] = absolute ? fabs(g->tvc[r]) : g->tvc[r];
    }
    double g_su = 0.0, g_sv = 0.0, g_tu[3] = {0, 0, 0}, g_tv[3] = {0, 0, 0};
    for (int r = 0; r < 3; ++r) {
        g_su += g_col0[r] * tuc[r];
        g_sv += g_col1[r] * tvc[r];
    }
    for (int j = 0; j < 3; ++j) {
        g_mean[j] = R[0 + j] * g_pc[0] + R[3 + j] * g_pc[1] + R[6 + j] * g_pc[2];
        g_tu[j] = g->s_u * (R[0 + j] * g_col0[0] + R[3 + j] * g_col0[1] + R[6 + j] * g_col0[2]);
        g_tv[j] = g->s_v * (R[0 + j] * g_col1[0] + R[3 + j] * g_col1[1] + R[6 + j] * g_col1[2]);
    }
    g_ls[0] = g->su_clamped ? 0.0 : g_su * g->s_u;
    g_ls[1] = g->sv_clamped ? 0.0 : g_sv * g->s_v;
    double w = g->qn[0], x = g->qn[1], y = g->qn[2], z = g->qn[3];
    double gq[4];
    if (!absolute) {
        gq[0] = g_tu[1] * 2 * z - g_tu[2] * 2 * y - g_tv[0] * 2 * z + g_tv[2] * 2 * x;
        gq[1] = g_tu[1] * 2 * y + g_tu[2] * 2 * z + g_tv[0] * 2 * y - g_tv[1] * 4 * x + g_tv[2] * 2 * w;
        gq[2] = -g_tu[0] * 4 * y + g_tu[1] * 2 * x - g_tu[2] * 2 * w + g_tv[0] * 2 * x + g_tv[2] * 2 * z;
        gq[3] = -g_tu[0] * 4 * z + g_tu[1] * 2 * w + g_tu[2] * 2 * x - g_tv[0] * 2 * w - g_tv[1] * 4 * z +
                g_tv[2] * 2 * y;
        const double dot = w * gq[0] + x * gq[1] + y * gq[2] + z * gq[3];
        for (int i = 0; i < 4; ++i) g_quat[i] = (gq[i] - g->qn[i] * dot) / g->qnorm;
    } else {
        w = fabs(w), x = fabs(x), y = fabs(y), z = fabs(z);
        gq[0] = g_tu[1] * 2 * z + g_tu[2] * 2 * y + g_tv[0] * 2 * z + g_tv[2] * 2 * x;
        gq[1] = g_tu[1] * 2 * y + g_tu[2] * 2 * z + g_tv[0] * 2 * y + g_tv[1] * 4 * x + g_tv[2] * 2 * w;
        gq[2] = g_tu[0] * 4 * y + g_tu[1] * 2 * x + g_tu[2] * 2 * w + g_tv[0] * 2 * x + g_tv[2] * 2 * z;
        gq[3] = g_tu[0] * 4 * z + g_tu[1] * 2 * w + g_tu[2] * 2 * x + g_tv[0] * 2 * w + g_tv[1] * 4 * z +
                g_tv[2] * 2 * y;
        const double dot = w * gq[0] + x * gq[1] + y * gq[2] + z * gq[3];
        const double q[4] = {w, x, y, z};
        for (int i = 0; i < 4; ++i) g_quat[i] = (gq[i] + q[i] * dot) / g->qnorm;
    }
}

static void zero_grads(orc_grads *gr, int64_t K, size_t tex_stride, int pin) {
    memset(gr->position, 0, sizeof(double) * (size_t)K * (pin ? 3 : 2));
    if (!pin) {
        if (gr->depth_key) memset(gr->depth_key, 0, sizeof(double) * (size_t)K);
        memset(gr->theta, 0, sizeof(double) * (size_t)K);
    } else {
        memset(gr->quat, 0, sizeof(double) * (size_t)K * 4);
    }
    memset(gr->log_scale, 0, sizeof(double) * (size_t)K * 2);
    memset(gr->opacity_logit, 0, sizeof(double) * (size_t)K);
    memset(gr->grid, 0, sizeof(double) * (size_t)K * tex_stride);
}

/* ordered reduction tile -> rank (raster.hpp:368-385) of one record family,
 * then (pinhole) the per-primitive chain. */
static void reduce_records(const orc_camera *cam, const orc_binning *b, const geom_t *geom, int64_t K,
                           size_t tex_stride, size_t stride, double **records, orc_grads *gr, int absolute) {
    const int pin = cam->mode == ORC_MODE_PINHOLE;
    const size_t gs = geom_slots(cam);
    const int nt = b->tiles_x * b->tiles_y;
    double *dM = pin ? calloc((size_t)(K > 0 ? K : 1) * 9, sizeof(double)) : NULL;
    for (int tile = 0; tile < nt; ++tile) {
        const double *partial = records[tile];
        if (!partial) continue;
        const int32_t *list = b->values + b->offsets[tile];
        const int64_t len = b->offsets[tile + 1] - b->offsets[tile];
        for (int64_t rank = 0; rank < len; ++rank) {
            const int32_t id = list[rank];
            const double *rec = partial + (size_t)rank * stride;
            if (!pin) {
                gr->position[2 * id + 0] += rec[0];
                gr->position[2 * id + 1] += rec[1];
                gr->theta[id] += rec[2];
                gr->log_scale[2 * id + 0] += rec[3];
                gr->log_scale[2 * id + 1] += rec[4];
                gr->opacity_logit[id] += rec[5];
            } else {
                for (int j = 0; j < 9; ++j) dM[9 * (size_t)id + j] += rec[j];
                gr->opacity_logit[id] += rec[9];
            }
            double *gg = gr->grid + (size_t)id * tex_stride;
            for (size_t i = 0; i < tex_stride; ++i) gg[i] += rec[gs + i];
        }
        free(records[tile]);
        records[tile] = NULL;
    }
    if (pin) {
        for (int64_t k = 0; k < K; ++k) {
            if (!geom[k].valid) continue;
            double *d = dM + 9 * k;
            if (absolute) {
                /* (|E|, |X|, |Y|) sums of the compositor's decomposition -> |dL/dM|:
                 * C0 = M0 x M1, Cx = M1 x M2, Cy = M2 x M0 with |cross| bounds */
                const geom_t *g = &geom[k];
                double aM[9], gC0[3], gCx[3], gCy[3], out[9];
                for (int j = 0; j < 9; ++j) aM[j] = fabs(g->M[j]);
                for (int j = 0; j < 3; ++j) {
                    gC0[j] = d[j];
                    gCx[j] = d[3 + j] + fabs(g->dxc) * d[j];
                    gCy[j] = d[6 + j] + fabs(g->dyc) * d[j];
                }
                const double *A0 = aM, *A1 = aM + 3, *A2 = aM + 6;
#define ACROSS(a, b, o)                                \
    do {                                               \
        (o)[0] = (a)[1] * (b)[2] + (a)[2] * (b)[1];    \
        (o)[1] = (a)[2] * (b)[0] + (a)[0] * (b)[2];    \
        (o)[2] = (a)[0] * (b)[1] + (a)[1] * (b)[0];    \
    } while (0)
                double t0[3], t1[3];
                ACROSS(A1, gC0, t0);
                ACROSS(gCy, A2, t1);
                for (int j = 0; j < 3; ++j) out[j] = t0[j] + t1[j];
                ACROSS(gC0, A0, t0);
                ACROSS(A2, gCx, t1);
                for (int j = 0; j < 3; ++j) out[3 + j] = t0[j] + t1[j];
                ACROSS(gCx, A1, t0);
                ACROSS(A0, gCy, t1);
                for (int j = 0; j < 3; ++j) out[6 + j] = t0[j] + t1[j];
#undef ACROSS
                memcpy(d, out, sizeof(out));
            }
            pinhole_chain(cam, &geom[k], d, gr->position + 3 * k, gr->quat + 4 * k, gr->log_scale + 2 * k, absolute);
        }
        free(dM);
    }
}

int orc_render_backward(const orc_splats *s, const orc_camera *cam, const orc_config *cfg, const orc_binning *b,
                        const double *trans, const int32_t *last, const double *image_grad, orc_grads *gr,
                        const uint8_t *kink_px, orc_grads *mag, orc_grads *slack, const orc_kink *kink) {
    return orc_render_backward_tm(s, cam, cfg, b, trans, last, image_grad, gr, kink_px, mag, slack, NULL, kink);
}

int orc_render_backward_tm(const orc_splats *s, const orc_camera *cam, const orc_config *cfg, const orc_binning *b,
                           const double *trans, const int32_t *last, const double *image_grad, orc_grads *gr,
                           const uint8_t *kink_px, orc_grads *mag, orc_grads *slack, orc_grads *tmag,
                           const orc_kink *kink) {
    int st = validate(cam, cfg, s);
    if (st) return st;
    if (b->tiles_x != (cam->width + cfg->tile_size - 1) / cfg->tile_size ||
        b->tiles_y != (cam->height + cfg->tile_size - 1) / cfg->tile_size)
        return ORC_INVALID_ARGUMENT; /* raster.hpp:283-285 */
    const int64_t K = s->count;
    const size_t tex_stride = (size_t)s->n * s->n * 3;
    const int pin = cam->mode == ORC_MODE_PINHOLE;
    /* zero the gradient buffer (core.hpp:154-163) */
    zero_grads(gr, K, tex_stride, pin);
    if (mag) zero_grads(mag, K, tex_stride, pin);
    if (slack) zero_grads(slack, K, tex_stride, pin);
    if (tmag) zero_grads(tmag, K, tex_stride, pin);

    geom_t *geom = build_all_geom(s, cam);
    const int nt = b->tiles_x * b->tiles_y;
    const size_t ntc = (size_t)(nt > 0 ? nt : 1);
    double **partials = calloc(ntc, sizeof(double *));
    double **mags = mag ? calloc(ntc, sizeof(double *)) : NULL;
    double **slacks = slack ? calloc(ntc, sizeof(double *)) : NULL;
    double **tmags = tmag ? calloc(ntc, sizeof(double *)) : NULL;
    if (!geom || !partials || (mag && !mags) || (slack && !slacks) || (tmag && !tmags)) {
        free(geom);
        free(partials);
        free(mags);
        free(slacks);
        free(tmags);
        return ORC_OOM;
    }
    raster_ctx_t c;
    memset(&c, 0, sizeof(c));
    c.s = s;
    c.cam = cam;
    c.cfg = cfg;
    c.b = b;
    c.geom = geom;
    c.kink = kink;
    c.trans = (double *)trans;
    c.last = (int32_t *)last;
    c.image_grad = image_grad;
    c.kink_px_in = kink_px;
    c.partials = partials;
    c.mags = mags;
    c.slacks = slacks;
    c.want_mag = mag != NULL;
    c.want_slack = slack != NULL;
    c.tmags = tmags;
    c.want_tmag = tmag != NULL;
    c.stride = geom_slots(cam) + tex_stride;
    for_each_tile(nt, cfg->threads, backward_tile, &c);

    reduce_records(cam, b, geom, K, tex_stride, c.stride, partials, gr, 0);
    if (mag) reduce_records(cam, b, geom, K, tex_stride, c.stride, mags, mag, 1);
    if (slack) reduce_records(cam, b, geom, K, tex_stride, c.stride, slacks, slack, 1);
    if (tmag) reduce_records(cam, b, geom, K, tex_stride, c.stride, tmags, tmag, 1);
    free(partials);
    free(mags);
    free(slacks);
    free(tmags);
    free(geom);
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* reference.hpp:20-105 -- naive renderer and FD gradient                     */
/* ------------------------------------------------------------------------- */

int orc_render_naive(const orc_splats *s, const orc_camera *cam, double *color, double *trans) {
    int st = validate(cam, NULL, s);
    if (st) return st;
    geom_t *geom = build_all_geom(s, cam);
    int32_t *order = malloc(sizeof(int32_t) * (size_t)(s->count > 0 ? s->count : 1));
    double *depth = malloc(sizeof(double) * (size_t)(s->count > 0 ? s->count : 1));
    if (!geom || !order || !depth) {
        free(geom);
        free(order);
        free(depth);
        return ORC_OOM;
    }
    int64_t cnt = 0;
    for (int64_t k = 0; k < s->count; ++k) {
        depth[k] = geom[k].depth;
        if (geom[k].valid) order[cnt++] = (int32_t)k; /* pinhole validity cull (near plane) */
    }
    pthread_mutex_lock(&g_sort_mu);
    g_sort_depth = depth;
    qsort(order, (size_t)cnt, sizeof(int32_t), cmp_depth_index); /* reference.hpp:22-27 */
    g_sort_depth = NULL;
    pthread_mutex_unlock(&g_sort_mu);
    raster_ctx_t c;
    memset(&c, 0, sizeof(c));
    c.s = s;
    c.cam = cam;
    const size_t tex_stride = (size_t)s->n * s->n * 3;
    for (int y = 0; y < cam->height; ++y) {
        for (int x = 0; x < cam->width; ++x) {
            const double px = x + 0.5, py = y + 0.5;
            double t = 1.0, acc[3] = {0.0, 0.0, 0.0};
            for (int64_t i = 0; i < cnt; ++i) {
                const int32_t id = order[i];
                double u, v, a[3], b[3], cz;
                if (!eval_uv(&c, &geom[id], px, py, &u, &v, a, b, &cz)) continue;
                const double alpha = dmin(sigmoid(s->opacity_logit[id]) * gaussian_weight(u, v), kMaxAlpha);
                double col[3];
                orc_bilinear(u, v, s->n, s->sigma, s->grid + (size_t)id * tex_stride, col);
                for (int ch = 0; ch < 3; ++ch) acc[ch] += col[ch] * alpha * t;
                t *= 1.0 - alpha;
            }
            const size_t p = (size_t)y * cam->width + x;
            for (int ch = 0; ch < 3; ++ch) color[p * 3 + ch] = acc[ch] + t * cam->background[ch];
            trans[p] = t;
        }
    }
    free(geom);
    free(order);
    free(depth);
    return ORC_OK;
}

static double linear_loss(const orc_splats *s, const orc_camera *cam, const double *w, double *color,
                          double *trans) {
    orc_render_naive(s, cam, color, trans);
    const size_t n = (size_t)cam->width * cam->height * 3;
    double acc = 0.0;
    for (size_t i = 0; i < n; ++i) acc += w[i] * color[i];
    return acc;
}

/* reference.hpp:69-80 (realised step in the denominator) */
static double fd_one(orc_splats *s, const orc_camera *cam, const double *w, double *param, double step,
                     double *color, double *trans) {
    const double saved = *param;
    const double hi = saved + step, lo = saved - step;
    *param = hi;
    const double lhi = linear_loss(s, cam, w, color, trans);
    *param = lo;
    const double llo = linear_loss(s, cam, w, color, trans);
    *param = saved;
    return (lhi - llo) / (hi - lo);
}

static void fd_group(orc_splats *s, const orc_camera *cam, const double *w, double step, double *arr, size_t n,
                     double *out, double *color, double *trans) {
    for (size_t i = 0; i < n; ++i) out[i] = fd_one(s, cam, w, &arr[i], step, color, trans);
}

/* reference.hpp:87-105 */
int orc_gradient_fd(const orc_splats *s0, const orc_camera *cam, const double *weights, double step, orc_grads *g) {
    if (!(step > 0.0)) return ORC_INVALID_ARGUMENT;
    const int64_t K = s0->count;
    const size_t tex = (size_t)K * s0->n * s0->n * 3;
    const int pin = cam->mode == ORC_MODE_PINHOLE;
    orc_splats s = *s0;
    /* private mutable copies */
    double *pos = malloc(sizeof(double) * (size_t)K * (pin ? 3 : 2) + 8);
    double *dk = malloc(sizeof(double) * (size_t)K + 8);
    double *th = malloc(sizeof(double) * (size_t)K + 8);
    double *qt = malloc(sizeof(double) * (size_t)K * 4 + 8);
    double *ls = malloc(sizeof(double) * (size_t)K * 2 + 8);
    double *op = malloc(sizeof(double) * (size_t)K + 8);
    double *gd = malloc(sizeof(double) * tex + 8);
    double *color = malloc(sizeof(double) * (size_t)cam->width * cam->height * 3);
    double *trans = malloc(sizeof(double) * (size_t)cam->width * cam->height);
    memcpy(pos, s0->position, sizeof(double) * (size_t)K * (pin ? 3 : 2));
    if (!pin) {
        memcpy(dk, s0->depth_key, sizeof(double) * (size_t)K);
        memcpy(th, s0->theta, sizeof(double) * (size_t)K);
    } else {
        memcpy(qt, s0->quat, sizeof(double) * (size_t)K * 4);
    }
    memcpy(ls, s0->log_scale, sizeof(double) * (size_t)K * 2);
    memcpy(op, s0->opacity_logit, sizeof(double) * (size_t)K);
    memcpy(gd, s0->grid, sizeof(double) * tex);
    s.position = pos;
    s.depth_key = pin ? NULL : dk;
    s.theta = pin ? NULL : th;
    s.quat = pin ? qt : NULL;
    s.log_scale = ls;
    s.opacity_logit = op;
    s.grid = gd;
    fd_group(&s, cam, weights, step, pos, (size_t)K * (pin ? 3 : 2), g->position, color, trans);
    if (!pin) {
        fd_group(&s, cam, weights, step, dk, (size_t)K, g->depth_key, color, trans);
        fd_group(&s, cam, weights, step, th, (size_t)K, g->theta, color, trans);
    } else {
        fd_group(&s, cam, weights, step, qt, (size_t)K * 4, g->quat, color, trans);
    }
    fd_group(&s, cam, weights, step, ls, (size_t)K * 2, g->log_scale, color, trans);
    fd_group(&s, cam, weights, step, op, (size_t)K, g->opacity_logit, color, trans);
    fd_group(&s, cam, weights, step, gd, tex, g->grid, color, trans);
    free(pos);
    free(dk);
    free(th);
    free(qt);
    free(ls);
    free(op);
    free(gd);
    free(color);
    free(trans);
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* optim.hpp:76-90 and the L1 photometric loss                                */
/* ------------------------------------------------------------------------- */

int64_t orc_adam_group(double *p, const double *g, double *m, double *v, int64_t n, double lr, double beta1,
                       double beta2, double eps, double bias1, double bias2) {
    for (int64_t i = 0; i < n; ++i) {
        const double gi = g[i];
        if (isnan(gi) || isinf(gi)) return i + 1;
        m[i] = beta1 * m[i] + (1.0 - beta1) * gi;
        v[i] = beta2 * v[i] + (1.0 - beta2) * gi * gi;
        const double m_hat = m[i] / bias1;
        const double v_hat = v[i] / bias2;
        p[i] -= lr * m_hat / (sqrt(v_hat) + eps);
    }
    return 0;
}

double orc_l1_loss(const double *c, const double *t, int64_t n, double scale, double *grad) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double d = c[i] - t[i];
        acc += fabs(d);
        if (grad) grad[i] = scale * (double)((d > 0.0) - (d < 0.0));
    }
    return acc * scale;
}

/* ---- seeded inputs (rng.hpp:12-46) --------------------------------------------
 * MT19937-64 as published by Matsumoto & Nishimura (the engine std::mt19937_64 names):
 * w=64, n=312, m=156, r=31, a=0xB5026F5AA96619E9, tempering (u,d)=(29,0x5555555555555555),
 * (s,b)=(17,0x71D67FFFEDA60000), (t,c)=(37,0xFFF7EEE000000000), l=43, init multiplier f=6364136223846793005. */
#define ORC_MT_N 312
#define ORC_MT_M 156
void orc_rng_seed(orc_rng *r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < ORC_MT_N; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = ORC_MT_N;
    r->have_spare = 0;
    r->spare = 0.0;
}

uint64_t orc_rng_next(orc_rng *r) {
    static const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL, a = 0xB5026F5AA96619E9ULL;
    if (r->idx >= ORC_MT_N) {
        for (int i = 0; i < ORC_MT_N; ++i) {
            const uint64_t x = (r->mt[i] & upper) | (r->mt[(i + 1) % ORC_MT_N] & lower);
            r->mt[i] = r->mt[(i + ORC_MT_M) % ORC_MT_N] ^ (x >> 1) ^ ((x & 1ULL) ? a : 0ULL);
        }
        r->idx = 0;
    }
    uint64_t y = r->mt[r->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

double orc_rng_uniform(orc_rng *r) { return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53; } /* rng.hpp:20-22 */

static double rng_uniform_in(orc_rng *r, double lo, double hi) { return lo + (hi - lo) * orc_rng_uniform(r); }

double orc_rng_normal(orc_rng *r, double mean, double stddev) { /* rng.hpp:26-40 */
    if (r->have_spare) {
        r->have_spare = 0;
        return mean + stddev * r->spare;
    }
    const double u1 = 1.0 - orc_rng_uniform(r);
    const double u2 = orc_rng_uniform(r);
    const double radius = sqrt(-2.0 * log(u1));
    const double angle = 2.0 * 3.14159265358979323846 * u2; /* M_PI */
    r->spare = radius * sin(angle);
    r->have_spare = 1;
    return mean + stddev * radius * cos(angle);
}

int orc_scene_generate_pinhole(int64_t count, int32_t n, uint64_t seed, double mean_lo, double mean_hi,
                               double mean_sigma, double log_scale_lo, double log_scale_hi, float *position,
                               float *quat, float *log_scale, float *opacity_logit, float *grid) {
    if (count < 0 || n < 1) return ORC_INVALID_ARGUMENT;
    orc_rng *geo = (orc_rng *)malloc(sizeof(orc_rng));
    if (!geo) return ORC_OOM;
    orc_rng_seed(geo, seed);
    for (int64_t k = 0; k < count; ++k) {
        for (int i = 0; i < 3; ++i)
            position[3 * k + i] = (float)(mean_sigma > 0.0 ? orc_rng_normal(geo, 0.0, mean_sigma)
                                                           : rng_uniform_in(geo, mean_lo, mean_hi));
        for (int i = 0; i < 2; ++i) log_scale[2 * k + i] = (float)rng_uniform_in(geo, log_scale_lo, log_scale_hi);
        double q[4], nn = 0.0;
        for (int i = 0; i < 4; ++i) {
            q[i] = orc_rng_normal(geo, 0.0, 1.0);
            nn += q[i] * q[i];
        }
        const double inv = 1.0 / sqrt(nn);
        for (int i = 0; i < 4; ++i) quat[4 * k + i] = (float)(q[i] * inv);
        opacity_logit[k] = (float)orc_rng_normal(geo, 0.0, 1.0);
    }
    orc_rng_seed(geo, seed + 1);
    const int64_t nt = count * (int64_t)n * n * 3;
    for (int64_t i = 0; i < nt; ++i) grid[i] = (float)orc_rng_uniform(geo);
    free(geo);
    return ORC_OK;
}

void orc_uniform_fill(uint64_t seed, int64_t n, float *out) {
    orc_rng r;
    orc_rng_seed(&r, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = (float)orc_rng_uniform(&r);
}
