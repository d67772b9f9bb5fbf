// gb_project.cu -- K1 (per-primitive projection + cull + tile rectangle); K5, the gradient chain, is in
// gb_chain.cu and shares the geometry of gb_geom.cuh.
//
// K1 runs in fp64 and this translation unit is compiled with -fmad=false so
// the binning decisions (opacity cull, 3-sigma box, pixel-centre coverage,
// raster.hpp:61-101) replay the fp64 operation sequence of the reference
// (ortho) and of the oracle's pinhole extension exactly; that is what makes
// the tile lists bit-exact.  Only CUDA's exp/sin/cos may differ
// from glibc by an ulp, which moves a box edge by ~1e-16 relative.
//
// HBM traffic: K1 reads 40 B of parameters and writes 48 B header + 8 B rect
// + 4 B count + 4 B depth key per binned primitive; K5 reads the parameters
// and the 48 B accumulator and read-modify-writes 40 B of gradients.
#include <math.h>

#include "gb_geom.cuh"

namespace gb {





// raster.hpp:61-86 + 93-101 (and the pinhole dual-conic box).  Writes the
// inclusive pixel range; returns false when culled.
__device__ bool cull_rect(const ProjParams& p, int64_t k, const Geom& g, int& x0, int& x1, int& y0, int& y1) {
    if (p.alpha_skip > 0.0 && g.alpha_k < p.alpha_skip) return false;  // g.alpha_k: the same expression
    double min_x, max_x, min_y, max_y;
    if (p.cutoff > 0.0) {
        if (p.mode == GB_MODE_ORTHO) {
            const double th = (double)p.theta[k];
            const double suc = g.s_u * cos(th);
            const double sus = g.s_u * sin(th);
            const double svc = g.s_v * cos(th);
            const double svs = g.s_v * sin(th);
            const double hx = p.cutoff * sqrt(suc * suc + svs * svs);
            const double hy = p.cutoff * sqrt(sus * sus + svc * svc);
            const double x = (double)p.position[2 * k];
            const double y = (double)p.position[2 * k + 1];
            min_x = x - hx;
            max_x = x + hx;
            min_y = y - hy;
            max_y = y + hy;
        } else {
            if (!g.valid) return false;
            const double r = p.cutoff;
            const double* M = g.M;
            const double lat = sqrt(M[6] * M[6] + M[7] * M[7]);
            if (!(M[8] - r * lat > p.near_plane)) return false;
            double H0[3], H1[3], H2[3];
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                H0[j] = p.fx * M[j] + p.cx * M[6 + j];
                H1[j] = p.fy * M[3 + j] + p.cy * M[6 + j];
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
            if (!(dx >= 0.0) || !(dy >= 0.0)) return false;
            const double sx = sqrt(dx), sy = sqrt(dy);
            const double xa = (C02 - sx) / C22, xb = (C02 + sx) / C22;
            const double ya = (C12 - sy) / C22, yb = (C12 + sy) / C22;
            min_x = dmin_(xa, xb);
            max_x = dmax_(xa, xb);
            min_y = dmin_(ya, yb);
            max_y = dmax_(ya, yb);
        }
    } else {
        if (!g.valid) return false;
        min_x = 0.0;
        max_x = (double)p.W;
        min_y = 0.0;
        max_y = (double)p.H;
    }
    min_x = dmax_(min_x, 0.0);
    min_y = dmax_(min_y, 0.0);
    max_x = dmin_(max_x, (double)p.W);
    max_y = dmin_(max_y, (double)p.H);
    if (!(min_x < max_x) || !(min_y < max_y)) return false;
    x0 = max(0, (int)ceil(min_x - 0.5));
    y0 = max(0, (int)ceil(min_y - 0.5));
    x1 = min(p.W - 1, (int)floor(max_x - 0.5));
    y1 = min(p.H - 1, (int)floor(max_y - 0.5));
    if (x0 > x1 || y0 > y1) return false;
    return true;
}

// Pixel box outside which alpha < alpha_skip is certain: the AABB of the uv
// ellipse u^2 + v^2 <= 2 ln(alpha_k / alpha_skip) (radius enlarged by 1e-3
// relative + 0.05 px), so the fp32 evaluation there sits > 0.1% below the
// threshold and skipping it cannot change a decision.  Whole image when the
// threshold is disabled or the ellipse is not entirely in front of the camera.
// uv radius of the alpha-skip region, enlarged as described above (alpha_box / alpha_ellipse)
__device__ __forceinline__ double alpha_radius(const ProjParams& p, const Geom& g) {
    return sqrt(2.0 * log(g.alpha_k / p.alpha_skip)) * 1.001 + 1e-3;
}

__device__ float4 alpha_box(const ProjParams& p, int64_t k, const Geom& g, double r) {
    const float4 all = make_float4(-1e30f, 1e30f, -1e30f, 1e30f);
    if (!(p.alpha_skip > 0.0)) return all;
    if (!(g.alpha_k > p.alpha_skip)) return make_float4(1e30f, -1e30f, 1e30f, -1e30f);  // never composited
    double min_x, max_x, min_y, max_y;
    if (p.mode == GB_MODE_ORTHO) {
        const double th = (double)p.theta[k];
        const double suc = g.s_u * cos(th), sus = g.s_u * sin(th), svc = g.s_v * cos(th), svs = g.s_v * sin(th);
        const double hx = r * sqrt(suc * suc + svs * svs), hy = r * sqrt(sus * sus + svc * svc);
        min_x = (double)p.position[2 * k] - hx;
        max_x = (double)p.position[2 * k] + hx;
        min_y = (double)p.position[2 * k + 1] - hy;
        max_y = (double)p.position[2 * k + 1] + hy;
    } else {
        const double* M = g.M;
        const double lat = sqrt(M[6] * M[6] + M[7] * M[7]);
        if (!(M[8] - r * lat > 0.0)) return all;
        double H0[3], H1[3], H2[3];
        for (int j = 0; j < 3; ++j) {
            H0[j] = p.fx * M[j] + p.cx * M[6 + j];
            H1[j] = p.fy * M[3 + j] + p.cy * M[6 + j];
            H2[j] = M[6 + j];
        }
        const double r2 = r * r;
        const double C00 = r2 * (H0[0] * H0[0] + H0[1] * H0[1]) - H0[2] * H0[2];
        const double C02 = r2 * (H0[0] * H2[0] + H0[1] * H2[1]) - H0[2] * H2[2];
        const double C11 = r2 * (H1[0] * H1[0] + H1[1] * H1[1]) - H1[2] * H1[2];
        const double C12 = r2 * (H1[0] * H2[0] + H1[1] * H2[1]) - H1[2] * H2[2];
        const double C22 = r2 * (H2[0] * H2[0] + H2[1] * H2[1]) - H2[2] * H2[2];
        const double dx = C02 * C02 - C00 * C22, dy = C12 * C12 - C11 * C22;
        if (!(dx >= 0.0) || !(dy >= 0.0) || !(C22 < 0.0)) return all;
        const double sx = sqrt(dx), sy = sqrt(dy), ic = 1.0 / C22;  // product-only box: reciprocal, not 4 divisions
        const double xa = (C02 - sx) * ic, xb = (C02 + sx) * ic;
        const double ya = (C12 - sy) * ic, yb = (C12 + sy) * ic;
        min_x = dmin_(xa, xb);
        max_x = dmax_(xa, xb);
        min_y = dmin_(ya, yb);
        max_y = dmax_(ya, yb);
    }
    const double m = 0.05;  // px
    if (!(min_x == min_x && max_x == max_x && min_y == min_y && max_y == max_y)) return all;
    return make_float4((float)fmax(-1e30, ceil(min_x - 0.5 - m)), (float)fmin(1e30, floor(max_x - 0.5 + m)),
                       (float)fmax(-1e30, ceil(min_y - 0.5 - m)), (float)fmin(1e30, floor(max_y - 0.5 + m)));
}


// The same alpha-skip region as a pixel-space ellipse, for the exact
// block-vs-entry test of the sub-warp compositors (gb_composite.cu):
// alpha < alpha_skip for certain outside (p - e)^T Q (p - e) <= 1, p in pixel
// index coordinates (pixel centre at index + 0.5), same radius margin as
// alpha_box.  Record: a = (e_x, e_y, Q11, Q22), b = (Q12, Q12/Q22, Q12/Q11, 0).
// All-zero Q passes everything (threshold disabled, or the region reaches
// behind the camera and is not an ellipse); e = +inf-like passes nothing.
__device__ CullRec alpha_ellipse(const ProjParams& p, int64_t k, const Geom& g, double r) {
    const CullRec all = {make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};
    const CullRec none = {make_float4(1e30f, 1e30f, 1.f, 1.f), make_float4(0.f, 0.f, 0.f, 0.f)};
    if (!(p.alpha_skip > 0.0)) return all;
    if (!(g.alpha_k > p.alpha_skip)) return none;
    const double r2 = r * r;
    double A11, A12, A22, ex, ey;
    if (p.mode == GB_MODE_ORTHO) {
        // u^2 + v^2 with u = (c dx + s dy)/s_u, v = (-s dx + c dy)/s_v (raster.hpp:36-42)
        const double th = (double)p.theta[k];
        const double c = cos(th), s = sin(th);
        const double iu2 = 1.0 / (g.s_u * g.s_u), iv2 = 1.0 / (g.s_v * g.s_v);
        A11 = (c * c * iu2 + s * s * iv2) / r2;
        A12 = (c * s * (iu2 - iv2)) / r2;
        A22 = (s * s * iu2 + c * c * iv2) / r2;
        ex = (double)p.position[2 * k] - 0.5;
        ey = (double)p.position[2 * k + 1] - 0.5;
    } else {
        const double* M = g.M;
        const double lat = sqrt(M[6] * M[6] + M[7] * M[7]);
        if (!(M[8] - r * lat > 0.0)) return all;
        // pixel ~ H (u, v, 1); (u, v, 1) ~ adj(H) pixel; region: w0^2 + w1^2 - r^2 w2^2 <= 0
        double H0[3], H1[3], H2[3], c0[3], c1[3], c2[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            H0[j] = p.fx * M[j] + p.cx * M[6 + j];
            H1[j] = p.fy * M[3 + j] + p.cy * M[6 + j];
            H2[j] = M[6 + j];
        }
        cross3(H1, H2, c0);
        cross3(H2, H0, c1);
        cross3(H0, H1, c2);
        // adj(H) has columns c0, c1, c2, so w_m = sum_j p_j c_j[m] and C[j][l] = <c_j, c_l> under diag(1, 1, -r^2)
        const double* col[3] = {c0, c1, c2};
        double C[3][3];
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int l = 0; l < 3; ++l)
                C[j][l] = col[j][0] * col[l][0] + col[j][1] * col[l][1] - r2 * col[j][2] * col[l][2];
        // C is over p = (x, y, 1) with x, y continuous pixel coordinates
        const double det2 = C[0][0] * C[1][1] - C[0][1] * C[0][1];
        if (!(C[0][0] > 0.0) || !(det2 > 0.0)) return all;
        const double idet = 1.0 / det2;  // product-only ellipse: reciprocals instead of divisions
        const double cx = -(C[1][1] * C[0][2] - C[0][1] * C[1][2]) * idet;
        const double cy = -(C[0][0] * C[1][2] - C[0][1] * C[0][2]) * idet;
        const double kk = -(C[2][2] + C[0][2] * cx + C[1][2] * cy);
        if (!(kk > 0.0)) return all;
        const double ikk = 1.0 / kk;
        A11 = C[0][0] * ikk;
        A12 = C[0][1] * ikk;
        A22 = C[1][1] * ikk;
        ex = cx - 0.5;
        ey = cy - 0.5;
    }
    if (!(isfinite(A11) && isfinite(A12) && isfinite(A22) && isfinite(ex) && isfinite(ey)) || !(A11 > 0.0) ||
        !(A22 > 0.0) || fabs(ex) > 1e7 || fabs(ey) > 1e7)
        return all;
    // The kernels evaluate the form in fp32, whose error near the boundary is ~eps32 * cond(Q); past
    // cond 4096 that would eat the 0.2 % margin (thin, grazing surfels).  Those fall back to the ellipse
    // circumscribing the alpha-box (axis-aligned, no cancellation).
    const double tr = 0.5 * (A11 + A22), dq = sqrt(fmax(tr * tr - (A11 * A22 - A12 * A12), 0.0));
    if (!(tr - dq > 0.0) || (tr + dq) > 4096.0 * (tr - dq)) {
        const float4 box = alpha_box(p, k, g, r);  // only here: the compositors test the ellipse
        if (box.x > box.y || box.z > box.w) return none;
        if (box.x < -1e29f || box.y > 1e29f || box.z < -1e29f || box.w > 1e29f) return all;
        const double hx = 0.5 * ((double)box.y - (double)box.x) + 0.5, hy = 0.5 * ((double)box.w - (double)box.z) + 0.5;
        CullRec out;
        out.a = make_float4((float)(0.5 * ((double)box.x + (double)box.y)), (float)(0.5 * ((double)box.z + (double)box.w)),
                            (float)(0.5 / (hx * hx)), (float)(0.5 / (hy * hy)));
        out.b = make_float4(0.f, 0.f, 0.f, 0.f);
        return out;
    }
    CullRec out;
    out.a = make_float4((float)ex, (float)ey, (float)A11, (float)A22);
    out.b = make_float4((float)A12, (float)(A12 / A22), (float)(A12 / A11), 0.f);
    return out;
}



// K1: one thread per primitive.
// 4 CTAs per SM (64 registers, with spills): K1 8 % faster than at 74 registers / 3 CTAs
#ifndef GB_K1_MINB
#define GB_K1_MINB 4
#endif
__global__ void __launch_bounds__(256, GB_K1_MINB) k_project(const ProjParams p, ScreenHeader* __restrict__ hdr,
                                                 CullRec* __restrict__ cull, uint2* __restrict__ rects,
                                                 uint32_t* __restrict__ counts, uint32_t* __restrict__ depth_bits) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= p.K) return;
    Geom g;
    build_geom<false>(p, k, g);
    int x0, x1, y0, y1;
    if (!cull_rect(p, k, g, x0, x1, y0, y1)) {
        counts[k] = 0;
        depth_bits[k] = 0xffffffffu;  // culled: sorts after every binned primitive (K2a)
        return;
    }
    const int tx0 = x0 / p.ts, tx1 = x1 / p.ts, ty0 = y0 / p.ts, ty1 = y1 / p.ts;
    counts[k] = (uint32_t)((tx1 - tx0 + 1) * (ty1 - ty0 + 1));
    rects[k] = make_uint2((uint32_t)tx0 | ((uint32_t)ty0 << 16), (uint32_t)tx1 | ((uint32_t)ty1 << 16));
    depth_bits[k] = float_order_key((float)g.depth);
    ScreenHeader h;
    if (p.mode == GB_MODE_ORTHO) {
        h.h0 = mk4(p.position[2 * k], p.position[2 * k + 1], g.cos_t, g.sin_t);
        h.h1 = mk4(1.0 / g.s_u, 1.0 / g.s_v, g.alpha_k, 0.0);
        h.h2 = mk4(0.0, 0.0, 0.0, 0.0);
    } else {
        int cxi, cyi;
        real hx, hy;
        double dxe, dye;
        // the header is product-only (no binning decision reads it): reciprocals instead of divisions
        pinhole_centre<true>(p, g, cxi, cyi, hx, hy, dxe, dye);
        PinholeCoeffs pc;
        pinhole_coeffs(g, dxe, dye, pc);
        const double iez = 1.0 / pc.E[2];
        const double sx = iez * p.inv_fx, sy = iez * p.inv_fy;
        const bool ok = pc.E[2] != 0.0 && isfinite(sx) && isfinite(sy);
        const double nan = (double)__int_as_float(0x7fc00000);
        // X = Cx/(E_z fx), Y = Cy/(E_z fy); a degenerate plane (through the camera centre) misses everywhere
        h.h0 = ok ? mk4(pc.Cx[0] * sx, pc.Cx[1] * sx, pc.Cx[2] * sx, pc.Cy[0] * sy) : mk4(0.0, 0.0, nan, 0.0);
        h.h1 = ok ? mk4(pc.Cy[1] * sy, pc.Cy[2] * sy, g.alpha_k, hx) : mk4(0.0, nan, g.alpha_k, hx);
        h.h2 = mk4(hy, 0.0, 0.0, 0.0);
        h.h2.y = hdr_from_int(cxi);
        h.h2.z = hdr_from_int(cyi);
    }
    const double ar = p.alpha_skip > 0.0 && g.alpha_k > p.alpha_skip ? alpha_radius(p, g) : 0.0;
#ifdef GB_CULL_BOX
    h.h3 = alpha_box(p, k, g, ar);  // A/B variant: the compositors test the box
#else
    h.h3 = make_float4(0.f, 0.f, 0.f, 0.f);  // unread: the compositors test the ellipse (cull record)
#endif
    hdr[k] = h;
    cull[k] = alpha_ellipse(p, k, g, ar);
}


}  // namespace gb

// ---- host launchers (called from gb_capi.cu) -------------------------------
namespace gb {

ProjParams make_proj_params(const gb_splats* s, const gb_camera* cam, const gb_raster_config* cfg, int tiles_x,
                            int tiles_y) {
    ProjParams p;
    p.mode = cam->mode;
    p.n = s->grid.n;
    p.K = s->count;
    p.position = s->position;
    p.depth_key = s->depth_key;
    p.theta = s->theta;
    p.quat = s->quat;
    p.log_scale = s->log_scale;
    p.opacity = s->opacity_logit;
    p.W = cam->width;
    p.H = cam->height;
    p.fx = cam->fx;
    p.fy = cam->fy;
    p.cx = cam->cx;
    p.cy = cam->cy;
    p.inv_fx = 1.0 / cam->fx;
    p.inv_fy = 1.0 / cam->fy;
    for (int i = 0; i < 9; ++i) p.R[i] = cam->rot[i];
    for (int i = 0; i < 3; ++i) p.t[i] = cam->trans[i];
    p.near_plane = cam->near_plane;
    p.ts = cfg->tile_size;
    p.tiles_x = tiles_x;
    p.tiles_y = tiles_y;
    p.cutoff = cfg->cutoff_radius;
    p.alpha_skip = cfg->alpha_skip;
    return p;
}

cudaError_t launch_project(const ProjParams& p, ScreenHeader* hdr, CullRec* cull, uint2* rects, uint32_t* counts,
                           uint32_t* depth_bits, cudaStream_t st) {
    if (p.K == 0) return cudaSuccess;
    const int threads = 256;
    const unsigned blocks = (unsigned)((p.K + threads - 1) / threads);
    k_project<<<blocks, threads, 0, st>>>(p, hdr, cull, rects, counts, depth_bits);
    return cudaGetLastError();
}


}  // namespace gb
