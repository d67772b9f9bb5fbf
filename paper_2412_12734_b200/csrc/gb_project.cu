// gb_project.cu -- K1 (per-primitive projection + cull + tile rectangle) and
// K5 (per-primitive gradient chain to the raw parameters).
//
// Both run in fp64 and this translation unit is compiled with -fmad=false so
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

#include "gb_internal.cuh"

namespace gb {



struct Geom {
    bool valid;
    double alpha_k, s_u, s_v;
    bool su_clamped, sv_clamped;
    double cos_t, sin_t;  // ortho
    double qn[4], qnorm;  // pinhole
    double tuc[3], tvc[3];
    double M[9];
    double depth;
};

__device__ __forceinline__ double dmax_(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double dmin_(double a, double b) { return (b < a) ? b : a; }

// core.hpp:95-100 + raster.hpp:157-175 (ortho); SURVEY Appendix C (pinhole).
// Operation order mirrors oracle/gb_oracle.c build_geom().
__device__ void build_geom(const ProjParams& p, int64_t k, Geom& g) {
    g.valid = false;
    g.alpha_k = 1.0 / (1.0 + exp(-(double)p.opacity[k]));
    // SoA fields are read as one vector per primitive (log-scales 8 B, quaternion 16 B; the C-ABI requires
    // the caller's buffers to be at least 16-B aligned, as every device allocator provides)
    const float2 ls = __ldg(reinterpret_cast<const float2*>(p.log_scale) + k);
    const double eu = exp((double)ls.x);
    const double ev = exp((double)ls.y);
    g.s_u = dmax_(eu, 1e-8);
    g.s_v = dmax_(ev, 1e-8);
    g.su_clamped = eu < 1e-8;
    g.sv_clamped = ev < 1e-8;
    if (p.mode == GB_MODE_ORTHO) {
        g.valid = true;
        const double th = (double)p.theta[k];
        g.cos_t = cos(th);
        g.sin_t = sin(th);
        g.depth = (double)p.depth_key[k];
        return;
    }
    const float4 q4 = __ldg(reinterpret_cast<const float4*>(p.quat) + k);
    const double q0 = q4.x, q1 = q4.y, q2 = q4.z, q3 = q4.w;
    const double nn = q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3;
    g.qnorm = sqrt(nn);
    if (!(g.qnorm > 0.0)) return;
    g.qn[0] = q0 / g.qnorm;
    g.qn[1] = q1 / g.qnorm;
    g.qn[2] = q2 / g.qnorm;
    g.qn[3] = q3 / g.qnorm;
    const double w = g.qn[0], x = g.qn[1], y = g.qn[2], z = g.qn[3];
    double tu[3], tv[3];
    tu[0] = 1.0 - 2.0 * (y * y + z * z);
    tu[1] = 2.0 * (x * y + w * z);
    tu[2] = 2.0 * (x * z - w * y);
    tv[0] = 2.0 * (x * y - w * z);
    tv[1] = 1.0 - 2.0 * (x * x + z * z);
    tv[2] = 2.0 * (y * z + w * x);
    const double m0 = p.position[3 * k + 0], m1 = p.position[3 * k + 1], m2 = p.position[3 * k + 2];
    double pc[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        pc[r] = p.R[3 * r + 0] * m0 + p.R[3 * r + 1] * m1 + p.R[3 * r + 2] * m2 + p.t[r];
        g.tuc[r] = p.R[3 * r + 0] * tu[0] + p.R[3 * r + 1] * tu[1] + p.R[3 * r + 2] * tu[2];
        g.tvc[r] = p.R[3 * r + 0] * tv[0] + p.R[3 * r + 1] * tv[1] + p.R[3 * r + 2] * tv[2];
        g.M[3 * r + 0] = g.s_u * g.tuc[r];
        g.M[3 * r + 1] = g.s_v * g.tvc[r];
        g.M[3 * r + 2] = pc[r];
    }
    g.depth = (double)(float)pc[2];
    g.valid = pc[2] > p.near_plane;
}

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
        const double sx = sqrt(dx), sy = sqrt(dy);
        const double xa = (C02 - sx) / C22, xb = (C02 + sx) / C22;
        const double ya = (C12 - sy) / C22, yb = (C12 + sy) / C22;
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

__device__ __forceinline__ void cross3(const double* a, const double* b, double* c) {
    c[0] = a[1] * b[2] - a[2] * b[1];
    c[1] = a[2] * b[0] - a[0] * b[2];
    c[2] = a[0] * b[1] - a[1] * b[0];
}

// The same alpha-skip region as a pixel-space ellipse, for the exact
// block-vs-entry test of the sub-warp compositors (gb_composite.cu):
// alpha < alpha_skip for certain outside (p - e)^T Q (p - e) <= 1, p in pixel
// index coordinates (pixel centre at index + 0.5), same radius margin as
// alpha_box.  Record: a = (e_x, e_y, Q11, Q22), b = (Q12, Q12/Q22, Q12/Q11, 0).
// All-zero Q passes everything (threshold disabled, or the region reaches
// behind the camera and is not an ellipse); e = +inf-like passes nothing.
__device__ CullRec alpha_ellipse(const ProjParams& p, int64_t k, const Geom& g, double r, const float4 box) {
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
        const double cx = -(C[1][1] * C[0][2] - C[0][1] * C[1][2]) / det2;
        const double cy = -(C[0][0] * C[1][2] - C[0][1] * C[0][2]) / det2;
        const double kk = -(C[2][2] + C[0][2] * cx + C[1][2] * cy);
        if (!(kk > 0.0)) return all;
        A11 = C[0][0] / kk;
        A12 = C[0][1] / kk;
        A22 = C[1][1] / kk;
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

// header slot values in the compositor's precision
__device__ __forceinline__ real4 mk4(double a, double b, double c, double d) {
#ifdef GB_PARITY_F64
    return make_double4(a, b, c, d);
#else
    return make_float4((float)a, (float)b, (float)c, (float)d);
#endif
}

// Effective projected centre used by the compositor (see ScreenHeader).
__device__ __forceinline__ void pinhole_centre(const ProjParams& p, const Geom& g, int& cxi, int& cyi, real& hx,
                                               real& hy, double& dxe, double& dye) {
    const double pz = g.M[8];
    const double cxp = p.fx * (g.M[2] / pz) + p.cx;
    const double cyp = p.fy * (g.M[5] / pz) + p.cy;
    const double fxi = floor(cxp), fyi = floor(cyp);
    cxi = (int)fxi;
    cyi = (int)fyi;
    hx = (real)(0.5 - (cxp - fxi));
    hy = (real)(0.5 - (cyp - fyi));
    const double c0x = fxi + 0.5 - (double)hx;
    const double c0y = fyi + 0.5 - (double)hy;
    dxe = (c0x - p.cx) / p.fx;
    dye = (c0y - p.cy) / p.fy;
}

// c = a x b with a = M0 - dxn M2, b = M1 - dyn M2 is exactly linear in the
// normalised pixel offset: c = C0 + dxn Cx + dyn Cy, C0 = M0 x M1,
// Cx = M1 x M2, Cy = M2 x M0 (the dxn*dyn term is M2 x M2 = 0).  Centred at
// the compositor's centre (dxe, dye): E = C0 + dxe Cx + dye Cy.
struct PinholeCoeffs {
    double C0[3], Cx[3], Cy[3], E[3];
};

__device__ __forceinline__ void pinhole_coeffs(const Geom& g, double dxe, double dye, PinholeCoeffs& pc) {
    const double* M0 = g.M;
    const double* M1 = g.M + 3;
    const double* M2 = g.M + 6;
    cross3(M0, M1, pc.C0);
    cross3(M1, M2, pc.Cx);
    cross3(M2, M0, pc.Cy);
#pragma unroll
    for (int j = 0; j < 3; ++j) pc.E[j] = pc.C0[j] + dxe * pc.Cx[j] + dye * pc.Cy[j];
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
    build_geom(p, k, g);
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
        pinhole_centre(p, g, cxi, cyi, hx, hy, dxe, dye);
        PinholeCoeffs pc;
        pinhole_coeffs(g, dxe, dye, pc);
        const double sx = 1.0 / (pc.E[2] * p.fx), sy = 1.0 / (pc.E[2] * p.fy);
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
    h.h3 = alpha_box(p, k, g, ar);
    hdr[k] = h;
    cull[k] = alpha_ellipse(p, k, g, ar, h.h3);
}

// K5: chain the K4 screen-space sums to the raw parameters and ADD into the
// gradient buffer with reds (red.global.add): several views' K5s run on
// different streams into one buffer (the trainer's view lanes), so a plain
// read-modify-write could lose updates.  Ortho: raster.hpp:350-360 with the per-eval products
// (u_hat*u, ...) summed by K4.  Pinhole: dL/dM from (S_A, S_B, S_D) then the
// camera/quaternion chain (oracle pinhole_chain()).
// 8 CTAs of 128 threads per SM (64 registers, with spills): fp64 latency hides better with more warps
// (+0.9 % end to end over 96-104 registers at 4-5 CTAs)
#ifndef GB_K5_MINB
#define GB_K5_MINB 8
#endif
__global__ void __launch_bounds__(128, GB_K5_MINB) k_chain(const ProjParams p, const uint32_t* __restrict__ counts,
                                               const real* __restrict__ accum, gb_grads g_out) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= p.K) return;
    if (counts[k] == 0) return;
    const real4* a4 = reinterpret_cast<const real4*>(accum + k * kAccumStride);
    const real4 A = a4[0], B = a4[1], C = a4[2];
    Geom g;
    build_geom(p, k, g);
    if (p.mode == GB_MODE_ORTHO) {
        const double su = A.x, sv = A.y, suv = A.z, svu = A.w, suu = B.x, svv = B.y, sop = B.z;
        const double inv_su = 1.0 / g.s_u, inv_sv = 1.0 / g.s_v;
        atomicAdd(reinterpret_cast<float2*>(g_out.position) + k,
                  make_float2((float)(su * (-g.cos_t * inv_su) + sv * (g.sin_t * inv_sv)),
                              (float)(su * (-g.sin_t * inv_su) + sv * (-g.cos_t * inv_sv))));
        atomicAdd(g_out.theta + k, (float)(suv * (g.s_v * inv_su) - svu * (g.s_u * inv_sv)));
        atomicAdd(reinterpret_cast<float2*>(g_out.log_scale) + k,
                  make_float2(g.su_clamped ? 0.0f : (float)(-suu), g.sv_clamped ? 0.0f : (float)(-svv)));
        atomicAdd(g_out.opacity_logit + k, (float)(sop * (g.alpha_k * (1.0 - g.alpha_k))));
        return;
    }
    if (!g.valid) return;
    int cxi, cyi;
    real hx, hy;
    double dxe, dye;
    pinhole_centre(p, g, cxi, cyi, hx, hy, dxe, dye);
    // K4 sums over pixels of gc' = dL/dc' (c' = c / E_z):  S_E = sum gc', S_X = sum dx gc', S_Y = sum dy gc'
    PinholeCoeffs pc;
    pinhole_coeffs(g, dxe, dye, pc);
    if (!(pc.E[2] != 0.0)) return;
    const double iez = 1.0 / pc.E[2];
    const double SE[3] = {A.x, A.y, A.z}, SX[3] = {A.w, B.x, B.y}, SY[3] = {B.z, B.w, C.x};
    const double sop = C.y;
    double gC0[3], gCx[3], gCy[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        const double gE = SE[j] * iez;  // dL/dc = dL/dc' / E_z (u, v are scale invariant)
        gC0[j] = gE;
        gCx[j] = SX[j] * iez / p.fx + dxe * gE;
        gCy[j] = SY[j] * iez / p.fy + dye * gE;
    }
    // C0 = M0 x M1, Cx = M1 x M2, Cy = M2 x M0  ->  dL/dM (rows)
    const double* M0 = g.M;
    const double* M1 = g.M + 3;
    const double* M2 = g.M + 6;
    double t0[3], t1[3], dM[9];
    cross3(M1, gC0, t0);
    cross3(gCy, M2, t1);
    for (int j = 0; j < 3; ++j) dM[j] = t0[j] + t1[j];
    cross3(gC0, M0, t0);
    cross3(M2, gCx, t1);
    for (int j = 0; j < 3; ++j) dM[3 + j] = t0[j] + t1[j];
    cross3(gCx, M1, t0);
    cross3(M0, gCy, t1);
    for (int j = 0; j < 3; ++j) dM[6 + j] = t0[j] + t1[j];
    double g_col0[3], g_col1[3], g_pc[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        g_col0[r] = dM[3 * r + 0];
        g_col1[r] = dM[3 * r + 1];
        g_pc[r] = dM[3 * r + 2];
    }
    double g_su = 0.0, g_sv = 0.0, g_tu[3], g_tv[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        g_su += g_col0[r] * g.tuc[r];
        g_sv += g_col1[r] * g.tvc[r];
    }
    const double* R = p.R;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        atomicAdd(g_out.position + 3 * k + j, (float)(R[0 + j] * g_pc[0] + R[3 + j] * g_pc[1] + R[6 + j] * g_pc[2]));
        g_tu[j] = g.s_u * (R[0 + j] * g_col0[0] + R[3 + j] * g_col0[1] + R[6 + j] * g_col0[2]);
        g_tv[j] = g.s_v * (R[0 + j] * g_col1[0] + R[3 + j] * g_col1[1] + R[6 + j] * g_col1[2]);
    }
    atomicAdd(reinterpret_cast<float2*>(g_out.log_scale) + k,
              make_float2(g.su_clamped ? 0.0f : (float)(g_su * g.s_u), g.sv_clamped ? 0.0f : (float)(g_sv * g.s_v)));
    const double w = g.qn[0], x = g.qn[1], y = g.qn[2], z = g.qn[3];
    double gq[4];
    gq[0] = g_tu[1] * 2 * z - g_tu[2] * 2 * y - g_tv[0] * 2 * z + g_tv[2] * 2 * x;
    gq[1] = g_tu[1] * 2 * y + g_tu[2] * 2 * z + g_tv[0] * 2 * y - g_tv[1] * 4 * x + g_tv[2] * 2 * w;
    gq[2] = -g_tu[0] * 4 * y + g_tu[1] * 2 * x - g_tu[2] * 2 * w + g_tv[0] * 2 * x + g_tv[2] * 2 * z;
    gq[3] = -g_tu[0] * 4 * z + g_tu[1] * 2 * w + g_tu[2] * 2 * x - g_tv[0] * 2 * w - g_tv[1] * 4 * z + g_tv[2] * 2 * y;
    const double dot = w * gq[0] + x * gq[1] + y * gq[2] + z * gq[3];
    atomicAdd(reinterpret_cast<float4*>(g_out.quat) + k,
              make_float4((float)((gq[0] - g.qn[0] * dot) / g.qnorm), (float)((gq[1] - g.qn[1] * dot) / g.qnorm),
                          (float)((gq[2] - g.qn[2] * dot) / g.qnorm), (float)((gq[3] - g.qn[3] * dot) / g.qnorm)));
    atomicAdd(g_out.opacity_logit + k, (float)(sop * (g.alpha_k * (1.0 - g.alpha_k))));
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

cudaError_t launch_chain(const ProjParams& p, const uint32_t* counts, const real* accum, const gb_grads& g,
                         cudaStream_t st) {
    if (p.K == 0) return cudaSuccess;
    const int threads = 128;  // 96 fp64-heavy registers per thread: finer blocks fill the SMs better (+1 %)
    const unsigned blocks = (unsigned)((p.K + threads - 1) / threads);
    k_chain<<<blocks, threads, 0, st>>>(p, counts, accum, g);
    return cudaGetLastError();
}

}  // namespace gb
