// gb_geom.cuh -- per-primitive fp64 geometry shared by K1 (gb_project.cu, no FMA contraction: bit-exact
// binning decisions) and K5 (gb_chain.cu, contraction on and reciprocals instead of divisions: gradients only).
#pragma once
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
// Operation order mirrors oracle/gb_oracle.c build_geom() (kFast = false: K1, whose binning decisions must be
// bit-exact).  kFast = true (K5, gradients only): one reciprocal of the quaternion norm instead of four
// divisions, in a translation unit with FMA contraction.
template <bool kFast>
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
    if (kFast) {
        const double iq = 1.0 / g.qnorm;
        g.qn[0] = q0 * iq;
        g.qn[1] = q1 * iq;
        g.qn[2] = q2 * iq;
        g.qn[3] = q3 * iq;
    } else {
        g.qn[0] = q0 / g.qnorm;
        g.qn[1] = q1 / g.qnorm;
        g.qn[2] = q2 / g.qnorm;
        g.qn[3] = q3 / g.qnorm;
    }
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

__device__ __forceinline__ void cross3(const double* a, const double* b, double* c) {
    c[0] = a[1] * b[2] - a[2] * b[1];
    c[1] = a[2] * b[0] - a[0] * b[2];
    c[2] = a[0] * b[1] - a[1] * b[0];
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
template <bool kFast>
__device__ __forceinline__ void pinhole_centre(const ProjParams& p, const Geom& g, int& cxi, int& cyi, real& hx,
                                               real& hy, double& dxe, double& dye) {
    const double pz = g.M[8];
    double cxp, cyp;
    if (kFast) {
        const double ipz = 1.0 / pz;
        cxp = p.fx * (g.M[2] * ipz) + p.cx;
        cyp = p.fy * (g.M[5] * ipz) + p.cy;
    } else {
        cxp = p.fx * (g.M[2] / pz) + p.cx;
        cyp = p.fy * (g.M[5] / pz) + p.cy;
    }
    const double fxi = floor(cxp), fyi = floor(cyp);
    cxi = (int)fxi;
    cyi = (int)fyi;
    hx = (real)(0.5 - (cxp - fxi));
    hy = (real)(0.5 - (cyp - fyi));
    const double c0x = fxi + 0.5 - (double)hx;
    const double c0y = fyi + 0.5 - (double)hy;
    dxe = kFast ? (c0x - p.cx) * p.inv_fx : (c0x - p.cx) / p.fx;
    dye = kFast ? (c0y - p.cy) * p.inv_fy : (c0y - p.cy) / p.fy;
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

}  // namespace gb
