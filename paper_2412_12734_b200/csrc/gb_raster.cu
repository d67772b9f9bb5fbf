// gb_raster.cu -- K3 (per-tile forward compositor) and K4 (per-tile
// back-to-front backward), fp32, sm_100a.
//
// One CTA per 16x16 tile (any tile size 1..32), one thread per pixel.  The
// tile's sorted list is walked in batches of B entries: each batch's 48 B
// screen headers and full n x n x 3 textures are staged in shared memory
// (the texture is the shared-memory cost that forced the
// A6000 implementation to 8x8 tiles at n=8; a B200 CTA has 227 KB).
//
// K3 restates render_forward (raster.hpp:201-261) + bilinear
// (texture.hpp:49-66); K4 restates render_backward (raster.hpp:277-387) +
// adj_bilinear_accum (texture.hpp:77-111).  Instead of the reference's
// per-(tile, rank) partial records and ordered reduction, K4 reduces each
// entry's contributions across the warp with shuffles and issues vector
// red.global.add into (a) the caller's texel gradients and (b) a 48 B
// per-primitive screen-space accumulator that K5 chains to the raw params.
#include "gb_internal.cuh"

namespace gb {

constexpr unsigned kFull = 0xffffffffu;

template <int NT>
__device__ __forceinline__ int tex_n(int n_rt) {
    return NT ? NT : n_rt;
}

struct Bilin {
    int o00;  // offset of texel (i_u, i_v) channel 0
    float fu, fv;
    float w00, w10, w01, w11;
};

template <int NT>
__device__ __forceinline__ void bilin_setup(float u, float v, int N, const RasterConst& rc, Bilin& b) {
    int iu, iv;
    float s = __fmaf_rn(u, rc.tex_scale, rc.tex_offset);
    s = fminf(fmaxf(s, 0.0f), (float)(N - 1));
    iu = min((int)floorf(s), N - 2);
    b.fu = __fsub_rn(s, (float)iu);
    float t = __fmaf_rn(v, rc.tex_scale, rc.tex_offset);
    t = fminf(fmaxf(t, 0.0f), (float)(N - 1));
    iv = min((int)floorf(t), N - 2);
    b.fv = __fsub_rn(t, (float)iv);
    b.o00 = (iu * N + iv) * 3;
    const float gu = 1.0f - b.fu, gv = 1.0f - b.fv;
    b.w00 = gu * gv;
    b.w10 = b.fu * gv;
    b.w01 = gu * b.fv;
    b.w11 = b.fu * b.fv;
}

// ---------------------------------------------------------------------------
// shared-memory batch staging
// ---------------------------------------------------------------------------
template <int NT>
__device__ __forceinline__ void stage_batch(const int32_t* __restrict__ values, const ScreenHeader* __restrict__ hdr,
                                            const float* __restrict__ tex, int64_t first, int nb, int N,
                                            ScreenHeader* s_hdr, int* s_id, float* s_tex) {
    const int nthr = blockDim.x;
    const int tid = threadIdx.x;
    for (int i = tid; i < nb; i += nthr) {
        const int id = values[first + i];
        s_id[i] = id;
        s_hdr[i] = hdr[id];
    }
    __syncthreads();
    const int F = 3 * N * N;
    if ((F & 3) == 0) {
        const int F4 = F >> 2;
        const float4* __restrict__ t4 = reinterpret_cast<const float4*>(tex);
        float4* s4 = reinterpret_cast<float4*>(s_tex);
        for (int i = tid; i < nb * F4; i += nthr) {
            const int e = i / F4;
            const int o = i - e * F4;
            s4[i] = __ldg(&t4[(size_t)s_id[e] * F4 + o]);
        }
    } else {
        for (int i = tid; i < nb * F; i += nthr) {
            const int e = i / F;
            const int o = i - e * F;
            s_tex[i] = __ldg(&tex[(size_t)s_id[e] * F + o]);
        }
    }
    __syncthreads();
}

__host__ __device__ inline size_t batch_smem_bytes(int B, int N) {
    return (size_t)B * (sizeof(ScreenHeader) + sizeof(int) + sizeof(float) * 3 * N * N);
}

// ---------------------------------------------------------------------------
// K3 forward
// ---------------------------------------------------------------------------
template <int MODE, int NT>
__global__ void __launch_bounds__(256) k_forward(const uint2* __restrict__ ranges, const int32_t* __restrict__ values,
                                                 const ScreenHeader* __restrict__ hdr, const float* __restrict__ tex,
                                                 const CamConst cc, const RasterConst rc, int n_rt, int B,
                                                 float* __restrict__ out_color, float* __restrict__ out_trans,
                                                 int32_t* __restrict__ out_last) {
    extern __shared__ float4 smem4[];
    const int N = tex_n<NT>(n_rt);
    const int F = 3 * N * N;
    ScreenHeader* s_hdr = reinterpret_cast<ScreenHeader*>(smem4);
    float* s_tex = reinterpret_cast<float*>(s_hdr + B);
    int* s_id = reinterpret_cast<int*>(s_tex + (size_t)B * F);

    const int tile = blockIdx.x;
    const int ts = rc.tile_size;
    const int tx = tile % rc.tiles_x, ty = tile / rc.tiles_x;
    int lx, ly;
    tile_pixel(threadIdx.x, ts, lx, ly);
    const int x = tx * ts + lx, y = ty * ts + ly;
    const bool inside = (int)threadIdx.x < ts * ts && x < cc.width && y < cc.height;
    const uint2 range = ranges[tile];

    float T = 1.0f;
    float acc0 = 0.0f, acc1 = 0.0f, acc2 = 0.0f;
    int last = -1;
    bool done = !inside;

    for (uint32_t base = range.x; base < range.y; base += B) {
        if (__syncthreads_count(!done) == 0) break;
        const int nb = (int)min((uint32_t)B, range.y - base);
        stage_batch<NT>(values, hdr, tex, base, nb, N, s_hdr, s_id, s_tex);
        if (!done) {
            for (int j = 0; j < nb; ++j) {
                const ScreenHeader h = s_hdr[j];
                float u, v;
                bool hit;
                if (MODE == GB_MODE_ORTHO) {
                    hit = eval_uv_ortho(h, x, y, u, v);
                } else {
                    PinholeTerms pt;
                    hit = eval_uv_pinhole(h, x, y, u, v, pt);
                }
                if (!hit) continue;
                const float alpha_k = h.h1.z;
                const float G = gauss_weight(u, v);
                const float alpha = fminf(__fmul_rn(alpha_k, G), kMaxAlphaF);
                if (alpha < rc.alpha_skip) continue;
                const float* t = s_tex + (size_t)j * F;
                float c0, c1, c2;
                if (N == 1) {
                    c0 = t[0];
                    c1 = t[1];
                    c2 = t[2];
                } else {
                    Bilin b;
                    bilin_setup<NT>(u, v, N, rc, b);
                    const float* p00 = t + b.o00;
                    const float* p10 = p00 + 3 * N;
                    c0 = p00[0] * b.w00 + p10[0] * b.w10 + p00[3] * b.w01 + p10[3] * b.w11;
                    c1 = p00[1] * b.w00 + p10[1] * b.w10 + p00[4] * b.w01 + p10[4] * b.w11;
                    c2 = p00[2] * b.w00 + p10[2] * b.w10 + p00[5] * b.w01 + p10[5] * b.w11;
                }
                const float w = alpha * T;
                acc0 = fmaf(c0, w, acc0);
                acc1 = fmaf(c1, w, acc1);
                acc2 = fmaf(c2, w, acc2);
                T = __fmul_rn(T, __fsub_rn(1.0f, alpha));
                last = (int)(base - range.x) + j;
                if (rc.early_stop > 0.0f && T < rc.early_stop) {
                    done = true;
                    break;
                }
            }
        }
    }
    if (inside) {
        const size_t p = (size_t)y * cc.width + x;
        out_color[p * 3 + 0] = fmaf(T, cc.bg[0], acc0);
        out_color[p * 3 + 1] = fmaf(T, cc.bg[1], acc1);
        out_color[p * 3 + 2] = fmaf(T, cc.bg[2], acc2);
        out_trans[p] = T;
        out_last[p] = last;
    }
}

// ---------------------------------------------------------------------------
// K4 backward
// ---------------------------------------------------------------------------
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

__device__ __forceinline__ void red_add(float* p, float v) {
    if (v != 0.0f) atomicAdd(p, v);
}

template <int MODE, int NT>
__global__ void __launch_bounds__(256) k_backward(const uint2* __restrict__ ranges, const int32_t* __restrict__ values,
                                                  const ScreenHeader* __restrict__ hdr, const float* __restrict__ tex,
                                                  const CamConst cc, const RasterConst rc, int n_rt, int B,
                                                  const float* __restrict__ in_trans,
                                                  const int32_t* __restrict__ in_last,
                                                  const float* __restrict__ image_grad, float* __restrict__ accum,
                                                  float* __restrict__ grid_grad) {
    extern __shared__ float4 smem4[];
    __shared__ int s_maxlast;
    const int N = tex_n<NT>(n_rt);
    const int F = 3 * N * N;
    ScreenHeader* s_hdr = reinterpret_cast<ScreenHeader*>(smem4);
    float* s_tex = reinterpret_cast<float*>(s_hdr + B);
    int* s_id = reinterpret_cast<int*>(s_tex + (size_t)B * F);

    const int tile = blockIdx.x;
    const int ts = rc.tile_size;
    const int tx = tile % rc.tiles_x, ty = tile / rc.tiles_x;
    int lx, ly;
    tile_pixel(threadIdx.x, ts, lx, ly);
    const int x = tx * ts + lx, y = ty * ts + ly;
    const bool inside = (int)threadIdx.x < ts * ts && x < cc.width && y < cc.height;
    const uint2 range = ranges[tile];
    const int lane = threadIdx.x & 31;

    // raster.hpp:313-322: skip pixels with nothing composited or zero cotangent
    int last = -1;
    float T = 1.0f, g0 = 0.0f, g1 = 0.0f, g2 = 0.0f;
    if (inside) {
        const size_t p = (size_t)y * cc.width + x;
        last = in_last[p];
        g0 = image_grad[p * 3 + 0];
        g1 = image_grad[p * 3 + 1];
        g2 = image_grad[p * 3 + 2];
        T = in_trans[p];
        if (g0 == 0.0f && g1 == 0.0f && g2 == 0.0f) last = -1;
    }
    float bh0 = cc.bg[0], bh1 = cc.bg[1], bh2 = cc.bg[2];
    if (threadIdx.x == 0) s_maxlast = -1;
    __syncthreads();
    const int wmax = __reduce_max_sync(kFull, last);
    if (lane == 0 && wmax >= 0) atomicMax(&s_maxlast, wmax);
    __syncthreads();
    const int count = s_maxlast + 1;
    const float sigma = rc.sigma;

    for (int bend = count; bend > 0; bend -= B) {
        const int bstart = max(0, bend - B);
        const int nb = bend - bstart;
        __syncthreads();  // previous batch fully consumed
        stage_batch<NT>(values, hdr, tex, (int64_t)range.x + bstart, nb, N, s_hdr, s_id, s_tex);
        for (int j = nb - 1; j >= 0; --j) {
            const int rank = bstart + j;
            bool on = rank <= last;
            const ScreenHeader h = s_hdr[j];
            float u = 0.f, v = 0.f, G = 0.f, alpha = 0.f, araw = 0.f;
            PinholeTerms pt;
            if (on) {
                bool hit;
                if (MODE == GB_MODE_ORTHO) {
                    hit = eval_uv_ortho(h, x, y, u, v);
                } else {
                    hit = eval_uv_pinhole(h, x, y, u, v, pt);
                }
                if (hit) {
                    const float alpha_k = h.h1.z;
                    G = gauss_weight(u, v);
                    araw = __fmul_rn(alpha_k, G);
                    alpha = fminf(araw, kMaxAlphaF);
                    on = !(alpha < rc.alpha_skip);
                } else {
                    on = false;
                }
            }
            const unsigned act = __ballot_sync(kFull, on);
            if (act == 0) continue;

            float sg[10];
#pragma unroll
            for (int i = 0; i < 10; ++i) sg[i] = 0.0f;
            float tg[12];
#pragma unroll
            for (int i = 0; i < 12; ++i) tg[i] = 0.0f;
            int tbase = -1;
            if (on) {
                T = __fdiv_rn(T, __fsub_rn(1.0f, alpha));  // raster.hpp:333
                const float* t = s_tex + (size_t)j * F;
                float c0, c1, c2, fu_hat = 0.0f, fv_hat = 0.0f;
                const float aT = alpha * T;
                const float ch0 = aT * g0, ch1 = aT * g1, ch2 = aT * g2;  // c_hat (raster.hpp:338-340)
                if (N == 1) {
                    c0 = t[0];
                    c1 = t[1];
                    c2 = t[2];
                    tg[0] = ch0;
                    tg[1] = ch1;
                    tg[2] = ch2;
                    tbase = 0;
                } else {
                    Bilin b;
                    bilin_setup<NT>(u, v, N, rc, b);
                    const float* p00 = t + b.o00;
                    const float* p10 = p00 + 3 * N;
                    const float gu = 1.0f - b.fu, gv = 1.0f - b.fv;
                    float cc_[3];
                    const float chat[3] = {ch0, ch1, ch2};
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const float c00 = p00[c], c10 = p10[c], c01 = p00[3 + c], c11 = p10[3 + c];
                        cc_[c] = c00 * b.w00 + c10 * b.w10 + c01 * b.w01 + c11 * b.w11;
                        tg[c] = chat[c] * b.w00;
                        tg[3 + c] = chat[c] * b.w10;
                        tg[6 + c] = chat[c] * b.w01;
                        tg[9 + c] = chat[c] * b.w11;
                        fu_hat = fmaf(chat[c], (c10 - c00) * gv + (c11 - c01) * b.fv, fu_hat);
                        fv_hat = fmaf(chat[c], (c01 - c00) * gu + (c11 - c10) * b.fu, fv_hat);
                    }
                    c0 = cc_[0];
                    c1 = cc_[1];
                    c2 = cc_[2];
                    tbase = b.o00;
                }
                // texture.hpp:106-109 (strict mask)
                float u_hat = (N > 1 && u > -sigma && u < sigma) ? rc.tex_scale * fu_hat : 0.0f;
                float v_hat = (N > 1 && v > -sigma && v < sigma) ? rc.tex_scale * fv_hat : 0.0f;
                // raster.hpp:344-346
                const float gT0 = g0 * T, gT1 = g1 * T, gT2 = g2 * T;
                const float alpha_hat = gT0 * (c0 - bh0) + gT1 * (c1 - bh1) + gT2 * (c2 - bh2);
                float op = 0.0f;
                if (araw < kMaxAlphaF) {  // raster.hpp:350-354
                    op = alpha_hat * G;
                    const float aa = alpha_hat * alpha;
                    u_hat -= aa * u;
                    v_hat -= aa * v;
                }
                if (MODE == GB_MODE_ORTHO) {
                    sg[0] = u_hat;
                    sg[1] = v_hat;
                    sg[2] = u_hat * v;
                    sg[3] = v_hat * u;
                    sg[4] = u_hat * u;
                    sg[5] = v_hat * v;
                    sg[6] = op;
                } else {
                    // (u, v) = (c_x, c_y) / c_z with c = E' + dx X + dy Y (K1 header)
                    const float iz = 1.0f / pt.cz;
                    const float gc0 = u_hat * iz, gc1 = v_hat * iz, gc2 = -(u_hat * u + v_hat * v) * iz;
                    sg[0] = gc0;
                    sg[1] = gc1;
                    sg[2] = gc2;
                    sg[3] = pt.dx * gc0;
                    sg[4] = pt.dx * gc1;
                    sg[5] = pt.dx * gc2;
                    sg[6] = pt.dy * gc0;
                    sg[7] = pt.dy * gc1;
                    sg[8] = pt.dy * gc2;
                    sg[9] = op;
                }
                // raster.hpp:362
                const float om = 1.0f - alpha;
                bh0 = alpha * c0 + om * bh0;
                bh1 = alpha * c1 + om * bh1;
                bh2 = alpha * c2 + om * bh2;
            }
            const int id = s_id[j];
            // screen-space sums -> accum (one vector red per 4 floats)
            constexpr int NS = MODE == GB_MODE_ORTHO ? 7 : 10;
#pragma unroll
            for (int i = 0; i < NS; ++i) sg[i] = warp_sum(sg[i]);
            if (lane == 0) {
                float4* a4 = reinterpret_cast<float4*>(accum + (size_t)id * kAccumStride);
                atomicAdd(&a4[0], make_float4(sg[0], sg[1], sg[2], sg[3]));
                atomicAdd(&a4[1], make_float4(sg[4], sg[5], sg[6], MODE == GB_MODE_ORTHO ? 0.0f : sg[7]));
                if (MODE != GB_MODE_ORTHO) atomicAdd(reinterpret_cast<float2*>(&a4[2]), make_float2(sg[8], sg[9]));
            }
            // texel gradients: one warp reduction per distinct bilinear base
            float* gg = grid_grad + (size_t)id * F;
            unsigned pending = act;
            while (pending) {
                const int leader = __ffs(pending) - 1;
                const int b = __shfl_sync(kFull, tbase, leader);
                const bool mine = on && tbase == b;
                pending &= ~__ballot_sync(kFull, mine);
                if (N == 1) {
                    float s0 = warp_sum(mine ? tg[0] : 0.0f);
                    float s1 = warp_sum(mine ? tg[1] : 0.0f);
                    float s2 = warp_sum(mine ? tg[2] : 0.0f);
                    if (lane == leader) {
                        red_add(gg + 0, s0);
                        red_add(gg + 1, s1);
                        red_add(gg + 2, s2);
                    }
                } else {
                    float s[12];
#pragma unroll
                    for (int i = 0; i < 12; ++i) s[i] = warp_sum(mine ? tg[i] : 0.0f);
                    if (lane == leader) {
                        float* p00 = gg + b;
                        float* p10 = p00 + 3 * N;
#pragma unroll
                        for (int c = 0; c < 3; ++c) {
                            red_add(p00 + c, s[c]);
                            red_add(p10 + c, s[3 + c]);
                            red_add(p00 + 3 + c, s[6 + c]);
                            red_add(p10 + 3 + c, s[9 + c]);
                        }
                    }
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
int pick_batch(int N, int tile_threads) {
    const size_t per = batch_smem_bytes(1, N);
    int B = (int)(49152 / per);
    if (B > 256) B = 256;
    B &= ~3;  // keep the smem carve-up 16 B aligned
    if (B < 4) B = 4;
    (void)tile_threads;
    return B;
}

template <typename K>
static cudaError_t set_smem(K kernel, size_t bytes) {
    if (bytes <= 48 * 1024) return cudaSuccess;
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <int MODE, int NT>
static cudaError_t fwd_t(int tiles, int threads, size_t smem, cudaStream_t st, const uint2* ranges,
                         const int32_t* values, const ScreenHeader* hdr, const float* tex, const CamConst& cc,
                         const RasterConst& rc, int n, int B, float* color, float* trans, int32_t* last) {
    cudaError_t e = set_smem(k_forward<MODE, NT>, smem);
    if (e != cudaSuccess) return e;
    k_forward<MODE, NT><<<tiles, threads, smem, st>>>(ranges, values, hdr, tex, cc, rc, n, B, color, trans, last);
    return cudaGetLastError();
}

template <int MODE, int NT>
static cudaError_t bwd_t(int tiles, int threads, size_t smem, cudaStream_t st, const uint2* ranges,
                         const int32_t* values, const ScreenHeader* hdr, const float* tex, const CamConst& cc,
                         const RasterConst& rc, int n, int B, const float* trans, const int32_t* last,
                         const float* image_grad, float* accum, float* grid_grad) {
    cudaError_t e = set_smem(k_backward<MODE, NT>, smem);
    if (e != cudaSuccess) return e;
    k_backward<MODE, NT><<<tiles, threads, smem, st>>>(ranges, values, hdr, tex, cc, rc, n, B, trans, last,
                                                        image_grad, accum, grid_grad);
    return cudaGetLastError();
}

#define GB_DISPATCH_N(FN, MODE, ...)                    \
    switch (n) {                                        \
        case 1: return FN<MODE, 1>(__VA_ARGS__);        \
        case 2: return FN<MODE, 2>(__VA_ARGS__);        \
        case 4: return FN<MODE, 4>(__VA_ARGS__);        \
        case 8: return FN<MODE, 8>(__VA_ARGS__);        \
        case 16: return FN<MODE, 16>(__VA_ARGS__);      \
        default: return FN<MODE, 0>(__VA_ARGS__);       \
    }

cudaError_t launch_forward(int mode, int n, int tiles, int ts, const uint2* ranges, const int32_t* values,
                           const ScreenHeader* hdr, const float* tex, const CamConst& cc, const RasterConst& rc,
                           float* color, float* trans, int32_t* last, cudaStream_t st) {
    if (tiles == 0) return cudaSuccess;
    const int threads = ((ts * ts + 31) / 32) * 32;
    const int B = pick_batch(n, threads);
    const size_t smem = batch_smem_bytes(B, n);
    if (mode == GB_MODE_ORTHO) {
        GB_DISPATCH_N(fwd_t, GB_MODE_ORTHO, tiles, threads, smem, st, ranges, values, hdr, tex, cc, rc, n, B, color,
                      trans, last)
    } else {
        GB_DISPATCH_N(fwd_t, GB_MODE_PINHOLE, tiles, threads, smem, st, ranges, values, hdr, tex, cc, rc, n, B,
                      color, trans, last)
    }
}

cudaError_t launch_backward(int mode, int n, int tiles, int ts, const uint2* ranges, const int32_t* values,
                            const ScreenHeader* hdr, const float* tex, const CamConst& cc, const RasterConst& rc,
                            const float* trans, const int32_t* last, const float* image_grad, float* accum,
                            float* grid_grad, cudaStream_t st) {
    if (tiles == 0) return cudaSuccess;
    const int threads = ((ts * ts + 31) / 32) * 32;
    const int B = pick_batch(n, threads);
    const size_t smem = batch_smem_bytes(B, n);
    if (mode == GB_MODE_ORTHO) {
        GB_DISPATCH_N(bwd_t, GB_MODE_ORTHO, tiles, threads, smem, st, ranges, values, hdr, tex, cc, rc, n, B, trans,
                      last, image_grad, accum, grid_grad)
    } else {
        GB_DISPATCH_N(bwd_t, GB_MODE_PINHOLE, tiles, threads, smem, st, ranges, values, hdr, tex, cc, rc, n, B,
                      trans, last, image_grad, accum, grid_grad)
    }
}

}  // namespace gb
