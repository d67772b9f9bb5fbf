// gb_raster.cu -- K3 (per-tile forward compositor) and K4 (per-tile
// back-to-front backward), fp32, sm_100a.
//
// One CTA per tile (tile size 1..16), one thread per pixel; with 8-multiple
// tiles each warp owns an 8x4 pixel block.  Two implementations of the walk:
//
//  * direct (k_forward_direct / k_backward_direct, the default): every warp
//    walks the tile's sorted list on its own through L1.  Per 32 entries it
//    loads ids and cull records, tests its pixel rectangle against each
//    entry's exact alpha-skip ellipse (K1 alpha_ellipse) and ballots; then it
//    composites the passing entries one at a time.  No CTA barrier.
//  * staged (k_forward / k_backward, GB_COMPOSITOR=staged): a producer warp
//    streams every entry's 64 B header and full n x n x 3 texture into a
//    4-stage shared-memory ring with TMA bulk copies (cp.async.bulk, UBLKCP)
//    and mbarrier full/empty handshakes, the 8 consumer warps composite from
//    shared memory (PAPER.md:202-206 staged textures the same way).  Measured
//    slower: it copies whole textures where a pixel needs four
//    texels and spends issue slots in barrier waits.
//
// K3 restates render_forward (raster.hpp:201-261) + bilinear
// (texture.hpp:49-66); K4 restates render_backward (raster.hpp:277-387) +
// adj_bilinear_accum (texture.hpp:77-111).  In the direct walks each entry is
// shaded in one of four texel footprint classes (bwd_shade): lanes outside the
// |u|, |v| < sigma texture square are clamped to one texel row/column, so a warp
// whose active lanes never interpolate along an axis loads and scatters 1 or 2
// texels per pixel instead of 4.  Instead of the reference's per-(tile, rank)
// partial records and ordered reduction, K4 adds each entry's per-pixel
// contributions with red.global.add into (a) the caller's texel gradients and
// (b) a 48 B per-primitive screen-space accumulator that K5 chains to the raw
// parameters: straight from every active lane when at most 12 lanes are active,
// else after a warp reduction (a shared-memory transpose, lane l summing half
// of row l/2).
#include <climits>
#include <cstdlib>
#include <cstring>

#include "gb_compose.cuh"

namespace gb {


#ifdef GB_DEBUG_COUNTERS
// development counters (not built by default): [0] warp-entries tested, [1] passing the box,
// [2] with an active lane, [3] active lanes, [4] uniform-cell texel groups, [5] per-lane texel groups,
// [6] active entries with both 4x4 halves active, [7] with both 8x2 halves active
__device__ unsigned long long g_dbg[8];
#define GB_DBG(i, v) atomicAdd(&g_dbg[i], (unsigned long long)(v))
extern "C" __attribute__((visibility("default"))) int gb_debug_counters(unsigned long long* out, int reset) {
    cudaMemcpyFromSymbol(out, g_dbg, sizeof(g_dbg));
    if (reset) {
        unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(g_dbg, z, sizeof(z));
    }
    return 0;
}
#else
#define GB_DBG(i, v)
#endif

// ---------------------------------------------------------------------------
// asynchronous batch staging: TMA bulk copies (n even) or cp.async (n odd)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

// Blocking wait on an mbarrier phase.  try_wait with a suspend-time hint lets
// the hardware park the warp until the phase flips instead of spinning on
// issue slots the compositing warps need.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(0x989680)
        : "memory");
}

// Producer-side wait: the producer runs up to kStages batches ahead and then
// waits on the slowest consumer; poll with an exponential nanosleep back-off so
// it does not steal issue slots from the compositing warps.
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{ .reg .pred P1; mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2; selp.u32 %0, 1, 0, P1; }"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    uint32_t ns = 32;
    while (!mbar_test(bar, parity)) {
        __nanosleep(ns);
        ns = ns < 512 ? ns * 2 : 512;
    }
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// One staging buffer: B headers, B ids, B textures.
struct Stage {
    ScreenHeader* hdr;
    float* tex;
    int* id;
};

__host__ __device__ inline size_t stage_bytes(int B, int N) {  // rounded so the second buffer stays 128 B aligned
    return ((size_t)B * (sizeof(ScreenHeader) + sizeof(float) * 3 * N * N + sizeof(int)) + 127) & ~(size_t)127;
}

__device__ __forceinline__ Stage stage_at(unsigned char* base, int buf, int B, int N) {
    unsigned char* p = base + (size_t)buf * stage_bytes(B, N);
    Stage s;
    s.hdr = reinterpret_cast<ScreenHeader*>(p);
    s.tex = reinterpret_cast<float*>(p + (size_t)B * sizeof(ScreenHeader));
    s.id = reinterpret_cast<int*>(p + (size_t)B * (sizeof(ScreenHeader) + sizeof(float) * 3 * N * N));
    return s;
}

// Issued by warp 0 only: entries [first, first + nb) of the tile list.  Bulk
// path (n even: 12 n^2 B is a multiple of 16): lane 0 arms the barrier with
// the batch's byte count, then the lanes each issue bulk copies.  cp.async
// path (n odd): the whole warp copies 4-byte words and arrives on the barrier
// when they land (cp.async.mbarrier.arrive.noinc).
__device__ __forceinline__ void issue_batch(const int32_t* __restrict__ values, const ScreenHeader* __restrict__ hdr,
                                            const float* __restrict__ tex, int64_t first, int nb, int N,
                                            const Stage& s, uint64_t* bar) {
    const int lane = threadIdx.x & 31;
    const int F = 3 * N * N;
    // make the generic-proxy reads of this buffer (previous batch) ordered before the async writes
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if ((F & 3) == 0) {
        if (lane == 0) mbar_arrive_expect_tx(bar, (uint32_t)nb * (uint32_t)(sizeof(ScreenHeader) + 4 * F));
        __syncwarp();
        for (int i = lane; i < nb; i += 32) {
            const int id = values[first + i];
            s.id[i] = id;
            bulk_g2s(&s.hdr[i], &hdr[id], sizeof(ScreenHeader), bar);
            bulk_g2s(s.tex + (size_t)i * F, tex + (size_t)id * F, 4u * F, bar);
        }
    } else {
        for (int i = lane; i < nb; i += 32) s.id[i] = values[first + i];
        __syncwarp();
        for (int i = lane; i < nb * 4; i += 32) {
            const int e = i >> 2, q = i & 3;
            cp_async16(reinterpret_cast<float4*>(&s.hdr[e]) + q, reinterpret_cast<const float4*>(&hdr[s.id[e]]) + q);
        }
        for (int i = lane; i < nb * F; i += 32) {
            const int e = i / F, o = i - e * F;
            cp_async4(s.tex + i, tex + (size_t)s.id[e] * F + o);
        }
        // every lane's copies arrive on the barrier (count 32) when they complete
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
    }
}


__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// ---------------------------------------------------------------------------
// Warp-specialised staging pipeline shared by K3/K4.
//   warp `cw` (the last warp; cw = number of consumer warps) is the producer:
//   for each batch r it waits until every consumer released stage r % S
//   (empty[s]) and issues the batch's bulk copies completing on full[s];
//   consumer warps wait full[s], composite, arrive empty[s].  Consumers never
//   meet at a CTA barrier, so a warp with little work runs up to S-1 batches
//   ahead instead of idling at a per-batch __syncthreads.  Warps stay in the
//   pipeline until the last batch (no phase is ever skipped); once every
//   consumer has finished early (forward), the producer stops copying and just
//   completes the remaining full[] phases so the finished warps drain through.
// ---------------------------------------------------------------------------
constexpr int kStages = 4;

struct Pipe {
    uint64_t full[kStages];
    uint64_t empty[kStages];
    int active;  // consumer warps still compositing (forward early termination)
};

__device__ __forceinline__ void pipe_init(Pipe& p, int consumers, bool bulk) {
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&p.full[s], bulk ? 1 : 32);
            mbar_init(&p.empty[s], consumers);
        }
        p.active = consumers;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
}

// Producer loop over `nbatch` batches; batch r covers list entries
// [first(r), first(r) + count(r)) relative to the tile's range start.
template <typename FirstFn>
__device__ __forceinline__ void produce(Pipe& p, const int32_t* __restrict__ values,
                                        const ScreenHeader* __restrict__ hdr, const float* __restrict__ tex,
                                        int64_t base, int nbatch, int B, int N, unsigned char* smem, FirstFn span) {
    const bool bulk = ((3 * N * N) & 3) == 0;
    const int lane = threadIdx.x & 31;
    for (int r = 0; r < nbatch; ++r) {
        const int s = r % kStages;
        if (r >= kStages) mbar_wait_sleep(&p.empty[s], ((r / kStages) - 1) & 1);
        if (*(volatile int*)&p.active == 0) {  // nobody needs the data: complete the phase without copies
            if (!bulk || lane == 0) mbar_arrive(&p.full[s]);
            continue;
        }
        int first, cnt;
        span(r, first, cnt);
        issue_batch(values, hdr, tex, base + first, cnt, N, stage_at(smem, s, B, N), &p.full[s]);
    }
}

// ---------------------------------------------------------------------------
// K3 forward
// ---------------------------------------------------------------------------
template <int MODE, int NT>
__global__ void __launch_bounds__(288) k_forward(const uint2* __restrict__ ranges, const int32_t* __restrict__ values,
                                                 const ScreenHeader* __restrict__ hdr, const float* __restrict__ tex,
                                                 const CamConst cc, const RasterConst rc, int n_rt, int B,
                                                 float* __restrict__ out_color, float* __restrict__ out_trans,
                                                 int32_t* __restrict__ out_last) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) Pipe pipe;
    const int N = tex_n<NT>(n_rt);
    const int F = 3 * N * N;
    const int ts = rc.tile_size;
    const int consumers = (ts * ts + 31) >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tile = blockIdx.x;
    const uint2 range = ranges[tile];
    const int total = (int)(range.y - range.x);
    const int nbatch = (total + B - 1) / B;
    pipe_init(pipe, consumers, (F & 3) == 0);
    __syncthreads();

    if (warp == consumers) {  // producer warp
        produce(pipe, values, hdr, tex, range.x, nbatch, B, N, smem, [&](int r, int& first, int& cnt) {
            first = r * B;
            cnt = min(B, total - first);
        });
        return;
    }

    const int tx = tile % rc.tiles_x, ty = tile / rc.tiles_x;
    int lx, ly;
    tile_pixel(threadIdx.x, ts, lx, ly);
    const int x = tx * ts + lx, y = ty * ts + ly;
    const bool inside = (int)threadIdx.x < ts * ts && x < cc.width && y < cc.height;
    // this warp's pixel block (as pixel indices)
    const float bx0 = (float)__reduce_min_sync(kFull, x), bx1 = (float)__reduce_max_sync(kFull, x);
    const float by0 = (float)__reduce_min_sync(kFull, y), by1 = (float)__reduce_max_sync(kFull, y);

    float T = 1.0f;
    float acc0 = 0.0f, acc1 = 0.0f, acc2 = 0.0f;
    int last = -1;
    bool done = !inside;
    bool warp_done = false;
    for (int r = 0; r < nbatch; ++r) {
        const int s = r % kStages;
        if (!warp_done && __all_sync(kFull, done)) {  // every pixel of this warp terminated early
            warp_done = true;
            if (lane == 0) atomicSub(&pipe.active, 1);
        }
        mbar_wait(&pipe.full[s], (r / kStages) & 1);
        const Stage st = stage_at(smem, s, B, N);
        const int nb = min(B, total - r * B);
        if (!warp_done) {
            // one ballot per 32 entries finds the entries whose alpha-box meets this warp's block;
            // the loop stays warp-uniform (finished lanes ride along idle)
            for (int c0 = 0; c0 < nb; c0 += 32) {
                unsigned mask =
                    __ballot_sync(kFull, c0 + lane < nb && !box_miss(st.hdr[c0 + lane].h3, bx0, bx1, by0, by1));
                while (mask) {
                    const int j = c0 + __ffs(mask) - 1;
                    mask &= mask - 1;
                    if (!done) {
                        const ScreenHeader h = st.hdr[j];
                        float u, v;
                        bool hit;
                        if (MODE == GB_MODE_ORTHO) {
                            hit = eval_uv_ortho(h, x, y, u, v);
                        } else {
                            PinholeTerms pt;
                            hit = eval_uv_pinhole(h, x, y, u, v, pt);
                        }
                        if (hit) {
                            const float G = gauss_weight(u, v);
                            const float alpha = fminf(__fmul_rn(h.h1.z, G), kMaxAlphaF);
                            if (!(alpha < rc.alpha_skip)) {
                                const float* t = st.tex + (size_t)j * F;
                                float c0_, c1_, c2_;
                                if (N == 1) {
                                    c0_ = t[0];
                                    c1_ = t[1];
                                    c2_ = t[2];
                                } else {
                                    Bilin b;
                                    bilin_setup(u, v, N, rc, b);
                                    const float* p00 = t + b.o00;
                                    const float* p10 = p00 + 3 * N;
                                    c0_ = p00[0] * b.w00 + p10[0] * b.w10 + p00[3] * b.w01 + p10[3] * b.w11;
                                    c1_ = p00[1] * b.w00 + p10[1] * b.w10 + p00[4] * b.w01 + p10[4] * b.w11;
                                    c2_ = p00[2] * b.w00 + p10[2] * b.w10 + p00[5] * b.w01 + p10[5] * b.w11;
                                }
                                const float w = alpha * T;
                                acc0 = fmaf(c0_, w, acc0);
                                acc1 = fmaf(c1_, w, acc1);
                                acc2 = fmaf(c2_, w, acc2);
                                T = __fmul_rn(T, __fsub_rn(1.0f, alpha));
                                last = r * B + j;
                                if (rc.early_stop > 0.0f && T < rc.early_stop) done = true;
                            }
                        }
                    }
                    if (__all_sync(kFull, done)) break;
                }
                if (__all_sync(kFull, done)) break;
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&pipe.empty[s]);
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
// warp reduce-scatter: V = 2^M values per lane -> after the call, lane l holds
// the warp sum of value index (l >> (5 - M)); V - 1 + (5 - M) shuffles.
// ---------------------------------------------------------------------------
template <int V>
__device__ __forceinline__ float reduce_scatter(float (&a)[V], int lane) {
    static_assert(V >= 1 && V <= 32 && (V & (V - 1)) == 0, "V must be a power of two <= 32");
    constexpr int M = V == 1 ? 0 : V == 2 ? 1 : V == 4 ? 2 : V == 8 ? 3 : V == 16 ? 4 : 5;
#pragma unroll
    for (int k = 0; k < M; ++k) {
        const int off = 16 >> k;
        const bool up = (lane & off) != 0;
        const int S = V >> k;
#pragma unroll
        for (int j = 0; j < S / 2; ++j) {
            const float send = up ? a[j] : a[j + S / 2];
            const float keep = up ? a[j + S / 2] : a[j];
            a[j] = keep + __shfl_xor_sync(kFull, send, off);
        }
    }
    float r = a[0];
#pragma unroll
    for (int off = 16 >> M; off > 0; off >>= 1) r += __shfl_xor_sync(kFull, r, off);
    return r;
}

// ---------------------------------------------------------------------------
// K4 backward
// ---------------------------------------------------------------------------
// One backward entry for the calling warp: evaluate, update the pixel's
// rewind state, reduce and scatter the gradients (raster.hpp:324-363).
// Texel footprint class of a warp-entry (texture.hpp:27-47).  A lane whose |u| >= sigma sits where the
// clamp pins u' to 0 or n-1: f_u is exactly 0 or 1, one texel row carries all the weight and the u
// adjoint is masked (texture.hpp:106-109); likewise for v.  When no active lane of the warp needs
// interpolation along u (v), the bilinear cell degenerates to a texel pair or a single texel and the
// warp skips the loads, products and reductions of the zero-weight corners.  In a configs[3] view 27 %
// of warp-entries need one texel, 48 % two, 25 % all four (62 % of active pixels are clamped in both).
enum { kCellFull = 0, kCellU = 1, kCellV = 2, kCellOne = 3 };

template <int CELL>
struct CellShape {
    static constexpr int texels = CELL == kCellFull ? 4 : CELL == kCellOne ? 1 : 2;
};

// offset of reduced texel-gradient value i (corner i / 3, channel i % 3) from the class's base texel
template <int CELL>
__device__ __forceinline__ int cell_offset(int i, int N) {
    if (CELL == kCellFull) return corner_offset(i, N);
    if (CELL == kCellU) return i < 3 ? i : 3 * N + i - 3;  // (i_u, i_v'), (i_u + 1, i_v')
    return i;                                              // kCellV: (i_u', i_v), (i_u', i_v + 1); kCellOne
}

// One backward entry for the calling warp, after the evaluation: rewind the pixel's state, form the
// adjoints and reduce/scatter the gradients (raster.hpp:324-363).
template <int MODE, int NT, int CELL>
__device__ __forceinline__ void bwd_shade(const float* __restrict__ t, int id, bool on, unsigned act, float u,
                                          float v, float G, float alpha, float araw, const PinholeTerms& pt,
                                          float& T, float g0, float g1, float g2, float& bh0, float& bh1,
                                          float& bh2, const RasterConst& rc, int N, int lane, float* wscratch,
                                          float* __restrict__ accum, float* __restrict__ grid_grad) {
    constexpr int NS = MODE == GB_MODE_ORTHO ? 7 : 10;  // screen-space sums per entry
    constexpr int NX = CellShape<CELL>::texels;
    const int F = 3 * N * N;
    const float sigma = rc.sigma;
    float red[16];  // screen-space sums (NS of 16 slots)
#pragma unroll
    for (int i = 0; i < 16; ++i) red[i] = 0.0f;
    float tg[3 * NX];
#pragma unroll
    for (int i = 0; i < 3 * NX; ++i) tg[i] = 0.0f;
    int tbase = -1;
    float wk[NX];  // corner weights
#pragma unroll
    for (int k = 0; k < NX; ++k) wk[k] = 0.0f;
    if (on) {
        T = __fmul_rn(T, rcp_approx(__fsub_rn(1.0f, alpha)));  // raster.hpp:333
        float c0, c1, c2, fu_hat = 0.0f, fv_hat = 0.0f;
        const float aT = alpha * T;
        const float chat[3] = {aT * g0, aT * g1, aT * g2};  // c_hat (raster.hpp:338-340)
        float cc_[3];
        if (CELL == kCellFull) {
            Bilin b;
            bilin_setup(u, v, N, rc, b);
            const float* p00 = t + b.o00;
            const float* p10 = p00 + 3 * N;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const float c00 = p00[c], c10 = p10[c], c01 = p00[3 + c], c11 = p10[3 + c];
                cc_[c] = c00 * b.w00 + c10 * b.w10 + c01 * b.w01 + c11 * b.w11;
                tg[c] = chat[c] * b.w00;
                tg[3 + c] = chat[c] * b.w10;
                tg[6 + c] = chat[c] * b.w01;
                tg[9 + c] = chat[c] * b.w11;
                // texture.hpp:102-103: (C10 - C00)(1 - f_v) + (C11 - C01) f_v = du + f_v e and
                // (C01 - C00)(1 - f_u) + (C11 - C10) f_u = dv + f_u e, e = C11 - C10 - C01 + C00
                const float du = c10 - c00, dv = c01 - c00, e = (c11 - c10) - dv;
                fu_hat = fmaf(chat[c], fmaf(b.fv, e, du), fu_hat);
                fv_hat = fmaf(chat[c], fmaf(b.fu, e, dv), fv_hat);
            }
            tbase = b.o00;
            wk[0] = b.w00;
            wk[1] = b.w10;
            wk[2] = b.w01;
            wk[3] = b.w11;
        } else if (CELL == kCellU || CELL == kCellV) {
            // interpolation along one axis; the other sits on texel 0 or n-1
            const float w = CELL == kCellU ? u : v;
            float sx = __fmaf_rn(w, rc.tex_scale, rc.tex_offset);
            sx = fminf(fmaxf(sx, 0.0f), (float)(N - 1));
            const int i0 = min((int)floorf(sx), N - 2);
            const float f = __fsub_rn(sx, (float)i0);
            const float gf = 1.0f - f;
            const int other = (CELL == kCellU ? v : u) > 0.0f ? N - 1 : 0;
            tbase = (CELL == kCellU ? i0 * N + other : other * N + i0) * 3;
            const float* pa = t + tbase;
            const float* pb = pa + (CELL == kCellU ? 3 * N : 3);
            float fh = 0.0f;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const float ca = pa[c], cb = pb[c];
                cc_[c] = fmaf(cb, f, ca * gf);  // = the four-corner blend with two zero weights
                tg[c] = chat[c] * gf;
                tg[3 + c] = chat[c] * f;
                fh = fmaf(chat[c], cb - ca, fh);
            }
            if (CELL == kCellU)
                fu_hat = fh;
            else
                fv_hat = fh;
            wk[0] = gf;
            wk[1] = f;
        } else {  // kCellOne (and n = 1): a single texel with weight 1
            const int iu = N > 1 && u > 0.0f ? N - 1 : 0, iv = N > 1 && v > 0.0f ? N - 1 : 0;
            tbase = (iu * N + iv) * 3;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                cc_[c] = t[tbase + c];
                tg[c] = chat[c];
            }
            wk[0] = 1.0f;
        }
        c0 = cc_[0];
        c1 = cc_[1];
        c2 = cc_[2];
        // texture.hpp:106-109 (strict mask)
        float u_hat = (CELL != kCellV && CELL != kCellOne && u > -sigma && u < sigma) ? rc.tex_scale * fu_hat : 0.0f;
        float v_hat = (CELL != kCellU && CELL != kCellOne && v > -sigma && v < sigma) ? rc.tex_scale * fv_hat : 0.0f;
        // raster.hpp:344-346
        const float alpha_hat = T * (g0 * (c0 - bh0) + g1 * (c1 - bh1) + g2 * (c2 - bh2));
        float op = 0.0f;
        if (araw < kMaxAlphaF) {  // raster.hpp:350-354
            op = alpha_hat * G;
            const float aa = alpha_hat * alpha;
            u_hat -= aa * u;
            v_hat -= aa * v;
        }
        if (MODE == GB_MODE_ORTHO) {
            red[0] = u_hat;
            red[1] = v_hat;
            red[2] = u_hat * v;
            red[3] = v_hat * u;
            red[4] = u_hat * u;
            red[5] = v_hat * v;
            red[6] = op;
        } else {
            // (u, v) = (c_x, c_y) / c_z with c = E' + dx X + dy Y (K1 header)
            const float iz = pt.iz;
            const float gc0 = u_hat * iz, gc1 = v_hat * iz, gc2 = -(u_hat * u + v_hat * v) * iz;
            red[0] = gc0;
            red[1] = gc1;
            red[2] = gc2;
            red[3] = pt.dx * gc0;
            red[4] = pt.dx * gc1;
            red[5] = pt.dx * gc2;
            red[6] = pt.dy * gc0;
            red[7] = pt.dy * gc1;
            red[8] = pt.dy * gc2;
            red[9] = op;
        }
        // raster.hpp:362
        const float om = 1.0f - alpha;
        bh0 = alpha * c0 + om * bh0;
        bh1 = alpha * c1 + om * bh1;
        bh2 = alpha * c2 + om * bh2;
    }
    float* gg = grid_grad + (size_t)id * F;
    // this lane's non-zero texels straight to memory: one float2 + one float red each
    auto texel_reds = [&]() {
#pragma unroll
        for (int k = 0; k < NX; ++k)  // a zero corner weight (clamped or on-grid uv) adds nothing
            if (wk[k] != 0.0f)
                red3(gg + tbase + cell_offset<CELL>(3 * k, N), tg[3 * k], tg[3 * k + 1], tg[3 * k + 2]);
    };
    if (__popc(act) <= rc.direct_lanes) {
        // few active lanes: each adds its own terms with vector reds -- ~20 instructions for the warp
        // instead of two ~35-instruction warp reductions (12 % of warp-entries have one active lane)
        if (on) {
            float* a = accum + (size_t)id * kAccumStride;  // 48-B records: 16-B aligned
            red4(a, red[0], red[1], red[2], red[3]);
            if (NS == 10) {
                red4(a + 4, red[4], red[5], red[6], red[7]);
                atomicAdd(reinterpret_cast<float2*>(a + 8), make_float2(red[8], red[9]));
            } else {
                atomicAdd(reinterpret_cast<float2*>(a + 4), make_float2(red[4], red[5]));
                atomicAdd(a + 6, red[6]);
            }
            texel_reds();
        }
        return;
    }
    {  // screen-space sums: lane l owns value l >> 1
        float sv[NS];
#pragma unroll
        for (int i = 0; i < NS; ++i) sv[i] = red[i];
        const float r2 = smem_reduce<NS>(sv, wscratch, lane);
        if ((lane & 1) == 0 && (lane >> 1) < NS) red_add(accum + (size_t)id * kAccumStride + (lane >> 1), r2);
    }
    if (CELL == kCellOne && NT != 1 && N > 1) {
        // one texel per lane, and it is one of the four grid corners (by the signs of u, v): one warp
        // reduction over the 4 corners x 3 channels instead of up to 32 reds on at most 4 addresses
        const int q = on ? ((u > 0.0f) ? 2 : 0) + ((v > 0.0f) ? 1 : 0) : -1;
        float tq[12];
#pragma unroll
        for (int i = 0; i < 12; ++i) tq[i] = (q == i / 3) ? tg[i % 3] : 0.0f;
        const float r2 = smem_reduce<12>(tq, wscratch, lane);
        const int row = lane >> 1, qc = row / 3;
        if ((lane & 1) == 0 && row < 12)
            red_add(gg + 3 * (((qc >> 1) ? N - 1 : 0) * N + ((qc & 1) ? N - 1 : 0)) + row % 3, r2);
        return;
    }
    // texel gradients: one warp reduction when every active lane has the same base texel;
    // otherwise each lane adds its own texels -- cheaper than a reduction per distinct cell
    const int b0 = __shfl_sync(kFull, tbase, __ffs(act) - 1);
    if (__all_sync(kFull, !on || tbase == b0)) {
        if (lane == 0) GB_DBG(4, 1);
        const float r2 = smem_reduce<3 * NX>(tg, wscratch, lane);
        if ((lane & 1) == 0 && (lane >> 1) < 3 * NX) red_add(gg + b0 + cell_offset<CELL>(lane >> 1, N), r2);
    } else if (on) {
        if (lane == 0) GB_DBG(5, 1);
        texel_reds();
    }
}

// One backward entry for the calling warp: evaluate, pick the warp's texel footprint class, then
// bwd_shade (raster.hpp:324-363).
template <int MODE, int NT>
__device__ __forceinline__ void bwd_entry(const ScreenHeader& h, const float* __restrict__ t, int id, int rank,
                                          int last, int x, int y, float& T, float g0, float g1, float g2,
                                          float& bh0, float& bh1, float& bh2, const RasterConst& rc, int N,
                                          int lane, float* wscratch, float* __restrict__ accum,
                                          float* __restrict__ grid_grad) {
    const float sigma = rc.sigma;
    bool on = rank <= last;
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
            G = gauss_weight(u, v);
            araw = __fmul_rn(h.h1.z, G);
            alpha = fminf(araw, kMaxAlphaF);
            on = !(alpha < rc.alpha_skip);
        } else {
            on = false;
        }
    }
    const unsigned act = __ballot_sync(kFull, on);
    if (act == 0) return;
    if (lane == 0) {
        GB_DBG(2, 1);
        GB_DBG(3, __popc(act));
        GB_DBG(6, (act & 0x0F0F0F0Fu) && (act & 0xF0F0F0F0u));  // both 4x4 halves active
        GB_DBG(7, (act & 0x0000FFFFu) && (act & 0xFFFF0000u));  // both 8x2 halves active
    }
#define GB_SHADE(CELL)                                                                                          \
    bwd_shade<MODE, NT, CELL>(t, id, on, act, u, v, G, alpha, araw, pt, T, g0, g1, g2, bh0, bh1, bh2, rc, N, \
                              lane, wscratch, accum, grid_grad)
    if (N == 1) {
        GB_SHADE(kCellOne);
        return;
    }
    const bool au = __any_sync(kFull, on && u > -sigma && u < sigma);
    const bool av = __any_sync(kFull, on && v > -sigma && v < sigma);
    if (au && av)
        GB_SHADE(kCellFull);
    else if (au)
        GB_SHADE(kCellU);
    else if (av)
        GB_SHADE(kCellV);
    else
        GB_SHADE(kCellOne);
#undef GB_SHADE
}

template <int MODE, int NT>
__global__ void __launch_bounds__(288, 4) k_backward(const uint2* __restrict__ ranges, const int32_t* __restrict__ values,
                                                  const ScreenHeader* __restrict__ hdr, const float* __restrict__ tex,
                                                  const CamConst cc, const RasterConst rc, int n_rt, int B,
                                                  const float* __restrict__ in_trans,
                                                  const int32_t* __restrict__ in_last,
                                                  const float* __restrict__ image_grad, float* __restrict__ accum,
                                                  float* __restrict__ grid_grad) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) Pipe pipe;
    __shared__ int s_maxlast;
    const int N = tex_n<NT>(n_rt);
    const int F = 3 * N * N;
    const int ts = rc.tile_size;
    const int consumers = (ts * ts + 31) >> 5;
    const int tile = blockIdx.x;
    const int tx = tile % rc.tiles_x, ty = tile / rc.tiles_x;
    int lx, ly;
    tile_pixel(threadIdx.x, ts, lx, ly);
    const int x = tx * ts + lx, y = ty * ts + ly;
    const bool inside = (int)threadIdx.x < ts * ts && x < cc.width && y < cc.height;
    const uint2 range = ranges[tile];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;

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
    if (threadIdx.x == 0) s_maxlast = -1;
    pipe_init(pipe, consumers, (F & 3) == 0);
    __syncthreads();
    const int wmax = __reduce_max_sync(kFull, last);
    if (lane == 0 && wmax >= 0) atomicMax(&s_maxlast, wmax);
    __syncthreads();
    const int count = s_maxlast + 1;  // entries [0, count) are walked back to front
    const int nbatch = (count + B - 1) / B;
    // batch r covers ranks [max(0, count - (r+1) B), count - r B)

    if (warp == consumers) {  // producer warp
        produce(pipe, values, hdr, tex, range.x, nbatch, B, N, smem, [&](int r, int& first, int& cnt) {
            first = max(0, count - (r + 1) * B);
            cnt = count - r * B - first;
        });
        return;
    }

    const float bx0 = (float)__reduce_min_sync(kFull, x), bx1 = (float)__reduce_max_sync(kFull, x);
    const float by0 = (float)__reduce_min_sync(kFull, y), by1 = (float)__reduce_max_sync(kFull, y);
    const int wlast = wmax;  // this warp never needs ranks above its own max
    // per-warp reduction scratch after the staging ring
    float* wscratch = reinterpret_cast<float*>(smem + kStages * stage_bytes(B, N)) + warp * kRedRows * kRedStride;
    float bh0 = cc.bg[0], bh1 = cc.bg[1], bh2 = cc.bg[2];

    for (int r = 0; r < nbatch; ++r) {
        const int s = r % kStages;
        const int bstart = max(0, count - (r + 1) * B);
        const int nb = count - r * B - bstart;
        mbar_wait(&pipe.full[s], (r / kStages) & 1);
        const Stage st = stage_at(smem, s, B, N);
        const int jmax = min(nb - 1, wlast - bstart);
        for (int c0 = jmax & ~31; c0 >= 0; c0 -= 32) {
          // one ballot per 32 entries: in rank range for this warp and alpha-box meets its block
          unsigned mask = __ballot_sync(kFull, c0 + lane <= jmax &&
                                                   !box_miss(st.hdr[c0 + lane].h3, bx0, bx1, by0, by1));
          if (lane == 0) GB_DBG(1, __popc(mask));
          while (mask) {
            const int bit = 31 - __clz(mask);
            mask &= ~(1u << bit);
            const int j = c0 + bit;
            const int rank = bstart + j;
            bwd_entry<MODE, NT>(st.hdr[j], st.tex + (size_t)j * F, st.id[j], rank, last, x, y, T, g0, g1, g2, bh0,
                                bh1, bh2, rc, N, lane, wscratch, accum, grid_grad);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&pipe.empty[s]);
    }
}

// ---------------------------------------------------------------------------
// Direct variants (no shared-memory staging): each warp walks the tile list on
// its own, reading ids, headers and texels through L1 (__ldg).  No producer,
// no CTA-level synchronisation; warps finish independently.  The walks are
// device functions shared by the forward, the backward and the fused
// forward + loss + backward kernel, so all three run the same arithmetic.
// ---------------------------------------------------------------------------
struct WarpPixel {
    int x, y;
    bool inside;
    float bx0, bx1, by0, by1;  // the warp's pixel rectangle
};

__device__ __forceinline__ WarpPixel warp_pixel(const RasterConst& rc, const CamConst& cc, int tile) {
    WarpPixel w;
    const int ts = rc.tile_size;
    const int tx = tile % rc.tiles_x, ty = tile / rc.tiles_x;
    int lx, ly;
    tile_pixel(threadIdx.x, ts, lx, ly);
    w.x = tx * ts + lx;
    w.y = ty * ts + ly;
    w.inside = (int)threadIdx.x < ts * ts && w.x < cc.width && w.y < cc.height;
    w.bx0 = (float)__reduce_min_sync(kFull, w.x);
    w.bx1 = (float)__reduce_max_sync(kFull, w.x);
    w.by0 = (float)__reduce_min_sync(kFull, w.y);
    w.by1 = (float)__reduce_max_sync(kFull, w.y);
    return w;
}

// one lane's test of list entry `idl` against its warp's rectangle: exact alpha-skip ellipse (K1) or,
// with a null cull array, the alpha-box
__device__ __forceinline__ bool entry_meets_warp(const ScreenHeader* __restrict__ hdr, const CullRec* __restrict__ cull,
                                                 int idl, const WarpPixel& w) {
    return cull ? ellipse_meets_rect(__ldg(&cull[idl].a), __ldg(&cull[idl].b), w.bx0 - 0.05f, w.bx1 + 0.05f,
                                     w.by0 - 0.05f, w.by1 + 0.05f)
                : !box_miss(__ldg(&hdr[idl].h3), w.bx0, w.bx1, w.by0, w.by1);
}

// The warp rectangle of the lanes still in play (the forward's pixels not yet past early termination):
// entries that meet only the other pixels change nothing.
__device__ __forceinline__ WarpPixel live_rect(const WarpPixel& wp, bool live) {
    WarpPixel r = wp;
    r.bx0 = (float)__reduce_min_sync(kFull, live ? wp.x : INT_MAX);
    r.bx1 = (float)__reduce_max_sync(kFull, live ? wp.x : INT_MIN);
    r.by0 = (float)__reduce_min_sync(kFull, live ? wp.y : INT_MAX);
    r.by1 = (float)__reduce_max_sync(kFull, live ? wp.y : INT_MIN);
    return r;
}

// render_forward's per-pixel loop (raster.hpp:237-250) for the calling warp's pixels
template <int MODE, int NT>
__device__ __forceinline__ void fwd_walk(const uint2 range, const int32_t* __restrict__ values,
                                         const ScreenHeader* __restrict__ hdr, const CullRec* __restrict__ cull,
                                         const float* __restrict__ tex, const RasterConst& rc, int N,
                                         const WarpPixel& wp, float& T, float& acc0, float& acc1, float& acc2,
                                         int& last) {
    const int F = 3 * N * N;
    const int lane = threadIdx.x & 31;
    const int total = (int)(range.y - range.x);
    const int x = wp.x, y = wp.y;
    T = 1.0f;
    acc0 = acc1 = acc2 = 0.0f;
    last = -1;
    bool done = !wp.inside;
    const float early = rc.early_stop > 0.0f ? rc.early_stop : -1.0f;  // T >= 0: a disabled stop never fires
    for (int c0 = 0; c0 < total && !__all_sync(kFull, done); c0 += 32) {
        const WarpPixel lr = live_rect(wp, !done);
        int idl = -1;
        bool pass = false;
        if (c0 + lane < total) {
            idl = __ldg(&values[range.x + c0 + lane]);
            pass = entry_meets_warp(hdr, cull, idl, lr);
        }
        unsigned mask = __ballot_sync(kFull, pass);
        while (mask) {
            const int bit = __ffs(mask) - 1;
            mask &= mask - 1;
            const int id = __shfl_sync(kFull, idl, bit);
            // every lane evaluates (the warp runs the instructions anyway); finished pixels just do not
            // composite -- no branch around the evaluation
            float u, v;
            ScreenHeader h;
            h.h0 = __ldg(&hdr[id].h0);
            h.h1 = __ldg(&hdr[id].h1);
            h.h2 = __ldg(&hdr[id].h2);
            bool hit;
            if (MODE == GB_MODE_ORTHO) {
                hit = eval_uv_ortho(h, x, y, u, v);
            } else {
                PinholeTerms pt;
                hit = eval_uv_pinhole(h, x, y, u, v, pt);
            }
            const float G = gauss_weight(u, v);
            const float alpha = fminf(__fmul_rn(h.h1.z, G), kMaxAlphaF);  // raster.hpp:241
            const bool comp = !done && hit && !(alpha < rc.alpha_skip);     // raster.hpp:242
            // texel footprint class of the warp (see bwd_shade): clamped axes read one texel row
            const float sigma = rc.sigma;
            const bool au = N > 1 && __any_sync(kFull, comp && u > -sigma && u < sigma);
            const bool av = N > 1 && __any_sync(kFull, comp && v > -sigma && v < sigma);
            if (comp) {
                const float* t = tex + (size_t)id * F;
                float c0_, c1_, c2_;
                if (au && av) {
                    Bilin b;
                    bilin_setup(u, v, N, rc, b);
                    const float* p00 = t + b.o00;
                    const float* p10 = p00 + 3 * N;
                    c0_ = __ldg(p00) * b.w00 + __ldg(p10) * b.w10 + __ldg(p00 + 3) * b.w01 + __ldg(p10 + 3) * b.w11;
                    c1_ = __ldg(p00 + 1) * b.w00 + __ldg(p10 + 1) * b.w10 + __ldg(p00 + 4) * b.w01 +
                          __ldg(p10 + 4) * b.w11;
                    c2_ = __ldg(p00 + 2) * b.w00 + __ldg(p10 + 2) * b.w10 + __ldg(p00 + 5) * b.w01 +
                          __ldg(p10 + 5) * b.w11;
                } else if (au || av) {  // the four-corner blend with two zero weights
                    // (separate uniform branches: each keeps its index arithmetic free of selects)
                    const float* pa;
                    const float* pb;
                    float f;
                    if (au) {
                        float sx = __fmaf_rn(u, rc.tex_scale, rc.tex_offset);
                        sx = fminf(fmaxf(sx, 0.0f), (float)(N - 1));
                        const int i0 = min((int)floorf(sx), N - 2);
                        f = __fsub_rn(sx, (float)i0);
                        pa = t + (i0 * N + (v > 0.0f ? N - 1 : 0)) * 3;
                        pb = pa + 3 * N;
                    } else {
                        float sx = __fmaf_rn(v, rc.tex_scale, rc.tex_offset);
                        sx = fminf(fmaxf(sx, 0.0f), (float)(N - 1));
                        const int i0 = min((int)floorf(sx), N - 2);
                        f = __fsub_rn(sx, (float)i0);
                        pa = t + ((u > 0.0f ? N - 1 : 0) * N + i0) * 3;
                        pb = pa + 3;
                    }
                    const float gf = 1.0f - f;
                    c0_ = fmaf(__ldg(pb), f, __ldg(pa) * gf);
                    c1_ = fmaf(__ldg(pb + 1), f, __ldg(pa + 1) * gf);
                    c2_ = fmaf(__ldg(pb + 2), f, __ldg(pa + 2) * gf);
                } else {  // one texel (and n = 1)
                    const float* p = t + (N > 1 ? ((u > 0.0f ? N - 1 : 0) * N + (v > 0.0f ? N - 1 : 0)) * 3 : 0);
                    c0_ = __ldg(p);
                    c1_ = __ldg(p + 1);
                    c2_ = __ldg(p + 2);
                }
                const float w = alpha * T;  // raster.hpp:244-249
                acc0 = fmaf(c0_, w, acc0);
                acc1 = fmaf(c1_, w, acc1);
                acc2 = fmaf(c2_, w, acc2);
                T = __fmul_rn(T, __fsub_rn(1.0f, alpha));
                last = c0 + bit;
                if (T < early) done = true;  // raster.hpp:250
            }
            if (__all_sync(kFull, done)) break;
        }
    }
}

// render_backward's per-pixel loop (raster.hpp:313-364) for the calling warp's pixels
template <int MODE, int NT>
__device__ __forceinline__ void bwd_walk(const uint2 range, const int32_t* __restrict__ values,
                                         const ScreenHeader* __restrict__ hdr, const CullRec* __restrict__ cull,
                                         const float* __restrict__ tex, const CamConst& cc, const RasterConst& rc,
                                         int N, const WarpPixel& wp, int last, float T, float g0, float g1, float g2,
                                         float* wscratch, float* __restrict__ accum, float* __restrict__ grid_grad) {
    const int F = 3 * N * N;
    const int lane = threadIdx.x & 31;
    if (g0 == 0.0f && g1 == 0.0f && g2 == 0.0f) last = -1;  // raster.hpp:315-317
    float bh0 = cc.bg[0], bh1 = cc.bg[1], bh2 = cc.bg[2];
    const int wlast = __reduce_max_sync(kFull, last);
    for (int c0 = wlast & ~31; c0 >= 0; c0 -= 32) {
        // (a live rectangle here -- lanes with last >= c0 -- measured 1 % slower: few entries drop out)
        const WarpPixel& lr = wp;
        int idl = -1;
        bool pass = false;
        if (c0 + lane <= wlast) {
            idl = __ldg(&values[range.x + c0 + lane]);
            pass = entry_meets_warp(hdr, cull, idl, lr);
        }
        unsigned mask = __ballot_sync(kFull, pass);
        if (lane == 0) GB_DBG(1, __popc(mask));
        while (mask) {
            const int bit = 31 - __clz(mask);
            mask &= ~(1u << bit);
            const int id = __shfl_sync(kFull, idl, bit);
            ScreenHeader h;
            h.h0 = __ldg(&hdr[id].h0);
            h.h1 = __ldg(&hdr[id].h1);
            h.h2 = __ldg(&hdr[id].h2);
            bwd_entry<MODE, NT>(h, tex + (size_t)id * F, id, c0 + bit, last, wp.x, wp.y, T, g0, g1, g2, bh0, bh1,
                                bh2, rc, N, lane, wscratch, accum, grid_grad);
        }
    }
}

template <int MODE, int NT>
__global__ void __launch_bounds__(256) k_forward_direct(const uint2* __restrict__ ranges,
                                                        const int32_t* __restrict__ values,
                                                        const ScreenHeader* __restrict__ hdr,
                                                        const CullRec* __restrict__ cull, const float* __restrict__ tex,
                                                        const CamConst cc, const RasterConst rc, int n_rt,
                                                        float* __restrict__ out_color, float* __restrict__ out_trans,
                                                        int32_t* __restrict__ out_last) {
    const WarpPixel wp = warp_pixel(rc, cc, blockIdx.x);
    float T, a0, a1, a2;
    int last;
    fwd_walk<MODE, NT>(ranges[blockIdx.x], values, hdr, cull, tex, rc, tex_n<NT>(n_rt), wp, T, a0, a1, a2, last);
    if (wp.inside) {  // raster.hpp:253-254
        const size_t p = (size_t)wp.y * cc.width + wp.x;
        out_color[p * 3 + 0] = fmaf(T, cc.bg[0], a0);
        out_color[p * 3 + 1] = fmaf(T, cc.bg[1], a1);
        out_color[p * 3 + 2] = fmaf(T, cc.bg[2], a2);
        out_trans[p] = T;
        out_last[p] = last;
    }
}

// render_forward with the photometric loss (KIND 0 = L1, 1 = MSE; K6) in its epilogue: the pixel's
// colour turns into the loss cotangent in registers, so the image is written only when asked for and
// no separate loss pass runs.  T and the last rank are always written (the backward rewinds from them).
template <int MODE, int NT, int KIND>
__global__ void __launch_bounds__(256) k_forward_loss(const uint2* __restrict__ ranges,
                                                      const int32_t* __restrict__ values,
                                                      const ScreenHeader* __restrict__ hdr,
                                                      const CullRec* __restrict__ cull, const float* __restrict__ tex,
                                                      const CamConst cc, const RasterConst rc, int n_rt,
                                                      const float* __restrict__ target, float scale,
                                                      float* __restrict__ out_color, float* __restrict__ out_trans,
                                                      int32_t* __restrict__ out_last, float* __restrict__ out_grad,
                                                      float* __restrict__ loss) {
    const WarpPixel wp = warp_pixel(rc, cc, blockIdx.x);
    float T, a0, a1, a2;
    int last;
    fwd_walk<MODE, NT>(ranges[blockIdx.x], values, hdr, cull, tex, rc, tex_n<NT>(n_rt), wp, T, a0, a1, a2, last);
    float l = 0.0f;
    if (wp.inside) {
        const size_t p = (size_t)wp.y * cc.width + wp.x;
        const float c[3] = {fmaf(T, cc.bg[0], a0), fmaf(T, cc.bg[1], a1), fmaf(T, cc.bg[2], a2)};
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {  // K6 (gb_misc.cu k_loss), per pixel
            const float d = c[ch] - target[p * 3 + ch];
            float g;
            if (KIND == 0) {
                l += fabsf(d);
                g = scale * (float)((d > 0.0f) - (d < 0.0f));
            } else {
                l = fmaf(d, d, l);
                g = 2.0f * scale * d;
            }
            out_grad[p * 3 + ch] = g;
            if (out_color) out_color[p * 3 + ch] = c[ch];
        }
        out_trans[p] = T;
        out_last[p] = last;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(kFull, l, o);
    if ((threadIdx.x & 31) == 0 && loss && l != 0.0f) atomicAdd(loss, l * scale);
}

// <= 48 registers: 5 CTAs (40 warps) per SM -- with 32 B of spills, measured 1.3 % faster than 64
// registers at 4 CTAs (6 CTAs at 40 registers: no gain)
#ifndef GB_K4_MINB
#define GB_K4_MINB 5
#endif
template <int MODE, int NT>
__global__ void __launch_bounds__(256, GB_K4_MINB) k_backward_direct(const uint2* __restrict__ ranges,
                                                         const int32_t* __restrict__ values,
                                                         const ScreenHeader* __restrict__ hdr,
                                                         const CullRec* __restrict__ cull, const float* __restrict__ tex,
                                                         const CamConst cc, const RasterConst rc, int n_rt,
                                                         const float* __restrict__ in_trans,
                                                         const int32_t* __restrict__ in_last,
                                                         const float* __restrict__ image_grad,
                                                         float* __restrict__ accum, float* __restrict__ grid_grad) {
    extern __shared__ __align__(16) float red_scratch[];
    const WarpPixel wp = warp_pixel(rc, cc, blockIdx.x);
    int last = -1;
    float T = 1.0f, g0 = 0.0f, g1 = 0.0f, g2 = 0.0f;
    if (wp.inside) {  // raster.hpp:313-322
        const size_t p = (size_t)wp.y * cc.width + wp.x;
        last = in_last[p];
        g0 = image_grad[p * 3 + 0];
        g1 = image_grad[p * 3 + 1];
        g2 = image_grad[p * 3 + 2];
        T = in_trans[p];
    }
    bwd_walk<MODE, NT>(ranges[blockIdx.x], values, hdr, cull, tex, cc, rc, tex_n<NT>(n_rt), wp, last, T, g0, g1, g2,
                       red_scratch + (threadIdx.x >> 5) * kRedRows * kRedStride, accum, grid_grad);
}

// render_forward + the photometric loss (KIND 0 = L1, 1 = MSE; K6) + render_backward of one view in one
// kernel.  Every warp composites its pixels, turns them into the loss cotangent in registers and walks the
// same entries back to front while their headers and texels are still in L1/L2; colour, transmittance,
// last rank and the cotangent are stored only when asked for.
template <int MODE, int NT, int KIND>
__global__ void __launch_bounds__(256) k_fused_direct(const uint2* __restrict__ ranges,
                                                      const int32_t* __restrict__ values,
                                                      const ScreenHeader* __restrict__ hdr,
                                                      const CullRec* __restrict__ cull, const float* __restrict__ tex,
                                                      const CamConst cc, const RasterConst rc, int n_rt,
                                                      const float* __restrict__ target, float scale,
                                                      float* __restrict__ out_color, float* __restrict__ out_trans,
                                                      int32_t* __restrict__ out_last, float* __restrict__ out_grad,
                                                      float* __restrict__ loss, float* __restrict__ accum,
                                                      float* __restrict__ grid_grad) {
    extern __shared__ __align__(16) float red_scratch[];
    const int N = tex_n<NT>(n_rt);
    const WarpPixel wp = warp_pixel(rc, cc, blockIdx.x);
    const uint2 range = ranges[blockIdx.x];
    float T, a0, a1, a2;
    int last;
    fwd_walk<MODE, NT>(range, values, hdr, cull, tex, rc, N, wp, T, a0, a1, a2, last);
    float g0 = 0.0f, g1 = 0.0f, g2 = 0.0f, l = 0.0f;
    if (wp.inside) {
        const size_t p = (size_t)wp.y * cc.width + wp.x;
        const float c[3] = {fmaf(T, cc.bg[0], a0), fmaf(T, cc.bg[1], a1), fmaf(T, cc.bg[2], a2)};
        float g[3];
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {  // K6 (gb_misc.cu k_loss), per pixel
            const float d = c[ch] - target[p * 3 + ch];
            if (KIND == 0) {
                l += fabsf(d);
                g[ch] = scale * (float)((d > 0.0f) - (d < 0.0f));
            } else {
                l = fmaf(d, d, l);
                g[ch] = 2.0f * scale * d;
            }
        }
        g0 = g[0];
        g1 = g[1];
        g2 = g[2];
        if (out_color) {
            out_color[p * 3 + 0] = c[0];
            out_color[p * 3 + 1] = c[1];
            out_color[p * 3 + 2] = c[2];
            out_trans[p] = T;
            out_last[p] = last;
        }
        if (out_grad) {
            out_grad[p * 3 + 0] = g0;
            out_grad[p * 3 + 1] = g1;
            out_grad[p * 3 + 2] = g2;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(kFull, l, o);
    if ((threadIdx.x & 31) == 0 && loss && l != 0.0f) atomicAdd(loss, l * scale);
    bwd_walk<MODE, NT>(range, values, hdr, cull, tex, cc, rc, N, wp, last, T, g0, g1, g2,
                       red_scratch + (threadIdx.x >> 5) * kRedRows * kRedStride, accum, grid_grad);
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
static int tune_env(const char* name, int dflt) {  // development knob: GB_TUNE_* overrides
    const char* v = getenv(name);
    return v ? atoi(v) : dflt;
}

// Compositor variant: 1 = one warp per entry reading through L1 (default),
// 0 = sub-warp groups (gb_composite.cu; tile sizes 8 and 16), 2 = one warp per
// entry with TMA bulk-copy staging.  GB_COMPOSITOR=direct|grp|staged selects
// one explicitly (A/B measurements and parity tests); GB_COMPOSITOR_BWD
// overrides it for the backward only.
static int compositor_variant(bool backward = false) {
    const char* v = backward && getenv("GB_COMPOSITOR_BWD") ? getenv("GB_COMPOSITOR_BWD") : getenv("GB_COMPOSITOR");
    if (!v) return 1;
    if (!strcmp(v, "grp")) return 0;
    if (!strcmp(v, "staged")) return 2;
    return 1;
}

int pick_batch(int N, int stage_budget = 13312) {
    // kStages staging buffers within ~52 KB (K3) / ~37 KB + reduction scratch (K4) keep 4 CTAs per SM
    const size_t per = stage_bytes(1, N);
    int B = (int)(stage_budget / per);
    if (B > 64) B = 64;
    if (B < 2) B = 2;
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

template <int MODE, int NT>
static cudaError_t fwdd_t(int tiles, int threads, cudaStream_t st, const uint2* ranges, const int32_t* values,
                          const ScreenHeader* hdr, const CullRec* cull, const float* tex, const CamConst& cc, const RasterConst& rc, int n,
                          float* color, float* trans, int32_t* last) {
    if (tune_env("GB_CULL_BOX", 0)) cull = nullptr;  // A/B: alpha-box test instead of the exact ellipse
    k_forward_direct<MODE, NT><<<tiles, threads, 0, st>>>(ranges, values, hdr, cull, tex, cc, rc, n, color, trans, last);
    return cudaGetLastError();
}

template <int MODE, int NT>
static cudaError_t bwdd_t(int tiles, int threads, cudaStream_t st, const uint2* ranges, const int32_t* values,
                          const ScreenHeader* hdr, const CullRec* cull, const float* tex, const CamConst& cc, const RasterConst& rc, int n,
                          const float* trans, const int32_t* last, const float* image_grad, float* accum,
                          float* grid_grad) {
    const size_t smem = (size_t)(threads / 32) * kRedRows * kRedStride * 4;
    if (tune_env("GB_CULL_BOX", 0)) cull = nullptr;
    k_backward_direct<MODE, NT><<<tiles, threads, smem, st>>>(ranges, values, hdr, cull, tex, cc, rc, n, trans, last,
                                                               image_grad, accum, grid_grad);
    return cudaGetLastError();
}

cudaError_t launch_forward(int mode, int n, int tiles, int ts, const uint2* ranges, const int32_t* values,
                           const ScreenHeader* hdr, const CullRec* cull, const float* tex, const CamConst& cc, const RasterConst& rc,
                           float* color, float* trans, int32_t* last, cudaStream_t st) {
    if (tiles == 0) return cudaSuccess;
    const int variant = compositor_variant();
    if (variant == 0 && grp_supported(ts))
        return launch_forward_grp(mode, n, tiles, ts, ranges, values, hdr, cull, tex, cc, rc, color, trans, last, st);
    if (variant != 2) {
        const int threads = ((ts * ts + 31) / 32) * 32;
        if (mode == GB_MODE_ORTHO) {
            GB_DISPATCH_N(fwdd_t, GB_MODE_ORTHO, tiles, threads, st, ranges, values, hdr, cull, tex, cc, rc, n, color,
                          trans, last)
        } else {
            GB_DISPATCH_N(fwdd_t, GB_MODE_PINHOLE, tiles, threads, st, ranges, values, hdr, cull, tex, cc, rc, n, color,
                          trans, last)
        }
    }
    const int threads = ((ts * ts + 31) / 32) * 32 + 32;  // + the producer warp
    const int B = pick_batch(n, tune_env("GB_TUNE_FWD_BUDGET", 13312));
    const size_t smem = kStages * stage_bytes(B, n);
    if (mode == GB_MODE_ORTHO) {
        GB_DISPATCH_N(fwd_t, GB_MODE_ORTHO, tiles, threads, smem, st, ranges, values, hdr, tex, cc, rc, n, B, color,
                      trans, last)
    } else {
        GB_DISPATCH_N(fwd_t, GB_MODE_PINHOLE, tiles, threads, smem, st, ranges, values, hdr, tex, cc, rc, n, B,
                      color, trans, last)
    }
}

cudaError_t launch_backward(int mode, int n, int tiles, int ts, const uint2* ranges, const int32_t* values,
                            const ScreenHeader* hdr, const CullRec* cull, const float* tex, const CamConst& cc, const RasterConst& rc,
                            const float* trans, const int32_t* last, const float* image_grad, float* accum,
                            float* grid_grad, cudaStream_t st) {
    if (tiles == 0) return cudaSuccess;
    const int variant = compositor_variant(true);
    if (variant == 0 && grp_supported(ts))
        return launch_backward_grp(mode, n, tiles, ts, ranges, values, hdr, cull, tex, cc, rc, trans, last, image_grad,
                                   accum, grid_grad, st);
    if (variant != 2) {
        const int threads = ((ts * ts + 31) / 32) * 32;
        if (mode == GB_MODE_ORTHO) {
            GB_DISPATCH_N(bwdd_t, GB_MODE_ORTHO, tiles, threads, st, ranges, values, hdr, cull, tex, cc, rc, n, trans, last,
                          image_grad, accum, grid_grad)
        } else {
            GB_DISPATCH_N(bwdd_t, GB_MODE_PINHOLE, tiles, threads, st, ranges, values, hdr, cull, tex, cc, rc, n, trans,
                          last, image_grad, accum, grid_grad)
        }
    }
    const int threads = ((ts * ts + 31) / 32) * 32 + 32;  // + the producer warp
    const int B = pick_batch(n, tune_env("GB_TUNE_BWD_BUDGET", 9216));
    const size_t smem = kStages * stage_bytes(B, n) + (size_t)(threads / 32 - 1) * kRedRows * kRedStride * 4;
    if (mode == GB_MODE_ORTHO) {
        GB_DISPATCH_N(bwd_t, GB_MODE_ORTHO, tiles, threads, smem, st, ranges, values, hdr, tex, cc, rc, n, B, trans,
                      last, image_grad, accum, grid_grad)
    } else {
        GB_DISPATCH_N(bwd_t, GB_MODE_PINHOLE, tiles, threads, smem, st, ranges, values, hdr, tex, cc, rc, n, B,
                      trans, last, image_grad, accum, grid_grad)
    }
}

template <int MODE, int NT>
static cudaError_t fused_t(int tiles, int threads, cudaStream_t st, const uint2* ranges, const int32_t* values,
                           const ScreenHeader* hdr, const CullRec* cull, const float* tex, const CamConst& cc,
                           const RasterConst& rc, int n, int kind, const float* target, float scale, float* color,
                           float* trans, int32_t* last, float* image_grad, float* loss, float* accum,
                           float* grid_grad) {
    const size_t smem = (size_t)(threads / 32) * kRedRows * kRedStride * 4;
    if (tune_env("GB_CULL_BOX", 0)) cull = nullptr;
    if (kind == 0)
        k_fused_direct<MODE, NT, 0><<<tiles, threads, smem, st>>>(ranges, values, hdr, cull, tex, cc, rc, n, target,
                                                                  scale, color, trans, last, image_grad, loss, accum,
                                                                  grid_grad);
    else
        k_fused_direct<MODE, NT, 1><<<tiles, threads, smem, st>>>(ranges, values, hdr, cull, tex, cc, rc, n, target,
                                                                  scale, color, trans, last, image_grad, loss, accum,
                                                                  grid_grad);
    return cudaGetLastError();
}

template <int MODE, int NT>
static cudaError_t fwdl_t(int tiles, int threads, cudaStream_t st, const uint2* ranges, const int32_t* values,
                          const ScreenHeader* hdr, const CullRec* cull, const float* tex, const CamConst& cc,
                          const RasterConst& rc, int n, int kind, const float* target, float scale, float* color,
                          float* trans, int32_t* last, float* image_grad, float* loss) {
    if (tune_env("GB_CULL_BOX", 0)) cull = nullptr;
    if (kind == 0)
        k_forward_loss<MODE, NT, 0><<<tiles, threads, 0, st>>>(ranges, values, hdr, cull, tex, cc, rc, n, target,
                                                               scale, color, trans, last, image_grad, loss);
    else
        k_forward_loss<MODE, NT, 1><<<tiles, threads, 0, st>>>(ranges, values, hdr, cull, tex, cc, rc, n, target,
                                                               scale, color, trans, last, image_grad, loss);
    return cudaGetLastError();
}

// K3 + K6 (direct compositor only): trans, last and image_grad are required, color optional
cudaError_t launch_forward_loss(int mode, int n, int tiles, int ts, const uint2* ranges, const int32_t* values,
                                const ScreenHeader* hdr, const CullRec* cull, const float* tex, const CamConst& cc,
                                const RasterConst& rc, int kind, const float* target, float scale, float* color,
                                float* trans, int32_t* last, float* image_grad, float* loss, cudaStream_t st) {
    if (tiles == 0) return cudaSuccess;
    const int threads = ((ts * ts + 31) / 32) * 32;
    if (mode == GB_MODE_ORTHO) {
        GB_DISPATCH_N(fwdl_t, GB_MODE_ORTHO, tiles, threads, st, ranges, values, hdr, cull, tex, cc, rc, n, kind,
                      target, scale, color, trans, last, image_grad, loss)
    } else {
        GB_DISPATCH_N(fwdl_t, GB_MODE_PINHOLE, tiles, threads, st, ranges, values, hdr, cull, tex, cc, rc, n, kind,
                      target, scale, color, trans, last, image_grad, loss)
    }
}

// the single-kernel forward + loss + backward (k_fused_direct) instead of K3+K6 then K4: measured slower
bool fused_single_kernel() { return tune_env("GB_FUSED_KERNEL", 0) != 0; }

// true when launch_fused runs (the direct compositors are selected); otherwise the caller composes
// launch_forward + launch_loss + launch_backward
bool fused_available() { return compositor_variant() == 1 && compositor_variant(true) == 1 && !getenv("GB_NO_FUSE"); }

cudaError_t launch_fused(int mode, int n, int tiles, int ts, const uint2* ranges, const int32_t* values,
                         const ScreenHeader* hdr, const CullRec* cull, const float* tex, const CamConst& cc,
                         const RasterConst& rc, int kind, const float* target, float scale, float* color, float* trans,
                         int32_t* last, float* image_grad, float* loss, float* accum, float* grid_grad,
                         cudaStream_t st) {
    if (tiles == 0) return cudaSuccess;
    const int threads = ((ts * ts + 31) / 32) * 32;
    if (mode == GB_MODE_ORTHO) {
        GB_DISPATCH_N(fused_t, GB_MODE_ORTHO, tiles, threads, st, ranges, values, hdr, cull, tex, cc, rc, n, kind,
                      target, scale, color, trans, last, image_grad, loss, accum, grid_grad)
    } else {
        GB_DISPATCH_N(fused_t, GB_MODE_PINHOLE, tiles, threads, st, ranges, values, hdr, cull, tex, cc, rc, n, kind,
                      target, scale, color, trans, last, image_grad, loss, accum, grid_grad)
    }
}

}  // namespace gb
