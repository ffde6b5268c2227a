// blend.cu -- stage (d) "Blending" with the GEMM-compatible
// exponent of GEMM-GS (Eq. 6-8; Alg. 2), and
// the CUDA-core direct form (Alg. 1) as an A/B baseline.
//
// k_blend_tc: persistent, warp-specialised tcgen05 kernel, 2 CTAs per SM.
//   warp 8 (producer + MMA issuer): per batch of NB = 32 Gaussians of a tile's
//     sorted list, lane j gathers Gaussian j (mean, conic, opacity, colour),
//     builds v_g (Eq. 6) scaled by log2(e) with log2(o) folded into
//     the constant term (reading R-10), splits it into TF32 hi + lo (reading
//     R-11) and writes the row [hi(6) | lo(6) | 0(4)] of M_g into shared memory;
//     one lane then issues 4 x tcgen05.mma.kind::tf32 (M=128 pixels, N=32,
//     K=8; 2 pixel halves x 2 K-steps) that multiply the constant pixel matrix
//     M_p (rows [v_p | v_p | 0], precomputed once per CTA, the
//     "offline" M_p of P:302) by M_g^T into TMEM, and commits to an mbarrier.
//   warps 0-7 (compositors, one pixel per thread): tcgen05.ld 32x32b.x32 gives
//     each thread its own pixel's 32 exponents m = log2(alpha); then alpha =
//     min(0.99, 2^m), alpha-skip below 1/255, T' = T(1-alpha), stop when
//     T' < 1e-4 (not composited), C += alpha T c (Eq. 1; readings R-1..R-4).
//     A warp skips a Gaussian with one vote when none of its 32 pixels keeps it.
//   A tile ends when its list is exhausted or all 256 pixels have terminated;
//   tiles come from an atomic work queue.
// Reference pixel p_c = tile centre (16 t_x + 7.5, 16 t_y + 7.5) (reading R-6),
// x_bar = x_c - x_p (Eq. 4; reading R-7).
#include <algorithm>

#include "gs_common.cuh"

namespace gs {

constexpr int NB = 32;        // Gaussians per batch (MMA N)
constexpr int STAGES = 4;     // smem / TMEM ring depth
constexpr int NCW = 8;        // compositor warps: 256 pixels
constexpr int TC_THREADS = (NCW + 1) * 32;
constexpr int TMEM_COLS = STAGES * 2 * NB;   // 256
static_assert(TMEM_COLS == 256, "TMEM allocation must be a power of two");

struct __align__(1024) SmemTC {
    uint8_t A[2][128 * 64];       // M_p halves: 128 rows x 16 tf32, interleaved core matrices
    uint8_t B[STAGES][NB * 64];   // M_g rows
    float4 rgb[STAGES][NB];
    int4 hdr[STAGES];             // {tile, seq, count, list offset}
    uint64_t full[STAGES];
    uint64_t empty[STAGES];
    uint32_t tmem_base;
    uint32_t warp_done_seq[NCW];
};

// byte offset of (row r, 16-byte K-chunk c) in a K-major no-swizzle operand
// with 4 K-chunks per row: core matrix = 8 rows x 16 B, LBO = 128, SBO = 512
__device__ __forceinline__ uint32_t op_off(int r, int c) { return (r >> 3) * 512 + c * 128 + (r & 7) * 16; }

// pixel of compositor thread p = 32*w + lane inside the 16x16 tile: warp w
// covers the 8x4 block at (8*(w%2), 4*(w/2)) (compact blocks maximise the
// warp-uniform skip).
__device__ __forceinline__ void pixel_of(int p, int &x, int &y) {
    const int w = p >> 5, l = p & 31;
    x = 8 * (w & 1) + (l & 7);
    y = 4 * (w >> 1) + (l >> 3);
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}

struct Rec {
    float2 m;     // projected mean
    float4 co;    // (A, B, C, opacity)
    float4 col;   // (r, g, b, 0)
};

__device__ __forceinline__ void gather(Rec &r, const float2 *__restrict__ xy, const float4 *__restrict__ conic_o,
                                       const float4 *__restrict__ rgb, uint32_t gi, bool ok) {
    if (ok) {
        r.m = __ldg(xy + gi);
        r.co = __ldg(conic_o + gi);
        r.col = __ldg(rgb + gi);
    } else {
        r.m = make_float2(0.f, 0.f);
        r.co = make_float4(0.f, 0.f, 0.f, 1.f);
        r.col = make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

template <bool DUMP, bool STATS>
__global__ void __launch_bounds__(TC_THREADS, 2)
    k_blend_tc(const float2 *__restrict__ xy, const float4 *__restrict__ conic_o, const float4 *__restrict__ rgb,
               const uint32_t *__restrict__ vals, const uint2 *__restrict__ ranges, int ntiles, int gx, int W,
               int H, float bg0, float bg1, float bg2, float *__restrict__ out_rgb, float *__restrict__ out_T,
               float *__restrict__ dump_m, uint32_t *tile_queue, unsigned long long *stat_eval,
               unsigned long long *stat_kept) {
    extern __shared__ uint8_t smem_raw[];
    SmemTC &sm = *reinterpret_cast<SmemTC *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // ---- one-time setup -------------------------------------------------
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; s++) {
            mbar_init(&sm.full[s], 33);          // 32 producer lanes + 1 MMA commit
            mbar_init(&sm.empty[s], NCW);        // one arrival per compositor warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp < NCW) {
        // M_p row for pixel p (Eq. 7): [xb^2, yb^2, xb*yb, xb, yb, 1] twice (hi/lo), then 0
        const int p = threadIdx.x;
        int x, y;
        pixel_of(p, x, y);
        const float xb = 7.5f - (float)x, yb = 7.5f - (float)y;
        const float v[6] = {xb * xb, yb * yb, xb * yb, xb, yb, 1.0f};   // exact in TF32
        uint32_t u[16];
#pragma unroll
        for (int k = 0; k < 6; k++) u[k] = u[6 + k] = __float_as_uint(v[k]);
        u[12] = u[13] = u[14] = u[15] = 0u;
        const int h = p >> 7, r = p & 127;
        const uint32_t base = smem_u32(&sm.A[h][0]);
#pragma unroll
        for (int c = 0; c < 4; c++) st_shared_v4(base + op_off(r, c), u[4 * c], u[4 * c + 1], u[4 * c + 2], u[4 * c + 3]);
        if (lane == 0) sm.warp_done_seq[warp] = 0;
        fence_proxy_async_smem();
    } else {
        tmem_alloc(&sm.tmem_base, TMEM_COLS);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;

    if (warp == NCW) {
        // =================== producer + MMA issuer ===================
        // Software pipeline over the flattened stream of (tile, batch):
        //   indices of batch k+1 and the records of batch k were requested one
        //   iteration earlier, and the first batch of the next tile is fetched
        //   in four steps spread over the current tile's iterations, so the
        //   compositors never wait for a full gather latency (~1 us).
        constexpr uint32_t IDESC = idesc_tf32(128, NB);
        const uint32_t a_base = smem_u32(&sm.A[0][0]);
        const uint32_t b_base = smem_u32(&sm.B[0][0]);
        uint32_t s = 0, ph = 0;
        unsigned long long n_eval = 0;
        // current tile
        int tile = 0;
        if (lane == 0) tile = (int)atomicAdd(tile_queue, 1u);
        tile = __shfl_sync(0xffffffffu, tile, 0);
        uint2 rg = tile < ntiles ? ranges[tile] : make_uint2(0u, 0u);
        uint32_t seq = 1;
        uint32_t b = rg.x;
        Rec cur;
        uint32_t inext;
        {
            const uint32_t i0 = (b + lane < rg.y) ? vals[b + lane] : 0u;
            inext = (b + NB + lane < rg.y) ? vals[b + NB + lane] : 0u;
            gather(cur, xy, conic_o, rgb, i0, b + lane < rg.y);
        }
        // next-tile head
        int hstate = 0, ntile = 0, ntile_l0 = 0;
        uint2 nrg = make_uint2(0u, 0u);
        uint32_t hidx0 = 0, hidx1 = 0;
        Rec h0;
        auto head_step = [&]() {
            switch (hstate) {
                case 0:
                    if (lane == 0) ntile_l0 = (int)atomicAdd(tile_queue, 1u);
                    break;
                case 1:
                    ntile = __shfl_sync(0xffffffffu, ntile_l0, 0);
                    nrg = ntile < ntiles ? ranges[ntile] : make_uint2(0u, 0u);
                    break;
                case 2:
                    hidx0 = (nrg.x + lane < nrg.y) ? vals[nrg.x + lane] : 0u;
                    hidx1 = (nrg.x + NB + lane < nrg.y) ? vals[nrg.x + NB + lane] : 0u;
                    break;
                case 3:
                    gather(h0, xy, conic_o, rgb, hidx0, nrg.x + lane < nrg.y);
                    break;
                default:
                    return;
            }
            hstate++;
        };
        for (;;) {
            if (tile >= ntiles) {
                mbar_wait(&sm.empty[s], ph ^ 1);
                if (lane == 0) sm.hdr[s] = make_int4(-1, 0, 0, 0);
                mbar_arrive(&sm.full[s]);
                if (lane == 0) mbar_arrive(&sm.full[s]);
                if (STATS && lane == 0) atomicAdd(stat_eval, n_eval);
                break;
            }
            head_step();
            bool end = b >= rg.y;
            if (!DUMP && !end) {
                const uint32_t dseq = lane < NCW ? *((volatile uint32_t *)&sm.warp_done_seq[lane]) : seq;
                end = __all_sync(0xffffffffu, dseq >= seq);   // every pixel of the tile terminated
            }
            if (end) {
                mbar_wait(&sm.empty[s], ph ^ 1);
                if (lane == 0) sm.hdr[s] = make_int4(tile, (int)seq, 0, 0);
                mbar_arrive(&sm.full[s]);
                if (lane == 0) mbar_arrive(&sm.full[s]);
                if (++s == STAGES) { s = 0; ph ^= 1; }
                while (hstate < 4) head_step();
                tile = ntile;
                rg = nrg;
                b = rg.x;
                seq++;
                cur = h0;
                inext = hidx1;
                hstate = 0;
                continue;
            }
            // prefetch: records of batch b+NB, indices of batch b+2NB
            Rec nx;
            gather(nx, xy, conic_o, rgb, inext, b + NB + lane < rg.y);
            const uint32_t inext2 = (b + 2 * NB + lane < rg.y) ? vals[b + 2 * NB + lane] : 0u;
            const uint32_t cnt = min((uint32_t)NB, rg.y - b);
            const float xc = (float)(GS_TILE * (tile % gx)) + 7.5f;
            const float yc = (float)(GS_TILE * (tile / gx)) + 7.5f;
            uint32_t u[16];
            if ((uint32_t)lane < cnt) {
                // Eq. (6): v_g with xh = x_g - x_c, yh = y_g - y_c, times log2(e); + log2(o)
                const float xh = cur.m.x - xc, yh = cur.m.y - yc;
                const float A = cur.co.x, B = cur.co.y, C = cur.co.z;
                float v[6];
                v[0] = -0.5f * A * LOG2E;
                v[1] = -0.5f * C * LOG2E;
                v[2] = -B * LOG2E;
                v[3] = -(A * xh + B * yh) * LOG2E;
                v[4] = -(C * yh + B * xh) * LOG2E;
                v[5] = -(0.5f * A * xh * xh + 0.5f * C * yh * yh + B * xh * yh) * LOG2E + lg2_approx(cur.co.w);
#pragma unroll
                for (int k = 0; k < 6; k++) {
                    const uint32_t hi = f32_to_tf32_rna(v[k]);
                    const uint32_t lo = f32_to_tf32_rna(v[k] - __uint_as_float(hi));
                    u[k] = hi;
                    u[6 + k] = lo;
                }
            } else {
                // padding column: exponent -1e30, never kept by any pixel
#pragma unroll
                for (int k = 0; k < 12; k++) u[k] = 0u;
                u[5] = __float_as_uint(-1e30f);
            }
            u[12] = u[13] = u[14] = u[15] = 0u;
            mbar_wait(&sm.empty[s], ph ^ 1);
            const uint32_t rb = b_base + s * (NB * 64);
#pragma unroll
            for (int c = 0; c < 4; c++)
                st_shared_v4(rb + op_off(lane, c), u[4 * c], u[4 * c + 1], u[4 * c + 2], u[4 * c + 3]);
            sm.rgb[s][lane] = cur.col;
            if (lane == 0) sm.hdr[s] = make_int4(tile, (int)seq, (int)cnt, (int)b);
            if (STATS && lane == 0) n_eval += (unsigned long long)cnt * GS_TILE_PIX;
            fence_proxy_async_smem();
            mbar_arrive(&sm.full[s]);
            __syncwarp();
            if (lane == 0) {
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < 2; kk++)
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        const uint64_t ad = umma_desc(a_base + h * (128 * 64) + kk * 256, 128, 512);
                        const uint64_t bd = umma_desc(b_base + s * (NB * 64) + kk * 256, 128, 512);
                        mma_tf32(tmem + s * (2 * NB) + h * NB, ad, bd, IDESC, kk);
                    }
                mma_commit(&sm.full[s]);
            }
            __syncwarp();
            if (++s == STAGES) { s = 0; ph ^= 1; }
            cur = nx;
            inext = inext2;
            b += NB;
        }
    } else {
        // =================== compositors ===================
        const int p = threadIdx.x;
        int x, y;
        pixel_of(p, x, y);
        const uint32_t t_lane = (uint32_t)(32 * (warp & 3)) << 16;
        const uint32_t t_half = (uint32_t)(warp >> 2) * NB;
        uint32_t s = 0, ph = 0;
        float T = 1.0f, C0 = 0.f, C1 = 0.f, C2 = 0.f;
        bool done = false, wdone = false;
        uint32_t n_kept = 0;
        for (;;) {
            mbar_wait(&sm.full[s], ph);
            tc_fence_after();
            const int4 hd = sm.hdr[s];
            if (hd.z == 0) {
                if (hd.x < 0) {
                    if (STATS) {
                        unsigned long long k = n_kept;
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
                        if (lane == 0) atomicAdd(stat_kept, k);
                    }
                    break;
                }
                if (!DUMP) {
                    const int px = GS_TILE * (hd.x % gx) + x, py = GS_TILE * (hd.x / gx) + y;
                    if (px < W && py < H) {
                        const size_t pix = (size_t)py * W + px, plane = (size_t)W * H;
                        out_rgb[pix] = C0 + T * bg0;
                        out_rgb[plane + pix] = C1 + T * bg1;
                        out_rgb[2 * plane + pix] = C2 + T * bg2;
                        out_T[pix] = T;
                    }
                }
                T = 1.0f; C0 = C1 = C2 = 0.f; done = false; wdone = false;
            } else if (!wdone) {
                float m[NB];
                tmem_ld32(tmem + t_lane + s * (2 * NB) + t_half, m);
                tmem_wait_ld();
                const int cnt = hd.z;
                if (DUMP) {
                    for (int j = 0; j < cnt; j++) dump_m[((size_t)hd.w + j) * GS_TILE_PIX + p] = m[j];
                } else {
                    // columns j >= cnt hold the padding exponent -1e30: no count checks needed
#pragma unroll
                    for (int j = 0; j < NB; j++) {
                        const float mj = m[j];
                        const bool live = (mj >= LOG2_ALPHA_MIN) && !done;
                        if (__any_sync(0xffffffffu, live)) {
                            const float4 c = sm.rgb[s][j];
                            const float a = fminf(ALPHA_MAX, ex2_approx(mj));
                            const float tT = T * (1.0f - a);
                            if (live) {
                                if (STATS) n_kept++;
                                if (tT < T_MIN) {
                                    done = true;
                                } else {
                                    const float wgt = a * T;
                                    C0 += wgt * c.x;
                                    C1 += wgt * c.y;
                                    C2 += wgt * c.z;
                                    T = tT;
                                }
                            }
                        }
                    }
                    if (__all_sync(0xffffffffu, done)) {
                        wdone = true;
                        if (lane == 0) *((volatile uint32_t *)&sm.warp_done_seq[warp]) = (uint32_t)hd.y;
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.empty[s]);
            if (++s == STAGES) { s = 0; ph ^= 1; }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == NCW) {
        tc_fence_after();
        tmem_dealloc(tmem, TMEM_COLS);
    }
}

void launch_blend_tc(const Workspace &ws, cudaStream_t st, const float2 *xy, const float4 *conic_o,
                     const float4 *rgb, const uint32_t *vals, const uint2 *ranges, int ntiles, int gx, int W,
                     int H, const float bg[3], float *out_rgb, float *out_T, float *dump_m, int num_sms,
                     bool stats) {
    const size_t smem = sizeof(SmemTC) + 1024;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_blend_tc<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_blend_tc<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_blend_tc<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr_set = true;
    }
    const int grid = std::max(1, std::min(2 * num_sms, ntiles));
    uint32_t *queue = &ws.counters->tile_queue;
    unsigned long long *se = &ws.counters->pairs_eval, *sk = &ws.counters->pairs_kept;
    if (dump_m)
        k_blend_tc<true, false><<<grid, TC_THREADS, smem, st>>>(xy, conic_o, rgb, vals, ranges, ntiles, gx, W, H,
                                                                 bg[0], bg[1], bg[2], out_rgb, out_T, dump_m, queue,
                                                                 se, sk);
    else if (stats)
        k_blend_tc<false, true><<<grid, TC_THREADS, smem, st>>>(xy, conic_o, rgb, vals, ranges, ntiles, gx, W, H,
                                                                 bg[0], bg[1], bg[2], out_rgb, out_T, dump_m, queue,
                                                                 se, sk);
    else
        k_blend_tc<false, false><<<grid, TC_THREADS, smem, st>>>(xy, conic_o, rgb, vals, ranges, ntiles, gx, W, H,
                                                                  bg[0], bg[1], bg[2], out_rgb, out_T, dump_m, queue,
                                                                  se, sk);
}

// ===========================================================================
// CUDA-core direct blend (Alg. 1 with Eq. 3 per pixel): one 256-thread CTA per
// tile, batches of 256 Gaussians staged in shared memory.
// ===========================================================================
__global__ void __launch_bounds__(256) k_blend_direct(const float2 *__restrict__ xy, const float4 *__restrict__ conic_o,
                                                      const float4 *__restrict__ rgb, const uint32_t *__restrict__ vals,
                                                      const uint2 *__restrict__ ranges, int gx, int W, int H,
                                                      float bg0, float bg1, float bg2, float *__restrict__ out_rgb,
                                                      float *__restrict__ out_T) {
    __shared__ float4 s_g[256];     // (x, y, A, B)
    __shared__ float2 s_g2[256];    // (C, log2 o)
    __shared__ float4 s_c[256];
    const int tile = blockIdx.x;
    const int p = threadIdx.x;
    int x, y;
    pixel_of(p, x, y);
    const int px = GS_TILE * (tile % gx) + x, py = GS_TILE * (tile / gx) + y;
    const float fx = (float)px, fy = (float)py;
    const uint2 rg = ranges[tile];
    float T = 1.0f, C0 = 0.f, C1 = 0.f, C2 = 0.f;
    bool done = false;
    for (uint32_t b0 = rg.x; b0 < rg.y; b0 += 256) {
        if (__syncthreads_count(done) == 256) break;
        const uint32_t cnt = min(256u, rg.y - b0);
        if ((uint32_t)p < cnt) {
            const uint32_t gi = vals[b0 + p];
            const float2 m = xy[gi];
            const float4 co = conic_o[gi];
            s_g[p] = make_float4(m.x, m.y, co.x, co.y);
            s_g2[p] = make_float2(co.z, lg2_approx(co.w));
            s_c[p] = rgb[gi];
        }
        __syncthreads();
        for (uint32_t j = 0; j < cnt && !done; j++) {
            const float4 g = s_g[j];
            const float2 g2 = s_g2[j];
            const float dx = g.x - fx, dy = g.y - fy;
            const float power = -0.5f * (g.z * dx * dx + g2.x * dy * dy) - g.w * dx * dy;   // Eq. (3)
            const float mj = power * LOG2E + g2.y;
            if (mj < LOG2_ALPHA_MIN) continue;
            const float a = fminf(ALPHA_MAX, ex2_approx(mj));
            const float tT = T * (1.0f - a);
            if (tT < T_MIN) { done = true; break; }
            const float4 c = s_c[j];
            const float wgt = a * T;
            C0 += wgt * c.x; C1 += wgt * c.y; C2 += wgt * c.z;
            T = tT;
        }
    }
    if (px < W && py < H) {
        const size_t pix = (size_t)py * W + px, plane = (size_t)W * H;
        out_rgb[pix] = C0 + T * bg0;
        out_rgb[plane + pix] = C1 + T * bg1;
        out_rgb[2 * plane + pix] = C2 + T * bg2;
        out_T[pix] = T;
    }
}

void launch_blend_direct(cudaStream_t st, const float2 *xy, const float4 *conic_o, const float4 *rgb,
                         const uint32_t *vals, const uint2 *ranges, int ntiles, int gx, int W, int H,
                         const float bg[3], float *out_rgb, float *out_T, const Counters *) {
    if (ntiles <= 0) return;
    k_blend_direct<<<ntiles, 256, 0, st>>>(xy, conic_o, rgb, vals, ranges, gx, W, H, bg[0], bg[1], bg[2], out_rgb,
                                           out_T);
}

}  // namespace gs
