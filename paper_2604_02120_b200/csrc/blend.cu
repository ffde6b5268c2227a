// blend.cu -- stage (d) "Blending" with the GEMM-compatible
// exponent of GEMM-GS (Eq. 6-8; Alg. 2), and
// the CUDA-core direct form (Alg. 1) as an A/B baseline.
//
// k_blend_tc: persistent, warp-specialised tcgen05 kernel, 4 CTAs per SM
// (10 warps, <= 51 registers, 128 TMEM columns each: 4 x 128 = the SM's 512).
//   warp 8 (producer): per batch of NB = 32 Gaussians of a tile's sorted list,
//     lane j gathers Gaussian j (mean, conic+opacity, colour) with cp.async into
//     a raw-record ring RAW batches deep; tiles come from an atomic work queue.
//   warp 9 (builder + MMA issuer): builds v_g (Eq. 6) scaled by
//     log2(e) with log2(o) folded into the constant term (reading R-10), splits
//     it into TF32 hi + lo (reading R-11), writes the row [hi(6) | lo(6) | 0(4)]
//     of M_g into shared memory, then one lane issues 4 x tcgen05.mma.kind::tf32
//     (M=128 pixels, N=32, K=8; 2 pixel halves x 2 K-steps) that multiply the
//     constant pixel matrix M_p (rows [v_p | v_p | 0], built once per
//     CTA: the "offline" M_p of P:302) by M_g^T into TMEM, committing to an
//     mbarrier. The TMEM ring is STAGES = 2 batches deep.
//   warps 0-7 (compositors, one pixel per thread): tcgen05.ld 32x32b.x16 gives
//     each thread its own pixel's exponents m = log2(alpha), 16 at a time; then
//     alpha = min(0.99, 2^m), alpha-skip below 1/255, T' = T(1-alpha), stop when
//     T' < 1e-4 (not composited), C += alpha T c (Eq. 1; readings R-1..R-4).
//     A warp skips a Gaussian with one vote when none of its 32 pixels keeps it.
//     Per batch, warp 0 polls the batch's mbarriers and warps 1-7 wait for it in a
//     named barrier, so the waiting costs no issue slots (GS_BLEND_NAMED_WAIT).
//   The compositor loop is a serial dependency chain per pixel, so the kernel is
//   latency-bound: occupancy (CTAs per SM) is what sets its speed, and the pipe-
//   line shape (one helper warp each for gathers and rows+MMA, 2 TMEM stages,
//   16-column loads) is the one that fits 4 CTAs per SM (blend).
//   A tile ends when its list is exhausted or all 256 pixels have terminated.
// Reference pixel p_c = tile centre (16 t_x + 7.5, 16 t_y + 7.5) (reading R-6),
// x_bar = x_c - x_p (Eq. 4; reading R-7).
#include <algorithm>
#include <type_traits>

#include <cuda.h>   // CUtensorMap (the TMA descriptors of the frame stores)

#include "gs_common.cuh"

namespace gs {

// Pipeline shape; overridable with -D for tuning sweeps (tools/sweep_blend.py).
#ifndef GS_BLEND_STAGES
#define GS_BLEND_STAGES 2
#endif
#ifndef GS_BLEND_NBLD
#define GS_BLEND_NBLD 1
#endif
#ifndef GS_BLEND_RAW
#define GS_BLEND_RAW 1   // raw-record ring depth (round-1 sweep: 1 / 2 / 3 / 4 -> blend 0.267 / 0.270 / 0.274 / 0.279 ms
                         // per view; round 2 with the supertile producer: 1 vs 2 -> 0.253 vs 0.260-0.263, r2_sweep_m/n)
#endif
#ifndef GS_BLEND_MINB
#define GS_BLEND_MINB 4      // resident CTAs per SM (registers, TMEM = MINB * TMEM_COLS <= 512)
#endif
#ifndef GS_BLEND_GRID_X100
#define GS_BLEND_GRID_X100 (100 * GS_BLEND_MINB)   // persistent grid: CTAs per SM x 100 (sweep knob)
#endif
#ifndef GS_BLEND_CH
#define GS_BLEND_CH 16
#endif
#ifndef GS_BLEND_NAMED_WAIT
#define GS_BLEND_NAMED_WAIT 1   // 1: compositor warps 1-7 wait in a named barrier behind warp 0's mbarrier poll (0: every warp polls)
#endif
#ifndef GS_BLEND_NB
#define GS_BLEND_NB 32
#endif
#ifndef GS_BLEND_STALE_THR
#define GS_BLEND_STALE_THR 1   // 1: the compositors' skip threshold changes only between 16-column chunks
#endif
constexpr int NB = GS_BLEND_NB;         // Gaussians per batch (MMA N: 16 or 32)
#ifndef GS_BLEND_KSTEPS
#define GS_BLEND_KSTEPS 2   // K = 8 * KSTEPS: 2 = TF32 hi/lo (R-11); 1 = single TF32 pass (A/B evidence only)
#endif
static_assert(GS_BLEND_KSTEPS == 1 || GS_BLEND_KSTEPS == 2, "K = 8 (single TF32) or 16 (hi/lo)");
static_assert(NB == 16 || NB == 32, "batch = MMA N = 16 or 32 (one producer / builder lane per Gaussian)");
constexpr int CH = GS_BLEND_CH;         // TMEM columns per compositor load (16 or 32)
constexpr int STAGES = GS_BLEND_STAGES; // M_g / TMEM ring depth
constexpr int NCW = 8;                  // compositor warps: 256 pixels
constexpr int NBLD = GS_BLEND_NBLD;     // builder warps (alternate batches)
constexpr int RAW = GS_BLEND_RAW;       // raw-record ring (producer -> builders): gathers in flight
constexpr int RING = 2 * STAGES;   // colour / header slots (see SLOTS below)
#ifndef GS_BLEND_LPF
#define GS_BLEND_LPF 1
#endif
#ifndef GS_BLEND_L1PF
#define GS_BLEND_L1PF 0    // 1: prefetch the list round after the held one into L1 (no gain: r2_sweep_k)
#endif
#ifndef GS_BLEND_HPF
#define GS_BLEND_HPF 1     // 1: fetch the next tile's first list round during the current tile
#endif
constexpr int LPF = GS_BLEND_LPF;  // list rounds (128 entries) the producer holds ahead
constexpr int LQ = 256;            // producer queue of kept entries (>= NB + 128, power of two)
// warp roles: 0..NCW-1 compositors, NCW producer, NCW+1.. builders (each also issues
// the MMAs of the batches it built, and builder 0 owns the TMEM allocation)
constexpr int WARP_PRODUCER = NCW, WARP_BUILD0 = NCW + 1, WARP_TMEM = NCW + 1;
constexpr int TC_THREADS = (NCW + 1 + NBLD) * 32;
static_assert(STAGES % NBLD == 0, "all batches of a TMEM stage must come from one builder");
constexpr int TMEM_COLS = STAGES * 2 * NB;   // 256
static_assert(TMEM_COLS >= 32 && (TMEM_COLS & (TMEM_COLS - 1)) == 0 && GS_BLEND_MINB * TMEM_COLS <= 512,
              "TMEM allocation must be a power of two >= 32 and fit MINB CTAs per SM");
// Batch b of a CTA's stream (data batch, end-of-tile marker or terminal)
//   raw slot b % RAW  (producer -> builder b % NBLD),
//   M_g/TMEM stage b % STAGES (builder -> MMA warp -> compositors),
//   colour/header slot b % RING. A builder writes stage/slot of batch b only
// after the MMA of batch b - STAGES completed, which required every compositor
// warp to release batch b - 2*STAGES: RING = 2*STAGES slots need no extra wait.
// Header: {ty << 16 | tx, seq, count, list offset}; count 0 = end-of-tile marker,
// count -1 = batch of an already terminated tile (skipped), tile -1 = terminal.

#ifndef GS_BLEND_BULK
#define GS_BLEND_BULK 0   // 1: one cp.async.bulk (TMA engine, UBLKCP) per 48-B record; 0: three cp.async (LDGSTS).
                          // A/B (profiles/r2_sweep_bulk.txt, C5 orbit): bulk 1353 / 1360 fps, blend 0.284 / 0.287 ms;
                          // cp.async 1390 / 1393 fps, 0.266 / 0.269 ms: 48-B bulk copies cost more than they save
#endif
using RawRec = Splat;   // one gathered Gaussian: the preprocess's 48-B record, copied as is
#ifndef GS_BLEND_TMA_STORE
#define GS_BLEND_TMA_STORE 1   // 1: frames leave through a TMA tensor store per tile (UTMASTG); 0: per-thread stores
#endif
#if GS_BLEND_TMA_STORE && !GS_BLEND_NAMED_WAIT
#error "the TMA store epilogue relies on the per-batch named barrier of the compositors"
#endif

struct __align__(1024) SmemTC {
    uint8_t A[2][128 * 64];       // M_p halves: 128 rows x 16 tf32, interleaved core matrices
    uint8_t B[STAGES][NB * 64];   // M_g rows
    float4 rgb[RING][NB];
    int4 hdr[RING];
    RawRec raw[RAW][NB];
    int4 raw_hdr[RAW];
    uint64_t full[STAGES];        // MMA done (commit), or marker -> compositors
    uint64_t empty[STAGES];       // compositors released the TMEM stage -> MMA warp
    uint64_t slot_ready[RING];    // colours/header written -> compositors
    uint64_t raw_full[RAW];       // producer -> builder
    uint64_t raw_empty[RAW];      // builder -> producer
    uint32_t lq[LQ];              // producer: kept list entries waiting for a batch
    uint32_t tmem_base;
    uint32_t warp_done_seq[NCW];
#if GS_BLEND_TMA_STORE
    alignas(128) float outb[2][4][GS_TILE_PIX];   // finished tile (R, G, B, T planes, row-major 16 x 16), double-
                                                  // buffered; a TMA source must be 128-B aligned
#endif
};

// N4 (GS_BLEND_TC_COLOR): the colour sum C = sum_i c_i alpha_i T_i (Eq. 1) as a second
// tensor-core product per batch, C[pixels x 16] += W[pixels x NB] . Col[16 x NB]^T with
// W = alpha T (0 for Gaussians not composited), rounded to TF32 by the compositors into
// shared memory, and Col = the batch's colours split TF32 hi | lo (rows r, g, b, r_lo, g_lo,
// b_lo, 0...). The accumulators (2 halves x 16 columns) live in TMEM for the whole tile;
// 160 columns round the allocation up to 256, so 2 CTAs per SM.
struct __align__(1024) SmemTCC : SmemTC {
    uint8_t Wb[2][2][128 * 128];   // W per colour-batch parity and pixel half: 128 rows x 32 tf32 (K-major)
    uint8_t Cb[RING][16 * 128];    // colour operand per slot: 16 rows x 32 tf32 (K-major)
    uint64_t wfull[2];             // compositors wrote W of colour batch n (parity n % 2)
    uint64_t cdone[2];             // the colour MMA of batch n read W[n % 2] (commit)
    uint64_t cacc;                 // the tile's colour accumulators are complete (commit at its marker)
};
constexpr int CM_TMEM_COLS = 256;
constexpr int CM_COL0 = STAGES * 2 * NB;   // first accumulator column (after the exponent stages)

// byte offset of (row r, 16-byte K-chunk c) in a K-major no-swizzle operand
// with 4 K-chunks per row: core matrix = 8 rows x 16 B, LBO = 128, SBO = 512
__device__ __forceinline__ uint32_t op_off(int r, int c) { return (r >> 3) * 512 + c * 128 + (r & 7) * 16; }
// the same with 8 K-chunks per row (K = 32): LBO = 128, SBO = 1024
__device__ __forceinline__ uint32_t op_off32(int r, int c) { return (r >> 3) * 1024 + c * 128 + (r & 7) * 16; }

// pixel of compositor thread p = 32*w + lane inside the 16x16 tile: warp w
// covers the 8x4 block at (8*(w%2), 4*(w/2)) (compact blocks maximise the
// warp-uniform skip).
__device__ __forceinline__ void pixel_of(int p, int &x, int &y) {
    const int w = p >> 5, l = p & 31;
    x = 8 * (w & 1) + (l & 7);
    y = 4 * (w >> 1) + (l >> 3);
}

__device__ __forceinline__ float4 ld_shared_f4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}

__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, float (&v)[32]) { tmem_ld32(taddr, v); }
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, float (&v)[16]) { tmem_ld16(taddr, v); }

__device__ __forceinline__ bool tile_done(const SmemTC &sm, int lane, uint32_t seq) {
    const uint32_t dseq = lane < NCW ? *((volatile const uint32_t *)&sm.warp_done_seq[lane]) : seq;
    return __all_sync(0xffffffffu, dseq >= seq);
}

// Row j of M_g for batch `hd` (lane j): Eq. (6) v_g with xh = x_g - x_c, yh = y_g - y_c,
// scaled by log2(e), log2(o) folded into the constant term (R-10), split into TF32
// hi + lo (R-11); padding rows get the exponent -1e30 (never kept).
__device__ __forceinline__ void build_row(SmemTC &sm, int stage, int slot, const int4 &hd, const RawRec &rr, int lane,
                                          int gx) {
    uint32_t u[16];
    if (lane < hd.z) {
        const float xc = (float)(GS_TILE * (hd.x & 0xffff)) + 7.5f;   // hd.x = ty << 16 | tx
        const float yc = (float)(GS_TILE * (hd.x >> 16)) + 7.5f;
        const float xh = rr.m.x - xc, yh = rr.m.y - yc;
        const float A = rr.co.x, B = rr.co.y, C = rr.co.z;
        float v[6];
        v[0] = -0.5f * A * LOG2E;
        v[1] = -0.5f * C * LOG2E;
        v[2] = -B * LOG2E;
        v[3] = -(A * xh + B * yh) * LOG2E;
        v[4] = -(C * yh + B * xh) * LOG2E;
        v[5] = -(0.5f * A * xh * xh + 0.5f * C * yh * yh + B * xh * yh) * LOG2E + lg2_approx(rr.co.w);
#pragma unroll
        for (int k = 0; k < 6; k++) {
            const uint32_t hi = f32_to_tf32_rna(v[k]);
            const uint32_t lo = f32_to_tf32_rna(v[k] - __uint_as_float(hi));
            u[k] = hi;
            u[6 + k] = GS_BLEND_KSTEPS == 2 ? lo : 0u;   // K = 8: hi only, the lo columns stay zero
        }
    } else {
#pragma unroll
        for (int k = 0; k < 12; k++) u[k] = 0u;
        u[5] = __float_as_uint(-1e30f);
    }
    u[12] = u[13] = u[14] = u[15] = 0u;
    const uint32_t rb = smem_u32(&sm.B[stage][0]);
#pragma unroll
    for (int c = 0; c < 4; c++) st_shared_v4(rb + op_off(lane, c), u[4 * c], u[4 * c + 1], u[4 * c + 2], u[4 * c + 3]);
    sm.rgb[slot][lane] = rr.col;
}

// optional per-batch event trace of CTA 0 (debug builds of the timeline): trace[b*16 + ev] = clock64
#define TRACE_EV(ev, b)                                                                                   \
    do {                                                                                                  \
        if (TRACE && blockIdx.x == 0 && (b) < 1024u && lane == 0) trace[(size_t)(b) * 16 + (ev)] = clock64(); \
    } while (0)

template <bool DUMP, bool STATS, bool TRACE, bool CM>
__global__ void __launch_bounds__(TC_THREADS, CM ? 2 : GS_BLEND_MINB)
    k_blend_tc(const Splat *__restrict__ splat, const TileLists lists, int tile0, int ntiles, int gx,
               int W, int H, float bg0, float bg1, float bg2, float *__restrict__ out_rgb, float *__restrict__ out_T,
               float *__restrict__ dump_m, uint32_t *tile_queue, unsigned long long *stat_eval,
               unsigned long long *stat_kept, long long *trace, const __grid_constant__ CUtensorMap tm_rgb,
               const __grid_constant__ CUtensorMap tm_T, int tma_out) {
    // used as is (no pointer arithmetic), so every access compiles to LDS/STS rather than
    // generic loads; the dynamic window starts 1024-B aligned (checked: TMA needs 128 B)
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    using SM = std::conditional_t<CM, SmemTCC, SmemTC>;
    SM &sm = *reinterpret_cast<SM *>(smem_raw);
    if (threadIdx.x == 0 && (smem_u32(smem_raw) & 1023u)) __trap();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int NCOLS = CM ? CM_TMEM_COLS : TMEM_COLS;
    static_assert(!CM || NBLD == 1, "the colour MMA follows the single builder's batch order");

    // ---- one-time setup -------------------------------------------------
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; s++) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], NCW);
        }
        for (int r = 0; r < RING; r++) mbar_init(&sm.slot_ready[r], 1);
        for (int r = 0; r < RAW; r++) {
            mbar_init(&sm.raw_full[r], GS_BLEND_BULK ? 1 : 33);   // header arrive (+ expect_tx) | 32 cp.async + header
            mbar_init(&sm.raw_empty[r], 1);
        }
        if constexpr (CM) {
            for (int q = 0; q < 2; q++) {
                mbar_init(&sm.wfull[q], NCW);
                mbar_init(&sm.cdone[q], 1);
            }
            mbar_init(&sm.cacc, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if constexpr (CM) {   // colour operand rows 6..15 stay zero
        for (int i = threadIdx.x; i < RING * 16 * 128 / 16; i += TC_THREADS)
            reinterpret_cast<uint4 *>(&sm.Cb[0][0])[i] = make_uint4(0u, 0u, 0u, 0u);
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
    } else if (warp == WARP_TMEM) {
        tmem_alloc(&sm.tmem_base, NCOLS);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;
    pdl_wait();   // the setup above overlapped the binning's tail

    if (warp == WARP_PRODUCER) {
        // =================== producer: list filter + asynchronous gathers ===================
        // A tile's list is its supertile's list filtered by the tile's mask bit (per-tile
        // lists: every entry). Entries are read 128 per round, LPF rounds ahead in registers
        // (the next tile's first round is fetched during the current tile); the kept
        // Gaussians, in list order, pass through a 64-entry queue in shared memory and leave
        // in batches of NB (the last one of a list may be partial). Lane j of batch b copies
        // record j with cp.async straight into raw slot b % RAW; the slot's barrier completes
        // when the copies land, so RAW batches of gathers are in flight.
        uint32_t b_idx = 0;
        const bool st_mode = lists.keys != nullptr;
        // list range of tile t and the key bit that selects it (per-tile lists: any bit)
        auto tile_list = [&](int t, uint2 &r, uint32_t &kbit) {
            if (t >= ntiles) {
                r = make_uint2(0u, 0u);
                kbit = 1u;
            } else if (st_mode) {
                const int tx = t % gx, ty = t / gx;
                r = lists.ranges[(ty >> 2) * lists.sgx + (tx >> 2)];
                kbit = 1u << (16 + 4 * (ty & 3) + (tx & 3));
            } else {
                r = lists.ranges[t];
                kbit = 1u;
            }
        };
        // One round = 128 list entries from position p (a multiple of 4): lane L holds entries
        // p + 4L .. p + 4L + 3 (one 16-B load of keys and one of values when all four lie
        // inside the range, else per entry); entries outside [r.x, r.y) read as key 0.
        auto fetch = [&](const uint2 &r, uint32_t p, uint4 &k, uint4 &v) {
            const uint32_t e = p + 4u * lane;
            if (e >= r.x && e + 3u < r.y) {
                v = __ldg(reinterpret_cast<const uint4 *>(lists.vals + e));
                k = st_mode ? __ldg(reinterpret_cast<const uint4 *>(lists.keys + e))
                            : make_uint4(~0u, ~0u, ~0u, ~0u);
            } else {
                uint32_t kk[4], vv[4];
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const bool ok = e + j >= r.x && e + j < r.y;
                    vv[j] = ok ? lists.vals[e + j] : 0u;
                    kk[j] = ok ? (st_mode ? lists.keys[e + j] : ~0u) : 0u;
                }
                v = make_uint4(vv[0], vv[1], vv[2], vv[3]);
                k = make_uint4(kk[0], kk[1], kk[2], kk[3]);
            }
        };
        int tile = 0;
        if (lane == 0) tile = tile0 + (int)atomicAdd(tile_queue, 1u);   // tiles [tile0, ntiles)
        tile = __shfl_sync(0xffffffffu, tile, 0);
        // headers carry the tile as ty << 16 | tx (one division per tile here, none per batch)
        auto tcode_of = [&](int t) { return ((t / gx) << 16) | (t % gx); };
        int tcode = tcode_of(tile);
        uint2 rg;
        uint32_t kbit;
        tile_list(tile, rg, kbit);
        uint32_t seq = 1, pos = rg.x & ~3u, head = 0, tail = 0, taken = 0;
        uint4 lk[LPF], lv[LPF];
#pragma unroll
        for (int j = 0; j < LPF; j++) fetch(rg, pos + 128u * j, lk[j], lv[j]);
        int hstate = 0, ntile = 0, ntile_l0 = 0;
        uint2 nrg = make_uint2(0u, 0u);
        uint32_t nkbit = 1u;
        uint4 hk = make_uint4(0u, 0u, 0u, 0u), hv = hk;   // the next tile's first round
        auto head_step = [&]() {
            switch (hstate) {
                case 0:
                    if (lane == 0) ntile_l0 = tile0 + (int)atomicAdd(tile_queue, 1u);
                    break;
                case 1:
                    ntile = __shfl_sync(0xffffffffu, ntile_l0, 0);
                    tile_list(ntile, nrg, nkbit);
                    break;
                case 2:
                    if (GS_BLEND_HPF) fetch(nrg, nrg.x & ~3u, hk, hv);
                    break;
                default:
                    return;
            }
            hstate++;
        };
        // stage batch b_idx: header (+ records of lanes < hd.z) into raw slot
        auto push = [&](const int4 &hd, uint32_t gi) {
            const int r = b_idx % RAW;
            TRACE_EV(0, b_idx);
            mbar_wait(&sm.raw_empty[r], ((b_idx / RAW) & 1u) ^ 1u);
            TRACE_EV(1, b_idx);
#if GS_BLEND_BULK
            // the header arrives with the batch's byte count; each lane's bulk copy of its
            // 48-B record completes its share of the transaction bytes (the phase completes
            // when all have landed)
            if (lane == 0) {
                sm.raw_hdr[r] = hd;
                mbar_arrive_expect_tx(&sm.raw_full[r], hd.z > 0 ? (uint32_t)hd.z * (uint32_t)sizeof(Splat) : 0u);
            }
            __syncwarp();
            if (lane < hd.z) bulk_g2s(&sm.raw[r][lane], splat + gi, (uint32_t)sizeof(Splat), &sm.raw_full[r]);
#else
            if (lane < hd.z) {
                RawRec &d = sm.raw[r][lane];
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&d.m)), "l"(&splat[gi].m)
                             : "memory");
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&d.co)), "l"(&splat[gi].co)
                             : "memory");
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&d.col)), "l"(&splat[gi].col)
                             : "memory");
            }
            if (lane == 0) {
                sm.raw_hdr[r] = hd;
                mbar_arrive(&sm.raw_full[r]);
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&sm.raw_full[r]))
                         : "memory");
#endif
            b_idx++;
        };
        for (;;) {
            if (tile >= ntiles) {
                for (int t = 0; t < NBLD; t++) push(make_int4(-1, 0, 0, 0), 0u);   // one per builder
                break;
            }
            head_step();
            // fill the queue up to NB kept Gaussians (or the end of the list)
            while (tail - head < (uint32_t)NB && pos < rg.y) {
                // ordered compaction of the round: lane L's kept entries go to the queue after
                // those of lanes < L (exclusive scan of the per-lane counts)
                const uint32_t km = ((lk[0].x & kbit) ? 1u : 0u) | ((lk[0].y & kbit) ? 2u : 0u) |
                                    ((lk[0].z & kbit) ? 4u : 0u) | ((lk[0].w & kbit) ? 8u : 0u);
                const uint32_t c = (uint32_t)__popc(km);
                // exclusive prefix of the per-lane counts (0..4) from three ballots of their bits:
                // independent votes instead of a 5-step dependent shuffle scan
                const uint32_t b0 = __ballot_sync(0xffffffffu, c & 1u), b1 = __ballot_sync(0xffffffffu, c & 2u),
                               b2 = __ballot_sync(0xffffffffu, c & 4u);
                if (b0 | b1 | b2) {
                    const uint32_t lt = lanemask_lt_u32();
                    uint32_t w = tail + __popc(b0 & lt) + 2u * __popc(b1 & lt) + 4u * __popc(b2 & lt);
                    if (km & 1u) sm.lq[w++ & (LQ - 1)] = lv[0].x;
                    if (km & 2u) sm.lq[w++ & (LQ - 1)] = lv[0].y;
                    if (km & 4u) sm.lq[w++ & (LQ - 1)] = lv[0].z;
                    if (km & 8u) sm.lq[w & (LQ - 1)] = lv[0].w;
                    tail += __popc(b0) + 2u * __popc(b1) + 4u * __popc(b2);
                }
                if (GS_BLEND_L1PF) {   // the round after the next one into L1 (no registers held)
                    const uint32_t e = pos + 128u * (LPF + 1) + 4u * lane;
                    if (e < rg.y) {
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(lists.vals + e));
                        if (st_mode) asm volatile("prefetch.global.L1 [%0];" ::"l"(lists.keys + e));
                    }
                }
#pragma unroll
                for (int j = 0; j + 1 < LPF; j++) {
                    lk[j] = lk[j + 1];
                    lv[j] = lv[j + 1];
                }
                fetch(rg, pos + 128u * LPF, lk[LPF - 1], lv[LPF - 1]);
                pos += 128u;
            }
            __syncwarp();
            bool end = tail == head;   // list exhausted, queue empty
            if (!DUMP && !end) end = tile_done(sm, lane, seq);
            if (end) {
                push(make_int4(tcode, (int)seq, 0, 0), 0u);   // end-of-tile marker
                while (hstate < 3) head_step();
                tile = ntile;
                tcode = tcode_of(tile);
                rg = nrg;
                kbit = nkbit;
                pos = rg.x & ~3u;
                head = tail = taken = 0;
                seq++;
                if (GS_BLEND_HPF) {
                    lk[0] = hk;
                    lv[0] = hv;
                } else {
                    fetch(rg, pos, lk[0], lv[0]);
                }
#pragma unroll
                for (int j = 1; j < LPF; j++) fetch(rg, pos + 128u * j, lk[j], lv[j]);
                hstate = 0;
                continue;
            }
            const uint32_t cnt = min((uint32_t)NB, tail - head);
            const uint32_t gi = lane < cnt ? sm.lq[(head + lane) & (LQ - 1)] : 0u;
            __syncwarp();   // (the queue slots read here are refilled by later rounds)
            push(make_int4(tcode, (int)seq, (int)cnt, (int)(rg.x + taken)), gi);
            head += cnt;
            taken += cnt;
        }
    } else if (warp >= WARP_BUILD0 && warp < WARP_BUILD0 + NBLD) {
        // =================== builders: M_g rows (Eq. 6-7) ===================
        // STATS: the exponents the MMA computes, (Gaussian, pixel) pairs of the batches built
        // (batches of a tile found terminated before their build are dropped, not counted)
        unsigned long long n_eval = 0;
        // CM: the colour MMA of data batch n is issued once the compositors wrote its W, i.e.
        // while the next batch is built (pend_*: the batch waiting for it)
        int pend_slot = -1;
        uint32_t n_col = 0, pend_n = 0;
        bool first_of_tile = true, pend_first = false;
        auto flush_colour = [&]() {
            if constexpr (CM) {
                if (pend_slot < 0) return;
                mbar_wait(&sm.wfull[pend_n & 1u], (pend_n >> 1) & 1u);
                tc_fence_after();
                if (lane == 0) {
                    constexpr uint32_t IDESC = idesc_tf32(128, 16);
                    const uint32_t b_base = smem_u32(&sm.Cb[pend_slot][0]);
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        const uint32_t a_base = smem_u32(&sm.Wb[pend_n & 1u][h][0]);
#pragma unroll
                        for (int kk = 0; kk < NB / 8; kk++)
                            mma_tf32(tmem + CM_COL0 + h * 16, umma_desc(a_base + kk * 256, 128, 1024),
                                     umma_desc(b_base + kk * 256, 128, 1024), IDESC,
                                     (pend_first && kk == 0) ? 0u : 1u);
                    }
                    mma_commit(&sm.cdone[pend_n & 1u]);
                }
                __syncwarp();
                pend_slot = -1;
            }
        };
        for (uint32_t kb = warp - WARP_BUILD0;; kb += NBLD) {
            const int r = kb % RAW, s = kb % STAGES, slot = kb % RING;
            mbar_wait(&sm.raw_full[r], (kb / RAW) & 1u);
            TRACE_EV(2, kb);
            int4 hd = sm.raw_hdr[r];
            // stage s / slot are reusable once batch kb-STAGES went through the MMA warp
            // (for every batch kind: this also keeps the slot_ready phases in step)
            if (kb >= STAGES) mbar_wait(&sm.full[s], ((kb / STAGES) - 1) & 1u);
            TRACE_EV(3, kb);
            if (hd.z > 0) {
                if (!DUMP && tile_done(sm, lane, (uint32_t)hd.y)) hd.z = -1;   // tile already terminated
            }
            if (hd.z > 0) {
                if (lane < NB) build_row(sm, s, slot, hd, sm.raw[r][lane], lane, gx);
                if constexpr (CM) {   // colour operand of the slot: K index = lane, rows r g b hi | lo
                    const float4 c = sm.raw[r][lane].col;
                    const float cv[3] = {c.x, c.y, c.z};
                    const uint32_t cb = smem_u32(&sm.Cb[slot][0]) + (lane >> 2) * 128 + (lane & 3) * 4;
#pragma unroll
                    for (int ch = 0; ch < 3; ch++) {
                        const uint32_t hi = lane < hd.z ? f32_to_tf32_rna(cv[ch]) : 0u;
                        const uint32_t lo = lane < hd.z ? f32_to_tf32_rna(cv[ch] - __uint_as_float(hi)) : 0u;
                        asm volatile("st.shared.b32 [%0], %1;" ::"r"(cb + ch * 16), "r"(hi) : "memory");
                        asm volatile("st.shared.b32 [%0], %1;" ::"r"(cb + (3 + ch) * 16), "r"(lo) : "memory");
                    }
                }
                fence_proxy_async_smem();
                if (STATS) n_eval += (unsigned long long)hd.z * GS_TILE_PIX;
            }
            if (lane == 0) sm.hdr[slot] = hd;
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&sm.raw_empty[r]);
                mbar_arrive(&sm.slot_ready[slot]);
            }
            TRACE_EV(4, kb);
            {
                const uint32_t ph = (kb / STAGES) & 1u;
                mbar_wait(&sm.empty[s], ph ^ 1u);   // batch kb - STAGES no longer read from TMEM
                if (hd.z > 0) {
                    tc_fence_after();
                    if (lane == 0) {
                        constexpr uint32_t IDESC = idesc_tf32(128, NB);
                        const uint32_t a_base = smem_u32(&sm.A[0][0]);
                        const uint32_t b_base = smem_u32(&sm.B[s][0]);
#pragma unroll
                        for (int kk = 0; kk < GS_BLEND_KSTEPS; kk++)
#pragma unroll
                            for (int h = 0; h < 2; h++)
                                mma_tf32(tmem + s * (2 * NB) + h * NB,
                                         umma_desc(a_base + h * (128 * 64) + kk * 256, 128, 512),
                                         umma_desc(b_base + kk * 256, 128, 512), IDESC, kk);
                        mma_commit(&sm.full[s]);
                    }
                } else if (lane == 0) {
                    mbar_arrive(&sm.full[s]);   // marker / skipped batch: no MMA
                }
                __syncwarp();
            }
            if constexpr (CM) {
                flush_colour();   // the previous data batch (its W is written while this one computes)
                if (hd.z > 0) {
                    pend_slot = slot;
                    pend_n = n_col++;
                    pend_first = first_of_tile;
                    first_of_tile = false;
                } else if (hd.z == 0 && hd.x >= 0) {   // end of tile: accumulators complete
                    // (only for tiles with a colour batch: their last W implies the compositors
                    // read the previous tile's accumulators, so cacc is never two phases ahead)
                    if (!first_of_tile && lane == 0) mma_commit(&sm.cacc);
                    __syncwarp();
                    first_of_tile = true;
                }
            }
            if (hd.x < 0) {
                if (STATS && lane == 0) atomicAdd(stat_eval, n_eval);
                break;
            }
        }
    } else {
        // =================== compositors ===================
        const int p = threadIdx.x;
        int x, y;
        pixel_of(p, x, y);
        const uint32_t t_lane = (uint32_t)(32 * (warp & 3)) << 16;
        const uint32_t t_half = (uint32_t)(warp >> 2) * NB;
        // Pixel state. Termination is encoded in the skip threshold: thr = +inf once the
        // pixel has stopped (R-2), so "live" is a single compare and no bool is carried.
        float T = 1.0f, C0 = 0.f, C1 = 0.f, C2 = 0.f, thr = LOG2_ALPHA_MIN;
        float tmin = T_MIN;   // GS_BLEND_STALE_THR: the stop threshold of T (+inf once stopped)
        bool wdone = false;
        uint32_t n_kept = 0, n_tiles = 0;
        uint32_t n_col = 0, n_acc = 0;    // CM: data batches (W buffers) and tiles with accumulators so far
        bool tile_col = false;            // CM: the tile had a colour batch
        const int crow_w = p & 127;       // CM: this pixel's row in its half's W operand
        for (uint32_t k = 0;; k++) {
            const int s = k % STAGES;
            const int c_slot = k % RING;
#if GS_BLEND_NAMED_WAIT
            // one warp polls the barriers, the other compositor warps sleep in a named
            // barrier (no issue slots spent spinning); tc_fence_after orders their TMEM loads
            if (warp == 0) {
                mbar_wait(&sm.slot_ready[c_slot], (k / RING) & 1u);
                mbar_wait(&sm.full[s], (k / STAGES) & 1u);
                if constexpr (CM) {
                    const int4 h0 = sm.hdr[c_slot];
                    if (h0.z > 0 && n_col >= 2)   // W[n % 2] free: the colour MMA of batch n - 2 read it
                        mbar_wait(&sm.cdone[n_col & 1u], ((n_col - 2) >> 1) & 1u);
                    else if (h0.z == 0 && h0.x >= 0 && tile_col)   // the tile's accumulators are complete
                        mbar_wait(&sm.cacc, n_acc & 1u);
                }
            }
            asm volatile("bar.sync 1, 256;" ::: "memory");
#else
            mbar_wait(&sm.slot_ready[c_slot], (k / RING) & 1u);
            mbar_wait(&sm.full[s], (k / STAGES) & 1u);
#endif
            if (warp == 0) TRACE_EV(7, k);
            if (warp == 7) TRACE_EV(9, k);
            tc_fence_after();
            const int4 hd = sm.hdr[c_slot];
            if (hd.z == 0) {
                if (hd.x < 0) {
                    if (STATS) {
                        unsigned long long kk = n_kept;
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) kk += __shfl_xor_sync(0xffffffffu, kk, o);
                        if (lane == 0) atomicAdd(stat_kept, kk);
                    }
                    break;
                }
                if constexpr (CM) {   // C from the tile's colour accumulators: hi + lo columns
                    if (tile_col) {
                        float cv[16];
                        tmem_ld16(tmem + t_lane + CM_COL0 + (uint32_t)(warp >> 2) * 16, cv);
                        tmem_wait_ld();
                        C0 = cv[0] + cv[3];
                        C1 = cv[1] + cv[4];
                        C2 = cv[2] + cv[5];
                        n_acc++;
                    }
                    tile_col = false;
                }
#if GS_BLEND_TMA_STORE
                if (!DUMP && tma_out) {
                    // a9 through the TMA engine: the tile's four planes go to shared memory,
                    // then ONE thread stores them with two tensor copies (3-D RGB box, 2-D T
                    // box) that clip the frame edge themselves. Double-buffered: the store of
                    // the tile before last must have read its buffer (wait_group.read 1), which
                    // thread 0 checked right after issuing the previous tile's store, before
                    // it joined this tile's batch barriers.
                    float *ob = &sm.outb[n_tiles & 1][0][0];
                    const int pi = y * GS_TILE + x;
                    ob[pi] = C0 + T * bg0;
                    ob[GS_TILE_PIX + pi] = C1 + T * bg1;
                    ob[2 * GS_TILE_PIX + pi] = C2 + T * bg2;
                    ob[3 * GS_TILE_PIX + pi] = T;
                    fence_proxy_async_smem();
                    asm volatile("bar.sync 2, 256;" ::: "memory");
                    if (threadIdx.x == 0) {
                        const int x0 = GS_TILE * (hd.x & 0xffff), y0 = GS_TILE * (hd.x >> 16);
                        tma_store_3d(&tm_rgb, ob, x0, y0, 0);
                        tma_store_2d(&tm_T, ob + 3 * GS_TILE_PIX, x0, y0);
                        bulk_commit_group();
                        bulk_wait_group_read1();
                    }
                    n_tiles++;
                } else
#endif
                if (!DUMP) {
                    const int px = GS_TILE * (hd.x & 0xffff) + x, py = GS_TILE * (hd.x >> 16) + y;
                    if (px < W && py < H) {
                        const size_t pix = (size_t)py * W + px, plane = (size_t)W * H;
                        out_rgb[pix] = C0 + T * bg0;
                        out_rgb[plane + pix] = C1 + T * bg1;
                        out_rgb[2 * plane + pix] = C2 + T * bg2;
                        out_T[pix] = T;
                    }
                }
                T = 1.0f; C0 = C1 = C2 = 0.f; thr = LOG2_ALPHA_MIN; tmin = T_MIN; wdone = false;
            } else if (hd.z > 0 && wdone) {
                if constexpr (CM) {   // W of a finished warp: zeros
                    const uint32_t wb = smem_u32(&sm.Wb[n_col & 1u][warp >> 2][0]);
#pragma unroll
                    for (int c = 0; c < NB / 4; c++) st_shared_v4(wb + op_off32(crow_w, c), 0u, 0u, 0u, 0u);
                }
            } else if (hd.z > 0 && !wdone) {
                const int cnt = hd.z;
                const uint32_t crow = smem_u32(&sm.rgb[c_slot][0]);
                // exponents come out of TMEM CH columns at a time (CH = 16 keeps the
                // register count low enough for 4 CTAs per SM)
#pragma unroll
                for (int h0 = 0; h0 < NB; h0 += CH) {
                    float m[CH];
                    float wv[CM ? CH : 1];   // CM: this chunk's W = alpha T (0: not composited)
                    tmem_ld_cols(tmem + t_lane + s * (2 * NB) + t_half + h0, m);
                    tmem_wait_ld();
                    if (DUMP) {
                        for (int j = 0; j < CH && h0 + j < cnt; j++)
                            dump_m[((size_t)hd.w + h0 + j) * GS_TILE_PIX + p] = m[j];
                    } else {
                        // columns j >= cnt hold the padding exponent -1e30: no count checks needed.
                        // GS_BLEND_STALE_THR: the skip threshold is only updated between chunks
                        // and a pixel that stops inside the chunk is masked by its stop threshold `tmin`, so the
                        // skip vote of column j + 1 does not wait for column j's compositing
                        // (same frames: a stopped pixel never composites again either way)
#pragma unroll
                        for (int j = 0; j < CH; j++) {
                            const float mj = m[j];
                            const bool live = mj >= thr;                    // alpha >= 1/255 (R-1), pixel running
                            if constexpr (CM) wv[j] = 0.f;
                            if (__any_sync(0xffffffffu, live)) {            // warp-uniform skip
                                const float a = fminf(ALPHA_MAX, ex2_approx(mj));   // alpha = 2^m capped (R-4)
                                const float tT = fmaf(-a, T, T);                    // T (1 - alpha)
                                const float w = a * T;
#if GS_BLEND_STALE_THR
                                // tmin = +inf once the pixel stopped: one compare tests both
                                const bool acc = live && tT >= tmin;                // composite (Eq. 1, R-3)
                                if (STATS) n_kept += (live && tmin < 1.f) ? 1u : 0u;
#else
                                const bool acc = live && tT >= T_MIN;               // composite (Eq. 1, R-3)
                                if (STATS) n_kept += live ? 1u : 0u;
#endif
                                if constexpr (CM) {
                                    wv[j] = acc ? w : 0.f;
                                } else {
                                    // (predicated updates: a select-free form, w = (acc ? a : 0) T,
                                    // saves the register moves but lengthens the chain, measured slower)
                                    const float4 c = ld_shared_f4(crow + 16 * (h0 + j));
                                    C0 = acc ? fmaf(w, c.x, C0) : C0;
                                    C1 = acc ? fmaf(w, c.y, C1) : C1;
                                    C2 = acc ? fmaf(w, c.z, C2) : C2;
                                }
                                T = acc ? tT : T;
#if GS_BLEND_STALE_THR
                                tmin = (live && !acc) ? __int_as_float(0x7f800000) : tmin;   // stop (R-2)
#else
                                thr = (live && !acc) ? __int_as_float(0x7f800000) : thr;   // stop (R-2)
#endif
                            }
                        }
#if GS_BLEND_STALE_THR
                        thr = tmin > 1.f ? __int_as_float(0x7f800000) : thr;
#endif
                        if constexpr (CM) {   // this chunk's 16 W values, TF32 (round to nearest)
                            const uint32_t wb = smem_u32(&sm.Wb[n_col & 1u][warp >> 2][0]);
#pragma unroll
                            for (int q = 0; q < CH / 4; q++)
                                st_shared_v4(wb + op_off32(crow_w, h0 / 4 + q), f32_to_tf32_rna(wv[4 * q]),
                                             f32_to_tf32_rna(wv[4 * q + 1]), f32_to_tf32_rna(wv[4 * q + 2]),
                                             f32_to_tf32_rna(wv[4 * q + 3]));
                        }
                    }
                }
                if (!DUMP) {
                    if (__all_sync(0xffffffffu, thr > 0.f)) {
                        wdone = true;
                        if (lane == 0) *((volatile uint32_t *)&sm.warp_done_seq[warp]) = (uint32_t)hd.y;
                    }
                }
            }
            tc_fence_before();
            if constexpr (CM) {
                if (hd.z > 0) {   // W of this batch written (every warp, finished or not)
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&sm.wfull[n_col & 1u]);
                    n_col++;
                    tile_col = true;
                }
            }
            __syncwarp();
            if (warp == 0) TRACE_EV(8, k);
            if (warp == 7) TRACE_EV(10, k);
            if (lane == 0) mbar_arrive(&sm.empty[s]);
        }
    }
#if GS_BLEND_TMA_STORE
    if (threadIdx.x == 0 && tma_out) bulk_wait_group_all();   // the last stores complete before the CTA exits
#endif
    tc_fence_before();
    __syncthreads();
    if (warp == WARP_TMEM) {
        tc_fence_after();
        tmem_dealloc(tmem, NCOLS);
    }
}

long long *g_blend_trace = nullptr;   // set by gs_debug_set_trace (debug only)

// TMA descriptors of a frame: RGB planes as a 3-D tensor {W, H, 3} with 16 x 16 x 3 boxes,
// T as a 2-D tensor {W, H} with 16 x 16 boxes (row pitch W floats). cuTensorMapEncodeTiled
// comes from the driver through the runtime's entry-point query (no libcuda link). False
// when the layout does not allow a tensor map (row pitch or base not 16-B aligned): the
// kernel then stores per thread.
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static bool frame_tensor_maps(float *out_rgb, float *out_T, int W, int H, CUtensorMap &m_rgb, CUtensorMap &m_T) {
    static EncodeTiledFn encode = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            encode = reinterpret_cast<EncodeTiledFn>(fn);
        else
            cudaGetLastError();
    }
    if (!encode || !out_rgb || !out_T || (W & 3) || (reinterpret_cast<uintptr_t>(out_rgb) & 15) ||
        (reinterpret_cast<uintptr_t>(out_T) & 15))
        return false;
    const cuuint64_t dims3[3] = {(cuuint64_t)W, (cuuint64_t)H, 3};
    const cuuint64_t str3[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4};
    const cuuint32_t box3[3] = {GS_TILE, GS_TILE, 3}, es3[3] = {1, 1, 1};
    const cuuint64_t dims2[2] = {(cuuint64_t)W, (cuuint64_t)H};
    const cuuint64_t str2[1] = {(cuuint64_t)W * 4};
    const cuuint32_t box2[2] = {GS_TILE, GS_TILE}, es2[2] = {1, 1};
    return encode(&m_rgb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, out_rgb, dims3, str3, box3, es3,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS &&
           encode(&m_T, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, out_T, dims2, str2, box2, es2,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void launch_blend_tc(const Workspace &ws, cudaStream_t st, const Splat *splat, const TileLists &lists, int tile0,
                     int ntiles, int gx, int W, int H, const float bg[3], float *out_rgb, float *out_T, float *dump_m,
                     int num_sms, bool stats, bool colour_mma) {
    const size_t smem = sizeof(SmemTC) + 1024, smem_c = sizeof(SmemTCC) + 1024;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_blend_tc<false, false, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        cudaFuncSetAttribute(k_blend_tc<false, true, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        cudaFuncSetAttribute(k_blend_tc<true, false, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        cudaFuncSetAttribute(k_blend_tc<false, false, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        cudaFuncSetAttribute(k_blend_tc<false, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem_c);
        cudaFuncSetAttribute(k_blend_tc<false, true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem_c);
        attr_set = true;
    }
    colour_mma = colour_mma && !dump_m;
    const int grid = std::max(1, std::min(colour_mma ? 2 * num_sms : GS_BLEND_GRID_X100 * num_sms / 100, ntiles - tile0));
    uint32_t *queue = &ws.counters->tile_queue;
    unsigned long long *se = &ws.counters->pairs_eval, *sk = &ws.counters->pairs_kept;
    CUtensorMap m_rgb{}, m_T{};
    const int tma = (GS_BLEND_TMA_STORE && !dump_m && frame_tensor_maps(out_rgb, out_T, W, H, m_rgb, m_T)) ? 1 : 0;
#define ARGS splat, lists, tile0, ntiles, gx, W, H, bg[0], bg[1], bg[2], out_rgb, out_T, dump_m, queue, se, sk
    if (dump_m)
        launch_pdl(k_blend_tc<true, false, false, false>, grid, TC_THREADS, smem, st, ARGS, nullptr, m_rgb, m_T, tma);
    else if (colour_mma && stats)
        launch_pdl(k_blend_tc<false, true, false, true>, grid, TC_THREADS, smem_c, st, ARGS, nullptr, m_rgb, m_T, tma);
    else if (colour_mma)
        launch_pdl(k_blend_tc<false, false, false, true>, grid, TC_THREADS, smem_c, st, ARGS, nullptr, m_rgb, m_T,
                   tma);
    else if (stats)
        launch_pdl(k_blend_tc<false, true, false, false>, grid, TC_THREADS, smem, st, ARGS, nullptr, m_rgb, m_T, tma);
    else if (g_blend_trace)
        launch_pdl(k_blend_tc<false, false, true, false>, grid, TC_THREADS, smem, st, ARGS, g_blend_trace, m_rgb, m_T,
                   tma);
    else
        launch_pdl(k_blend_tc<false, false, false, false>, grid, TC_THREADS, smem, st, ARGS, nullptr, m_rgb, m_T, tma);
#undef ARGS
}

// ===========================================================================
// CUDA-core direct blend (Alg. 1 with Eq. 3 per pixel): one 256-thread CTA per
// tile, batches of 256 Gaussians staged in shared memory.
// ===========================================================================
__global__ void __launch_bounds__(256) k_blend_direct(const Splat *__restrict__ splat, const uint32_t *__restrict__ vals,
                                                      const uint2 *__restrict__ ranges, int tile0, int gx, int W, int H,
                                                      float bg0, float bg1, float bg2, float *__restrict__ out_rgb,
                                                      float *__restrict__ out_T) {
    pdl_wait();
    __shared__ float4 s_g[256];     // (x, y, A, B)
    __shared__ float2 s_g2[256];    // (C, log2 o)
    __shared__ float4 s_c[256];
    const int tile = tile0 + blockIdx.x;
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
            const float2 m = splat[gi].m;
            const float4 co = splat[gi].co;
            s_g[p] = make_float4(m.x, m.y, co.x, co.y);
            s_g2[p] = make_float2(co.z, lg2_approx(co.w));
            s_c[p] = splat[gi].col;
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

void launch_blend_direct(cudaStream_t st, const Splat *splat, const uint32_t *vals, const uint2 *ranges, int tile0, int ntiles, int gx, int W, int H,
                         const float bg[3], float *out_rgb, float *out_T, const Counters *) {
    if (ntiles - tile0 <= 0) return;
    launch_pdl(k_blend_direct, ntiles - tile0, 256, 0, st, splat, vals, ranges, tile0, gx, W, H, bg[0], bg[1], bg[2], out_rgb,
                                           out_T);
}

// ===========================================================================
// Warp-level tensor-core blend (the paper's own kernel shape, on sm_100a):
// mma.sync.m16n8k8 TF32 (HMMA.1688) instead of tcgen05. A/B against k_blend_tc for
// the north star's "mma.sync or tcgen05, whichever ncu shows wins".
//   One 256-thread CTA per tile at a time (persistent, atomic tile queue), batches of
//   BATCH Gaussians (256): every thread gathers one Gaussian and writes its row
//   of M_g (Eq. 6, TF32 hi/lo, K = 16) into shared memory (Stage 2).
//   Each warp then owns its 32 pixels and, 16 Gaussians at a time, issues 2 (pixel
//   halves) x 2 (8-Gaussian n-blocks) x 2 (K-steps) mma.m16n8k8 (Stage 3)
//   with the constant M_p fragments in registers. The accumulator fragment spreads a
//   pixel's exponents over a lane quad, so they go through a per-warp shared buffer
//   (conflict-free: MMA row r is stored in buffer row 2r (r < 8) / 2(r-8)+1 of its
//   half, rows 20 words apart) and each lane reads back its own pixel's 16 values.
//   Compositing is the same as k_blend_tc's (Eq. 1, R-1..R-4, warp-uniform skip).
// Output is bit-identical for every BATCH (each exponent is the same MMA sum).
// ===========================================================================
constexpr int MMA_THREADS = 256;
constexpr int MMA_SUB = 16;            // Gaussians per MMA step (two n8 blocks)
constexpr int MMA_TS = 20;             // transpose-buffer row stride (words)

template <int BATCH>
struct SmemMMA {
    uint32_t Mg[BATCH][16];            // rows: word 4q + j holds K index q + 4j
    float4 rgb[BATCH];
    float tr[MMA_THREADS / 32][32 * MMA_TS];   // per-warp transpose buffer
    int tile;
};

__device__ __forceinline__ void mma_tf32_16x8x8(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// K index k of the pixel row [v_p | v_p | 0] (Eq. 7) for the pixel (x, y)
__device__ __forceinline__ uint32_t mp_word(int x, int y, int k) {
    const float xb = 7.5f - (float)x, yb = 7.5f - (float)y;
    const int kk = k < 6 ? k : (k < 12 ? k - 6 : -1);
    float v = 0.f;
    switch (kk) {
        case 0: v = xb * xb; break;
        case 1: v = yb * yb; break;
        case 2: v = xb * yb; break;
        case 3: v = xb; break;
        case 4: v = yb; break;
        case 5: v = 1.0f; break;
        default: v = 0.f;
    }
    return __float_as_uint(v);   // exact in TF32
}

#ifndef GS_MMA_MINB
#define GS_MMA_MINB 4
#endif
template <int BATCH>
__global__ void __launch_bounds__(MMA_THREADS, GS_MMA_MINB)
    k_blend_mma(const Splat *__restrict__ splat, const uint32_t *__restrict__ vals, const uint2 *__restrict__ ranges, int tile0, int ntiles, int gx,
                int W, int H, float bg0, float bg1, float bg2, float *__restrict__ out_rgb, float *__restrict__ out_T,
                uint32_t *tile_queue) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    SmemMMA<BATCH> &sm = *reinterpret_cast<SmemMMA<BATCH> *>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane & 3, r4 = lane >> 2;
    // compositor pixel of this thread = buffer row `lane` of its warp
    int x, y;
    pixel_of(threadIdx.x, x, y);
    // A fragments (M_p rows): MMA row r of pixel half h is buffer row 16h + (r < 8 ? 2r : 2(r-8)+1)
    uint32_t afr[2][2][4];
#pragma unroll
    for (int h = 0; h < 2; h++) {
        int px0, py0, px1, py1;
        pixel_of(warp * 32 + 16 * h + 2 * r4, px0, py0);       // MMA row r4
        pixel_of(warp * 32 + 16 * h + 2 * r4 + 1, px1, py1);   // MMA row r4 + 8
#pragma unroll
        for (int ks = 0; ks < 2; ks++) {
            afr[h][ks][0] = mp_word(px0, py0, 8 * ks + q);
            afr[h][ks][1] = mp_word(px1, py1, 8 * ks + q);
            afr[h][ks][2] = mp_word(px0, py0, 8 * ks + q + 4);
            afr[h][ks][3] = mp_word(px1, py1, 8 * ks + q + 4);
        }
    }
    float *tr = sm.tr[warp];
    pdl_wait();
    for (;;) {
        if (threadIdx.x == 0) sm.tile = tile0 + (int)atomicAdd(tile_queue, 1u);
        __syncthreads();
        const int tile = sm.tile;
        if (tile >= ntiles) break;
        const uint2 rg = ranges[tile];
        const float xc = (float)(GS_TILE * (tile % gx)) + 7.5f, yc = (float)(GS_TILE * (tile / gx)) + 7.5f;
        float T = 1.0f, C0 = 0.f, C1 = 0.f, C2 = 0.f, thr = LOG2_ALPHA_MIN;
        float tmin = T_MIN;   // GS_BLEND_STALE_THR: the stop threshold of T (+inf once stopped)
        bool wdone = false;
        // the record of Gaussian b + threadIdx.x is fetched one batch ahead, into registers,
        // so the gathers of batch k+1 overlap the MMAs and compositing of batch k
        float2 pm = make_float2(0.f, 0.f);
        float4 pco = make_float4(0.f, 0.f, 0.f, 1.f), pcol = make_float4(0.f, 0.f, 0.f, 0.f);
        auto fetch = [&](uint32_t b) {
            if (threadIdx.x < BATCH && b + threadIdx.x < rg.y) {
                const uint32_t gi = vals[b + threadIdx.x];
                pm = splat[gi].m;
                pco = splat[gi].co;
                pcol = splat[gi].col;
            }
        };
        fetch(rg.x);
        for (uint32_t b0 = rg.x; b0 < rg.y; b0 += BATCH) {
            if (__syncthreads_and(wdone)) break;   // every warp terminated (also: batch b0-1 consumed)
            const int cnt = (int)min((uint32_t)BATCH, rg.y - b0);
            const int i = threadIdx.x;
            if (i < ((cnt + MMA_SUB - 1) & ~(MMA_SUB - 1))) {
                uint32_t u[16];
                float4 col = make_float4(0.f, 0.f, 0.f, 0.f);
                if (i < cnt) {   // Eq. (6) row, log2 e and log2 o folded in (R-10), TF32 hi/lo (R-11)
                    col = pcol;
                    const float xh = pm.x - xc, yh = pm.y - yc;
                    const float A = pco.x, B = pco.y, C = pco.z;
                    float v[6];
                    v[0] = -0.5f * A * LOG2E;
                    v[1] = -0.5f * C * LOG2E;
                    v[2] = -B * LOG2E;
                    v[3] = -(A * xh + B * yh) * LOG2E;
                    v[4] = -(C * yh + B * xh) * LOG2E;
                    v[5] = -(0.5f * A * xh * xh + 0.5f * C * yh * yh + B * xh * yh) * LOG2E + lg2_approx(pco.w);
#pragma unroll
                    for (int k = 0; k < 6; k++) {
                        const uint32_t hi = f32_to_tf32_rna(v[k]);
                        u[k] = hi;
                        u[6 + k] = f32_to_tf32_rna(v[k] - __uint_as_float(hi));
                    }
                } else {   // padding row: exponent -1e30, never kept
#pragma unroll
                    for (int k = 0; k < 12; k++) u[k] = 0u;
                    u[5] = __float_as_uint(-1e30f);
                }
                u[12] = u[13] = u[14] = u[15] = 0u;
                uint4 *row = reinterpret_cast<uint4 *>(&sm.Mg[i][0]);
#pragma unroll
                for (int qq = 0; qq < 4; qq++) row[qq] = make_uint4(u[qq], u[qq + 4], u[qq + 8], u[qq + 12]);
                sm.rgb[i] = col;
            }
            fetch(b0 + BATCH);
            __syncthreads();
            if (wdone) continue;
            for (int g0 = 0; g0 < cnt; g0 += MMA_SUB) {
                // ---- exponents of 16 Gaussians for the warp's 32 pixels ----
                float d[2][2][4];
#pragma unroll
                for (int nb = 0; nb < 2; nb++) {
                    const uint4 bw = *reinterpret_cast<const uint4 *>(&sm.Mg[g0 + 8 * nb + r4][4 * q]);
#pragma unroll
                    for (int h = 0; h < 2; h++) {
#pragma unroll
                        for (int e = 0; e < 4; e++) d[h][nb][e] = 0.f;
                        mma_tf32_16x8x8(d[h][nb], afr[h][0], bw.x, bw.y);
                        mma_tf32_16x8x8(d[h][nb], afr[h][1], bw.z, bw.w);
                    }
                }
                __syncwarp();
#pragma unroll
                for (int h = 0; h < 2; h++)
#pragma unroll
                    for (int nb = 0; nb < 2; nb++) {
                        float *r0 = tr + (16 * h + 2 * r4) * MMA_TS + 8 * nb + 2 * q;
                        *reinterpret_cast<float2 *>(r0) = make_float2(d[h][nb][0], d[h][nb][1]);
                        *reinterpret_cast<float2 *>(r0 + MMA_TS) = make_float2(d[h][nb][2], d[h][nb][3]);
                    }
                __syncwarp();
                float m[MMA_SUB];
#pragma unroll
                for (int j = 0; j < MMA_SUB / 4; j++) {
                    const float4 t4 = *reinterpret_cast<const float4 *>(tr + lane * MMA_TS + 4 * j);
                    m[4 * j] = t4.x; m[4 * j + 1] = t4.y; m[4 * j + 2] = t4.z; m[4 * j + 3] = t4.w;
                }
                // ---- compositing, as k_blend_tc ----
                const uint32_t crow = smem_u32(&sm.rgb[g0]);
#pragma unroll
                for (int j = 0; j < MMA_SUB; j++) {
                    const float mj = m[j];
                    const bool live = mj >= thr;
                    if (__any_sync(0xffffffffu, live)) {
                        const float4 c = ld_shared_f4(crow + 16 * j);
                        const float a = fminf(ALPHA_MAX, ex2_approx(mj));
                        const float tT = fmaf(-a, T, T);
                        const float w = a * T;
                        const bool acc = live && tT >= T_MIN;
                        C0 = acc ? fmaf(w, c.x, C0) : C0;
                        C1 = acc ? fmaf(w, c.y, C1) : C1;
                        C2 = acc ? fmaf(w, c.z, C2) : C2;
                        T = acc ? tT : T;
                        thr = (live && !acc) ? __int_as_float(0x7f800000) : thr;
                    }
                }
                if (__all_sync(0xffffffffu, thr > 0.f)) {
                    wdone = true;
                    break;
                }
            }
        }
        const int px = GS_TILE * (tile % gx) + x, py = GS_TILE * (tile / gx) + y;
        if (px < W && py < H) {
            const size_t pix = (size_t)py * W + px, plane = (size_t)W * H;
            out_rgb[pix] = C0 + T * bg0;
            out_rgb[plane + pix] = C1 + T * bg1;
            out_rgb[2 * plane + pix] = C2 + T * bg2;
            out_T[pix] = T;
        }
        __syncthreads();   // sm.tile / the batch buffers are reused by the next tile
    }
}

template <int BATCH>
static void launch_mma_b(cudaStream_t st, int grid, const Splat *splat, const uint32_t *vals, const uint2 *ranges, int tile0, int ntiles, int gx, int W, int H,
                         const float bg[3], float *out_rgb, float *out_T, uint32_t *queue) {
    const size_t smem = sizeof(SmemMMA<BATCH>) + 128;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_blend_mma<BATCH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    launch_pdl(k_blend_mma<BATCH>, grid, MMA_THREADS, smem, st, splat, vals, ranges, tile0, ntiles, gx, W, H,
               bg[0], bg[1], bg[2], out_rgb, out_T, queue);
}

void launch_blend_mma(const Workspace &ws, cudaStream_t st, const Splat *splat, const uint32_t *vals, const uint2 *ranges, int tile0, int ntiles, int gx,
                      int W, int H, const float bg[3], float *out_rgb, float *out_T, int num_sms, int batch) {
    if (ntiles - tile0 <= 0) return;
    const int grid = std::max(1, std::min(GS_MMA_MINB * num_sms, ntiles - tile0));
    uint32_t *queue = &ws.counters->tile_queue;
    switch (batch) {
        case 32: launch_mma_b<32>(st, grid, splat, vals, ranges, tile0, ntiles, gx, W, H, bg, out_rgb, out_T, queue); break;
        case 64: launch_mma_b<64>(st, grid, splat, vals, ranges, tile0, ntiles, gx, W, H, bg, out_rgb, out_T, queue); break;
        case 128: launch_mma_b<128>(st, grid, splat, vals, ranges, tile0, ntiles, gx, W, H, bg, out_rgb, out_T, queue); break;
        default: launch_mma_b<256>(st, grid, splat, vals, ranges, tile0, ntiles, gx, W, H, bg, out_rgb, out_T, queue); break;
    }
}

}  // namespace gs
