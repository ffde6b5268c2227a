// gs_common.cuh -- shared definitions of the CUDA path (device workspace,
// constants, PTX wrappers for mbarrier / tcgen05 / TMEM on sm_100a).
// Product code only: nothing here is shared with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <utility>
#include <stdint.h>

#include "../../include/gs_render.h"

#define GS_TILE 16
#define GS_TILE_PIX 256

namespace gs {

// ---- per-frame device counters (zeroed once per frame) --------------------
struct Counters {
    uint32_t n_visible;        // compaction output
    uint32_t err;              // device-side error bits (1 = key capacity)
    uint64_t n_keys;           // K (64-bit: the capacity check is exact)
    uint32_t tile_queue;       // blend persistent work queue
    uint32_t n_rent;           // row entries (two-level binning): kept tile rows summed over Gaussians
    uint32_t n_cchunks;        // column-pass chunks (row-aligned, <= 4096 pairs each)
    uint32_t wide_depth;       // some visible depth key >= 2^27 above the near plane: 4th depth pass
    uint32_t n_spairs;         // supertile binning: (supertile, Gaussian) pairs
    unsigned long long pairs_eval;   // GS_FLAG_STATS: exponents computed by the blend
    unsigned long long pairs_kept;   // GS_FLAG_STATS: pairs composited or terminating
};

// errors of a multi-view call, accumulated over its views (each view's counters are
// reused by later views of the call): reset at the call's start, read by gs_last_stats
struct Sticky {
    uint32_t err;
    uint32_t pad;
    unsigned long long max_keys;   // largest K of the call's views (the capacity a retry needs)
};

constexpr int MAX_TILES = 1 << 20;   // 16384 x 16384 px; one-level binning sorts ceil(tile bits / 8) passes

// ---- the blend's per-Gaussian record ----------------------------------------
// One 48-byte record per visible Gaussian (slot-addressed), written by the preprocess:
// everything the blend reads of a Gaussian in one contiguous, 16-B aligned block, so
// the tcgen05 blend's producer fetches it with ONE bulk copy (cp.async.bulk, the TMA
// engine's 1-D form) straight into its shared-memory ring, and the other blends with
// three vector loads from two 32-B sectors (the SoA form touched three).
struct __align__(16) Splat {
    float2 m;      // projected mean (pixels)
    float2 aux;    // (0, 0): padding to the 16-B granule of the bulk copy
    float4 co;     // (A, B, C, opacity): conic of Eq. 3 and opacity
    float4 col;    // (r, g, b, 0): SH colour
};
static_assert(sizeof(Splat) == 48, "48-byte splat record");

// ---- what the blend reads for a tile -----------------------------------------
// Per-tile lists (the two-level / one-level binning, or a caller's lists): the tile's
// Gaussian slots vals[ranges[t].x .. ranges[t].y). Supertile lists (the tcgen05 blend's
// default, binning.cu "Supertile binning"): the range of the tile's 4 x 4-tile supertile
// (sgx supertiles per row) and keys with the tile mask in bits 16-31; the tile's list is
// the entries whose mask has bit 16 + 4 (ty % 4) + tx % 4, in list order.
struct TileLists {
    const uint32_t *vals;
    const uint32_t *keys;     // nullptr: per-tile lists
    const uint2 *ranges;
    int sgx;
};

__device__ __forceinline__ uint32_t lanemask_lt_u32() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ---- device workspace owned by the context ---------------------------------
struct Workspace {
    // per Gaussian SLOT (max_points): the preprocess packs the visible Gaussians of each
    // warp of 32 (index order) at the start of the warp's 32 slots (culled ones write
    // nothing); slot s is used iff s % 32 < wcount[s / 32]. The per-Gaussian arrays below
    // are slot-addressed; the binning's values, and hence the blend's gathers, are slots.
    uint32_t *wcount;          // [N/32+1] visible Gaussians per warp of 32
    uint32_t *orig;            // [N] Gaussian index of each used slot (debug outputs)
    uint32_t *depth_bits;      // [N] raw IEEE bits of the camera depth
    Splat *splat;              // [N] what the blend reads: mean, conic + opacity, colour (48 B AoS)
    ushort4 *rect;             // [N] (xmin, ymin, xmax, ymax) tiles, half-open
    uint32_t *touched;         // [N] tiles touched (0 = culled); with GS_FLAG_TIGHT: tiles kept
    unsigned long long *tmask; // [N] GS_FLAG_TIGHT: kept tiles of the rect (bit ty*w+tx), ~0 = all
    int32_t *radius;           // [N] pixel radius (debug output)
    uint32_t *sk[2];           // [N] depth keys of the visible Gaussians, ping-pong
    uint32_t *sv[2];           // [N] their indices; sv[0] = depth order after the sort
    uint32_t *off;             // [N] first pair of each depth-ordered Gaussian
    ushort4 *rect_r;           // [N] rect of each depth-ordered Gaussian
    unsigned long long *tmask_r;   // [N] its tile mask (GS_FLAG_TIGHT)
    // per key (max_keys)
    uint32_t *kt[2];           // [K] tile ids, ping-pong; kt[0] final
    uint32_t *kv[2];           // [K] Gaussian indices, ping-pong; kv[0] final
    uint32_t *chunk_first;     // [K/4096+1] Gaussian holding the first pair of each chunk
    // per tile
    uint2 *ranges;             // [tiles] [start, end) into kv[0]
    // two-level binning (tile rows, then columns)
    uint4 *cdesc;              // [max_chunks] column chunk: (tile row, first pair, pairs, first entry)
    uint32_t *cdesc_last;      // [max_chunks] last row entry of the chunk
    uint32_t *tile_cnt;        // [tiles] pairs per tile
    uint32_t *rowinfo;         // [3][513] per tile row: first entry, first pair, first column chunk
    // reduce-then-scan scratch (4096-element chunks)
    uint32_t *sums;            // [max_chunks] chunk sums of the order-preserving scans
    uint32_t *cmat;            // [512][max_chunks] per-chunk digit counts -> offsets
    uint32_t *row_total;       // [512] digit totals
    size_t max_chunks;
    int list_sgx;              // lists of the last binning: supertiles per row, 0 = per-tile lists
    Counters *counters;
    Sticky *sticky;            // the context's (shared by every workspace)
    // scene staging for the host-pointer entry point
    float *stage;
    size_t stage_bytes;
};

// intersection mode of the preprocess: 0 vanilla rect, 1 GS_FLAG_TIGHT (box + per-row
// column runs, tile masks), 2 GS_FLAG_OBOX (vanilla rect clipped to the opacity-aware box)
inline int intersect_mode(unsigned flags) {
    return (flags & GS_FLAG_TIGHT) ? 1 : ((flags & GS_FLAG_OBOX) ? 2 : 0);
}

// ---- per-view outputs of the preprocess (a view group shares one scene read) ----
struct PreOut {
    uint32_t *wcount;
    uint32_t *orig;
    uint32_t *depth_bits;
    Splat *splat;
    ushort4 *rect;
    uint32_t *touched;
    unsigned long long *tmask;
    int32_t *radius;           // nullptr: not written (debug output only)
    Counters *counters;        // zeroed by the preprocess
};
#ifndef GS_MAX_VIEW_GROUP
#define GS_MAX_VIEW_GROUP 16
#endif
constexpr int MAX_VIEW_GROUP = GS_MAX_VIEW_GROUP;  // views per preprocess launch (gs_set_view_group; default 4)
struct PreViews {
    gs_camera cam[MAX_VIEW_GROUP];
    PreOut out[MAX_VIEW_GROUP];
    int n;
    int band_y0, band_y1;      // tile rows rendered (row band of a split frame; 0, gy = all)
};

// tile rows [y0, y1) of band `band` of n_bands (n_bands <= 1: the whole grid of gy rows)
inline void band_rows(int gy, int band, int n_bands, int &y0, int &y1) {
    if (n_bands <= 1) {
        y0 = 0;
        y1 = gy;
        return;
    }
    y0 = (int)((long long)band * gy / n_bands);
    y1 = (int)((long long)(band + 1) * gy / n_bands);
}

// Chunk geometry of the single-pass scans / onesweep radix passes.
#ifndef GS_SORT_THREADS
#define GS_SORT_THREADS 256
#endif
constexpr int SORT_THREADS = GS_SORT_THREADS;
#ifndef GS_SORT_ITEMS
#define GS_SORT_ITEMS 12
#endif
constexpr int SORT_ITEMS = GS_SORT_ITEMS;   // elements per thread of a radix / scan chunk
constexpr int SORT_CHUNK = SORT_THREADS * SORT_ITEMS;   // 3072 keys per chunk (sweep: 12 items/thread beats 8, 10, 14, 16, 32)

__host__ __device__ inline int ceil_div_i(long long a, long long b) { return (int)((a + b - 1) / b); }

// ---- programmatic dependent launch ------------------------------------------
// Every kernel of the frame path is launched with programmatic stream
// serialisation and calls pdl_wait() before it touches its predecessor's results,
// so its launch (and any setup before the wait) overlaps the predecessor's tail.
// Without the launch attribute griddepcontrol.wait is a no-op.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

extern int g_pdl;   // 1 (default): programmatic dependent launch on; GS_PDL=0 turns it off (A/B)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---- small PTX helpers ------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// mbarrier
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cnt(uint64_t *bar, uint32_t cnt) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(cnt) : "memory");
}
// arrive (count 1) and raise the phase's expected transaction bytes by `bytes`
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// 1-D bulk copy global -> shared by the TMA engine (SASS UBLKCP): `bytes` (multiple of 16,
// both addresses 16-B aligned) land in dst, then complete `bytes` transaction bytes on bar
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// TMA tensor stores shared -> global (SASS UTMASTG), tracked by the issuing thread's bulk
// async-groups; the source must be made visible to the async proxy first
// (fence_proxy_async_smem + a barrier). Out-of-range box elements are not written.
__device__ __forceinline__ void tma_store_3d(const void *tmap, const void *src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(tmap),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
__device__ __forceinline__ void tma_store_2d(const void *tmap, const void *src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(tmap),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit_group() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// all but the most recent group have finished READING their shared-memory source
__device__ __forceinline__ void bulk_wait_group_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
// every group has completed (its global writes performed)
__device__ __forceinline__ void bulk_wait_group_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// Waits for the phase with the given parity. The suspend-time hint lets a
// waiting warp sleep in hardware until the phase completes instead of
// spinning (spinning warps took a third of the blend's issue slots).
#ifndef GS_MBAR_SUSPEND_NS
#define GS_MBAR_SUSPEND_NS 0x100000
#endif
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
#if GS_MBAR_SUSPEND_NS > 0
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"((uint32_t)GS_MBAR_SUSPEND_NS)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
#endif
}

// tcgen05 / TMEM
__device__ __forceinline__ void tmem_alloc(uint32_t *dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
}
__device__ __forceinline__ void tmem_relinquish() {
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, kind::tf32, both K-major
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 32 lanes x 32 consecutive columns: thread i receives row (lane base + i), cols c..c+31
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
#pragma unroll
    for (int i = 0; i < 16; i++) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
#pragma unroll
    for (int i = 0; i < 32; i++) v[i] = __uint_as_float(r[i]);
}

// UMMA shared-memory descriptor, K-major, no swizzle (core matrix = 8 rows x 16 B).
//   LBO = byte distance between the two core matrices adjacent in K,
//   SBO = byte distance between core-matrix groups adjacent in M/N.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;     // descriptor version (sm100)
    // base offset 0, lbo mode 0, layout type 0 = SWIZZLE_NONE
    return d;
}

// Instruction descriptor for kind::tf32: D f32, A/B tf32, both K-major.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4)                 // D format f32
           | (2u << 7)               // A format tf32
           | (2u << 10)              // B format tf32
           | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float lg2_approx(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// Round to TF32 (10 explicit mantissa bits), to nearest with ties away from zero:
// add half of the dropped 13-bit ulp to the magnitude bits and truncate. Same bits
// as cvt.rna.tf32.f32 for every finite input (ptxas expands that instruction into
// this plus an Inf/NaN guard; the operands here are always finite).
__device__ __forceinline__ uint32_t f32_to_tf32_rna(float x) {
    return (__float_as_uint(x) + 0x1000u) & 0xffffe000u;
}

// log2(1/255) in binary32: the alpha-skip threshold in the log2 domain (R-1)
constexpr float LOG2_ALPHA_MIN = -7.99435329f;
constexpr float LOG2E = 1.4426950408889634f;
constexpr float T_MIN = 1e-4f;    // early termination (R-2)
constexpr float ALPHA_MAX = 0.99f; // alpha cap (R-4)

}  // namespace gs

// host-side launch helpers (defined in the respective .cu files)
namespace gs {
void launch_preprocess(const Workspace &ws, cudaStream_t st, int N, const float *means, const float *scales,
                       const float *rots, const float *opacity, const float *shs, int sh_degree,
                       int sh_stride, float scale_mod, const gs_camera &cam, int W, int H, int imode,
                       bool with_radius, int band_y0, int band_y1);
PreOut pre_out_of(const Workspace &ws, bool with_radius);
void launch_preprocess_views(const PreViews &pv, cudaStream_t st, int N, const float *means, const float *scales,
                             const float *rots, const float *opacity, const float *shs, int sh_degree,
                             int sh_stride, float scale_mod, int W, int H, int imode);
int launch_binning(Workspace &ws, cudaStream_t st, int N, int64_t max_keys, int ntiles, int gx,
                   uint32_t &epoch, bool tight, float znear, bool concurrent, bool supertile);
int supertile_count(int gx, int gy);   // 4 x 4-tile supertiles of a gx x gy tile grid
void launch_blend_tc(const Workspace &ws, cudaStream_t st, const Splat *splat, const TileLists &lists, int tile0,
                     int ntiles, int gx, int W, int H, const float bg[3], float *out_rgb, float *out_T, float *dump_m,
                     int num_sms, bool stats, bool colour_mma);
extern long long *g_blend_trace;
void launch_blend_mma(const Workspace &ws, cudaStream_t st, const Splat *splat, const uint32_t *vals, const uint2 *ranges, int tile0, int ntiles, int gx,
                      int W, int H, const float bg[3], float *out_rgb, float *out_T, int num_sms, int batch);
void launch_blend_direct(cudaStream_t st, const Splat *splat, const uint32_t *vals, const uint2 *ranges, int tile0, int ntiles, int gx, int W, int H,
                         const float bg[3], float *out_rgb, float *out_T, const Counters *counters);
}  // namespace gs
