// binning.cu -- stages (b) "Duplication" and (c) "Sorting"
// and the per-tile ranges, as hand-written kernels (no CUB, no host
// synchronisation: every count stays on the device, so a frame is
// graph-capturable).
//
// Canonical result (R-12/R-13): each tile's Gaussians in the order of
// key = tile << 32 | depth bits, ties by Gaussian index. The paper's "duplicate
// with a concatenated key, then radix-sort" over 64-bit keys costs
// ~6 LSD passes over every pair; here the depth half is sorted once per
// *Gaussian* instead of once per pair:
//   1. compaction of the visible Gaussians (order-preserving scan), keys relative
//      to the near plane
//   2. stable LSD sort of the N_vis depth keys, 3 passes of 9 bits (a 4th pass
//      only if a depth key reaches 2^27; ties keep index order); the last pass
//      gathers each Gaussian's rect into depth order
//   3. the tile grouping, in one of two forms:
//      a. supertile lists (the tcgen05 blend, grids <= 512 supertiles): the
//         depth-ordered Gaussians expanded to (4x4-tile supertile, Gaussian) pairs
//         with a 16-bit tile mask each, ONE stable 9-bit pass on the supertile id
//         (expansion fused into its count and scatter), ranges from the digit
//         totals; a tile's list is its supertile's list filtered by its mask bit,
//         which the blend's producer does on the fly;
//      b. per-tile lists (the other blends, larger grids): two-level -- tile-row
//         entries, one stable pass on the row, pair offsets, one stable pass on the
//         column with the tile ranges from the column counts -- or, for grids wider
//         or taller than 512 tiles, one-level (all K (tile, index) pairs, ceil(tile
//         bits / 8) stable passes, ranges by boundary detection).
// Every scan / radix pass is reduce-then-scan over 3072-element chunks: count
// (shared-memory histograms, or run-length difference arrays for the expanding
// loaders) -> scan of the [digit][chunk] count matrix (one block per digit) ->
// stable scatter through shared memory with warp-ballot ranks. No block ever
// waits on another block (a decoupled look-back variant spent most of its time
// spinning on its predecessors).
#include <algorithm>
#include <cstring>

#include "gs_common.cuh"

namespace gs {

constexpr int NWARP = SORT_THREADS / 32;
// radix / scan grids: at most this many blocks per SM (grid-stride over chunks). A chain
// running alone (gs_render) wants wide grids; the concurrent chains of a view group share
// the GPU, and narrower grids let them interleave (sweep: 8 -> 4 is +1.5 % orbit fps).
#ifndef GS_GRID_MULT
#define GS_GRID_MULT 8
#endif
#ifndef GS_SCATTER_MINB
#define GS_SCATTER_MINB 3   // resident blocks per SM of the unpacked radix scatter (register cap)
#endif
#ifndef GS_SCATTER_MINB_PK
#define GS_SCATTER_MINB_PK 5   // the packed (column) scatter
#endif
#ifndef GS_SCAN_MINB
#define GS_SCAN_MINB 6   // minimum resident blocks of the scan kernels (0: not specified; 6: 40 registers, +0.8 % orbit fps)
#endif
#if GS_SCAN_MINB > 0
#define GS_SCAN_BOUNDS __launch_bounds__(SORT_THREADS, GS_SCAN_MINB)
#else
#define GS_SCAN_BOUNDS __launch_bounds__(SORT_THREADS)
#endif
#ifndef GS_COUNT_ILP
#define GS_COUNT_ILP 4   // Gaussians / row entries per thread per round in the run-count loops
#endif
constexpr int COUNT_ILP = GS_COUNT_ILP;
#ifndef GS_COUNT_NH
#define GS_COUNT_NH 4          // privatised shared histograms of the count kernel
#endif
#ifndef GS_GRID_MULT_CONCURRENT
#define GS_GRID_MULT_CONCURRENT 3   // r2 sweep: 3 vs 4 -> 1688 / 1688 / 1685 vs 1679 / 1680 / 1675 fps (profiles/r2_sweep_ac.txt)
#endif

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Element e of a 4096-element chunk lives in warp e/512, round (e/32)%16, lane e%32:
// each warp owns a contiguous range, so warp-local ranking in round order is stable.
__device__ __forceinline__ int elem_of(int w, int r, int lane) { return w * (SORT_ITEMS * 32) + r * 32 + lane; }

// Warp multisplit on a DBITS-bit digit: mask of the lanes holding the same digit.
// Ballots: 0.46 ns/element/SM on sm_100a for 8 bits with distinct digits, vs 1.0
// for match.any (tools/microbench_rank.cu); counting alone uses shared atomics
// (0.04 ns/element/SM). Each bit is 4 SASS instructions (LOP3->P, VOTE, predicated
// NOT, AND); the plain C++ form compiled to 7. Only the digit's significant bits
// are voted on, so the last, narrow pass of a sort costs proportionally less.
template <int DBITS>
__device__ __forceinline__ uint32_t peers_of(uint32_t d, bool valid) {
    uint32_t peers = __ballot_sync(0xffffffffu, valid);
    if (!valid) peers = ~peers;
#pragma unroll
    for (int b = 0; b < DBITS; b++) {
        asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
            "and.b32 t, %1, %2;\n\t"
            "setp.ne.u32 p, t, 0;\n\t"
            "vote.sync.ballot.b32 t, p, 0xffffffff;\n\t"
            "@!p not.b32 t, t;\n\t"
            "and.b32 %0, %0, t;\n\t}"
            : "+r"(peers)
            : "r"(d), "r"(1u << b));
    }
    return peers;
}

// ---------------------------------------------------------------------------
// element counts (device-resident)
// ---------------------------------------------------------------------------
enum : int { CNT_POINTS = 0, CNT_VISIBLE = 1, CNT_KEYS = 2, CNT_RENT = 3, CNT_VISIBLE_WIDE = 4, CNT_SPAIRS = 5 };
__device__ __forceinline__ uint32_t count_of(const Counters *c, int which, uint32_t n_points, uint64_t max_keys) {
    if (which == CNT_POINTS) return n_points;
    if (which == CNT_VISIBLE) return c->n_visible;
    if (which == CNT_VISIBLE_WIDE) return c->wide_depth ? c->n_visible : 0u;   // 4th depth pass only if needed
    if (which == CNT_RENT) return c->err ? 0u : c->n_rent;   // > max_keys sets err
    if (which == CNT_SPAIRS) return c->err ? 0u : c->n_spairs;   // K > max_keys sets err
    const uint64_t k = c->n_keys;
    return c->err ? 0u : (uint32_t)(k < max_keys ? k : max_keys);
}

// ---------------------------------------------------------------------------
// order-preserving scans (reduce -> scan sums -> apply)
// ---------------------------------------------------------------------------
// The depth key is stored relative to the near plane: key = bits(z) - bits(znear).
// Every visible z > znear > 0, so the subtraction keeps the order of the raw bits
// (R-13), and depths below znear * 2^16 (13107 at znear 0.2) give keys < 2^27:
// three 9-bit passes sort them; a larger key sets wide_depth and a 4th pass runs.
struct CompactOp {   // used slots -> (depth key, slot) of the visible Gaussians, index order
    const uint32_t *wcount, *depth_bits;   // slot s is used iff s % 32 < wcount[s / 32]
    uint32_t *out_k, *out_v;
    Counters *cnt;
    uint32_t dbase;   // bits(znear) if znear > 0, else 0 (raw bits, always 4 passes)
    static constexpr int WHICH = CNT_POINTS;
    static constexpr bool SIDE = false;
    struct Aux {
        uint32_t depth;
    };
    __device__ uint32_t load(uint32_t i) const { return (i & 31u) < wcount[i >> 5] ? 1u : 0u; }
    __device__ uint32_t load(uint32_t i, Aux &a) const {
        a.depth = depth_bits[i];   // unconditional: both loads in flight at once
        return (i & 31u) < wcount[i >> 5] ? 1u : 0u;
    }
    __device__ void emit(uint32_t i, uint64_t pos, uint32_t v, const Aux &a) const {
        if (v) {
            const uint32_t k = a.depth - dbase;
            out_k[pos] = k;
            out_v[pos] = i;
            if (k >= (1u << 27)) cnt->wide_depth = 1u;
        }
    }
    __device__ void finish(uint64_t total) const { cnt->n_visible = (uint32_t)total; }
};

struct OffsetsOp {   // tiles_touched in depth order -> pair offsets (+ chunk heads)
    const uint32_t *sorted_idx, *touched;
    uint32_t *off;
    uint32_t *chunk_first;
    Counters *cnt;
    uint64_t max_keys;
    static constexpr int WHICH = CNT_VISIBLE;
    static constexpr bool SIDE = false;
    struct Aux {};
    __device__ uint32_t load(uint32_t r) const { return touched[sorted_idx[r]]; }
    __device__ uint32_t load(uint32_t r, Aux &) const { return touched[sorted_idx[r]]; }
    __device__ void emit(uint32_t r, uint64_t o, uint32_t v, const Aux &) const {
        off[r] = (uint32_t)(o < 0xFFFFFFFFull ? o : 0xFFFFFFFFull);
        // every 4096-pair chunk boundary inside [o, o+v) belongs to Gaussian r
        for (uint64_t c = (o + SORT_CHUNK - 1) / SORT_CHUNK; c * SORT_CHUNK < o + v; c++)
            if (c * SORT_CHUNK < max_keys) chunk_first[c] = r;
    }
    __device__ void finish(uint64_t total) const {
        cnt->n_keys = total;
        if (total > max_keys) atomicOr(&cnt->err, 1u);
    }
};

template <class Op>
__global__ void GS_SCAN_BOUNDS k_scan_reduce(Op op, uint32_t n_points, uint32_t *sums, uint32_t *sums2) {
    pdl_wait();
    __shared__ uint32_t s_w[NWARP], s_w2[NWARP];
    const uint32_t n = count_of(op.cnt, Op::WHICH, n_points, 0);
    const uint32_t nchunks = (n + SORT_CHUNK - 1) / SORT_CHUNK;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        uint32_t acc = 0, acc2 = 0;
#pragma unroll
        for (int r = 0; r < SORT_ITEMS; r++) {
            const uint32_t e = c * SORT_CHUNK + elem_of(warp, r, lane);
            if (e < n) {
                acc += op.load(e);
                if constexpr (Op::SIDE) acc2 += op.side(e);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if constexpr (Op::SIDE) acc2 += __shfl_xor_sync(0xffffffffu, acc2, o);
        }
        if (lane == 0) {
            s_w[warp] = acc;
            s_w2[warp] = acc2;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t t = 0, t2 = 0;
            for (int w = 0; w < NWARP; w++) {
                t += s_w[w];
                t2 += s_w2[w];
            }
            sums[c] = t;
            if constexpr (Op::SIDE) sums2[c] = t2;
        }
        __syncthreads();
    }
}

// Each block computes its chunk's exclusive prefix itself, as the 64-bit sum of the
// chunk sums before it (at most a few thousand L2-resident words: no separate
// single-block scan of the sums, one launch and one dependency fewer); the block of
// the last chunk also reports the total (op.finish).
template <class Op>
__global__ void GS_SCAN_BOUNDS k_scan_apply(Op op, uint32_t n_points, const uint32_t *sums, const uint32_t *sums2) {
    pdl_wait();
    __shared__ uint32_t s_w[NWARP];
    __shared__ unsigned long long s_pre[NWARP], s_tot[NWARP], s_tot2[NWARP], s_base;
    const uint32_t n = count_of(op.cnt, Op::WHICH, n_points, 0);
    const uint32_t nchunks = (n + SORT_CHUNK - 1) / SORT_CHUNK;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        uint32_t v[SORT_ITEMS], rex[SORT_ITEMS], wrun = 0;
        typename Op::Aux aux[SORT_ITEMS];
#pragma unroll
        for (int r = 0; r < SORT_ITEMS; r++) {
            const uint32_t e = c * SORT_CHUNK + elem_of(warp, r, lane);
            v[r] = e < n ? op.load(e, aux[r]) : 0u;
        }
        // (the element loads above are in flight meanwhile)
        {   // prefix of the chunk sums before c (and, for the last chunk, the total)
            const bool last = c + 1 == nchunks;
            unsigned long long acc = 0, tot = 0, tot2 = 0;
            for (uint32_t k = threadIdx.x; k < (last ? nchunks : c); k += SORT_THREADS) {
                const unsigned long long x = sums[k];
                if (k < c) acc += x;
                tot += x;
                if constexpr (Op::SIDE) {
                    if (last) tot2 += sums2[k];
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                acc += __shfl_xor_sync(0xffffffffu, acc, o);
                tot += __shfl_xor_sync(0xffffffffu, tot, o);
                if constexpr (Op::SIDE) tot2 += __shfl_xor_sync(0xffffffffu, tot2, o);
            }
            if (lane == 0) {
                s_pre[warp] = acc;
                s_tot[warp] = tot;
                s_tot2[warp] = tot2;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                unsigned long long p = 0, t = 0, t2 = 0;
                for (int w = 0; w < NWARP; w++) {
                    p += s_pre[w];
                    t += s_tot[w];
                    t2 += s_tot2[w];
                }
                s_base = p;
                if (last) {
                    if constexpr (Op::SIDE) op.finish(t, t2);
                    else op.finish(t);
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int r = 0; r < SORT_ITEMS; r++) {
            uint32_t x = v[r];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            rex[r] = wrun + x - v[r];
            wrun += __shfl_sync(0xffffffffu, x, 31);
        }
        if (lane == 0) s_w[warp] = wrun;
        __syncthreads();
        uint64_t base = s_base;
        for (int w = 0; w < warp; w++) base += s_w[w];
#pragma unroll
        for (int r = 0; r < SORT_ITEMS; r++) {
            const uint32_t e = c * SORT_CHUNK + elem_of(warp, r, lane);
            if (e < n) op.emit(e, base + rex[r], v[r], aux[r]);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// loaders: a chunk's keys (and values) into shared memory
// ---------------------------------------------------------------------------
// Chunking of a radix pass: linear 4096-element chunks over n elements; the digit
// bases come from the digit totals (s_dbase). Loaders derive from this unless they
// define their own chunks (ColLoader).
struct LinearChunks {
    __device__ void epilogue(uint32_t, uint32_t) const {}   // per scattered element (g = slot, v = value)
    bool keys_if_wide = false;   // the last depth pass: its keys are only read by the 4th (wide) pass
    static constexpr bool PACKED = false;       // key = digit | value << PACK_SHIFT, no separate values
    static constexpr int PACK_SHIFT = 0;
    static constexpr bool EXPANDS = false;      // keys via key(i) from global memory
    static constexpr bool RUN_COUNTS = false;   // digit counts from runs (count_runs)
    __device__ uint32_t nchunks(uint32_t n) const { return (n + SORT_CHUNK - 1) / SORT_CHUNK; }
    __device__ void chunk(uint32_t c, uint32_t n, uint32_t &cbase, uint32_t &cvalid) const {
        cbase = c * SORT_CHUNK;
        cvalid = min((uint32_t)SORT_CHUNK, n - cbase);
    }
    __device__ uint32_t digit_base(uint32_t, uint32_t d, const uint32_t *s_dbase) const { return s_dbase[d]; }
};

struct PlainLoader : LinearChunks {
    const uint32_t *keys, *vals;
    // final depth pass: gather each Gaussian's rect (and tile mask) into depth order
    // as it is scattered, so later passes read them contiguously (nullptr: off)
    const ushort4 *g_rect = nullptr;
    ushort4 *g_rect_out = nullptr;
    const unsigned long long *g_tmask = nullptr;
    unsigned long long *g_tmask_out = nullptr;
    static constexpr int SCRATCH_WORDS = 0;
    __device__ void epilogue(uint32_t g, uint32_t v) const {
        if (g_rect_out) {
            g_rect_out[g] = g_rect[v];
            if (g_tmask_out) g_tmask_out[g] = g_tmask[v];
        }
    }
    __device__ uint32_t key(uint32_t i) const { return __ldcs(keys + i); }
    __device__ void load(uint32_t, uint32_t cbase, uint32_t cvalid, uint32_t *sk, uint32_t *sv, uint32_t *) const {
        uint32_t k[SORT_ITEMS], v[SORT_ITEMS];   // all loads in flight before the first use
#pragma unroll
        for (int q = 0; q < SORT_ITEMS; q++) {
            const uint32_t e = threadIdx.x + q * SORT_THREADS;
            if (e < cvalid) {
                k[q] = __ldcs(keys + cbase + e);
                if (sv) v[q] = __ldcs(vals + cbase + e);
            }
        }
#pragma unroll
        for (int q = 0; q < SORT_ITEMS; q++) {
            const uint32_t e = threadIdx.x + q * SORT_THREADS;
            if (e < cvalid) {
                sk[e] = k[q];
                if (sv) sv[e] = v[q];
            }
        }
    }
};

// Pairs cbase .. cbase+cvalid-1 of the depth-ordered duplication: pair p belongs
// to the Gaussian r with off[r] <= p < off[r+1]; it is the (p - off[r])-th tile
// of rect_r[r] in row-major order; value = sorted_idx[r].
// q-th set bit of a 64-bit mask
__device__ __forceinline__ uint32_t nth_set64(unsigned long long m, uint32_t q) {
    const uint32_t lo = (uint32_t)m, hi = (uint32_t)(m >> 32);
    const uint32_t c = __popc(lo);
    return q < c ? __fns(lo, 0, (int)q + 1) : 32u + __fns(hi, 0, (int)(q - c) + 1);
}

struct Expander {
    const uint32_t *off, *sorted_idx, *chunk_first;
    const ushort4 *rect_r;
    const unsigned long long *tmask_r;   // GS_FLAG_TIGHT: the q-th pair is the q-th kept tile
    const Counters *cnt;
    int gx;
    static constexpr int STAGE = 1024;                            // Gaussians staged in shared memory
    static constexpr int SCRATCH_WORDS = SORT_CHUNK + 6 * STAGE;  // owner map + (off, rect, idx, mask)
    __device__ void load(uint32_t cbase, uint32_t cvalid, uint32_t *sk, uint32_t *sv, uint32_t *scratch) const {
        uint32_t *s_owner = scratch;
        uint32_t *s_off = scratch + SORT_CHUNK;
        ushort4 *s_rect = reinterpret_cast<ushort4 *>(scratch + SORT_CHUNK + STAGE);
        uint32_t *s_idx = scratch + SORT_CHUNK + 3 * STAGE;
        unsigned long long *s_msk = reinterpret_cast<unsigned long long *>(scratch + SORT_CHUNK + 4 * STAGE);
        const uint32_t nv = cnt->n_visible;
        const uint32_t chunk = cbase / SORT_CHUNK;
        const uint32_t nchunks = (uint32_t)((cnt->n_keys + SORT_CHUNK - 1) / SORT_CHUNK);
        const uint32_t r_lo = chunk_first[chunk];
        const uint32_t r_hi = chunk + 1 < nchunks ? min(nv - 1, chunk_first[chunk + 1]) : nv - 1;
        const uint32_t n_g = r_hi - r_lo + 1;
        const bool staged = n_g <= (uint32_t)STAGE;
        for (uint32_t e = threadIdx.x; e < SORT_CHUNK; e += SORT_THREADS) s_owner[e] = 0u;
        if (staged) {
            for (uint32_t j = threadIdx.x; j < n_g; j += SORT_THREADS) {
                s_off[j] = off[r_lo + j];
                s_rect[j] = rect_r[r_lo + j];
                s_idx[j] = sorted_idx[r_lo + j];
                s_msk[j] = tmask_r ? tmask_r[r_lo + j] : ~0ull;
            }
        }
        __syncthreads();
        // segment heads: the Gaussian starting at pair cbase+e owns e, e+1, ...
        for (uint32_t j = 1 + threadIdx.x; j < n_g; j += SORT_THREADS) {
            const uint32_t o = staged ? s_off[j] : off[r_lo + j];
            if (o < cbase + cvalid) s_owner[o - cbase] = j;   // >= 1 pair each: heads are distinct
        }
        __syncthreads();
        {   // inclusive max-scan over the chunk (thread-blocked, 16 consecutive each)
            __shared__ uint32_t s_w[NWARP];
            const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
            const int e0 = threadIdx.x * SORT_ITEMS;
            uint32_t m = 0, loc[SORT_ITEMS];
#pragma unroll
            for (int q = 0; q < SORT_ITEMS; q++) {
                m = max(m, s_owner[e0 + q]);
                loc[q] = m;
            }
            uint32_t x = m;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x = max(x, y);
            }
            if (lane == 31) s_w[w] = x;
            __syncthreads();
            uint32_t pre = __shfl_up_sync(0xffffffffu, x, 1);
            if (lane == 0) pre = 0;
            for (int ww = 0; ww < w; ww++) pre = max(pre, s_w[ww]);
#pragma unroll
            for (int q = 0; q < SORT_ITEMS; q++) s_owner[e0 + q] = max(pre, loc[q]);
            __syncthreads();
        }
        for (uint32_t e = threadIdx.x; e < cvalid; e += SORT_THREADS) {
            const uint32_t j = s_owner[e];
            const uint32_t o = staged ? s_off[j] : off[r_lo + j];
            const ushort4 rc = staged ? s_rect[j] : rect_r[r_lo + j];
            uint32_t q = cbase + e - o;
            const uint32_t w = (uint32_t)(rc.z - rc.x);
            if (tmask_r) {
                const unsigned long long msk = staged ? s_msk[j] : tmask_r[r_lo + j];
                if (msk != ~0ull) q = nth_set64(msk, q);   // q-th kept tile of the rect
            }
            // q / w through a float reciprocal (q < 2^24), corrected to the exact quotient
            uint32_t qy = (uint32_t)((float)q * __frcp_rn((float)w));
            if (qy * w > q) qy--;
            else if ((qy + 1) * w <= q) qy++;
            const uint32_t ty = rc.y + qy, tx = rc.x + (q - qy * w);
            sk[cbase + e] = ty * (uint32_t)gx + tx;
            sv[cbase + e] = staged ? s_idx[j] : sorted_idx[r_lo + j];
        }
    }
};

// writes the K (tile, index) pairs in depth order: one 4096-pair chunk per iteration
__global__ void __launch_bounds__(SORT_THREADS) k_expand(Expander ex, uint64_t max_keys, uint32_t *kout,
                                                         uint32_t *vout) {
    pdl_wait();
    extern __shared__ uint32_t dyn[];
    const uint32_t n = count_of(ex.cnt, CNT_KEYS, 0, max_keys);
    const uint32_t nchunks = (n + SORT_CHUNK - 1) / SORT_CHUNK;
    for (uint32_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        const uint32_t cbase = c * SORT_CHUNK, cvalid = min((uint32_t)SORT_CHUNK, n - cbase);
        ex.load(cbase, cvalid, kout, vout, dyn);
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// radix pass, step 1: per-chunk digit counts -> cmat[digit][chunk]
// ---------------------------------------------------------------------------
template <class Loader, int NDIG>
__global__ void __launch_bounds__(SORT_THREADS) k_rs_count(Loader ld, const Counters *cnt, int which,
                                                           uint64_t max_keys, int shift, uint32_t *cmat,
                                                           uint32_t ldm) {
    pdl_wait();
    static_assert(NDIG == 256 || NDIG == 512, "8- or 9-bit digits");
    constexpr int DPT = NDIG / SORT_THREADS;   // digits per thread
    extern __shared__ uint32_t dyn[];          // expanding loaders: the chunk's keys + loader scratch
    constexpr int NH = GS_COUNT_NH;            // privatised histograms (warp % NH)
    __shared__ uint32_t s_h[NH][NDIG];
    __shared__ uint32_t s_w[NWARP];
    const uint32_t n = count_of(cnt, which, 0, max_keys);
    const uint32_t nchunks = ld.nchunks(n);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (uint32_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        uint32_t cbase, cvalid;
        ld.chunk(c, n, cbase, cvalid);
        if constexpr (Loader::RUN_COUNTS) {
            int *s_diff = reinterpret_cast<int *>(&s_h[0][0]);   // NDIG + 1 entries
            for (int i = threadIdx.x; i <= NDIG; i += SORT_THREADS) s_diff[i] = 0;
            __syncthreads();
            ld.count_runs(c, cbase, cvalid, s_diff);
            __syncthreads();
            // inclusive scan of the difference array = the digit counts (DPT digits per thread)
            uint32_t loc[DPT], x = 0;
#pragma unroll
            for (int i = 0; i < DPT; i++) {
                x += (uint32_t)s_diff[threadIdx.x * DPT + i];
                loc[i] = x;
            }
            uint32_t sc = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, sc, o);
                if (lane >= o) sc += y;
            }
            if (lane == 31) s_w[warp] = sc;
            __syncthreads();
            uint32_t base = sc - x;
            for (int w = 0; w < warp; w++) base += s_w[w];
#pragma unroll
            for (int i = 0; i < DPT; i++) cmat[(size_t)(threadIdx.x * DPT + i) * ldm + c] = base + loc[i];
            __syncthreads();
            continue;
        }
        for (int i = threadIdx.x; i < NH * NDIG; i += SORT_THREADS) (&s_h[0][0])[i] = 0;
        uint32_t k[SORT_ITEMS];
        if constexpr (Loader::EXPANDS) {
            ld.load(c, cbase, cvalid, dyn, nullptr, dyn + SORT_CHUNK);
            __syncthreads();
#pragma unroll
            for (int q = 0; q < SORT_ITEMS; q++) {
                const uint32_t e = threadIdx.x + q * SORT_THREADS;
                k[q] = e < cvalid ? dyn[e] : 0u;
            }
        } else {
#pragma unroll
            for (int q = 0; q < SORT_ITEMS; q++) {
                const uint32_t e = threadIdx.x + q * SORT_THREADS;
                k[q] = e < cvalid ? ld.key(cbase + e) : 0u;
            }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < SORT_ITEMS; q++) {
            const uint32_t e = threadIdx.x + q * SORT_THREADS;
            if (e < cvalid) atomicAdd(&s_h[warp % NH][(k[q] >> shift) & (NDIG - 1)], 1u);
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < DPT; i++) {
            const int d = threadIdx.x * DPT + i;
            uint32_t t = 0;
#pragma unroll
            for (int h = 0; h < NH; h++) t += s_h[h][d];
            cmat[(size_t)d * ldm + c] = t;
        }
        __syncthreads();
    }
}

// step 2: exclusive scan of each digit's row over the chunks; row totals. One block per
// digit; its SCANROWS_WARPS warps split the row into segments: each warp sums its segment
// (8 coalesced loads per lane in flight), the block adds up the segment totals, then each
// warp scans its segment from its offset (a row of 1042 chunks: 2 load round trips, where
// one warp walking the whole row took 5).
constexpr int SCANROWS_WARPS = 8;
__global__ void __launch_bounds__(SCANROWS_WARPS * 32) k_rs_scanrows(const Counters *cnt, int which, uint64_t max_keys,
                                                                   uint32_t *cmat, uint32_t ldm, uint32_t *row_total,
                                                                   int ndig) {
    pdl_wait();
    __shared__ uint32_t s_tot[SCANROWS_WARPS];
    const uint32_t n = count_of(cnt, which, 0, max_keys);
    const uint32_t nchunks = (n + SORT_CHUNK - 1) / SORT_CHUNK;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const int d = blockIdx.x;
    if (d >= ndig) return;
    uint32_t *row = cmat + (size_t)d * ldm;
    constexpr int U = 8;
    const uint32_t seg = ((nchunks + SCANROWS_WARPS - 1) / SCANROWS_WARPS + 31u) & ~31u;
    const uint32_t c0 = min(nchunks, warp * seg), c1 = min(nchunks, c0 + seg);
    uint32_t sum = 0;
    for (uint32_t base = c0; base < c1; base += 32 * U) {
        uint32_t v[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint32_t c = base + u * 32 + lane;
            v[u] = c < c1 ? row[c] : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; u++) sum += v[u];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) s_tot[warp] = sum;
    __syncthreads();
    uint32_t carry = 0, total = 0;
#pragma unroll
    for (int w = 0; w < SCANROWS_WARPS; w++) {
        const uint32_t t = s_tot[w];
        carry += (uint32_t)w < warp ? t : 0u;
        total += t;
    }
    for (uint32_t base = c0; base < c1; base += 32 * U) {
        uint32_t v[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint32_t c = base + u * 32 + lane;
            v[u] = c < c1 ? row[c] : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            uint32_t x = v[u];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= (uint32_t)o) x += y;
            }
            const uint32_t c = base + u * 32 + lane;
            if (c < c1) row[c] = carry + x - v[u];
            carry += __shfl_sync(0xffffffffu, x, 31);
        }
    }
    if (threadIdx.x == 0) row_total[d] = total;
}

// step 3: stable scatter. position = (all smaller digits) + (this digit in
// earlier chunks) + (rank among this chunk's elements of the digit)
template <class Loader, int DBITS>
__global__ void __launch_bounds__(SORT_THREADS, Loader::PACKED ? GS_SCATTER_MINB_PK : GS_SCATTER_MINB)
    k_rs_scatter(Loader ld, uint32_t *__restrict__ kout, uint32_t *__restrict__ vout, const Counters *cnt,
                 int which, uint64_t max_keys, int shift, const uint32_t *__restrict__ cmat, uint32_t ldm,
                 const uint32_t *__restrict__ row_total) {
    pdl_wait();
    constexpr int NDIG = DBITS > 8 ? 512 : 256;
    constexpr int DPT = NDIG / SORT_THREADS;   // digits owned per thread (consecutive)
    extern __shared__ uint32_t dyn[];
    // PACKED loaders carry the value in the key's upper bits (key = digit | value << PACK_SHIFT):
    // one word per element, half the shared memory, more resident blocks
    constexpr bool PK = Loader::PACKED;
    uint32_t *s_k = dyn, *s_v = PK ? nullptr : dyn + SORT_CHUNK;                    // loaded chunk
    uint32_t *s_ok = dyn + (PK ? 1 : 2) * SORT_CHUNK, *s_ov = PK ? nullptr : dyn + 3 * SORT_CHUNK;   // digit order
    // loader scratch: expanding loaders are done with it before s_ok is written
    uint32_t *s_scr = Loader::EXPANDS ? s_ok : dyn + 4 * SORT_CHUNK;
    __shared__ uint16_t s_whist[NWARP][NDIG];
    __shared__ uint32_t s_dbase[NDIG], s_blk[NDIG], s_base[NDIG], s_tot[NWARP];
    const uint32_t n = count_of(cnt, which, 0, max_keys);
    const uint32_t nchunks = ld.nchunks(n);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int d0 = threadIdx.x * DPT;
    if (kout && ld.keys_if_wide && !cnt->wide_depth) kout = nullptr;   // nobody reads these keys
    // exclusive scan over all NDIG digits; v[i] belongs to digit d0 + i
    auto block_excl_scan = [&](const uint32_t (&v)[DPT], uint32_t (&out)[DPT]) {
        uint32_t t = 0;
#pragma unroll
        for (int i = 0; i < DPT; i++) t += v[i];
        uint32_t x = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_tot[warp] = x;
        __syncthreads();
        uint32_t wb = x - t;
        for (int w = 0; w < warp; w++) wb += s_tot[w];
        __syncthreads();
#pragma unroll
        for (int i = 0; i < DPT; i++) {
            out[i] = wb;
            wb += v[i];
        }
    };
    {
        uint32_t v[DPT], o[DPT];
#pragma unroll
        for (int i = 0; i < DPT; i++) v[i] = row_total[d0 + i];
        block_excl_scan(v, o);
#pragma unroll
        for (int i = 0; i < DPT; i++) s_dbase[d0 + i] = o[i];
    }
    __syncthreads();
    for (uint32_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        uint32_t cbase, cvalid;
        ld.chunk(c, n, cbase, cvalid);
#pragma unroll
        for (int i = 0; i < DPT; i++) {
#pragma unroll
            for (int w = 0; w < NWARP; w++) s_whist[w][d0 + i] = 0;
            s_base[d0 + i] = ld.digit_base(c, d0 + i, s_dbase) + cmat[(size_t)(d0 + i) * ldm + c];
        }
        ld.load(c, cbase, cvalid, s_k, s_v, s_scr);
        __syncthreads();
        // warp-local stable ranks
        uint32_t rank[SORT_ITEMS];
#pragma unroll
        for (int r = 0; r < SORT_ITEMS; r++) {
            const int e = elem_of(warp, r, lane);
            const bool valid = (uint32_t)e < cvalid;
            const uint32_t d = valid ? ((s_k[e] >> shift) & (NDIG - 1)) : 0u;
            const uint32_t peers = peers_of<DBITS>(d, valid);
            uint32_t before = 0;
            if (valid) before = s_whist[warp][d];
            __syncwarp();
            if (valid && (__ffs(peers) - 1) == lane) s_whist[warp][d] = (uint16_t)(before + __popc(peers));
            __syncwarp();
            rank[r] = before + __popc(peers & lanemask_lt());
        }
        __syncthreads();
        {
            uint32_t tot[DPT], o[DPT];
#pragma unroll
            for (int i = 0; i < DPT; i++) {
                uint32_t total = 0;
#pragma unroll
                for (int w = 0; w < NWARP; w++) {
                    const uint32_t t = s_whist[w][d0 + i];
                    s_whist[w][d0 + i] = (uint16_t)total;
                    total += t;
                }
                tot[i] = total;
            }
            block_excl_scan(tot, o);
#pragma unroll
            for (int i = 0; i < DPT; i++) s_blk[d0 + i] = o[i];
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < SORT_ITEMS; r++) {
            const int e = elem_of(warp, r, lane);
            if ((uint32_t)e < cvalid) {
                const uint32_t k = s_k[e];
                const uint32_t d = (k >> shift) & (NDIG - 1);
                const uint32_t pos = s_blk[d] + s_whist[warp][d] + rank[r];
                s_ok[pos] = k;
                if (!PK) s_ov[pos] = s_v[e];
            }
        }
        __syncthreads();
        // runs of one digit are consecutive in shared and in global memory
#pragma unroll 4
        for (uint32_t p = threadIdx.x; p < cvalid; p += SORT_THREADS) {
            const uint32_t k = s_ok[p];
            const uint32_t d = (k >> shift) & (NDIG - 1);
            const uint32_t g = s_base[d] + (p - s_blk[d]);
            if constexpr (PK) {
                vout[g] = k >> Loader::PACK_SHIFT;
            } else {
                if (kout) kout[g] = k;
                const uint32_t v = s_ov[p];
                vout[g] = v;
                ld.epilogue(g, v);
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// tile ranges: boundary detection over the sorted tile ids
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_ranges(const uint32_t *__restrict__ keys, const Counters *cnt,
                                                uint64_t max_keys, uint2 *ranges, int which, uint32_t kmask) {
    pdl_wait();
    const uint32_t n = count_of(cnt, which, 0, max_keys);
    auto tiles_at = [&](uint32_t k) { return keys[k] & kmask; };
    const uint32_t stride = gridDim.x * blockDim.x * 4;
    for (uint32_t k0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4; k0 < n; k0 += stride) {
        uint32_t t[6];
        t[0] = k0 > 0 ? tiles_at(k0 - 1) : 0xFFFFFFFFu;
        if (k0 + 4 <= n) {
            const uint4 v = *reinterpret_cast<const uint4 *>(keys + k0);
            t[1] = v.x & kmask; t[2] = v.y & kmask; t[3] = v.z & kmask; t[4] = v.w & kmask;
        } else {
#pragma unroll
            for (int j = 0; j < 4; j++) t[1 + j] = k0 + j < n ? tiles_at(k0 + j) : 0xFFFFFFFFu;
        }
        t[5] = k0 + 4 < n ? tiles_at(k0 + 4) : 0xFFFFFFFFu;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const uint32_t k = k0 + j;
            if (k >= n) break;
            if (t[j + 1] != t[j]) ranges[t[j + 1]].x = k;
            if (t[j + 1] != t[j + 2]) ranges[t[j + 1]].y = k + 1;
        }
    }
}

// ---------------------------------------------------------------------------
// Two-level binning (tile grids up to 512 x 512): the stable sort by tile of the
// depth-ordered pairs is done MSD-style without materialising the K tile keys.
//   rows:    each depth-ordered Gaussian r contributes one entry per tile row it
//            keeps; one stable 8-bit pass on the row ty puts the entries in
//            (ty, depth) order (values r, keys ty).
//   columns: an entry of row ty holds a contiguous run of tile columns (the rect's
//            columns, or the kept run of a GS_FLAG_TIGHT row). Its pairs are
//            enumerated run by run, in row-aligned 4096-pair chunks, and one stable
//            pass on the column tx, segmented by row, writes each Gaussian index
//            straight to its final slot. Tile ranges follow from the column counts.
// The result is the same (tile, depth, index) order as a full stable sort.
// ---------------------------------------------------------------------------

// kept tile rows of a rect (bit ry of the result; rows without a kept tile are
// skipped); the full-rect case is all h rows
__device__ __forceinline__ uint32_t kept_rows(const ushort4 &rc, unsigned long long m) {
    const uint32_t w = rc.z - rc.x, h = rc.w - rc.y;
    if (m == ~0ull || w * h > 64u || h > 32u) return h >= 32u ? 0xFFFFFFFFu : ((1u << h) - 1u);
    const unsigned long long wmask = (w >= 64u) ? ~0ull : ((1ull << w) - 1ull);
    uint32_t rows = 0;
    for (uint32_t ry = 0; ry < h; ry++)
        if ((m >> (ry * w)) & wmask) rows |= 1u << ry;
    return rows;
}

struct RowOffsetsOp {   // kept rows per depth-ordered Gaussian -> row-entry offsets (+ kept-row masks)
    const ushort4 *rect_r;                 // rects in depth order (gathered by the last depth pass)
    const unsigned long long *tmask_r;     // GS_FLAG_TIGHT masks in depth order (nullptr: whole rects)
    uint32_t *roff, *rowmask_r;
    uint32_t *chunk_first;
    Counters *cnt;
    uint64_t max_keys;
    static constexpr int WHICH = CNT_VISIBLE;
    static constexpr bool SIDE = false;
    struct Aux {};   // emit re-reads (L1-hot): nothing is held across the scan, for occupancy
    __device__ uint32_t nrows(const ushort4 &rc, unsigned long long m, uint32_t &rows) const {
        if (!tmask_r) {
            rows = 0xFFFFFFFFu;
            return (uint32_t)(rc.w - rc.y);
        }
        rows = kept_rows(rc, m);
        return (uint32_t)(rc.w - rc.y) > 32u ? (uint32_t)(rc.w - rc.y) : (uint32_t)__popc(rows);
    }
    __device__ uint32_t load(uint32_t r) const {
        uint32_t rows;
        return nrows(rect_r[r], tmask_r ? tmask_r[r] : ~0ull, rows);
    }
    __device__ uint32_t load(uint32_t r, Aux &) const { return load(r); }
    __device__ void emit(uint32_t r, uint64_t o, uint32_t v, const Aux &) const {
        roff[r] = (uint32_t)(o < 0xFFFFFFFFull ? o : 0xFFFFFFFFull);
        if (tmask_r) {
            uint32_t rows;
            nrows(rect_r[r], tmask_r[r], rows);
            rowmask_r[r] = rows;
        }
        for (uint64_t c = (o + SORT_CHUNK - 1) / SORT_CHUNK; c * SORT_CHUNK < o + v; c++)
            if (c * SORT_CHUNK < max_keys) chunk_first[c] = r;
    }
    __device__ void finish(uint64_t total) const {
        cnt->n_rent = (uint32_t)(total < 0xFFFFFFFFull ? total : 0xFFFFFFFFull);
        if (total > max_keys) atomicOr(&cnt->err, 1u);
    }
};

// Warp-cooperative run expansion. Lane L holds a run of len_L >= 0 consecutive output
// slots; the non-empty runs are laid out back to back from slot 0 in lane order. Each
// round maps 32 slots to their runs with one OR-reduction of the run heads, so the work
// is balanced whatever the run lengths.
// emit(valid, owner, j, t): slot t is element j of the run of lane `owner`
// (every lane calls it, so it may shuffle the owner's data).
template <class F>
__device__ __forceinline__ void warp_expand(uint32_t len, F &&emit) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t nz = __ballot_sync(0xffffffffu, len != 0u);   // lanes with a run
    uint32_t pre = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, pre, o);
        if (lane >= (uint32_t)o) pre += y;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, pre, 31);
    pre -= len;   // exclusive
    int carry = -1;   // run (among the non-empty ones) of the slot before this round
    for (uint32_t g = 0; g < total; g += 32) {
        const uint32_t head = (len && pre >= g && pre < g + 32u) ? (1u << (pre - g)) : 0u;
        const uint32_t heads = __reduce_or_sync(0xffffffffu, head);
        const int run = min(31, carry + __popc(heads & (0xFFFFFFFFu >> (31u - lane))));
        carry += __popc(heads);
        const int owner = (int)min(31u, __fns(nz, 0, run + 1));   // the lane of that run
        const uint32_t t = g + lane;
        const uint32_t opre = __shfl_sync(0xffffffffu, pre, owner);
        emit(t < total, owner, t - opre, t);
    }
}

// Row entries cbase .. cbase+cvalid-1: entry e belongs to the depth-ordered Gaussian r
// with roff[r] <= e < roff[r+1] and is r's (e - roff[r])-th kept tile row ty. Its key
// packs the row and the row's run of kept tile columns: ty | x0 << 9 | width << 18
// (a GS_FLAG_TIGHT row keeps one contiguous run of columns); value = Gaussian index.
struct RowLoader : LinearChunks {
    const uint32_t *roff, *chunk_first, *rowmask_r, *sorted_idx;   // rowmask_r: GS_FLAG_TIGHT only
    const ushort4 *rect_r;
    const unsigned long long *tmask_r;                              // GS_FLAG_TIGHT only
    const Counters *cnt;
    bool tight;
    static constexpr bool EXPANDS = true;
    static constexpr bool RUN_COUNTS = true;   // k_rs_count uses count_runs (no expansion)
    static constexpr int SCRATCH_WORDS = 0;
    __device__ void count_runs(uint32_t c, uint32_t cbase, uint32_t cvalid, int *s_diff) const;
    __device__ void load(uint32_t c, uint32_t cbase, uint32_t cvalid, uint32_t *sk, uint32_t *sv, uint32_t *) const {
        const uint32_t nv = cnt->n_visible;
        const uint32_t nchunks = (cnt->n_rent + SORT_CHUNK - 1) / SORT_CHUNK;
        const uint32_t r_lo = chunk_first[c];
        const uint32_t r_hi = c + 1 < nchunks ? min(nv - 1, chunk_first[c + 1]) : nv - 1;
        const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
        const uint32_t cend = cbase + cvalid;
        const uint32_t n_rent = cnt->n_rent;
        // the next group's Gaussians are fetched while this group expands (latency hiding)
        uint32_t n_o = 0, n_o1 = 0, n_idx = 0, n_rows = 0xFFFFFFFFu;
        ushort4 n_rc = make_ushort4(0, 0, 0, 0);
        unsigned long long n_m = ~0ull;
        auto fetch = [&](uint32_t g) {
            const uint32_t r = g + lane;
            if (r <= r_hi) {
                n_o = roff[r];
                n_o1 = r + 1 < nv ? roff[r + 1] : n_rent;
                n_rc = rect_r[r];
                n_idx = sorted_idx[r];
                if (tight) {
                    n_rows = rowmask_r[r];
                    n_m = tmask_r[r];
                }
            }
        };
        fetch(r_lo + 32u * warp);
        for (uint32_t g0 = r_lo + 32u * warp; g0 <= r_hi; g0 += 32u * NWARP) {
            const uint32_t r = g0 + lane;
            const uint32_t o = n_o, o1 = n_o1, idx = n_idx, rows = n_rows;
            const ushort4 rc = n_rc;
            const unsigned long long m = n_m;
            if (g0 + 32u * NWARP <= r_hi) fetch(g0 + 32u * NWARP);
            uint32_t len = 0, q0 = 0, slot0 = 0, rxy = 0, rzw = 0;
            if (r <= r_hi) {
                rxy = (uint32_t)rc.x | ((uint32_t)rc.y << 16);
                rzw = (uint32_t)rc.z | ((uint32_t)rc.w << 16);
                q0 = o < cbase ? cbase - o : 0u;
                len = min(o1, cend) - (o + q0);
                slot0 = o + q0 - cbase;
            }
            const uint32_t wslot = __shfl_sync(0xffffffffu, slot0, 0);
            warp_expand(len, [&](bool valid, int owner, uint32_t j, uint32_t t) {
                const uint32_t oq0 = __shfl_sync(0xffffffffu, q0, owner);
                const uint32_t oxy = __shfl_sync(0xffffffffu, rxy, owner);
                const uint32_t ozw = __shfl_sync(0xffffffffu, rzw, owner);
                const uint32_t oidx = __shfl_sync(0xffffffffu, idx, owner);
                uint32_t orows = 0xFFFFFFFFu;
                unsigned long long om = ~0ull;
                if (tight) {
                    orows = __shfl_sync(0xffffffffu, rows, owner);
                    om = ((unsigned long long)__shfl_sync(0xffffffffu, (uint32_t)(m >> 32), owner) << 32) |
                         __shfl_sync(0xffffffffu, (uint32_t)m, owner);
                }
                if (!valid) return;
                const uint32_t x0r = oxy & 0xFFFFu, y0 = oxy >> 16, w = (ozw & 0xFFFFu) - x0r, h = (ozw >> 16) - y0;
                uint32_t q = oq0 + j;                                                   // q-th kept row
                if (orows != 0xFFFFFFFFu) q = __fns(orows, 0, (int)q + 1);
                uint32_t x0 = x0r, wr = w;
                if (om != ~0ull && w * h <= 64u) {   // the kept run of this row
                    const uint32_t bits = (uint32_t)((om >> (q * w)) & ((1ull << w) - 1ull));
                    x0 = x0r + (uint32_t)(__ffs(bits) - 1);
                    wr = (uint32_t)__popc(bits);
                }
                sk[wslot + t] = (y0 + q) | (x0 << 9) | (wr << 18);
                if (sv) sv[wslot + t] = oidx;
            });
        }
    }
};

// Digit counts of a chunk without expanding it: each Gaussian's rows in the chunk
// window are a run of consecutive digits (kept rows of a GS_FLAG_TIGHT box are
// counted one by one), added to the difference array s_diff[257].
__device__ __forceinline__ void row_count_runs(const RowLoader &ld, uint32_t c, uint32_t cbase, uint32_t cvalid,
                                               int *s_diff) {
    const uint32_t nv = ld.cnt->n_visible, n_rent = ld.cnt->n_rent;
    const uint32_t nchunks = (n_rent + SORT_CHUNK - 1) / SORT_CHUNK;
    const uint32_t r_lo = ld.chunk_first[c];
    const uint32_t r_hi = c + 1 < nchunks ? min(nv - 1, ld.chunk_first[c + 1]) : nv - 1;
    const uint32_t cend = cbase + cvalid;
    // COUNT_ILP Gaussians per thread per round: their loads are issued together
    for (uint32_t r0 = r_lo + threadIdx.x; r0 <= r_hi; r0 += COUNT_ILP * SORT_THREADS) {
        uint32_t o[COUNT_ILP], o1[COUNT_ILP], y0[COUNT_ILP], rows[COUNT_ILP];
#pragma unroll
        for (int u = 0; u < COUNT_ILP; u++) {
            const uint32_t r = r0 + (uint32_t)u * SORT_THREADS;
            o[u] = o1[u] = y0[u] = 0;
            rows[u] = 0xFFFFFFFFu;
            if (r <= r_hi) {
                o[u] = ld.roff[r];
                o1[u] = r + 1 < nv ? ld.roff[r + 1] : n_rent;
                y0[u] = ld.rect_r[r].y;
                if (ld.tight) rows[u] = ld.rowmask_r[r];
            }
        }
#pragma unroll
        for (int u = 0; u < COUNT_ILP; u++) {
            const uint32_t q0 = o[u] < cbase ? cbase - o[u] : 0u;
            const uint32_t len = min(o1[u], cend) - (o[u] + q0);
            if (o1[u] <= o[u] + q0 || len == 0) continue;
            if (rows[u] == 0xFFFFFFFFu) {
                atomicAdd(&s_diff[y0[u] + q0], 1);
                atomicAdd(&s_diff[y0[u] + q0 + len], -1);
            } else {
                for (uint32_t q = q0; q < q0 + len; q++) {
                    const uint32_t ty = y0[u] + (uint32_t)__fns(rows[u], 0, (int)q + 1);
                    atomicAdd(&s_diff[ty], 1);
                    atomicAdd(&s_diff[ty + 1], -1);
                }
            }
        }
    }
}

__device__ void RowLoader::count_runs(uint32_t c, uint32_t cbase, uint32_t cvalid, int *s_diff) const {
    row_count_runs(*this, c, cbase, cvalid, s_diff);
}

struct PairOffsetsOp {   // row entries in (ty, depth) order -> pair offsets (run widths from the packed keys)
    const uint32_t *e_key;
    uint32_t *poff;
    Counters *cnt;
    uint64_t max_keys;
    static constexpr int WHICH = CNT_RENT;
    static constexpr bool SIDE = false;
    struct Aux {};
    __device__ uint32_t load(uint32_t e) const { return e_key[e] >> 18; }
    __device__ uint32_t load(uint32_t e, Aux &) const { return e_key[e] >> 18; }
    __device__ void emit(uint32_t e, uint64_t o, uint32_t, const Aux &) const {
        poff[e] = (uint32_t)(o < 0xFFFFFFFFull ? o : 0xFFFFFFFFull);
    }
    __device__ void finish(uint64_t total) const {
        cnt->n_keys = total;
        if (total > max_keys) atomicOr(&cnt->err, 1u);
    }
};

// Pairs of one row-aligned chunk (cdesc): pair p belongs to the entry e with
// poff[e] <= p < poff[e+1] and is column x0 + (p - poff[e]) of its run. key = tile
// column tx, value = Gaussian index; digit bases are the tile starts (ranges[.].x).
template <bool PK, int RB>
struct ColLoader {
    static constexpr bool PACKED = PK;    // Gaussian indices < 2^(32 - RB): key = tx | index << RB
    static constexpr int PACK_SHIFT = RB;
    const uint32_t *poff, *e_key, *e_idx, *cdesc_last;
    const uint4 *cdesc;
    const uint2 *ranges;
    const Counters *cnt;
    int gx;
    static constexpr bool EXPANDS = true;
    static constexpr int SCRATCH_WORDS = 0;
    bool keys_if_wide = false;
    __device__ void epilogue(uint32_t, uint32_t) const {}
    __device__ uint32_t nchunks(uint32_t) const { return cnt->err ? 0u : cnt->n_cchunks; }
    __device__ void chunk(uint32_t c, uint32_t, uint32_t &cbase, uint32_t &cvalid) const {
        const uint4 d = cdesc[c];
        cbase = d.y;
        cvalid = d.z;
    }
    __device__ uint32_t digit_base(uint32_t c, uint32_t d, const uint32_t *) const {
        return d < (uint32_t)gx ? ranges[cdesc[c].x * (uint32_t)gx + d].x : 0u;
    }
    static constexpr bool RUN_COUNTS = true;
    __device__ void count_runs(uint32_t c, uint32_t cbase, uint32_t cvalid, int *s_diff) const {
        const uint32_t e_lo = cdesc[c].w, e_hi = cdesc_last[c], cend = cbase + cvalid;
        for (uint32_t e0 = e_lo + threadIdx.x; e0 <= e_hi; e0 += COUNT_ILP * SORT_THREADS) {
            uint32_t o[COUNT_ILP], k[COUNT_ILP];
#pragma unroll
            for (int u = 0; u < COUNT_ILP; u++) {
                const uint32_t e = e0 + (uint32_t)u * SORT_THREADS;
                o[u] = cend;   // (no run)
                k[u] = 0;
                if (e <= e_hi) {
                    o[u] = poff[e];
                    k[u] = e_key[e];
                }
            }
#pragma unroll
            for (int u = 0; u < COUNT_ILP; u++) {
                if (e0 + (uint32_t)u * SORT_THREADS > e_hi) continue;
                const uint32_t q0 = o[u] < cbase ? cbase - o[u] : 0u;
                const uint32_t len = min(o[u] + (k[u] >> 18), cend) - (o[u] + q0);
                const uint32_t x = ((k[u] >> 9) & 0x1FFu) + q0;
                atomicAdd(&s_diff[x], 1);
                atomicAdd(&s_diff[x + len], -1);
            }
        }
    }
    __device__ void load(uint32_t c, uint32_t cbase, uint32_t cvalid, uint32_t *sk, uint32_t *sv, uint32_t *) const {
        const uint32_t e_lo = cdesc[c].w, e_hi = cdesc_last[c];
        const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
        const uint32_t cend = cbase + cvalid;
        // the next group's entries are fetched while this group expands (latency hiding)
        uint32_t n_o = 0, n_k = 0, n_i = 0;
        auto fetch = [&](uint32_t g) {
            const uint32_t e = g + lane;
            if (e <= e_hi) {
                n_o = poff[e];
                n_k = e_key[e];
                n_i = e_idx[e];
            }
        };
        fetch(e_lo + 32u * warp);
        for (uint32_t g0 = e_lo + 32u * warp; g0 <= e_hi; g0 += 32u * NWARP) {
            const uint32_t e = g0 + lane;
            const uint32_t o = n_o, k = n_k, idx = n_i;
            if (g0 + 32u * NWARP <= e_hi) fetch(g0 + 32u * NWARP);
            uint32_t len = 0, x = 0, slot0 = 0;
            if (e <= e_hi) {
                const uint32_t q0 = o < cbase ? cbase - o : 0u;
                len = min(o + (k >> 18), cend) - (o + q0);
                x = ((k >> 9) & 0x1FFu) + q0;
                slot0 = o + q0 - cbase;
            }
            const uint32_t wslot = __shfl_sync(0xffffffffu, slot0, 0);
            warp_expand(len, [&](bool valid, int owner, uint32_t j, uint32_t t) {
                const uint32_t ox = __shfl_sync(0xffffffffu, x, owner);
                const uint32_t oidx = __shfl_sync(0xffffffffu, idx, owner);
                if (!valid) return;
                if (PK) {
                    sk[wslot + t] = (ox + j) | (oidx << RB);
                } else {
                    sk[wslot + t] = ox + j;
                    if (sv) sv[wslot + t] = oidx;
                }
            });
        }
    }
};

// Wide depth range only (a visible depth key >= 2^27, see CompactOp): the 4th pass
// left the order in sv[1]; move it back to sv[0] and gather the rects / masks.
__global__ void __launch_bounds__(256) k_depth_wide_copy(const Counters *cnt, const uint32_t *__restrict__ v_in,
                                                         uint32_t *__restrict__ v_out, const ushort4 *__restrict__ rect,
                                                         ushort4 *__restrict__ rect_r,
                                                         const unsigned long long *__restrict__ tmask,
                                                         unsigned long long *__restrict__ tmask_r) {
    pdl_wait();
    const uint32_t n = count_of(cnt, CNT_VISIBLE_WIDE, 0, 0);
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        const uint32_t v = v_in[r];
        v_out[r] = v;
        rect_r[r] = rect[v];
        if (tmask) tmask_r[r] = tmask[v];
    }
}


// one block: per tile row, first entry / first pair / first column chunk; chunk count
// (Capacity error path: when the row entries alone overflowed max_keys, the pair offsets
// were not computed; K = the sum of tiles touched is still reported, summed here.)
__global__ void __launch_bounds__(512) k_row_bounds(const uint32_t *__restrict__ rows_per_ty,
                                                    const uint32_t *__restrict__ poff, Counters *cnt, int gy,
                                                    uint64_t max_keys, uint32_t *rowinfo,
                                                    const uint32_t *__restrict__ sorted_idx,
                                                    const uint32_t *__restrict__ touched) {
    pdl_wait();
    __shared__ uint32_t s_w[16];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (cnt->err && cnt->n_keys == 0) {
        const uint32_t nv = cnt->n_visible;
        unsigned long long acc = 0;
        for (uint32_t r = t; r < nv; r += blockDim.x) acc += touched[sorted_idx[r]];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0 && acc) atomicAdd((unsigned long long *)&cnt->n_keys, acc);
    }
    auto excl = [&](uint32_t v) -> uint32_t {
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_w[warp] = x;
        __syncthreads();
        uint32_t b = 0;
        for (int w = 0; w < warp; w++) b += s_w[w];
        __syncthreads();
        return b + x - v;
    };
    const bool ok = cnt->err == 0u;
    const uint32_t R = ok ? cnt->n_rent : 0u;
    const uint32_t K = ok ? (uint32_t)cnt->n_keys : 0u;
    const uint32_t ne = (ok && t < gy) ? rows_per_ty[t] : 0u;
    const uint32_t rs = excl(ne);
    const uint32_t P = (t <= gy && rs < R) ? poff[rs] : K;
    // pairs of row t: next row's first pair - P (rows are contiguous in pair order)
    __shared__ uint32_t s_P[513];
    s_P[t] = P;
    if (t == 0) s_P[512] = K;
    __syncthreads();
    const uint32_t np = t < gy ? s_P[t + 1] - P : 0u;
    const uint32_t nch = (np + SORT_CHUNK - 1) / SORT_CHUNK;
    const uint32_t cb = excl(nch);
    if (t < gy) {
        rowinfo[t] = rs;
        rowinfo[513 + t] = P;
        rowinfo[2 * 513 + t] = cb;
    }
    if (t == gy - 1) {   // sentinels of row gy
        rowinfo[gy] = R;
        rowinfo[513 + gy] = K;
        rowinfo[2 * 513 + gy] = cb + nch;
        cnt->n_cchunks = cb + nch;
    }
}

// column chunk descriptors: (ty, first pair, pairs, first entry) and last entry
__global__ void __launch_bounds__(256) k_chunk_desc(const uint32_t *__restrict__ rowinfo,
                                                    const uint32_t *__restrict__ poff, const Counters *cnt, int gy,
                                                    uint4 *cdesc, uint32_t *cdesc_last) {
    pdl_wait();
    const uint32_t nch = cnt->err ? 0u : cnt->n_cchunks;
    const uint32_t *rs = rowinfo, *P = rowinfo + 513, *cb = rowinfo + 2 * 513;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < nch; c += gridDim.x * blockDim.x) {
        int lo = 0, hi = gy - 1;   // last row with cb[row] <= c
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (cb[mid] <= c) lo = mid;
            else hi = mid - 1;
        }
        const uint32_t ty = (uint32_t)lo;
        const uint32_t pbase = P[ty] + (c - cb[ty]) * SORT_CHUNK;
        const uint32_t pcount = min((uint32_t)SORT_CHUNK, P[ty + 1] - pbase);
        auto entry_of = [&](uint32_t p) {   // last entry of row ty with poff <= p
            uint32_t a = rs[ty], b = rs[ty + 1] - 1;
            while (a < b) {
                const uint32_t m = (a + b + 1) >> 1;
                if (poff[m] <= p) a = m;
                else b = m - 1;
            }
            return a;
        };
        cdesc[c] = make_uint4(ty, pbase, pcount, entry_of(pbase));
        cdesc_last[c] = entry_of(pbase + pcount - 1);
    }
}

// per (tile row, column digit): exclusive scan of the digit's counts over the row's
// chunks (in place in cmat) and the tile's pair count
__global__ void __launch_bounds__(32) k_col_scan(const uint32_t *__restrict__ rowinfo, const Counters *cnt,
                                                 uint32_t *cmat, uint32_t ldm, int gx, uint32_t *tile_cnt) {
    pdl_wait();
    const uint32_t ty = blockIdx.x, d = blockIdx.y, lane = threadIdx.x;
    const uint32_t *cb = rowinfo + 2 * 513;
    const uint32_t c0 = cnt->err ? 0u : cb[ty], c1 = cnt->err ? 0u : cb[ty + 1];
    uint32_t *row = cmat + (size_t)d * ldm;
    uint32_t carry = 0;
    for (uint32_t base = c0; base < c1; base += 32) {
        const uint32_t c = base + lane;
        const uint32_t v = c < c1 ? row[c] : 0u;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        if (c < c1) row[c] = carry + x - v;
        carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) tile_cnt[ty * (uint32_t)gx + d] = carry;
}

// per tile row: tile starts = row's first pair + exclusive scan of the tile counts
__global__ void __launch_bounds__(512) k_tile_ranges(const uint32_t *__restrict__ rowinfo,
                                                     const uint32_t *__restrict__ tile_cnt, int gx, uint2 *ranges) {
    pdl_wait();
    __shared__ uint32_t s_w[16];
    const uint32_t ty = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint32_t n = t < (uint32_t)gx ? tile_cnt[ty * gx + t] : 0u;
    uint32_t x = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    uint32_t b = 0;
    for (uint32_t w = 0; w < warp; w++) b += s_w[w];
    const uint32_t start = rowinfo[513 + ty] + b + x - n;
    if (t < (uint32_t)gx) ranges[ty * gx + t] = n ? make_uint2(start, start + n) : make_uint2(0u, 0u);
}


// ---------------------------------------------------------------------------
// Supertile binning (the tcgen05 blend's lists). A supertile is a block of
// ST_SIDE x ST_SIDE tiles. The depth-ordered Gaussians are expanded to
// (supertile, Gaussian) pairs -- one per supertile their rect overlaps, in
// row-major order -- and ONE stable radix pass on the supertile id groups them:
// each supertile's list is
// in (depth, index) order (up to 512 supertiles, 9 bits: e.g. 1080p has 30 x 17;
// larger grids take the per-tile two-level path). Each pair carries the 16-bit mask of the supertile's
// tiles the Gaussian's rect (GS_FLAG_TIGHT: its kept tiles) covers, so a tile's
// list (the pairs of that tile, sorted by depth) is its supertile's list
// filtered by one mask bit; the blend's producer warp filters it on the fly.
// Versus per-tile lists this sorts S ~ 0.31 K pairs once (C5: 5.4M vs 17.1M) and
// skips the row pass, the pair offsets and the column pass; the blend reads ~5x
// more list entries than it keeps, but only up to its tiles' termination (~12 %
// of the lists at C5).
// key = supertile id | mask << 16, value = Gaussian slot.
// ---------------------------------------------------------------------------
constexpr uint32_t ST_SIDE = 4;
#ifndef GS_ST_SERIAL
#define GS_ST_SERIAL 1       // supertile expansion: lanes write their own short runs
#endif
#ifndef GS_ST_COUNT_FAST
#define GS_ST_COUNT_FAST 1   // supertile counts: whole rects without divisions
#endif

__device__ __forceinline__ uint32_t st_count(const ushort4 &rc) {
    const uint32_t sx0 = rc.x / ST_SIDE, sx1 = (rc.z - 1u) / ST_SIDE + 1u;
    const uint32_t sy0 = rc.y / ST_SIDE, sy1 = (rc.w - 1u) / ST_SIDE + 1u;
    return (sx1 - sx0) * (sy1 - sy0);
}

// q / w for q < 2^24, w >= 1: float reciprocal estimate, corrected to the exact quotient
__device__ __forceinline__ uint32_t udiv_small(uint32_t q, uint32_t w) {
    uint32_t d = (uint32_t)((float)q * __frcp_rn((float)w));
    if (d * w > q) d--;
    else if ((d + 1) * w <= q) d++;
    return d;
}

// tiles of supertile (sx, sy) that the rect [x0, x1) x [y0, y1) covers (bit 4 (ty % 4) + tx % 4);
// with a GS_FLAG_TIGHT tile mask tm (bit (ty - y0) w + tx - x0 of the rect; ~0 = every tile,
// also for rects of more than 64 tiles) only the kept ones
__device__ __forceinline__ uint32_t st_mask(uint32_t x0, uint32_t y0, uint32_t x1, uint32_t y1, uint32_t sx,
                                            uint32_t sy, unsigned long long tm) {
    const uint32_t bx = ST_SIDE * sx, by = ST_SIDE * sy;
    const uint32_t xb = max(x0, bx), xe = min(x1, bx + ST_SIDE), yb = max(y0, by), ye = min(y1, by + ST_SIDE);
    const uint32_t w = x1 - x0;
    if (tm == ~0ull || w * (y1 - y0) > 64u) {
        const uint32_t cols = ((1u << (xe - xb)) - 1u) << (xb - bx);
        return cols * ((0x1111u >> (4u * (ST_SIDE - (ye - yb)))) << (4u * (yb - by)));
    }
    uint32_t m = 0;
    for (uint32_t ty = yb; ty < ye; ty++) {
        const uint32_t bits = (uint32_t)(tm >> ((ty - y0) * w + (xb - x0))) & ((1u << (xe - xb)) - 1u);
        m |= bits << (4u * (ty - by) + (xb - bx));
    }
    return m;
}

struct StOffsetsOp {   // supertiles per depth-ordered Gaussian -> pair offsets (+ chunk heads); side sum: K
    const ushort4 *rect_r;                 // rects in depth order (gathered by the last depth pass)
    const uint32_t *sorted_idx, *touched;  // GS_FLAG_TIGHT: K counts the kept tiles (touched)
    bool tight;
    uint32_t *soff, *chunk_first;
    Counters *cnt;
    uint64_t max_keys;
    static constexpr int WHICH = CNT_VISIBLE;
    static constexpr bool SIDE = true;
    struct Aux {};
    __device__ uint32_t load(uint32_t r) const { return st_count(rect_r[r]); }
    __device__ uint32_t load(uint32_t r, Aux &) const { return load(r); }
    __device__ uint32_t side(uint32_t r) const {
        if (tight) return touched[sorted_idx[r]];
        const ushort4 rc = rect_r[r];
        return (uint32_t)(rc.z - rc.x) * (uint32_t)(rc.w - rc.y);
    }
    __device__ void emit(uint32_t r, uint64_t o, uint32_t v, const Aux &) const {
        soff[r] = (uint32_t)(o < 0xFFFFFFFFull ? o : 0xFFFFFFFFull);
        for (uint64_t c = (o + SORT_CHUNK - 1) / SORT_CHUNK; c * SORT_CHUNK < o + v; c++)
            if (c * SORT_CHUNK < max_keys) chunk_first[c] = r;
    }
    __device__ void finish(uint64_t s_total, uint64_t k_total) const {
        cnt->n_spairs = (uint32_t)(s_total < 0xFFFFFFFFull ? s_total : 0xFFFFFFFFull);
        cnt->n_keys = k_total;   // K = the (Gaussian, tile) pairs, S <= K
        if (k_total > max_keys) atomicOr(&cnt->err, 1u);
    }
};

// Supertile pairs cbase .. cbase+cvalid-1: pair p belongs to the depth-ordered Gaussian r
// with soff[r] <= p < soff[r+1] and is the (p - soff[r])-th supertile of its rect (row-major).
struct StLoader : LinearChunks {
    const uint32_t *soff, *chunk_first, *sorted_idx;
    const ushort4 *rect_r;
    const unsigned long long *tmask_r;   // GS_FLAG_TIGHT only
    const Counters *cnt;
    int sgx;
    bool tight;
    static constexpr bool EXPANDS = true;
    static constexpr bool RUN_COUNTS = true;
    static constexpr int SCRATCH_WORDS = 0;
    __device__ void window(uint32_t c, uint32_t &r_lo, uint32_t &r_hi) const {
        const uint32_t nv = cnt->n_visible;
        const uint32_t nch = (cnt->n_spairs + SORT_CHUNK - 1) / SORT_CHUNK;
        r_lo = chunk_first[c];
        r_hi = c + 1 < nch ? min(nv - 1, chunk_first[c + 1]) : nv - 1;
    }
    // digit counts from runs: the Gaussian's supertiles in the chunk window are runs of
    // consecutive ids, one per supertile row
    __device__ void count_runs(uint32_t c, uint32_t cbase, uint32_t cvalid, int *s_diff) const {
        uint32_t r_lo, r_hi;
        window(c, r_lo, r_hi);
        const uint32_t nv = cnt->n_visible, S = cnt->n_spairs, cend = cbase + cvalid;
        for (uint32_t r0 = r_lo + threadIdx.x; r0 <= r_hi; r0 += COUNT_ILP * SORT_THREADS) {
            uint32_t o[COUNT_ILP], o1[COUNT_ILP];
            ushort4 rc[COUNT_ILP];
#pragma unroll
            for (int u = 0; u < COUNT_ILP; u++) {
                const uint32_t r = r0 + (uint32_t)u * SORT_THREADS;
                o[u] = o1[u] = 0;
                rc[u] = make_ushort4(0, 0, 1, 1);
                if (r <= r_hi) {
                    o[u] = soff[r];
                    o1[u] = r + 1 < nv ? soff[r + 1] : S;
                    rc[u] = rect_r[r];
                }
            }
#pragma unroll
            for (int u = 0; u < COUNT_ILP; u++) {
                const uint32_t q0 = o[u] < cbase ? cbase - o[u] : 0u;
                if (o1[u] <= o[u] + q0) continue;
                const uint32_t end = min(o1[u], cend) - o[u];
                const uint32_t sx0 = rc[u].x / ST_SIDE, sy0 = rc[u].y / ST_SIDE;
                const uint32_t sw = (rc[u].z - 1u) / ST_SIDE + 1u - sx0;
                if (GS_ST_COUNT_FAST && q0 == 0 && end == o1[u] - o[u]) {   // whole rect in the chunk: a run per row
                    const uint32_t sy1 = (rc[u].w - 1u) / ST_SIDE + 1u;
                    for (uint32_t sy = sy0; sy < sy1; sy++) {
                        const uint32_t d = sy * (uint32_t)sgx + sx0;
                        atomicAdd(&s_diff[d], 1);
                        atomicAdd(&s_diff[d + sw], -1);
                    }
                    continue;
                }
                for (uint32_t q = q0; q < end;) {
                    const uint32_t qy = udiv_small(q, sw), qx = q - qy * sw;
                    const uint32_t run = min(end - q, sw - qx);
                    const uint32_t d = (sy0 + qy) * (uint32_t)sgx + sx0 + qx;   // < 512
                    atomicAdd(&s_diff[d], 1);
                    atomicAdd(&s_diff[d + run], -1);
                    q += run;
                }
            }
        }
    }
    // key of the q-th supertile pair of the rect [x0, x1) x [y0, y1) (row-major over its
    // supertiles, sw per row): supertile id | tile mask << 16
    __device__ __forceinline__ uint32_t key_of(uint32_t x0, uint32_t y0, uint32_t x1, uint32_t y1, uint32_t qx,
                                               uint32_t qy, unsigned long long tm) const {
        const uint32_t sx = x0 / ST_SIDE + qx, sy = y0 / ST_SIDE + qy;
        return (sy * (uint32_t)sgx + sx) | (st_mask(x0, y0, x1, y1, sx, sy, tm) << 16);
    }
    // Each lane writes its own Gaussian's pairs (position in the rect stepped without a
    // division); Gaussians with more than SERIAL_MAX pairs in the chunk are left to a
    // warp-cooperative expansion afterwards (balanced whatever their length).
    static constexpr uint32_t SERIAL_MAX = 6;
    __device__ void load(uint32_t c, uint32_t cbase, uint32_t cvalid, uint32_t *sk, uint32_t *sv, uint32_t *) const {
        uint32_t r_lo, r_hi;
        window(c, r_lo, r_hi);
        const uint32_t nv = cnt->n_visible, S = cnt->n_spairs;
        const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
        const uint32_t cend = cbase + cvalid;
        for (uint32_t g0 = r_lo + 32u * warp; g0 <= r_hi; g0 += 32u * NWARP) {
            const uint32_t r = g0 + lane;
            uint32_t len = 0, q0 = 0, slot0 = 0, rxy = 0, rzw = 0, idx = 0;
            unsigned long long m = ~0ull;
            if (r <= r_hi) {
                const uint32_t o = soff[r], o1 = r + 1 < nv ? soff[r + 1] : S;
                const ushort4 rc = rect_r[r];
                idx = sorted_idx[r];
                if (tight) m = tmask_r[r];
                rxy = (uint32_t)rc.x | ((uint32_t)rc.y << 16);
                rzw = (uint32_t)rc.z | ((uint32_t)rc.w << 16);
                q0 = o < cbase ? cbase - o : 0u;
                len = min(o1, cend) - (o + q0);
                slot0 = o + q0 - cbase;
            }
            const uint32_t x0 = rxy & 0xFFFFu, y0 = rxy >> 16, x1 = rzw & 0xFFFFu, y1 = rzw >> 16;
            if (GS_ST_SERIAL && len > 0 && len <= SERIAL_MAX) {
                const uint32_t sx0 = x0 / ST_SIDE, sx1 = (x1 - 1u) / ST_SIDE, sy0 = y0 / ST_SIDE;
                const uint32_t sy1 = (y1 - 1u) / ST_SIDE, sw = sx1 + 1u - sx0;
                uint32_t qy = q0 ? udiv_small(q0, sw) : 0u;
                uint32_t qx = q0 - qy * sw;
                const bool plain = m == ~0ull || (x1 - x0) * (y1 - y0) > 64u;
                // the rect's tiles in its first / last supertile column and row (the inner
                // ones hold all four): the mask of supertile (sx, sy) is a 4-bit column
                // pattern times a 0x1111-pattern of rows (no carries)
                const uint32_t cf = (0xFu << (x0 & 3u)) & 0xFu, cl = 0xFu >> (3u - ((x1 - 1u) & 3u));
                const uint32_t rf = (0x1111u << (4u * (y0 & 3u))) & 0xFFFFu;
                const uint32_t rl = 0xFFFFu >> (4u * (3u - ((y1 - 1u) & 3u)));
                for (uint32_t j = 0; j < len; j++) {
                    const uint32_t sx = sx0 + qx, sy = sy0 + qy;
                    uint32_t mk;
                    if (plain) {
                        const uint32_t cm = (sx == sx0 ? cf : 0xFu) & (sx == sx1 ? cl : 0xFu);
                        const uint32_t rm = (sy == sy0 ? rf : 0x1111u) & (sy == sy1 ? rl : 0xFFFFu);
                        mk = cm * rm;
                    } else {
                        mk = st_mask(x0, y0, x1, y1, sx, sy, m);
                    }
                    sk[slot0 + j] = (sy * (uint32_t)sgx + sx) | (mk << 16);
                    if (sv) sv[slot0 + j] = idx;
                    if (++qx == sw) {
                        qx = 0;
                        qy++;
                    }
                }
            }
            if (GS_ST_SERIAL && !__any_sync(0xffffffffu, len > SERIAL_MAX)) continue;
            // the long ones, balanced over the warp (slots of the others are skipped)
            const uint32_t llen = (!GS_ST_SERIAL || len > SERIAL_MAX) ? len : 0u;
            warp_expand(llen, [&](bool valid, int owner, uint32_t j, uint32_t) {
                const uint32_t oq0 = __shfl_sync(0xffffffffu, q0, owner);
                const uint32_t os0 = __shfl_sync(0xffffffffu, slot0, owner);
                const uint32_t oxy = __shfl_sync(0xffffffffu, rxy, owner);
                const uint32_t ozw = __shfl_sync(0xffffffffu, rzw, owner);
                const uint32_t oidx = __shfl_sync(0xffffffffu, idx, owner);
                unsigned long long om = ~0ull;
                if (tight)
                    om = ((unsigned long long)__shfl_sync(0xffffffffu, (uint32_t)(m >> 32), owner) << 32) |
                         __shfl_sync(0xffffffffu, (uint32_t)m, owner);
                if (!valid) return;
                const uint32_t ox0 = oxy & 0xFFFFu, oy0 = oxy >> 16, ox1 = ozw & 0xFFFFu, oy1 = ozw >> 16;
                const uint32_t sw = (ox1 - 1u) / ST_SIDE + 1u - ox0 / ST_SIDE;
                const uint32_t q = oq0 + j, qy = udiv_small(q, sw);
                sk[os0 + j] = key_of(ox0, oy0, ox1, oy1, q - qy * sw, qy, om);
                if (sv) sv[os0 + j] = oidx;
            });
        }
    }
};

// one pass: the supertile ranges are the exclusive scan of the pass's digit totals
__global__ void __launch_bounds__(512) k_st_ranges(const uint32_t *__restrict__ row_total, int nst, uint2 *ranges) {
    pdl_wait();
    __shared__ uint32_t s_w[16];
    const uint32_t t = threadIdx.x, lane = t & 31u, warp = t >> 5;
    const uint32_t n = t < (uint32_t)nst ? row_total[t] : 0u;
    uint32_t x = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    uint32_t b = 0;
    for (uint32_t w = 0; w < warp; w++) b += s_w[w];
    const uint32_t start = b + x - n;
    if (t < (uint32_t)nst) ranges[t] = make_uint2(start, start + n);
}
// ---------------------------------------------------------------------------
template <class Loader, int NDIG = 256>
static void launch_count(const Workspace &ws, cudaStream_t st, int grid, Loader ld, int which, uint64_t mk,
                         int shift) {
    const size_t smem =
        (Loader::EXPANDS && !Loader::RUN_COUNTS) ? (SORT_CHUNK + Loader::SCRATCH_WORDS) * sizeof(uint32_t) : 0;
    static bool attrs = false;
    if (!attrs && smem > 48 * 1024) {
        cudaFuncSetAttribute(k_rs_count<Loader, NDIG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attrs = true;
    }
    launch_pdl(k_rs_count<Loader, NDIG>, grid, SORT_THREADS, smem, st, ld, ws.counters, which, mk, shift, ws.cmat,
                                                         (uint32_t)ws.max_chunks);
}

template <class Loader, int DBITS>
static void launch_scatter(const Workspace &ws, cudaStream_t st, int grid, Loader ld, uint32_t *kout,
                           uint32_t *vout, int which, uint64_t mk, int shift) {
    const size_t ldm = ws.max_chunks;
    static_assert(!Loader::EXPANDS || Loader::SCRATCH_WORDS <= SORT_CHUNK, "scratch aliases s_ok");
    const size_t sc_smem =
        ((Loader::PACKED ? 2 : 4) * SORT_CHUNK + (Loader::EXPANDS ? 0 : Loader::SCRATCH_WORDS)) * sizeof(uint32_t);
    static bool attrs = false;
    if (!attrs) {
        cudaFuncSetAttribute(k_rs_scatter<Loader, DBITS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sc_smem);
        attrs = true;
    }
    launch_pdl(k_rs_scatter<Loader, DBITS>, grid, SORT_THREADS, sc_smem, st, ld, kout, vout, ws.counters, which, mk, shift,
                                                                     ws.cmat, (uint32_t)ldm, ws.row_total);
}

// One stable LSD pass on bits [shift, shift + dbits) (dbits <= 9; higher key bits
// must already be zero above shift + dbits or belong to later passes).
template <class Loader>
static int radix_pass(const Workspace &ws, cudaStream_t st, int grid, Loader ld, uint32_t *kout, uint32_t *vout,
                      int which, uint64_t mk, int shift, int dbits = 8) {
    const size_t ldm = ws.max_chunks;
    if (dbits > 8) launch_count<Loader, 512>(ws, st, grid, ld, which, mk, shift);
    else launch_count<Loader, 256>(ws, st, grid, ld, which, mk, shift);
    const int ndig = dbits > 8 ? 512 : 256;
    launch_pdl(k_rs_scanrows, ndig, SCANROWS_WARPS * 32, 0, st, ws.counters, which, mk, ws.cmat, (uint32_t)ldm,
               ws.row_total, ndig);
    switch (dbits) {
    case 1: launch_scatter<Loader, 1>(ws, st, grid, ld, kout, vout, which, mk, shift); break;
    case 2: launch_scatter<Loader, 2>(ws, st, grid, ld, kout, vout, which, mk, shift); break;
    case 3: launch_scatter<Loader, 3>(ws, st, grid, ld, kout, vout, which, mk, shift); break;
    case 4: launch_scatter<Loader, 4>(ws, st, grid, ld, kout, vout, which, mk, shift); break;
    case 5: launch_scatter<Loader, 5>(ws, st, grid, ld, kout, vout, which, mk, shift); break;
    case 6: launch_scatter<Loader, 6>(ws, st, grid, ld, kout, vout, which, mk, shift); break;
    case 7: launch_scatter<Loader, 7>(ws, st, grid, ld, kout, vout, which, mk, shift); break;
    case 9: launch_scatter<Loader, 9>(ws, st, grid, ld, kout, vout, which, mk, shift); break;
    default: launch_scatter<Loader, 8>(ws, st, grid, ld, kout, vout, which, mk, shift); break;
    }
    return 3;
}

template <class Op>
static int scan_pass(const Workspace &ws, cudaStream_t st, int grid, Op op, uint32_t n_points) {
    uint32_t *sums2 = ws.sums + ws.max_chunks;   // side sums (Op::SIDE)
    launch_pdl(k_scan_reduce<Op>, grid, SORT_THREADS, 0, st, op, n_points, ws.sums, sums2);
    launch_pdl(k_scan_apply<Op>, grid, SORT_THREADS, 0, st, op, n_points, (const uint32_t *)ws.sums,
               (const uint32_t *)sums2);
    return 2;
}

template <class L>
static void col_scatter(const Workspace &ws, cudaStream_t st, int grid, const L &col, int tbx, uint64_t mk) {
    switch (std::max(1, tbx)) {
    case 1: launch_scatter<L, 1>(ws, st, grid, col, nullptr, ws.kv[0], CNT_KEYS, mk, 0); break;
    case 2: launch_scatter<L, 2>(ws, st, grid, col, nullptr, ws.kv[0], CNT_KEYS, mk, 0); break;
    case 3: launch_scatter<L, 3>(ws, st, grid, col, nullptr, ws.kv[0], CNT_KEYS, mk, 0); break;
    case 4: launch_scatter<L, 4>(ws, st, grid, col, nullptr, ws.kv[0], CNT_KEYS, mk, 0); break;
    case 5: launch_scatter<L, 5>(ws, st, grid, col, nullptr, ws.kv[0], CNT_KEYS, mk, 0); break;
    case 6: launch_scatter<L, 6>(ws, st, grid, col, nullptr, ws.kv[0], CNT_KEYS, mk, 0); break;
    case 7: launch_scatter<L, 7>(ws, st, grid, col, nullptr, ws.kv[0], CNT_KEYS, mk, 0); break;
    case 9: launch_scatter<L, 9>(ws, st, grid, col, nullptr, ws.kv[0], CNT_KEYS, mk, 0); break;
    default: launch_scatter<L, 8>(ws, st, grid, col, nullptr, ws.kv[0], CNT_KEYS, mk, 0); break;
    }
}

// column pass of the two-level binning with RB-bit column digits
template <int RB>
static void column_pass(const Workspace &ws, cudaStream_t st, int grid, int N, int gx, int gy, int tbx,
                        uint64_t mk) {
    Counters *cnt = ws.counters;
    const ColLoader<false, RB> col{ws.kt[0], ws.kt[1], ws.kv[1], ws.cdesc_last, ws.cdesc, ws.ranges, cnt, gx};
    launch_count<ColLoader<false, RB>, (1 << RB)>(ws, st, grid, col, CNT_KEYS, mk, 0);
    launch_pdl(k_col_scan, dim3(gy, gx), 32, 0, st, ws.rowinfo, cnt, ws.cmat, (uint32_t)ws.max_chunks, gx,
               ws.tile_cnt);
    launch_pdl(k_tile_ranges, gy, 512, 0, st, ws.rowinfo, ws.tile_cnt, gx, ws.ranges);
    if ((int64_t)N < ((int64_t)1 << (32 - RB))) {   // key = tx | index << RB fits one word
        const ColLoader<true, RB> colp{ws.kt[0], ws.kt[1], ws.kv[1], ws.cdesc_last, ws.cdesc, ws.ranges, cnt, gx};
        col_scatter(ws, st, grid, colp, tbx, mk);
    } else {
        col_scatter(ws, st, grid, col, tbx, mk);
    }
}

// the view's capacity error and K into the context's per-call accumulator
__global__ void k_sticky(const Counters *cnt, Sticky *sticky) {
    pdl_wait();
    if (cnt->err) atomicOr(&sticky->err, cnt->err);
    atomicMax(&sticky->max_keys, (unsigned long long)cnt->n_keys);
}

static int binning_body(Workspace &ws, cudaStream_t st, int N, int64_t max_keys, int ntiles, int gx, bool tight,
                        float znear, int grid_mult, bool supertile);

int supertile_count(int gx, int gy) {
    return ceil_div_i(gx, (int)ST_SIDE) * ceil_div_i(gy, (int)ST_SIDE);
}

int launch_binning(Workspace &ws, cudaStream_t st, int N, int64_t max_keys, int ntiles, int gx, uint32_t &,
                   bool tight, float znear, bool concurrent, bool supertile) {
    int launches = binning_body(ws, st, N, max_keys, ntiles, gx, tight, znear,
                                concurrent ? GS_GRID_MULT_CONCURRENT : GS_GRID_MULT, supertile);
    if (ws.sticky) {
        launch_pdl(k_sticky, 1, 1, 0, st, (const Counters *)ws.counters, ws.sticky);
        launches++;
    }
    return launches;
}

static int binning_body(Workspace &ws, cudaStream_t st, int N, int64_t max_keys, int ntiles, int gx, bool tight,
                        float znear, int grid_mult, bool supertile) {
    Counters *cnt = ws.counters;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int grid_n = std::max(1, std::min(nsm * grid_mult, ceil_div_i(N, SORT_CHUNK)));
    const int grid_k = std::max(1, std::min(nsm * grid_mult, ceil_div_i(max_keys, SORT_CHUNK)));
    const uint64_t mk = (uint64_t)max_keys;
    const int gy = ntiles / gx;
    const int nst = supertile_count(gx, gy);
    supertile = supertile && nst <= 512;   // (the caller decides with the same rule)
    if (!supertile && !(gx <= 512 && gy <= 512)) cudaMemsetAsync(ws.ranges, 0, sizeof(uint2) * (size_t)ntiles, st);
    int launches = 0;   // (the two-level path writes every tile range: no memset node)
    // 1. compaction of the visible Gaussians (index order), keys relative to the near plane
    uint32_t dbase = 0;
    if (znear > 0.f) memcpy(&dbase, &znear, 4);
    launches += scan_pass(ws, st, grid_n, CompactOp{ws.wcount, ws.depth_bits, ws.sk[1], ws.sv[1], cnt, dbase},
                          (uint32_t)N);
    // 2. depth sort: 3 stable passes of 9 bits (sk/sv 1 -> 0 -> 1 -> 0); the last one also
    //    gathers each Gaussian's rect (and tile mask) into depth order. Keys >= 2^27 (a
    //    visible depth beyond znear * 2^16) take a 4th pass on bits 27-31 and a copy back;
    //    both launches are no-ops otherwise (device-side count, no host sync).
    const unsigned long long *tm = tight ? ws.tmask : nullptr;
    for (int p = 0; p < 3; p++) {
        PlainLoader ld{{}, ws.sk[(p + 1) & 1], ws.sv[(p + 1) & 1]};
        if (p == 2) {
            ld.g_rect = ws.rect;
            ld.g_rect_out = ws.rect_r;
            ld.g_tmask = tm;
            ld.g_tmask_out = tm ? ws.tmask_r : nullptr;
            ld.keys_if_wide = true;
        }
        launches += radix_pass(ws, st, grid_n, ld, ws.sk[p & 1], ws.sv[p & 1], CNT_VISIBLE, mk, 9 * p, 9);
    }
    launches += radix_pass(ws, st, grid_n, PlainLoader{{}, ws.sk[0], ws.sv[0]}, ws.sk[1], ws.sv[1], CNT_VISIBLE_WIDE,
                           mk, 27, 5);
    launch_pdl(k_depth_wide_copy, nsm * 2, 256, 0, st, (const Counters *)cnt, (const uint32_t *)ws.sv[1], ws.sv[0],
               (const ushort4 *)ws.rect, ws.rect_r, tm, ws.tmask_r);
    launches++;
    if (supertile) {
        // 3. supertile pairs per depth-ordered Gaussian (K on the side), 4. one stable pass on
        //    the supertile id with the expansion fused in (final lists in kt[0] / kv[0]),
        // 5. supertile ranges from the pass's digit totals
        int sbits = 1;
        while ((1 << sbits) < nst) sbits++;
        launches += scan_pass(ws, st, grid_n,
                              StOffsetsOp{ws.rect_r, ws.sv[0], ws.touched, tight, ws.off, ws.chunk_first, cnt, mk},
                              (uint32_t)N);
        launches += radix_pass(ws, st, grid_k,
                               StLoader{{}, ws.off, ws.chunk_first, ws.sv[0], ws.rect_r, ws.tmask_r, cnt,
                                        ceil_div_i(gx, (int)ST_SIDE), tight},
                               ws.kt[0], ws.kv[0], CNT_SPAIRS, mk, 0, sbits);
        launch_pdl(k_st_ranges, 1, 512, 0, st, (const uint32_t *)ws.row_total, nst, ws.ranges);
        return launches + 1;
    }
    int tbx = 0, tby = 0;
    while ((1 << tbx) < gx) tbx++;
    while ((1 << tby) < gy) tby++;
    if (gx <= 512 && gy <= 512) {
        // 3. row entries of the depth-ordered Gaussians
        uint32_t *roff = ws.off, *rowmask_r = ws.sk[1];
        launches += scan_pass(ws, st, grid_n,
                              RowOffsetsOp{ws.rect_r, tight ? ws.tmask_r : nullptr, roff, rowmask_r, ws.chunk_first,
                                           cnt, mk},
                              (uint32_t)N);
        // 4. rows: one stable pass on ty -> entries (ty | x0 << 8 | width << 16, index) in kt[1] / kv[1]
        launches += radix_pass(ws, st, grid_k,
                               RowLoader{{}, roff, ws.chunk_first, rowmask_r, ws.sv[0], ws.rect_r, ws.tmask_r, cnt,
                                         tight},
                               ws.kt[1], ws.kv[1], CNT_RENT, mk, 0, std::max(1, tby));
        // 5. pair offsets of the entries (kt[0])
        launches += scan_pass(ws, st, grid_k, PairOffsetsOp{ws.kt[1], ws.kt[0], cnt, mk}, (uint32_t)N);
        // 6. row bounds and row-aligned column chunks
        launch_pdl(k_row_bounds, 1, 512, 0, st, ws.row_total, ws.kt[0], cnt, gy, mk, ws.rowinfo,
                   (const uint32_t *)ws.sv[0], (const uint32_t *)ws.touched);
        launch_pdl(k_chunk_desc, nsm * 2, 256, 0, st, ws.rowinfo, ws.kt[0], cnt, gy, ws.cdesc, ws.cdesc_last);
        // 7. columns: counts, per-(row, column) scans, tile ranges, stable scatter of the indices
        if (tbx > 8) column_pass<9>(ws, st, grid_k, N, gx, gy, tbx, mk);
        else column_pass<8>(ws, st, grid_k, N, gx, gy, tbx, mk);
        return launches + 6;   // row bounds, chunk descriptors, column count / scan / ranges / scatter
    }
    // 3. pair offsets in depth order
    launches += scan_pass(ws, st, grid_n,
                          OffsetsOp{ws.sv[0], ws.touched, ws.off, ws.chunk_first, cnt, mk},
                          (uint32_t)N);
    // 4. tile sort with the expansion fused into the first pass; final order in kt[0]/kv[0]
    int tbits = 0;
    while ((1 << tbits) < ntiles) tbits++;
    const int tpasses = std::max(1, (tbits + 7) / 8);
    {
        const size_t xs = Expander::SCRATCH_WORDS * sizeof(uint32_t);
        static bool xattr = false;
        if (!xattr) {
            cudaFuncSetAttribute(k_expand, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xs);
            xattr = true;
        }
        const int e = tpasses & 1;   // the passes alternate buffers and end in kt[0]/kv[0]
        launch_pdl(k_expand, grid_k, SORT_THREADS, xs, st, 
            Expander{ws.off, ws.sv[0], ws.chunk_first, ws.rect_r, tight ? ws.tmask_r : nullptr, cnt, gx}, mk,
            ws.kt[e], ws.kv[e]);
        launches++;
        for (int p = 0; p < tpasses; p++) {
            const int src = (e + p) & 1;
            launches += radix_pass(ws, st, grid_k, PlainLoader{{}, ws.kt[src], ws.kv[src]}, ws.kt[src ^ 1],
                                   ws.kv[src ^ 1], CNT_KEYS, mk, 8 * p, std::min(8, std::max(1, tbits - 8 * p)));
        }
    }
    // 5. tile ranges
    launch_pdl(k_ranges, nsm * 4, 256, 0, st, (const uint32_t *)ws.kt[0], (const Counters *)cnt, mk, ws.ranges,
               (int)CNT_KEYS, 0xFFFFFFFFu);
    return launches + 1;
}

}  // namespace gs
