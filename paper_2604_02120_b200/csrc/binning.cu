// binning.cu -- stages (b) "Duplication" and (c) "Sorting"
// plus tile-range identification, as hand-written single-pass kernels.
//
// Canonical order (R-12/R-13): per tile, ascending (depth bits,
// Gaussian index); key = tile << 32 | depth bits. Instead of one 64-bit
// radix sort over (tile, depth) (vanilla: ~6 passes x 24 B/key), the path is
//   1. order-preserving compaction of visible Gaussians   (decoupled look-back scan)
//   2. stable LSD radix sort of the N_vis depth keys       (4 onesweep passes, 8-bit digits)
//   3. scan of tiles_touched in depth order + duplication  (one look-back scan kernel;
//      emits (tile, index) pairs in (depth, index) order)
//   4. stable LSD radix sort of the K tile ids             (1-2 onesweep passes)
//   5. tile ranges by boundary detection
// Stability of 2 and 4 gives exactly the canonical (tile, depth, index) order.
// All counts (N_vis, K) stay on the device: no host synchronisation, graph-capturable.
#include <algorithm>

#include "gs_common.cuh"

namespace gs {

// ---------------------------------------------------------------------------
// epoch-tagged look-back status word: [epoch:24 | flag:2 | value:38]
// ---------------------------------------------------------------------------
constexpr uint64_t ST_AGG = 1, ST_PREFIX = 2;
__device__ __forceinline__ unsigned long long st_make(uint32_t epoch, uint64_t flag, uint64_t v) {
    return ((unsigned long long)(epoch & 0xFFFFFF) << 40) | (flag << 38) | (v & ((1ull << 38) - 1));
}
__device__ __forceinline__ uint32_t st_flag(unsigned long long w, uint32_t epoch) {
    return ((uint32_t)(w >> 40) == (epoch & 0xFFFFFF)) ? (uint32_t)((w >> 38) & 3) : 0u;
}
__device__ __forceinline__ uint64_t st_val(unsigned long long w) { return w & ((1ull << 38) - 1); }

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ---------------------------------------------------------------------------
// single-pass exclusive scan with decoupled look-back (one warp looks back)
// ---------------------------------------------------------------------------
struct CompactOp {   // visible flags -> (depth bits, index) of visible Gaussians, in index order
    const uint32_t *touched, *depth_bits;
    uint32_t *out_k, *out_v;
    Counters *cnt;
    uint32_t n;
    __device__ uint32_t size() const { return n; }
    __device__ uint32_t load(uint32_t i) const { return touched[i] > 0 ? 1u : 0u; }
    __device__ void emit(uint32_t i, uint64_t pos, uint32_t v) const {
        if (v) { out_k[pos] = depth_bits[i]; out_v[pos] = i; }
    }
    __device__ void finish(uint64_t total) const { cnt->n_visible = (uint32_t)total; }
};

struct DuplicateOp {   // tiles_touched in depth order -> offsets, and the (tile, index) pairs
    const uint32_t *sorted_idx, *touched;
    const ushort4 *rect;
    uint32_t *out_tile, *out_idx;
    Counters *cnt;
    uint64_t max_keys;
    int gx;
    __device__ uint32_t size() const { return cnt->n_visible; }
    __device__ uint32_t load(uint32_t r) const { return touched[sorted_idx[r]]; }
    __device__ void emit(uint32_t r, uint64_t off, uint32_t v) const {
        if (v == 0) return;
        if (off + v > max_keys) return;              // capacity error is raised in finish()
        const uint32_t i = sorted_idx[r];
        const ushort4 rc = rect[i];
        for (uint32_t ty = rc.y; ty < rc.w; ty++)
            for (uint32_t tx = rc.x; tx < rc.z; tx++) {
                out_tile[off] = ty * (uint32_t)gx + tx;
                out_idx[off] = i;
                off++;
            }
    }
    __device__ void finish(uint64_t total) const {
        cnt->n_keys = total;
        if (total > max_keys) atomicOr(&cnt->err, 1u);
    }
};

template <class Op>
__global__ void __launch_bounds__(SORT_THREADS) k_scan(Op op, unsigned long long *status, uint32_t epoch,
                                                       uint32_t *ticket) {
    __shared__ uint32_t s_chunk;
    __shared__ uint64_t s_warp[SORT_THREADS / 32];
    __shared__ uint64_t s_prefix;
    const uint32_t n = op.size();
    const uint32_t nchunks = (n + SORT_CHUNK - 1) / SORT_CHUNK;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (;;) {
        if (threadIdx.x == 0) s_chunk = atomicAdd(ticket, 1u);
        __syncthreads();
        const uint32_t chunk = s_chunk;
        if (chunk >= nchunks) break;
        const uint32_t base = chunk * SORT_CHUNK + threadIdx.x * SORT_ITEMS;
        uint32_t v[SORT_ITEMS];
        uint64_t tsum = 0;
#pragma unroll
        for (int j = 0; j < SORT_ITEMS; j++) {
            v[j] = (base + j < n) ? op.load(base + j) : 0u;
            tsum += v[j];
        }
        // block exclusive scan of per-thread sums
        uint64_t x = tsum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_warp[warp] = x;
        __syncthreads();
        uint64_t wbase = 0, agg = 0;
#pragma unroll
        for (int w = 0; w < SORT_THREADS / 32; w++) {
            if (w < warp) wbase += s_warp[w];
            agg += s_warp[w];
        }
        const uint64_t texcl = wbase + x - tsum;
        // look-back
        if (warp == 0) {
            if (lane == 0)
                st_volatile_u64(&status[chunk], st_make(epoch, chunk == 0 ? ST_PREFIX : ST_AGG, agg));
            uint64_t excl = 0;
            if (chunk > 0) {
                int c = (int)chunk - 1 - lane;
                for (;;) {
                    unsigned long long w = c >= 0 ? ld_volatile_u64(&status[c]) : st_make(epoch, ST_PREFIX, 0);
                    uint32_t f = c >= 0 ? st_flag(w, epoch) : (uint32_t)ST_PREFIX;
                    const uint32_t mp = __ballot_sync(0xffffffffu, f == ST_PREFIX);
                    const uint32_t mi = __ballot_sync(0xffffffffu, f == 0);
                    const int fp = mp ? __ffs(mp) - 1 : 32;
                    const uint32_t need = fp == 32 ? 0xffffffffu : ((2u << fp) - 1u);
                    if (mi & need) continue;    // a predecessor in the window has not published yet
                    uint64_t s = (lane <= fp) ? st_val(w) : 0;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                    excl += s;
                    if (fp < 32) break;
                    c -= 32;
                }
                if (lane == 0) st_volatile_u64(&status[chunk], st_make(epoch, ST_PREFIX, excl + agg));
            }
            if (lane == 0) s_prefix = excl;
        }
        __syncthreads();
        uint64_t run = s_prefix + texcl;
#pragma unroll
        for (int j = 0; j < SORT_ITEMS; j++) {
            if (base + j < n) op.emit(base + j, run, v[j]);
            run += v[j];
        }
        if (chunk == nchunks - 1 && threadIdx.x == 0) op.finish(s_prefix + agg);
        __syncthreads();
    }
}

// n == 0 still has to publish its (empty) total
template <class Op>
__global__ void k_scan_empty_finish(Op op) {
    if (op.size() == 0) op.finish(0);
}

// ---------------------------------------------------------------------------
// digit histograms for all passes (warp-aggregated shared atomics)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t keys_in_play(const Counters *cnt, int which, uint64_t max_keys,
                                                  uint32_t n_static) {
    if (which == 0) return n_static;
    if (which == 1) return cnt->n_visible;
    { const uint64_t k = cnt->n_keys; return (cnt->err != 0u) ? 0u : (uint32_t)(k < max_keys ? k : max_keys); }
}

__global__ void __launch_bounds__(256) k_hist(const uint32_t *__restrict__ keys, const Counters *cnt, int which,
                                              uint64_t max_keys, int npasses, uint32_t *hist_out) {
    __shared__ uint32_t s_h[4][256];
    for (int t = threadIdx.x; t < 4 * 256; t += blockDim.x) (&s_h[0][0])[t] = 0;
    __syncthreads();
    const uint32_t n = keys_in_play(cnt, which, max_keys, 0);
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t base = blockIdx.x * blockDim.x; base < n; base += stride) {
        const uint32_t i = base + threadIdx.x;
        const bool valid = i < n;
        const uint32_t k = valid ? keys[i] : 0u;
        for (int p = 0; p < npasses; p++) {
            const uint32_t d = valid ? ((k >> (8 * p)) & 255u) : 0xFFFFFFFFu;
            const uint32_t peers = __match_any_sync(0xffffffffu, d);
            if (valid && (__ffs(peers) - 1) == (int)lane) atomicAdd(&s_h[p][d], (uint32_t)__popc(peers));
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < npasses * 256; t += blockDim.x) {
        const uint32_t v = (&s_h[0][0])[t];
        if (v) atomicAdd(&hist_out[t], v);
    }
}

// ---------------------------------------------------------------------------
// one stable LSD pass over 8 bits with decoupled look-back (onesweep)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(SORT_THREADS) k_onesweep(const uint32_t *__restrict__ kin,
                                                           const uint32_t *__restrict__ vin, uint32_t *kout,
                                                           uint32_t *vout, const Counters *cnt, int which,
                                                           uint64_t max_keys, int shift, const uint32_t *hist,
                                                           unsigned long long *status, uint32_t epoch,
                                                           uint32_t *ticket) {
    constexpr int NW = SORT_THREADS / 32;
    __shared__ uint32_t s_whist[NW][256];
    __shared__ uint32_t s_glob[256];
    __shared__ uint32_t s_blk[256];
    __shared__ uint32_t s_base[256];
    __shared__ uint32_t s_tot[NW];
    __shared__ uint32_t s_keys[SORT_CHUNK];
    __shared__ uint32_t s_vals[SORT_CHUNK];
    __shared__ uint32_t s_chunk;
    const uint32_t n = keys_in_play(cnt, which, max_keys, 0);
    const uint32_t nchunks = (n + SORT_CHUNK - 1) / SORT_CHUNK;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int d_own = threadIdx.x;   // SORT_THREADS == 256 digits

    // global exclusive digit offsets (block scan of the histogram)
    {
        const uint32_t h = hist[d_own];
        uint32_t x = h;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_tot[warp] = x;
        __syncthreads();
        uint32_t wb = 0;
        for (int w = 0; w < warp; w++) wb += s_tot[w];
        s_glob[d_own] = wb + x - h;
        __syncthreads();
    }

    for (;;) {
        if (threadIdx.x == 0) s_chunk = atomicAdd(ticket, 1u);
        for (int w = 0; w < NW; w++) s_whist[w][d_own] = 0;
        __syncthreads();
        const uint32_t chunk = s_chunk;
        if (chunk >= nchunks) break;
        const uint32_t cbase = chunk * SORT_CHUNK;
        const uint32_t cvalid = min((uint32_t)SORT_CHUNK, n - cbase);

        // 1. warp-local stable ranking (rounds of 32 consecutive keys)
        uint32_t key[SORT_ITEMS], val[SORT_ITEMS], rank[SORT_ITEMS];
#pragma unroll
        for (int r = 0; r < SORT_ITEMS; r++) {
            const uint32_t e = warp * (SORT_ITEMS * 32) + r * 32 + lane;
            const bool valid = e < cvalid;
            key[r] = valid ? kin[cbase + e] : 0xFFFFFFFFu;
            val[r] = valid ? vin[cbase + e] : 0u;
            const uint32_t d = valid ? ((key[r] >> shift) & 255u) : 0xFFFFFFFFu;
            const uint32_t peers = __match_any_sync(0xffffffffu, d);
            uint32_t before = 0;
            if (valid) before = s_whist[warp][d];
            __syncwarp();
            if (valid && (__ffs(peers) - 1) == lane) s_whist[warp][d] = before + __popc(peers);
            __syncwarp();
            rank[r] = before + __popc(peers & lanemask_lt());
        }
        __syncthreads();
        // 2. per digit: exclusive over warps, chunk total
        uint32_t total = 0;
        for (int w = 0; w < NW; w++) {
            const uint32_t t = s_whist[w][d_own];
            s_whist[w][d_own] = total;
            total += t;
        }
        // 3. publish aggregate, block-local exclusive digit starts
        unsigned long long *my_status = status + (size_t)chunk * 256 + d_own;
        st_volatile_u64(my_status, st_make(epoch, chunk == 0 ? ST_PREFIX : ST_AGG, total));
        {
            uint32_t x = total;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) s_tot[warp] = x;
            __syncthreads();
            uint32_t wb = 0;
            for (int w = 0; w < warp; w++) wb += s_tot[w];
            s_blk[d_own] = wb + x - total;
        }
        // 4. per-digit look-back
        uint64_t excl = 0;
        if (chunk > 0) {
            int c = (int)chunk - 1;
            while (c >= 0) {
                const unsigned long long w = ld_volatile_u64(status + (size_t)c * 256 + d_own);
                const uint32_t f = st_flag(w, epoch);
                if (f == 0) continue;
                excl += st_val(w);
                if (f == ST_PREFIX) break;
                c--;
            }
            st_volatile_u64(my_status, st_make(epoch, ST_PREFIX, excl + total));
        }
        s_base[d_own] = s_glob[d_own] + (uint32_t)excl;
        __syncthreads();
        // 5. scatter into shared memory in digit order (stable)
#pragma unroll
        for (int r = 0; r < SORT_ITEMS; r++) {
            const uint32_t e = warp * (SORT_ITEMS * 32) + r * 32 + lane;
            if (e < cvalid) {
                const uint32_t d = (key[r] >> shift) & 255u;
                const uint32_t pos = s_blk[d] + s_whist[warp][d] + rank[r];
                s_keys[pos] = key[r];
                s_vals[pos] = val[r];
            }
        }
        __syncthreads();
        // 6. coalesced runs to global memory
        for (uint32_t p = threadIdx.x; p < cvalid; p += SORT_THREADS) {
            const uint32_t k = s_keys[p];
            const uint32_t d = (k >> shift) & 255u;
            const uint32_t g = s_base[d] + (p - s_blk[d]);
            kout[g] = k;
            vout[g] = s_vals[p];
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// tile ranges: boundary detection over the sorted tile ids
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_ranges(const uint32_t *__restrict__ tiles, const Counters *cnt,
                                                uint64_t max_keys, uint2 *ranges) {
    const uint32_t n = keys_in_play(cnt, 2, max_keys, 0);
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const uint32_t t = tiles[k];
        if (k == 0 || tiles[k - 1] != t) ranges[t].x = k;
        if (k == n - 1 || tiles[k + 1] != t) ranges[t].y = k + 1;
    }
}

// ---------------------------------------------------------------------------
void launch_binning(Workspace &ws, cudaStream_t st, int N, int64_t max_keys, int ntiles, int gx,
                    uint32_t &epoch) {
    Counters *cnt = ws.counters;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int persist = nsm * 4;
    const int max_chunks_n = ceil_div_i(N > 0 ? N : 1, SORT_CHUNK);
    const int max_chunks_k = ceil_div_i(max_keys > 0 ? max_keys : 1, SORT_CHUNK);
    cudaMemsetAsync(ws.ranges, 0, sizeof(uint2) * (size_t)ntiles, st);
    int tk = 0;   // ticket index

    // 1. compaction of visible Gaussians (index order)
    CompactOp cop{ws.touched, ws.depth_bits, ws.sk[0], ws.sv[0], cnt, (uint32_t)N};
    if (N > 0)
        k_scan<CompactOp><<<std::min(persist, max_chunks_n), SORT_THREADS, 0, st>>>(cop, ws.scan_status, ++epoch,
                                                                                     &cnt->tickets[tk++]);
    else
        k_scan_empty_finish<CompactOp><<<1, 1, 0, st>>>(cop);
    // 2. depth sort: 4 stable passes of 8 bits
    k_hist<<<nsm * 2, 256, 0, st>>>(ws.sk[0], cnt, 1, 0, 4, &cnt->hist_depth[0][0]);
    for (int p = 0; p < 4; p++) {
        k_onesweep<<<std::min(persist, max_chunks_n), SORT_THREADS, 0, st>>>(
            ws.sk[p & 1], ws.sv[p & 1], ws.sk[(p + 1) & 1], ws.sv[(p + 1) & 1], cnt, 1, 0, 8 * p,
            cnt->hist_depth[p], ws.sort_status, ++epoch, &cnt->tickets[tk++]);
    }
    // 3. offsets in depth order + duplication (sorted result is in sk[0]/sv[0])
    DuplicateOp dop{ws.sv[0], ws.touched, ws.rect, ws.kt[0], ws.kv[0], cnt, (uint64_t)max_keys, gx};
    k_scan<DuplicateOp><<<std::min(persist, max_chunks_n), SORT_THREADS, 0, st>>>(dop, ws.scan_status, ++epoch,
                                                                                   &cnt->tickets[tk++]);
    k_scan_empty_finish<DuplicateOp><<<1, 1, 0, st>>>(dop);
    // 4. stable sort of the tile ids
    int tbits = 0;
    while ((1 << tbits) < ntiles) tbits++;
    const int tpasses = tbits <= 8 ? 1 : (tbits <= 16 ? 2 : 3);
    k_hist<<<nsm * 2, 256, 0, st>>>(ws.kt[0], cnt, 2, (uint64_t)max_keys, tpasses, &cnt->hist_tile[0][0]);
    for (int p = 0; p < tpasses; p++) {
        k_onesweep<<<std::min(persist, max_chunks_k), SORT_THREADS, 0, st>>>(
            ws.kt[p & 1], ws.kv[p & 1], ws.kt[(p + 1) & 1], ws.kv[(p + 1) & 1], cnt, 2, (uint64_t)max_keys, 8 * p,
            cnt->hist_tile[p], ws.sort_status, ++epoch, &cnt->tickets[tk++]);
    }
    // swap so that kt[0]/kv[0] always hold the final order
    if (tpasses & 1) {
        std::swap(ws.kt[0], ws.kt[1]);
        std::swap(ws.kv[0], ws.kv[1]);
    }
    // 5. tile ranges
    k_ranges<<<nsm * 4, 256, 0, st>>>(ws.kt[0], cnt, (uint64_t)max_keys, ws.ranges);
}

}  // namespace gs
