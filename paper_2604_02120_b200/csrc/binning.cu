// binning.cu -- stages (b) "Duplication" and (c) "Sorting"
// and the per-tile ranges, as hand-written kernels (no CUB, no host sync).
//
// Canonical result (R-12/R-13): per tile, the indices of the
// Gaussians whose rectangle contains it, ascending in (depth bits, index);
// key = tile << 32 | depth bits. The paper's "duplicate with a concatenated
// key, then radix-sort" is realised B200-first as a bucket sort
// on the tile (the high key half) followed by per-tile shared-memory sorts on
// the depth (the low half), which yields exactly the same sorted key array:
//   1. k_count    : block-private shared-memory histograms of tile hits over a
//                   fixed contiguous partition of the Gaussians -> cnt[block][tile]
//   2. k_colscan  : per tile, exclusive prefix over blocks (coalesced over tiles)
//   3. k_tilescan : exclusive scan over tiles -> ranges, K, capacity check
//   4. k_scatter  : same partition; shared-memory cursors give every (Gaussian,
//                   tile) pair a slot inside its tile's segment (order within a
//                   segment is arbitrary at this point)
//   5. k_sort_*   : per tile, LSD radix sort of (depth bits, slot) pairs in
//                   shared memory (<= 4096 and <= 16384 entries), or a chunked
//                   global-memory block sort for longer lists; equal-depth runs
//                   are then ordered by Gaussian index.
// Traffic: ~24 B per Gaussian + ~16 B per key (vs ~150 B/key for a 6-pass LSD
// sort of 64-bit keys).
#include <algorithm>

#include "gs_common.cuh"

namespace gs {

constexpr int CNT_THREADS = 512;
constexpr int SMALL_CAP = 4096, SMALL_THREADS = 256;
constexpr int BIG_CAP = 16384, BIG_THREADS = 1024;

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ---------------------------------------------------------------------------
// 1. per-block tile histograms
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(CNT_THREADS) k_count(int N, const uint32_t *__restrict__ touched,
                                                       const ushort4 *__restrict__ rect, int gx, int ntiles,
                                                       uint32_t *__restrict__ cnt) {
    extern __shared__ uint32_t s_h[];
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) s_h[t] = 0;
    __syncthreads();
    const int per = ceil_div_i(N, gridDim.x);
    const int i0 = blockIdx.x * per, i1 = min(N, i0 + per);
    for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        if (touched[i] == 0) continue;
        const ushort4 r = rect[i];
        for (int ty = r.y; ty < r.w; ty++)
            for (int tx = r.x; tx < r.z; tx++) atomicAdd(&s_h[ty * gx + tx], 1u);
    }
    __syncthreads();
    uint32_t *row = cnt + (size_t)blockIdx.x * ntiles;
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) row[t] = s_h[t];
}

// ---------------------------------------------------------------------------
// 2. per tile: exclusive prefix over the count blocks
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_colscan(uint32_t *__restrict__ cnt, int nblocks, int ntiles,
                                                 uint32_t *__restrict__ total) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntiles) return;
    uint32_t run = 0;
    int b = 0;
    for (; b + 8 <= nblocks; b += 8) {
        uint32_t c[8];
#pragma unroll
        for (int j = 0; j < 8; j++) c[j] = cnt[(size_t)(b + j) * ntiles + t];
#pragma unroll
        for (int j = 0; j < 8; j++) {
            cnt[(size_t)(b + j) * ntiles + t] = run;
            run += c[j];
        }
    }
    for (; b < nblocks; b++) {
        const uint32_t c = cnt[(size_t)b * ntiles + t];
        cnt[(size_t)b * ntiles + t] = run;
        run += c;
    }
    total[t] = run;
}

// ---------------------------------------------------------------------------
// 3. exclusive scan over tiles (one block) -> ranges, K, capacity flag
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_tilescan(const uint32_t *__restrict__ total, int ntiles,
                                                   uint2 *__restrict__ ranges, uint32_t *__restrict__ start,
                                                   Counters *cnt, uint64_t max_keys) {
    __shared__ unsigned long long s_w[32];
    __shared__ unsigned long long s_carry;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int base = 0; base < ntiles; base += 1024) {
        const int t = base + threadIdx.x;
        const unsigned long long v = t < ntiles ? total[t] : 0;
        unsigned long long x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_w[warp] = x;
        __syncthreads();
        unsigned long long wb = 0, tot = 0;
        for (int w = 0; w < 32; w++) {
            if (w < warp) wb += s_w[w];
            tot += s_w[w];
        }
        const unsigned long long ex = s_carry + wb + x - v;
        if (t < ntiles) {
            const uint32_t s = (uint32_t)(ex < 0xFFFFFFFFull ? ex : 0xFFFFFFFFull);
            const unsigned long long e2 = ex + v;
            start[t] = s;
            ranges[t] = v ? make_uint2(s, (uint32_t)(e2 < 0xFFFFFFFFull ? e2 : 0xFFFFFFFFull)) : make_uint2(0u, 0u);
        }
        __syncthreads();
        if (threadIdx.x == 0) s_carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        cnt->n_keys = s_carry;
        if (s_carry > max_keys) atomicOr(&cnt->err, 1u);
    }
}

// ---------------------------------------------------------------------------
// 4. scatter Gaussian indices into their tiles' segments
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(CNT_THREADS) k_scatter(int N, const uint32_t *__restrict__ touched,
                                                         const ushort4 *__restrict__ rect, int gx, int ntiles,
                                                         const uint32_t *__restrict__ cnt,
                                                         const uint32_t *__restrict__ start,
                                                         uint32_t *__restrict__ vals, const Counters *counters) {
    extern __shared__ uint32_t s_cur[];
    if (counters->err) return;
    const uint32_t *row = cnt + (size_t)blockIdx.x * ntiles;
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) s_cur[t] = start[t] + row[t];
    __syncthreads();
    const int per = ceil_div_i(N, gridDim.x);
    const int i0 = blockIdx.x * per, i1 = min(N, i0 + per);
    for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        if (touched[i] == 0) continue;
        const ushort4 r = rect[i];
        for (int ty = r.y; ty < r.w; ty++)
            for (int tx = r.x; tx < r.z; tx++) {
                const uint32_t pos = atomicAdd(&s_cur[ty * gx + tx], 1u);
                vals[pos] = (uint32_t)i;
            }
    }
}

// ---------------------------------------------------------------------------
// 5. per-tile sort by (depth bits, Gaussian index)
// ---------------------------------------------------------------------------
// One stable LSD pass over an n-element chunk held by the block, 8-bit digit.
// Element e belongs to warp e / (ITEMS*32), round (e / 32) % ITEMS, lane e % 32,
// so a warp ranks a contiguous range in order (stability).
template <int NW, int ITEMS>
struct BlockRanker {
    uint16_t whist[NW][256];   // per-warp digit counts, then exclusive prefix over warps
    uint32_t tot[256];         // chunk digit totals
    uint32_t dstart[256];      // chunk exclusive digit starts
    uint32_t wsum[8];
    int all_same;

    // ranks keys src[e] (e < n); returns the chunk-local destination of each
    // item in pos[]; must be called by all NW*32 threads
    __device__ void rank(const uint32_t *src, int n, int shift, uint32_t (&key)[ITEMS], uint32_t (&pos)[ITEMS]) {
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        for (int i = threadIdx.x; i < NW * 256; i += NW * 32) (&whist[0][0])[i] = 0;
        if (threadIdx.x == 0) all_same = 0;
        __syncthreads();
        uint32_t rk[ITEMS];
#pragma unroll
        for (int r = 0; r < ITEMS; r++) {
            const int e = w * (ITEMS * 32) + r * 32 + lane;
            const bool valid = e < n;
            key[r] = valid ? src[e] : 0u;
            const uint32_t d = valid ? ((key[r] >> shift) & 255u) : 0xFFFFFFFFu;
            const uint32_t peers = __match_any_sync(0xffffffffu, d);
            uint32_t before = 0;
            if (valid) before = whist[w][d];
            __syncwarp();
            if (valid && (__ffs(peers) - 1) == lane) whist[w][d] = (uint16_t)(before + __popc(peers));
            __syncwarp();
            rk[r] = before + __popc(peers & lanemask_lt());
        }
        __syncthreads();
        // per digit: exclusive over warps, totals
        for (int d = threadIdx.x; d < 256; d += NW * 32) {
            uint32_t run = 0;
#pragma unroll
            for (int ww = 0; ww < NW; ww++) {
                const uint32_t c = whist[ww][d];
                whist[ww][d] = (uint16_t)run;
                run += c;
            }
            tot[d] = run;
            if ((int)run == n) all_same = 1;
        }
        __syncthreads();
        // exclusive scan of the 256 totals (first 8 warps)
        if (threadIdx.x < 256) {
            const uint32_t v = tot[threadIdx.x];
            uint32_t x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) wsum[w] = x;
            dstart[threadIdx.x] = x - v;   // warp-local for now
        }
        __syncthreads();
        if (threadIdx.x < 256) {
            uint32_t add = 0;
            for (int ww = 0; ww < (int)(threadIdx.x >> 5); ww++) add += wsum[ww];
            dstart[threadIdx.x] += add;
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < ITEMS; r++) {
            const int e = w * (ITEMS * 32) + r * 32 + lane;
            if (e < n) {
                const uint32_t d = (key[r] >> shift) & 255u;
                pos[r] = dstart[d] + whist[w][d] + rk[r];
            }
        }
    }
};

// order runs of equal keys by Gaussian index (insertion sort; runs are rare and short)
__device__ __forceinline__ void fix_ties(const uint32_t *keys, uint32_t *g, int n) {
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const bool head = (j == 0 || keys[j - 1] != keys[j]);
        if (!head || j + 1 >= n || keys[j + 1] != keys[j]) continue;
        int e = j + 1;
        while (e < n && keys[e] == keys[j]) e++;
        for (int a = j + 1; a < e; a++) {
            const uint32_t v = g[a];
            int b = a - 1;
            while (b >= j && g[b] > v) {
                g[b + 1] = g[b];
                b--;
            }
            g[b + 1] = v;
        }
    }
}

template <int NW, int ITEMS>
struct SortSmem {
    static constexpr int CAP = NW * 32 * ITEMS;
    uint32_t k[2][CAP];
    uint16_t p[2][CAP];
    BlockRanker<NW, ITEMS> rk;
};

// Sorts one tile list of n <= CAP entries: keys = depth bits of vals_in[start + j].
template <int NW, int ITEMS>
__device__ void sort_tile_smem(SortSmem<NW, ITEMS> &sm, const uint32_t *__restrict__ vals_in,
                               uint32_t *__restrict__ vals_out, const uint32_t *__restrict__ depth_bits,
                               uint32_t start, int n) {
    for (int j = threadIdx.x; j < n; j += NW * 32) {
        sm.k[0][j] = __ldg(&depth_bits[vals_in[start + j]]);
        sm.p[0][j] = (uint16_t)j;
    }
    __syncthreads();
    int cur = 0;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int pass = 0; pass < 4; pass++) {
        uint32_t key[ITEMS], pos[ITEMS];
        sm.rk.rank(sm.k[cur], n, 8 * pass, key, pos);
        if (sm.rk.all_same) {   // every key has the same digit: the pass is the identity
            __syncthreads();
            continue;
        }
        uint16_t pv[ITEMS];
#pragma unroll
        for (int r = 0; r < ITEMS; r++) {
            const int e = w * (ITEMS * 32) + r * 32 + lane;
            if (e < n) pv[r] = sm.p[cur][e];
        }
#pragma unroll
        for (int r = 0; r < ITEMS; r++) {
            const int e = w * (ITEMS * 32) + r * 32 + lane;
            if (e < n) {
                sm.k[cur ^ 1][pos[r]] = key[r];
                sm.p[cur ^ 1][pos[r]] = pv[r];
            }
        }
        cur ^= 1;
        __syncthreads();
    }
    // gather the Gaussian indices in sorted order into k[cur^1] (reused), fix ties, write out
    uint32_t *g = sm.k[cur ^ 1];
    for (int j = threadIdx.x; j < n; j += NW * 32) g[j] = vals_in[start + sm.p[cur][j]];
    __syncthreads();
    fix_ties(sm.k[cur], g, n);
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += NW * 32) vals_out[start + j] = g[j];
}

__global__ void __launch_bounds__(SMALL_THREADS) k_sort_small(const uint2 *__restrict__ ranges,
                                                              const uint32_t *__restrict__ vals_in,
                                                              uint32_t *__restrict__ vals_out,
                                                              const uint32_t *__restrict__ depth_bits,
                                                              uint32_t *__restrict__ big_list, Counters *counters) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    auto &sm = *reinterpret_cast<SortSmem<SMALL_THREADS / 32, SMALL_CAP / SMALL_THREADS> *>(smem_raw);
    if (counters->err) return;
    const int tile = blockIdx.x;
    const uint2 rg = ranges[tile];
    const int n = (int)(rg.y - rg.x);
    if (n <= 0) return;
    if (n > SMALL_CAP) {
        if (threadIdx.x == 0) big_list[atomicAdd(&counters->n_big, 1u)] = (uint32_t)tile;
        return;
    }
    if (n == 1) {
        if (threadIdx.x == 0) vals_out[rg.x] = vals_in[rg.x];
        return;
    }
    sort_tile_smem(sm, vals_in, vals_out, depth_bits, rg.x, n);
}

__global__ void __launch_bounds__(BIG_THREADS, 1) k_sort_big(const uint2 *__restrict__ ranges,
                                                             const uint32_t *__restrict__ vals_in,
                                                             uint32_t *__restrict__ vals_out,
                                                             const uint32_t *__restrict__ depth_bits,
                                                             const uint32_t *__restrict__ big_list,
                                                             uint32_t *__restrict__ huge_list, Counters *counters) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    auto &sm = *reinterpret_cast<SortSmem<BIG_THREADS / 32, BIG_CAP / BIG_THREADS> *>(smem_raw);
    if (counters->err) return;
    const uint32_t nbig = counters->n_big;
    for (uint32_t b = blockIdx.x; b < nbig; b += gridDim.x) {
        const int tile = (int)big_list[b];
        const uint2 rg = ranges[tile];
        const int n = (int)(rg.y - rg.x);
        if (n > BIG_CAP) {
            if (threadIdx.x == 0) huge_list[atomicAdd(&counters->n_huge, 1u)] = (uint32_t)tile;
            continue;
        }
        sort_tile_smem(sm, vals_in, vals_out, depth_bits, rg.x, n);
        __syncthreads();
    }
}

// Lists longer than BIG_CAP: chunked LSD sort in global memory by one block.
// Keys ping-pong between kbuf[0]/kbuf[1]; values between vals_in (used as
// scratch for its own segment) and vals_out (same segment offsets).
__global__ void __launch_bounds__(BIG_THREADS, 1) k_sort_huge(const uint2 *__restrict__ ranges,
                                                              uint32_t *vals_in, uint32_t *vals_out,
                                                              const uint32_t *__restrict__ depth_bits,
                                                              const uint32_t *__restrict__ huge_list, uint32_t *ka,
                                                              uint32_t *kb, Counters *counters) {
    constexpr int NW = BIG_THREADS / 32, ITEMS = BIG_CAP / BIG_THREADS;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    auto &sm = *reinterpret_cast<SortSmem<NW, ITEMS> *>(smem_raw);
    __shared__ uint32_t s_base[256];
    __shared__ uint32_t s_hist[256];
    __shared__ int s_same;
    if (counters->err) return;
    const uint32_t nh = counters->n_huge;
    for (uint32_t hI = blockIdx.x; hI < nh; hI += gridDim.x) {
        const uint2 rg = ranges[huge_list[hI]];
        const uint32_t s0 = rg.x;
        const int n = (int)(rg.y - rg.x);
        uint32_t *K[2] = {ka + s0, kb + s0};
        uint32_t *V[2] = {vals_in + s0, vals_out + s0};
        for (int j = threadIdx.x; j < n; j += BIG_THREADS) K[0][j] = depth_bits[V[0][j]];
        __syncthreads();
        int cur = 0;
        for (int pass = 0; pass < 4; pass++) {
            const int shift = 8 * pass;
            for (int d = threadIdx.x; d < 256; d += BIG_THREADS) s_hist[d] = 0;
            if (threadIdx.x == 0) s_same = 0;
            __syncthreads();
            for (int j = threadIdx.x; j < n; j += BIG_THREADS) atomicAdd(&s_hist[(K[cur][j] >> shift) & 255u], 1u);
            __syncthreads();
            if (threadIdx.x < 256) {
                uint32_t ex = 0;
                for (int d = 0; d < (int)threadIdx.x; d++) ex += s_hist[d];
                s_base[threadIdx.x] = ex;
                if ((int)s_hist[threadIdx.x] == n) s_same = 1;
            }
            __syncthreads();
            if (s_same) continue;
            for (int c0 = 0; c0 < n; c0 += BIG_CAP) {
                const int cn = min(BIG_CAP, n - c0);
                for (int j = threadIdx.x; j < cn; j += BIG_THREADS) sm.k[0][j] = K[cur][c0 + j];
                __syncthreads();
                uint32_t key[ITEMS], pos[ITEMS];
                sm.rk.rank(sm.k[0], cn, shift, key, pos);
                const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
                for (int r = 0; r < ITEMS; r++) {
                    const int e = w * (ITEMS * 32) + r * 32 + lane;
                    if (e < cn) {
                        const uint32_t d = (key[r] >> shift) & 255u;
                        const uint32_t g = s_base[d] + (pos[r] - sm.rk.dstart[d]);
                        K[cur ^ 1][g] = key[r];
                        V[cur ^ 1][g] = V[cur][c0 + e];
                    }
                }
                __syncthreads();
                if (threadIdx.x < 256) s_base[threadIdx.x] += sm.rk.tot[threadIdx.x];
                __syncthreads();
            }
            cur ^= 1;
            __syncthreads();
        }
        if (cur == 0)
            for (int j = threadIdx.x; j < n; j += BIG_THREADS) V[1][j] = V[0][j];
        __syncthreads();
        fix_ties(K[cur], V[1], n);
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
int launch_binning(Workspace &ws, cudaStream_t st, int N, int64_t max_keys, int ntiles, int gx, uint32_t &) {
    Counters *cnt = ws.counters;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    static bool attrs = false;
    const size_t small_smem = sizeof(SortSmem<SMALL_THREADS / 32, SMALL_CAP / SMALL_THREADS>);
    const size_t big_smem = sizeof(SortSmem<BIG_THREADS / 32, BIG_CAP / BIG_THREADS>);
    if (!attrs) {
        cudaFuncSetAttribute(k_count, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * MAX_TILES);
        cudaFuncSetAttribute(k_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * MAX_TILES);
        cudaFuncSetAttribute(k_sort_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)small_smem);
        cudaFuncSetAttribute(k_sort_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)big_smem);
        cudaFuncSetAttribute(k_sort_huge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)big_smem);
        attrs = true;
    }
    const int G = ws.count_blocks;
    const size_t hsmem = sizeof(uint32_t) * (size_t)ntiles;
    int launches = 0;
    if (N > 0) {
        k_count<<<G, CNT_THREADS, hsmem, st>>>(N, ws.touched, ws.rect, gx, ntiles, ws.cnt);
        launches++;
    } else {
        cudaMemsetAsync(ws.cnt, 0, sizeof(uint32_t) * (size_t)G * ntiles, st);
    }
    k_colscan<<<ceil_div_i(ntiles, 256), 256, 0, st>>>(ws.cnt, G, ntiles, ws.tile_total);
    k_tilescan<<<1, 1024, 0, st>>>(ws.tile_total, ntiles, ws.ranges, ws.tile_start, cnt, (uint64_t)max_keys);
    launches += 2;
    if (N > 0) {
        k_scatter<<<G, CNT_THREADS, hsmem, st>>>(N, ws.touched, ws.rect, gx, ntiles, ws.cnt, ws.tile_start,
                                                  ws.kv[0], cnt);
        k_sort_small<<<ntiles, SMALL_THREADS, small_smem, st>>>(ws.ranges, ws.kv[0], ws.kv[1], ws.depth_bits,
                                                                 ws.big_list, cnt);
        k_sort_big<<<nsm, BIG_THREADS, big_smem, st>>>(ws.ranges, ws.kv[0], ws.kv[1], ws.depth_bits, ws.big_list,
                                                       ws.huge_list, cnt);
        k_sort_huge<<<nsm, BIG_THREADS, big_smem, st>>>(ws.ranges, ws.kv[0], ws.kv[1], ws.depth_bits,
                                                        ws.huge_list, ws.kt[0], ws.kt[1], cnt);
        launches += 4;
    }
    return launches;
}

}  // namespace gs
