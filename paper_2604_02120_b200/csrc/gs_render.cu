// gs_render.cu -- the C-ABI of include/gs_render.h: context / workspace
// management and the per-frame orchestration of the four stages (PAPER.md
// P:109-117): preprocess -> compaction + depth sort -> duplication -> tile
// sort + ranges -> blend. All counts stay on the device (no host sync inside
// a frame); the only optional synchronisation is GS_FLAG_SYNC / gs_last_stats.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "gs_common.cuh"

struct gs_ctx {
    int device = 0;
    int num_sms = 148;
    int64_t max_points = 0, max_keys = 0;
    int max_w = 0, max_h = 0, max_tiles = 0;
    gs::Workspace ws{};
    uint32_t epoch = 0;
    cudaStream_t last_stream = nullptr;
    int64_t last_n = 0;
    int last_status = GS_OK;
    float *frame_rgb = nullptr, *frame_T = nullptr;   // staging for the host entry point
    int64_t launches = 0;                             // kernels launched (gs_stats.launches)
    // GS_FLAG_TIMING: a pool of events and (stage, start, end) spans, drained by gs_stage_times
    std::vector<cudaEvent_t> ev;
    int ev_used = 0;
    struct Span { int stage, e0, e1; };
    std::vector<Span> spans;
    double stage_ms[3] = {0, 0, 0};
    int64_t timed_frames = 0;
    // view groups (gs_render_views): per-view preprocess outputs + counters of every view slot
    int view_group = 4;
    // slot s*MAX_VIEW_GROUP + j = view j of a group in slot set s (two sets: the preprocess of
    // group g+1 runs while group g bins and blends). None of them is the context's own
    // workspace `ws`, which only the single-view calls (gs_render, gs_debug_*) use on the
    // caller's stream: a view group's preprocess may start before the caller's earlier work
    // (GS_FLAG_STATIC_SCENE, the host entry points), so the two must share no buffer.
    gs::Workspace vws[2 * gs::MAX_VIEW_GROUP] = {};
    bool vws_alloc[2 * gs::MAX_VIEW_GROUP] = {};
    gs::Counters *last_counters = nullptr;   // counters of the last rendered view
    gs::Sticky *sticky = nullptr;            // errors / largest K over the views of the last single-view call
    gs::Sticky *vsticky = nullptr;           // the same for the view-group calls (their own accumulator)
    gs::Sticky *last_sticky = nullptr;       // the accumulator of the last call (gs_last_stats)
    // gs_render_views_host: device -> host frame copies overlap the next view group
    cudaStream_t copy_stream = nullptr;
    // scene staging, double-buffered (the async entry point uploads call k+1's scene while
    // call k renders): up_stream copies, ev_scene_free[b] = the last preprocess reading b
    float *stage[2] = {};
    size_t stage_cap = 0;
    int stage_idx = 0;
    cudaStream_t up_stream = nullptr;
    cudaEvent_t ev_scene_ready[2] = {}, ev_scene_free[2] = {}, ev_copies_all = nullptr;
    // per staging slot (2 * MAX_VIEW_GROUP frames): the view's blend done / its copy done
    cudaEvent_t view_done[2 * gs::MAX_VIEW_GROUP] = {}, copies_done[2 * gs::MAX_VIEW_GROUP] = {};
    // gs_render_views, concurrent mode: preprocess on pre_stream, the binning chain of view j
    // of a group on bstream[j], blends on blend_stream (high priority); events per slot set
    bool concurrent = true;
    bool streams_ready = false;
    cudaStream_t pre_stream = nullptr, blend_stream = nullptr, bstream[gs::MAX_VIEW_GROUP] = {};
    cudaEvent_t ev_start = nullptr, ev_pre[2] = {}, ev_blended[2] = {}, ev_binned[2][gs::MAX_VIEW_GROUP] = {};
    // one event per view group of the last gs_render_views call, recorded after the group's
    // blends (gs_stream_wait_group: a consumer of the frames, e.g. the NCCL frame gather,
    // starts on group g while later groups still render)
    std::vector<cudaEvent_t> ev_group;
    int n_groups = 0;
    // one event per view of the last gs_render_views call, after its blend (gs_stream_wait_view)
    std::vector<cudaEvent_t> ev_view;
    int n_views_last = 0;
};

static constexpr int kMaxEvents = 4096;
#ifndef GS_CHAIN_STREAMS
#define GS_CHAIN_STREAMS 16   // concurrent binning chains of a view group (<= MAX_VIEW_GROUP)
#endif
static_assert(GS_CHAIN_STREAMS >= 1 && GS_CHAIN_STREAMS <= gs::MAX_VIEW_GROUP, "chain streams");
namespace gs {
int g_pdl = 1;
}

namespace {

template <class T>
cudaError_t alloc(T *&p, size_t count) {
    return cudaMalloc(reinterpret_cast<void **>(&p), std::max<size_t>(count, 1) * sizeof(T));
}

bool aligned16(const void *p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int check_cuda(cudaError_t e) {
    if (e != cudaSuccess) {
        fprintf(stderr, "gs_render: CUDA error %s\n", cudaGetErrorString(e));
        return GS_ERR_CUDA;
    }
    return GS_OK;
}

// every device buffer of one workspace (preprocess outputs, binning buffers, counters)
cudaError_t alloc_ws(gs::Workspace &w, size_t N, size_t K, size_t T) {
    // + 512: the row-aligned column chunks add at most one partial chunk per tile row
    w.max_chunks = (size_t)gs::ceil_div_i((int64_t)std::max(N, K) + 1, gs::SORT_CHUNK) + 1 + 512;
    cudaError_t e = cudaSuccess;
#define A(ptr, n) \
    if (e == cudaSuccess) e = alloc(ptr, n)
    A(w.wcount, N / 32 + 1); A(w.orig, N);
    A(w.depth_bits, N); A(w.splat, N); A(w.rect, N); A(w.touched, N);
    A(w.radius, N); A(w.tmask, N); A(w.tmask_r, N); A(w.sk[0], N); A(w.sk[1], N); A(w.sv[0], N); A(w.sv[1], N); A(w.off, N); A(w.rect_r, N);
    A(w.kt[0], K); A(w.kt[1], K); A(w.kv[0], K); A(w.kv[1], K); A(w.chunk_first, w.max_chunks);
    A(w.ranges, T); A(w.sums, 2 * w.max_chunks); A(w.cmat, w.max_chunks * 512); A(w.row_total, 512);
    A(w.cdesc, w.max_chunks); A(w.cdesc_last, w.max_chunks); A(w.tile_cnt, T); A(w.rowinfo, 3 * 513);
    A(w.counters, 1);
#undef A
    if (e == cudaSuccess) e = cudaMemset(w.counters, 0, sizeof(gs::Counters));
    // the compaction loads every slot's depth unconditionally (both loads in flight at
    // once) and discards those of unused slots: defined contents keep initcheck clean
    if (e == cudaSuccess) e = cudaMemset(w.depth_bits, 0, sizeof(uint32_t) * N);
    return e;
}

void free_ws(gs::Workspace &w) {
    void *ptrs[] = {w.wcount, w.orig, w.tmask, w.tmask_r, w.depth_bits, w.splat, w.rect, w.touched, w.radius, w.sk[0], w.sk[1],
                    w.sv[0], w.sv[1], w.off, w.rect_r, w.kt[0], w.kt[1], w.kv[0], w.kv[1], w.chunk_first,
                    w.ranges, w.sums, w.cmat, w.row_total, w.cdesc, w.cdesc_last, w.tile_cnt, w.rowinfo,
                    w.counters, w.stage};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    w = gs::Workspace{};
}

int validate(gs_ctx *c, int N, const void *means, const void *scales, const void *rots, const void *opacity,
             const void *shs, const gs_camera *cam, int W, int H, const gs_opts *o) {
    if (!c || !cam || !o || N < 0 || W <= 0 || H <= 0) return GS_ERR_INVALID_ARG;
    if (W > c->max_w || H > c->max_h) return GS_ERR_INVALID_ARG;
    if (N > c->max_points) return GS_ERR_CAPACITY;
    if (o->sh_degree > 3 || o->sh_degree < -1) return GS_ERR_INVALID_ARG;
    if (o->blend < GS_BLEND_TC || o->blend > GS_BLEND_TC_COLOR) return GS_ERR_INVALID_ARG;
    if (o->batch != 0 && o->batch != 32 && o->batch != 64 && o->batch != 128 && o->batch != 256)
        return GS_ERR_INVALID_ARG;
    if (o->n_bands < 0 || (o->n_bands > 1 && (o->band < 0 || o->band >= o->n_bands)))
        return GS_ERR_INVALID_ARG;
    if (o->sh_degree >= 0 && o->sh_stride < (o->sh_degree + 1) * (o->sh_degree + 1)) return GS_ERR_INVALID_ARG;
    if (N > 0 && (!means || !scales || !rots || !opacity || !shs)) return GS_ERR_INVALID_ARG;
    if (!aligned16(rots)) return GS_ERR_ALIGNMENT;
    return GS_OK;
}

void drain_events(gs_ctx *c) {
    for (const auto &sp : c->spans) cudaEventSynchronize(c->ev[sp.e1]);
    for (const auto &sp : c->spans) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, c->ev[sp.e0], c->ev[sp.e1]);
        c->stage_ms[sp.stage] += ms;
    }
    c->spans.clear();
    c->ev_used = 0;
}

// GS_FLAG_TIMING: records an event on st, returns its pool index (-1 when timing is off)
int mark(gs_ctx *c, cudaStream_t st, const gs_opts &o) {
    if (!(o.flags & GS_FLAG_TIMING)) return -1;
    if (c->ev.empty()) {
        c->ev.resize(kMaxEvents);
        for (auto &e : c->ev) cudaEventCreate(&e);
    }
    if (c->ev_used == kMaxEvents) drain_events(c);   // only between spans (see callers)
    cudaEventRecord(c->ev[c->ev_used], st);
    return c->ev_used++;
}
void span(gs_ctx *c, int stage, int e0, int e1) {
    if (e0 >= 0 && e1 > e0) c->spans.push_back({stage, e0, e1});
}

// the workspace of view slot v of a group: slot 0 is the context's own; slots 1..G-1
// get a full workspace of their own (~1 GB at C5), so the views' binning chains can run
// concurrently on their own streams
int view_ws(gs_ctx *c, int v, gs::Workspace **out) {
    gs::Workspace &w = c->vws[v];
    if (!c->vws_alloc[v]) {
        if (!c->vsticky) {
            cudaError_t e = alloc(c->vsticky, 1);
            if (e == cudaSuccess) e = cudaMemset(c->vsticky, 0, sizeof(gs::Sticky));
            if (e != cudaSuccess) {
                if (c->vsticky) cudaFree(c->vsticky);
                c->vsticky = nullptr;
                return check_cuda(e);
            }
        }
        if (int rc = check_cuda(alloc_ws(w, (size_t)c->max_points, (size_t)c->max_keys, (size_t)c->max_tiles))) {
            free_ws(w);   // a partial allocation is released; the slot stays unallocated (a retry re-allocates)
            cudaGetLastError();
            return rc;
        }
        w.sticky = c->vsticky;
        c->vws_alloc[v] = true;
    }
    *out = &w;
    return GS_OK;
}

// binning of one preprocessed view (its workspace) on st
void enqueue_binning(gs_ctx *c, gs::Workspace &w, cudaStream_t st, int N, const gs_camera &cam, int W, int H,
                     const gs_opts &o, bool concurrent = false) {
    const int gx = gs::ceil_div_i(W, GS_TILE), gy = gs::ceil_div_i(H, GS_TILE);
    // the tcgen05 blend filters supertile lists itself; the other blends read per-tile lists
    const bool super = (o.blend == GS_BLEND_TC || o.blend == GS_BLEND_TC_COLOR) && !(o.flags & GS_FLAG_TILE_LISTS) &&
                       gs::supertile_count(gx, gy) <= 512;
    w.list_sgx = super ? gs::ceil_div_i(gx, 4) : 0;
    c->launches += gs::launch_binning(w, st, N, c->max_keys, gx * gy, gx, c->epoch, (o.flags & GS_FLAG_TIGHT) != 0,
                                      cam.znear, concurrent, super);
}

// preprocess + binning of one view into the context's workspace (counters zeroed first)
int enqueue_front(gs_ctx *c, cudaStream_t st, int N, const float *means, const float *scales, const float *rots,
                  const float *opacity, const float *shs, const gs_camera &cam, int W, int H, const gs_opts &o,
                  bool debug = false) {
    const int e0 = mark(c, st, o);
    cudaMemsetAsync(c->sticky, 0, sizeof(gs::Sticky), st);   // this call's error accumulator
    c->last_sticky = c->sticky;
    if (N == 0) cudaMemsetAsync(c->ws.counters, 0, sizeof(gs::Counters), st);   // else k_preprocess zeroes them
    int y0 = 0, y1 = 0;
    gs::band_rows(gs::ceil_div_i(H, GS_TILE), o.band, o.n_bands, y0, y1);
    gs::launch_preprocess(c->ws, st, N, means, scales, rots, opacity, shs, o.sh_degree, o.sh_stride,
                          o.scale_modifier, cam, W, H, gs::intersect_mode(o.flags), debug, y0, y1);
    c->launches += N > 0 ? 1 : 0;
    const int e1 = mark(c, st, o);
    enqueue_binning(c, c->ws, st, N, cam, W, H, o);
    const int e2 = mark(c, st, o);
    span(c, 0, e0, e1);
    span(c, 1, e1, e2);
    c->last_counters = c->ws.counters;
    return e2;
}

// the lists a workspace's last binning produced
gs::TileLists lists_of(const gs::Workspace &w) {
    return gs::TileLists{w.kv[0], w.list_sgx ? w.kt[0] : nullptr, w.ranges, w.list_sgx};
}

void enqueue_blend(gs_ctx *c, const gs::Workspace &w, cudaStream_t st, const gs::Splat *splat,
                   const gs::TileLists &lists, int W, int H, const gs_opts &o, float *out_rgb, float *out_T,
                   float *dump) {
    const uint32_t *vals = lists.vals;
    const uint2 *ranges = lists.ranges;   // (per-tile lists for the mma.sync and direct blends)
    const int gx = gs::ceil_div_i(W, GS_TILE), gy = gs::ceil_div_i(H, GS_TILE);
    int y0 = 0, y1 = gy;   // the row band's tiles only (a split frame's other bands are untouched)
    gs::band_rows(gy, o.band, o.n_bands, y0, y1);
    const int t0 = y0 * gx, t1 = y1 * gx;
    if (o.blend == GS_BLEND_DIRECT && !dump)
        gs::launch_blend_direct(st, splat, vals, ranges, t0, t1, gx, W, H, o.bg, out_rgb, out_T,
                                w.counters);
    else if (o.blend == GS_BLEND_MMA && !dump)
        gs::launch_blend_mma(w, st, splat, vals, ranges, t0, t1, gx, W, H, o.bg, out_rgb, out_T,
                             c->num_sms, o.batch);
    else
        gs::launch_blend_tc(w, st, splat, lists, t0, t1, gx, W, H, o.bg, out_rgb, out_T, dump, c->num_sms,
                            (o.flags & GS_FLAG_STATS) != 0, o.blend == GS_BLEND_TC_COLOR);
    c->launches += 1;
}

int finish(gs_ctx *c, cudaStream_t st, const gs_opts &o, int64_t N) {
    c->last_stream = st;
    c->last_n = N;
    c->last_status = GS_OK;
    int rc = check_cuda(cudaGetLastError());
    if (rc) return c->last_status = rc;
    if (o.flags & GS_FLAG_SYNC) {
        gs_stats s;
        rc = gs_last_stats(c, &s);
        if (rc) return rc;
        return s.status;
    }
    return GS_OK;
}

// ---- small packing kernels for the debug / split entry points ------------
__global__ void k_pack_splats(int N, const float *xy, const float *conic, const float *opacity, const float *rgb,
                              gs::Splat *out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    gs::Splat s;
    s.m = make_float2(xy[2 * i], xy[2 * i + 1]);
    s.aux = make_float2(0.f, 0.f);
    s.co = make_float4(conic[3 * i], conic[3 * i + 1], conic[3 * i + 2], opacity[i]);
    s.col = rgb ? make_float4(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2], 0.f) : make_float4(0.f, 0.f, 0.f, 0.f);
    out[i] = s;
}

// debug preprocess: scatter the slot-addressed outputs back to Gaussian order (the
// outputs were zeroed first, so culled Gaussians read all zero)
__global__ void k_unpack_pre(int N, gs::Workspace ws, float *depth, float *xy, float *conic, float *rgb,
                             int32_t *rect, int32_t *radius, uint32_t *touched) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= N || (uint32_t)(s & 31) >= ws.wcount[s >> 5]) return;
    const uint32_t i = ws.orig[s];
    depth[i] = __uint_as_float(ws.depth_bits[s]);
    const gs::Splat sp = ws.splat[s];
    xy[2 * i] = sp.m.x;
    xy[2 * i + 1] = sp.m.y;
    const float4 co = sp.co;
    conic[3 * i] = co.x; conic[3 * i + 1] = co.y; conic[3 * i + 2] = co.z;
    const float4 c = sp.col;
    rgb[3 * i] = c.x; rgb[3 * i + 1] = c.y; rgb[3 * i + 2] = c.z;
    const ushort4 r = ws.rect[s];
    rect[4 * i] = r.x; rect[4 * i + 1] = r.y; rect[4 * i + 2] = r.z; rect[4 * i + 3] = r.w;
    radius[i] = ws.radius[s];
    touched[i] = ws.touched[s];
}

__global__ void k_keys_out(const uint2 *ranges, const uint32_t *idx, const uint32_t *depth_bits,
                           const uint32_t *orig, uint64_t *keys, uint32_t *vals) {
    const uint2 rg = ranges[blockIdx.x];
    for (uint32_t k = rg.x + threadIdx.x; k < rg.y; k += blockDim.x) {
        const uint32_t s = idx[k];   // slot -> (tile << 32 | depth bits, Gaussian index)
        keys[k] = ((uint64_t)blockIdx.x << 32) | depth_bits[s];
        vals[k] = orig[s];
    }
}

// debug binning of supertile lists: tile t's list = the entries of its supertile's list
// whose key has the tile's mask bit (the filter the tcgen05 blend's producer applies)
__device__ __forceinline__ void st_tile_of(const gs::TileLists &l, int gx, int t, uint2 &rg, uint32_t &kbit) {
    const int tx = t % gx, ty = t / gx;
    rg = l.ranges[(ty >> 2) * l.sgx + (tx >> 2)];
    kbit = 1u << (16 + 4 * (ty & 3) + (tx & 3));
}

__global__ void k_st_tile_count(gs::TileLists l, int gx, uint32_t *tile_cnt) {
    __shared__ uint32_t s_n;
    uint2 rg;
    uint32_t kbit;
    st_tile_of(l, gx, blockIdx.x, rg, kbit);
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    uint32_t n = 0;
    for (uint32_t k = rg.x + threadIdx.x; k < rg.y; k += blockDim.x) n += (l.keys[k] & kbit) ? 1u : 0u;
    atomicAdd(&s_n, n);
    __syncthreads();
    if (threadIdx.x == 0) tile_cnt[blockIdx.x] = s_n;
}

// one warp per tile: the kept entries in list order (ballot compaction) -> keys / values
__global__ void k_st_tile_fill(gs::TileLists l, int gx, const uint2 *tile_ranges, const uint32_t *depth_bits,
                               const uint32_t *orig, uint64_t *keys, uint32_t *vals) {
    uint2 rg;
    uint32_t kbit;
    st_tile_of(l, gx, blockIdx.x, rg, kbit);
    const uint32_t lane = threadIdx.x;
    uint32_t out = tile_ranges[blockIdx.x].x;
    for (uint32_t k0 = rg.x; k0 < rg.y; k0 += 32) {
        const uint32_t k = k0 + lane;
        const bool keep = k < rg.y && (l.keys[k] & kbit);
        const uint32_t bal = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            const uint32_t o = out + __popc(bal & ((1u << lane) - 1u));
            const uint32_t sl = l.vals[k];
            keys[o] = ((uint64_t)blockIdx.x << 32) | depth_bits[sl];
            vals[o] = orig[sl];
        }
        out += __popc(bal);
    }
}

}  // namespace

extern "C" {

const char *gs_status_string(int s) {
    switch (s) {
        case GS_OK: return "ok";
        case GS_ERR_INVALID_ARG: return "invalid argument";
        case GS_ERR_ALIGNMENT: return "pointer not 16-byte aligned";
        case GS_ERR_CAPACITY: return "capacity exceeded (N > max_points or K > max_keys)";
        case GS_ERR_CUDA: return "CUDA runtime error";
        case GS_ERR_UNSUPPORTED_ARCH: return "device is not sm_100 (B200)";
        case GS_ERR_NO_DEVICE: return "no CUDA device";
    }
    return "unknown status";
}

int gs_device_arch(int device) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return GS_ERR_NO_DEVICE;
    if (device < 0 || device >= n) return GS_ERR_INVALID_ARG;
    int ma = 0, mi = 0;
    cudaDeviceGetAttribute(&ma, cudaDevAttrComputeCapabilityMajor, device);
    cudaDeviceGetAttribute(&mi, cudaDevAttrComputeCapabilityMinor, device);
    return 10 * ma + mi;
}

int gs_ctx_create(gs_ctx **out, int device, int64_t max_points, int64_t max_keys, int max_w, int max_h) {
    if (!out || max_points < 0 || max_keys < 0 || max_w <= 0 || max_h <= 0) return GS_ERR_INVALID_ARG;
    if (max_keys >= (int64_t)1 << 32 || max_points >= (int64_t)1 << 31) return GS_ERR_INVALID_ARG;
    if ((int64_t)gs::ceil_div_i(max_w, GS_TILE) * gs::ceil_div_i(max_h, GS_TILE) > gs::MAX_TILES)
        return GS_ERR_INVALID_ARG;
    *out = nullptr;
    if (const char *e = getenv("GS_PDL")) gs::g_pdl = atoi(e) != 0;
    const int arch = gs_device_arch(device);
    if (arch < 0) return arch;
    if (arch != 100) return GS_ERR_UNSUPPORTED_ARCH;
    if (check_cuda(cudaSetDevice(device))) return GS_ERR_CUDA;
    gs_ctx *c = new (std::nothrow) gs_ctx();
    if (!c) return GS_ERR_INVALID_ARG;
    c->device = device;
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    c->max_points = max_points;
    c->max_keys = max_keys;
    c->max_w = max_w;
    c->max_h = max_h;
    c->max_tiles = gs::ceil_div_i(max_w, GS_TILE) * gs::ceil_div_i(max_h, GS_TILE);
    cudaError_t e = alloc_ws(c->ws, (size_t)max_points, (size_t)max_keys, (size_t)c->max_tiles);
    if (e == cudaSuccess) e = alloc(c->sticky, 1);
    if (e == cudaSuccess) e = cudaMemset(c->sticky, 0, sizeof(gs::Sticky));
    c->ws.sticky = c->sticky;
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        gs_ctx_destroy(c);
        return check_cuda(e);
    }
    *out = c;
    return GS_OK;
}

int gs_ctx_destroy(gs_ctx *c) {
    if (!c) return GS_ERR_INVALID_ARG;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    free_ws(c->ws);
    if (c->sticky) cudaFree(c->sticky);
    for (void *p : {(void *)c->frame_rgb, (void *)c->frame_T})
        if (p) cudaFree(p);
    for (int v = 0; v < 2 * gs::MAX_VIEW_GROUP; v++)
        if (c->vws_alloc[v]) free_ws(c->vws[v]);
    if (c->vsticky) cudaFree(c->vsticky);
    for (int k = 0; k < 2; k++) {
        for (int v = 0; v < gs::MAX_VIEW_GROUP; v++)
            if (c->ev_binned[k][v]) cudaEventDestroy(c->ev_binned[k][v]);
        if (c->ev_pre[k]) cudaEventDestroy(c->ev_pre[k]);
        if (c->ev_blended[k]) cudaEventDestroy(c->ev_blended[k]);
    }
    for (int v = 0; v < gs::MAX_VIEW_GROUP; v++)
        if (c->bstream[v]) cudaStreamDestroy(c->bstream[v]);
    if (c->ev_start) cudaEventDestroy(c->ev_start);
    for (auto e : c->ev_group) cudaEventDestroy(e);
    for (auto e : c->ev_view) cudaEventDestroy(e);
    if (c->blend_stream) cudaStreamDestroy(c->blend_stream);
    if (c->pre_stream) cudaStreamDestroy(c->pre_stream);
    for (auto &e : c->ev) cudaEventDestroy(e);
    for (int k = 0; k < 2 * gs::MAX_VIEW_GROUP; k++) {
        if (c->view_done[k]) cudaEventDestroy(c->view_done[k]);
        if (c->copies_done[k]) cudaEventDestroy(c->copies_done[k]);
    }
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    for (int k = 0; k < 2; k++) {
        if (c->stage[k]) cudaFree(c->stage[k]);
        if (c->ev_scene_ready[k]) cudaEventDestroy(c->ev_scene_ready[k]);
        if (c->ev_scene_free[k]) cudaEventDestroy(c->ev_scene_free[k]);
    }
    if (c->ev_copies_all) cudaEventDestroy(c->ev_copies_all);
    if (c->up_stream) cudaStreamDestroy(c->up_stream);
    delete c;
    return GS_OK;
}

int gs_render(gs_ctx *c, void *stream, int N, const float *means3D, const float *scales, const float *rots,
              const float *opacity, const float *shs, const gs_camera *cam, int W, int H, const gs_opts *o,
              float *out_rgb, float *out_T) {
    int rc = validate(c, N, means3D, scales, rots, opacity, shs, cam, W, H, o);
    if (rc) return rc;
    if (!out_rgb || !out_T) return GS_ERR_INVALID_ARG;
    cudaSetDevice(c->device);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int e2 = enqueue_front(c, st, N, means3D, scales, rots, opacity, shs, *cam, W, H, *o);
    enqueue_blend(c, c->ws, st, c->ws.splat, lists_of(c->ws), W, H, *o, out_rgb,
                  out_T, nullptr);
    const int e3 = mark(c, st, *o);
    span(c, 2, e2, e3);
    if (e3 >= 0) c->timed_frames++;
    return finish(c, st, *o, N);
}

// Optional per-group callbacks of render_views_impl (the host entry point's frame copies):
// pre_blend(v) runs before view v's blend is enqueued, post_blend(v) right after, both
// with the stream the blends run on.
struct GroupHooks {
    void *user;
    void (*pre_blend)(void *user, cudaStream_t bl, int v);
    void (*post_blend)(void *user, cudaStream_t bl, int v);
};

static int record_group(gs_ctx *c, cudaStream_t s, int g) {
    while ((int)c->ev_group.size() <= g) {
        cudaEvent_t e = nullptr;
        if (int rc = check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming))) return rc;
        c->ev_group.push_back(e);
    }
    c->n_groups = g + 1;
    return check_cuda(cudaEventRecord(c->ev_group[g], s));
}

static int record_view(gs_ctx *c, cudaStream_t s, int v) {
    while ((int)c->ev_view.size() <= v) {
        cudaEvent_t e = nullptr;
        if (int rc = check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming))) return rc;
        c->ev_view.push_back(e);
    }
    c->n_views_last = v + 1;
    return check_cuda(cudaEventRecord(c->ev_view[v], s));
}

static int ensure_streams(gs_ctx *c) {
    if (c->streams_ready) return GS_OK;
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaError_t e = cudaStreamCreateWithPriority(&c->pre_stream, cudaStreamNonBlocking, lo);
    // the blends run on a high-priority stream: a blend gets the SMs as soon as its chain is done
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&c->blend_stream, cudaStreamNonBlocking, hi);
    for (int j = 0; j < gs::MAX_VIEW_GROUP && e == cudaSuccess; j++)
        e = cudaStreamCreateWithPriority(&c->bstream[j], cudaStreamNonBlocking, lo);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming);
    for (int k = 0; k < 2 && e == cudaSuccess; k++) {
        e = cudaEventCreateWithFlags(&c->ev_pre[k], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_blended[k], cudaEventDisableTiming);
        for (int j = 0; j < gs::MAX_VIEW_GROUP && e == cudaSuccess; j++)
            e = cudaEventCreateWithFlags(&c->ev_binned[k][j], cudaEventDisableTiming);
    }
    if (int rc = check_cuda(e)) return rc;
    c->streams_ready = true;
    return GS_OK;
}

// n views of one scene in groups of view_group: one preprocess launch reads the scene
// once per group (k_preprocess), then each view is binned and blended (P:109-117 per view).
// Concurrent mode (default) is a three-stream software pipeline over two slot sets:
//   pre_stream:   pre(g) into slot set g%2, after the blends of group g-2 released it
//   bstream[j]:   binning chain of view j of group g, after pre(g) (the chains of a group
//                 run concurrently: they are latency-bound chains of small kernels)
//   blend_stream: blend of view j of group g, after chain (g, j)
// so pre(g+1) overlaps the chains and blends of group g. The caller's stream is joined at
// both ends (its earlier work before pre(0), the last blend before its later work).
// Serial mode runs everything on the caller's stream with slot set 0.
static int render_views_impl(gs_ctx *c, cudaStream_t st, int N, const float *means3D, const float *scales,
                             const float *rots, const float *opacity, const float *shs, const gs_camera *cams,
                             int n_views, int W, int H, const gs_opts &o, float *const *rgb_of, float *const *T_of,
                             const GroupHooks *hk = nullptr, cudaEvent_t after_last_pre = nullptr,
                             cudaEvent_t start_event = nullptr) {
    const int G = std::max(1, std::min(c->view_group, gs::MAX_VIEW_GROUP));
    const int imode = gs::intersect_mode(o.flags);
    const bool conc = c->concurrent && G > 1;
    if (conc) {
        if (int rc = ensure_streams(c)) return rc;
        if (start_event) {   // the caller orders the inputs itself (the host entry point's upload)
            cudaStreamWaitEvent(c->pre_stream, start_event, 0);
        } else {
            cudaEventRecord(c->ev_start, st);
            // GS_FLAG_STATIC_SCENE: no pending work on `stream` writes the scene, so the
            // preprocess (and binning) of this call may start while the caller's earlier
            // work -- e.g. the previous call's last blends -- still runs; the blends still
            // wait for it (they write the caller's frame buffers)
            if (!(o.flags & GS_FLAG_STATIC_SCENE)) cudaStreamWaitEvent(c->pre_stream, c->ev_start, 0);
            cudaStreamWaitEvent(c->blend_stream, c->ev_start, 0);
        }
    }
    // an error return after work was enqueued on the context streams joins them with the
    // caller's stream first, so `stream` never completes before work of this call
    auto fail = [&](int rc) {
        if (conc) {
            for (int k = 0; k < 2; k++) {
                cudaEventRecord(c->ev_blended[k], c->blend_stream);
                cudaStreamWaitEvent(st, c->ev_blended[k], 0);
            }
            cudaEventRecord(c->ev_pre[0], c->pre_stream);
            cudaStreamWaitEvent(st, c->ev_pre[0], 0);
            for (int j = 0; j < GS_CHAIN_STREAMS; j++) {
                cudaEventRecord(c->ev_binned[0][j], c->bstream[j]);
                cudaStreamWaitEvent(st, c->ev_binned[0][j], 0);
            }
        }
        return rc;
    };
    // the first slot's workspace (and the view accumulator) must exist before its reset
    {
        gs::Workspace *w0 = nullptr;
        if (int rc = view_ws(c, 0, &w0)) return fail(rc);
    }
    // the call's error accumulator: reset before any of its views bins (stream order: the
    // binning chains wait for the preprocess, which follows this reset on its stream)
    cudaMemsetAsync(c->vsticky, 0, sizeof(gs::Sticky), conc ? c->pre_stream : st);
    c->last_sticky = c->vsticky;
    int last_set = 0;
    for (int v0 = 0, g = 0; v0 < n_views; v0 += G, g++) {
        const int n = std::min(G, n_views - v0);
        const int set = conc ? (g & 1) : 0;
        last_set = set;
        gs::PreViews pv{};
        pv.n = n;
        gs::band_rows(gs::ceil_div_i(H, GS_TILE), o.band, o.n_bands, pv.band_y0, pv.band_y1);
        gs::Workspace *w[gs::MAX_VIEW_GROUP];
        for (int j = 0; j < n; j++) {
            if (int rc = view_ws(c, set * gs::MAX_VIEW_GROUP + j, &w[j])) return fail(rc);
            pv.cam[j] = cams[v0 + j];
            pv.out[j] = gs::pre_out_of(*w[j], false);
        }
        cudaStream_t ps = conc ? c->pre_stream : st;
        if (conc) cudaStreamWaitEvent(ps, c->ev_blended[set], 0);   // slot set free again (this or an earlier call)
        const int e0 = mark(c, ps, o);
        if (N == 0)
            for (int j = 0; j < n; j++) cudaMemsetAsync(w[j]->counters, 0, sizeof(gs::Counters), ps);
        gs::launch_preprocess_views(pv, ps, N, means3D, scales, rots, opacity, shs, o.sh_degree, o.sh_stride,
                                    o.scale_modifier, W, H, imode);
        c->launches += N > 0 ? 1 : 0;
        int e_prev = mark(c, ps, o);
        span(c, 0, e0, e_prev);
        if (after_last_pre && v0 + G >= n_views) cudaEventRecord(after_last_pre, ps);   // scene no longer read
        if (conc) {
            cudaEventRecord(c->ev_pre[set], ps);
            for (int j = 0; j < n; j++) {
                cudaStream_t bs = c->bstream[j % GS_CHAIN_STREAMS];   // chains beyond it queue up
                cudaStreamWaitEvent(bs, c->ev_pre[set], 0);
                const int b0 = mark(c, bs, o);
                enqueue_binning(c, *w[j], bs, N, cams[v0 + j], W, H, o, true);
                span(c, 1, b0, mark(c, bs, o));
                cudaEventRecord(c->ev_binned[set][j], bs);
            }
            cudaStream_t bl = c->blend_stream;
            for (int j = 0; j < n; j++) {
                cudaStreamWaitEvent(bl, c->ev_binned[set][j], 0);
                if (hk && hk->pre_blend) hk->pre_blend(hk->user, bl, v0 + j);
                const int e1 = mark(c, bl, o);
                enqueue_blend(c, *w[j], bl, w[j]->splat, lists_of(*w[j]), W, H,
                              o, rgb_of[v0 + j], T_of[v0 + j], nullptr);
                const int e2 = mark(c, bl, o);
                if (hk && hk->post_blend) hk->post_blend(hk->user, bl, v0 + j);
                if (int rc = record_view(c, bl, v0 + j)) return fail(rc);
                span(c, 2, e1, e2);
                if (e2 >= 0) c->timed_frames++;
                c->last_counters = w[j]->counters;
            }
            cudaEventRecord(c->ev_blended[set], bl);
            if (int rc = record_group(c, bl, g)) return fail(rc);
            continue;
        }
        for (int j = 0; j < n; j++) {
            enqueue_binning(c, *w[j], st, N, cams[v0 + j], W, H, o);
            if (hk && hk->pre_blend) hk->pre_blend(hk->user, st, v0 + j);
            const int e1 = mark(c, st, o);
            enqueue_blend(c, *w[j], st, w[j]->splat, lists_of(*w[j]), W, H, o,
                          rgb_of[v0 + j], T_of[v0 + j], nullptr);
            const int e2 = mark(c, st, o);
            if (hk && hk->post_blend) hk->post_blend(hk->user, st, v0 + j);
            if (int rc = record_view(c, st, v0 + j)) return fail(rc);
            span(c, 1, e_prev, e1);
            span(c, 2, e1, e2);
            e_prev = e2;
            if (e2 >= 0) c->timed_frames++;
            c->last_counters = w[j]->counters;
        }
        if (int rc = record_group(c, st, g)) return fail(rc);
    }
    if (conc) {   // the frames are complete in the caller's stream order
        cudaStreamWaitEvent(st, c->ev_blended[last_set], 0);
        cudaStreamWaitEvent(st, c->ev_blended[last_set ^ 1], 0);
    }
    return GS_OK;
}

int gs_render_views(gs_ctx *c, void *stream, int N, const float *means3D, const float *scales, const float *rots,
                    const float *opacity, const float *shs, const gs_camera *cams, int n_views, int W, int H,
                    const gs_opts *o, float *out_rgb, float *out_T) {
    if (!cams || n_views < 0) return GS_ERR_INVALID_ARG;
    if (n_views == 0) return GS_OK;
    for (int v = 0; v < n_views; v++) {
        int rc = validate(c, N, means3D, scales, rots, opacity, shs, &cams[v], W, H, o);
        if (rc) return rc;
    }
    if (!out_rgb || !out_T) return GS_ERR_INVALID_ARG;
    cudaSetDevice(c->device);
    const size_t plane = (size_t)W * H;
    std::vector<float *> prgb(n_views), pT(n_views);
    for (int v = 0; v < n_views; v++) {
        prgb[v] = out_rgb + (size_t)v * 3 * plane;
        pT[v] = out_T + (size_t)v * plane;
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (int rc = render_views_impl(c, st, N, means3D, scales, rots, opacity, shs, cams, n_views, W, H, *o,
                                   prgb.data(), pT.data()))
        return rc;
    return finish(c, st, *o, N);
}

// The host-buffer entry points. The scene is uploaded into one of two device staging
// buffers on the context's upload stream (after the last preprocess that read that buffer
// two calls ago), the views render as in gs_render_views, and every frame is copied back
// on the copy stream as soon as its blend is done (staging slot v % 2G, reused once its
// previous copy completed). sync: the call returns after `stream` and the copies are
// done. async: it returns at once; `stream` reaches completion only after the frames are
// on the host, and the next call's upload overlaps this call's rendering.
static int render_views_host_impl(gs_ctx *c, void *stream, int N, const float *means3D, const float *scales,
                                  const float *rots, const float *opacity, const float *shs, const gs_camera *cams,
                                  int n_views, int W, int H, const gs_opts *o, float *h_out_rgb, float *h_out_T,
                                  bool async) {
    if (!c || !o || !cams || n_views < 0 || N < 0) return GS_ERR_INVALID_ARG;
    if (N > c->max_points) return GS_ERR_CAPACITY;
    if (W <= 0 || H <= 0 || W > c->max_w || H > c->max_h) return GS_ERR_INVALID_ARG;
    if (!h_out_rgb || !h_out_T) return GS_ERR_INVALID_ARG;
    cudaSetDevice(c->device);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int ncoef = o->sh_degree < 0 ? 1 : o->sh_stride;
    const size_t f_means = 3 * (size_t)N, f_scales = 3 * (size_t)N, f_rots = 4 * (size_t)N, f_op = (size_t)N,
                 f_sh = 3 * (size_t)N * ncoef;
    auto pad4 = [](size_t x) { return (x + 3) & ~size_t(3); };
    const size_t total = pad4(f_means) + pad4(f_scales) + pad4(f_rots) + pad4(f_op) + pad4(f_sh);
    if (!c->up_stream) {
        if (check_cuda(cudaStreamCreateWithFlags(&c->up_stream, cudaStreamNonBlocking))) return GS_ERR_CUDA;
        for (int k = 0; k < 2; k++) {
            cudaEventCreateWithFlags(&c->ev_scene_ready[k], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&c->ev_scene_free[k], cudaEventDisableTiming);
        }
        cudaEventCreateWithFlags(&c->ev_copies_all, cudaEventDisableTiming);
    }
    if (total * sizeof(float) > c->stage_cap) {
        if (check_cuda(cudaDeviceSynchronize())) return GS_ERR_CUDA;   // staging in use by earlier calls
        // (re)allocation: on failure nothing stays half-allocated (stage_cap 0, null buffers),
        // so the next call retries instead of using a null staging buffer
        for (int k = 0; k < 2; k++) {
            if (c->stage[k]) cudaFree(c->stage[k]);
            c->stage[k] = nullptr;
        }
        c->stage_cap = 0;
        for (int k = 0; k < 2; k++) {
            if (cudaMalloc(&c->stage[k], total * sizeof(float)) != cudaSuccess) {
                cudaGetLastError();
                for (int j = 0; j < 2; j++) {
                    if (c->stage[j]) cudaFree(c->stage[j]);
                    c->stage[j] = nullptr;
                }
                return GS_ERR_CUDA;
            }
        }
        c->stage_cap = total * sizeof(float);
    }
    if (!c->copy_stream) {   // 2G staging frames (G <= MAX_VIEW_GROUP), a copy stream and its events
        const size_t fr = 2 * gs::MAX_VIEW_GROUP * (size_t)c->max_w * c->max_h;
        float *frgb = nullptr, *fT = nullptr;
        cudaStream_t cs = nullptr;
        cudaError_t e = cudaMalloc(&frgb, 3 * fr * sizeof(float));
        if (e == cudaSuccess) e = cudaMalloc(&fT, fr * sizeof(float));
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
        for (int k = 0; k < 2 * gs::MAX_VIEW_GROUP && e == cudaSuccess; k++) {
            if (!c->view_done[k]) e = cudaEventCreateWithFlags(&c->view_done[k], cudaEventDisableTiming);
            if (e == cudaSuccess && !c->copies_done[k])
                e = cudaEventCreateWithFlags(&c->copies_done[k], cudaEventDisableTiming);
        }
        if (e != cudaSuccess) {   // all or nothing: a retry starts from scratch
            if (frgb) cudaFree(frgb);
            if (fT) cudaFree(fT);
            if (cs) cudaStreamDestroy(cs);
            return check_cuda(e);
        }
        c->frame_rgb = frgb;
        c->frame_T = fT;
        c->copy_stream = cs;
    }
    const int b = c->stage_idx;
    c->stage_idx ^= 1;
    float *d = c->stage[b];
    float *dm = d, *ds = dm + pad4(f_means), *dr = ds + pad4(f_scales), *dop = dr + pad4(f_rots),
          *dsh = dop + pad4(f_op);
    for (int v = 0; v < n_views; v++)
        if (int rc = validate(c, N, dm, ds, dr, dop, dsh, &cams[v], W, H, o)) return rc;
    cudaStream_t up = c->up_stream;
    cudaStreamWaitEvent(up, c->ev_scene_free[b], 0);   // no preprocess still reads buffer b
    cudaMemcpyAsync(dm, means3D, f_means * 4, cudaMemcpyHostToDevice, up);
    cudaMemcpyAsync(ds, scales, f_scales * 4, cudaMemcpyHostToDevice, up);
    cudaMemcpyAsync(dr, rots, f_rots * 4, cudaMemcpyHostToDevice, up);
    cudaMemcpyAsync(dop, opacity, f_op * 4, cudaMemcpyHostToDevice, up);
    cudaMemcpyAsync(dsh, shs, f_sh * 4, cudaMemcpyHostToDevice, up);
    cudaEventRecord(c->ev_scene_ready[b], up);
    cudaStreamWaitEvent(st, c->ev_scene_ready[b], 0);
    const size_t plane = (size_t)W * H, mplane = (size_t)c->max_w * c->max_h;
    const int G = std::max(1, std::min(c->view_group, gs::MAX_VIEW_GROUP));
    gs_opts ov = *o;
    ov.flags &= ~GS_FLAG_SYNC;
    std::vector<float *> prgb(n_views), pT(n_views);
    for (int v = 0; v < n_views; v++) {
        const size_t slot = (size_t)(v % (2 * G));
        prgb[v] = c->frame_rgb + slot * 3 * mplane;
        pT[v] = c->frame_T + slot * mplane;
    }
    struct Copies {
        gs_ctx *c;
        float *h_rgb, *h_T;
        float *const *prgb, *const *pT;
        size_t plane;
        int nslots;
    } cp{c, h_out_rgb, h_out_T, prgb.data(), pT.data(), plane, 2 * G};
    GroupHooks hk;
    hk.user = &cp;
    hk.pre_blend = [](void *u, cudaStream_t bl, int v) {   // the staging slot's previous copy is done
        Copies &k = *static_cast<Copies *>(u);
        cudaStreamWaitEvent(bl, k.c->copies_done[v % k.nslots], 0);
    };
    hk.post_blend = [](void *u, cudaStream_t bl, int v) {
        Copies &k = *static_cast<Copies *>(u);
        const int sl = v % k.nslots;
        cudaEventRecord(k.c->view_done[sl], bl);
        cudaStreamWaitEvent(k.c->copy_stream, k.c->view_done[sl], 0);
        cudaMemcpyAsync(k.h_rgb + (size_t)v * 3 * k.plane, k.prgb[v], 3 * k.plane * 4, cudaMemcpyDeviceToHost,
                        k.c->copy_stream);
        cudaMemcpyAsync(k.h_T + (size_t)v * k.plane, k.pT[v], k.plane * 4, cudaMemcpyDeviceToHost, k.c->copy_stream);
        cudaEventRecord(k.c->copies_done[sl], k.c->copy_stream);
    };
    // the views' preprocess waits for this call's upload only (not for the caller's stream,
    // which still waits for the previous call's last copies), so back-to-back async calls
    // overlap; the slot sets and staging frames are protected by their own events
    if (int rc = render_views_impl(c, st, N, dm, ds, dr, dop, dsh, cams, n_views, W, H, ov, prgb.data(), pT.data(),
                                   &hk, c->ev_scene_free[b], c->ev_scene_ready[b]))
        return rc;
    cudaEventRecord(c->ev_copies_all, c->copy_stream);
    cudaStreamWaitEvent(st, c->ev_copies_all, 0);   // st completes only once the frames are on the host
    if (async) return finish(c, st, ov, N);
    int rc = check_cuda(cudaStreamSynchronize(st));
    if (rc) return rc;
    gs_opts os = *o;
    os.flags |= GS_FLAG_SYNC;
    return finish(c, st, os, N);
}

int gs_render_views_host(gs_ctx *c, void *stream, int N, const float *means3D, const float *scales,
                         const float *rots, const float *opacity, const float *shs, const gs_camera *cams,
                         int n_views, int W, int H, const gs_opts *o, float *h_out_rgb, float *h_out_T) {
    return render_views_host_impl(c, stream, N, means3D, scales, rots, opacity, shs, cams, n_views, W, H, o, h_out_rgb,
                                  h_out_T, false);
}

int gs_render_views_host_async(gs_ctx *c, void *stream, int N, const float *means3D, const float *scales,
                               const float *rots, const float *opacity, const float *shs, const gs_camera *cams,
                               int n_views, int W, int H, const gs_opts *o, float *h_out_rgb, float *h_out_T) {
    return render_views_host_impl(c, stream, N, means3D, scales, rots, opacity, shs, cams, n_views, W, H, o, h_out_rgb,
                                  h_out_T, true);
}

int gs_debug_timeline(gs_ctx *c, double *out, int max_spans, int *n_spans) {
    if (!c || !out || !n_spans || max_spans < 0) return GS_ERR_INVALID_ARG;
    cudaSetDevice(c->device);
    int n = 0;
    for (const auto &sp : c->spans) cudaEventSynchronize(c->ev[sp.e1]);
    for (const auto &sp : c->spans) {
        if (n >= max_spans) break;
        float t0 = 0.f, t1 = 0.f;
        cudaEventElapsedTime(&t0, c->ev[0], c->ev[sp.e0]);
        cudaEventElapsedTime(&t1, c->ev[0], c->ev[sp.e1]);
        out[3 * n] = sp.stage;
        out[3 * n + 1] = t0;
        out[3 * n + 2] = t1;
        n++;
    }
    *n_spans = n;
    return check_cuda(cudaGetLastError());
}

int gs_stream_wait_group(gs_ctx *c, void *stream, int g) {
    if (!c || g < 0 || g >= c->n_groups) return GS_ERR_INVALID_ARG;
    cudaSetDevice(c->device);
    return check_cuda(cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(stream), c->ev_group[g], 0));
}

int gs_stream_wait_view(gs_ctx *c, void *stream, int v) {
    if (!c || v < 0 || v >= c->n_views_last) return GS_ERR_INVALID_ARG;
    cudaSetDevice(c->device);
    return check_cuda(cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(stream), c->ev_view[v], 0));
}

int gs_set_view_group(gs_ctx *c, int g, int concurrent) {
    if (!c || g < 1 || g > gs::MAX_VIEW_GROUP) return GS_ERR_INVALID_ARG;
    c->view_group = g;
    c->concurrent = concurrent != 0;
    return GS_OK;
}

int gs_last_stats(gs_ctx *c, gs_stats *out) {
    if (!c || !out) return GS_ERR_INVALID_ARG;
    cudaSetDevice(c->device);
    if (check_cuda(cudaStreamSynchronize(c->last_stream))) return GS_ERR_CUDA;
    gs::Counters h;
    const gs::Counters *src = c->last_counters ? c->last_counters : c->ws.counters;
    if (check_cuda(cudaMemcpy(&h, src, sizeof(h), cudaMemcpyDeviceToHost))) return GS_ERR_CUDA;
    gs::Sticky sk{};
    const gs::Sticky *sks = c->last_sticky ? c->last_sticky : c->sticky;
    if (check_cuda(cudaMemcpy(&sk, sks, sizeof(sk), cudaMemcpyDeviceToHost))) return GS_ERR_CUDA;
    out->n_points = c->last_n;
    out->n_visible = h.n_visible;
    // K: the last view's, or the largest of the call's views if one of them overflowed
    out->n_keys = (sk.err & 1u) ? (int64_t)std::max<unsigned long long>(sk.max_keys, h.n_keys) : (int64_t)h.n_keys;
    out->capacity_keys = c->max_keys;
    out->status = ((h.err | sk.err) & 1u) ? GS_ERR_CAPACITY : c->last_status;
    out->launches = c->launches;
    out->pairs_evaluated = (int64_t)h.pairs_eval;
    out->pairs_kept = (int64_t)h.pairs_kept;
    c->last_status = out->status;
    return GS_OK;
}

int gs_stage_times(gs_ctx *c, double *ms, int64_t *frames) {
    if (!c || !ms) return GS_ERR_INVALID_ARG;
    cudaSetDevice(c->device);
    drain_events(c);
    for (int k = 0; k < 3; k++) {
        ms[k] = c->stage_ms[k];
        c->stage_ms[k] = 0;
    }
    if (frames) *frames = c->timed_frames;
    c->timed_frames = 0;
    return check_cuda(cudaGetLastError());
}

int gs_debug_preprocess(gs_ctx *c, void *stream, int N, const float *means3D, const float *scales,
                        const float *rots, const float *opacity, const float *shs, const gs_camera *cam, int W,
                        int H, const gs_opts *o, float *depth, float *xy, float *conic, float *rgb, int32_t *rect,
                        int32_t *radius, uint32_t *touched) {
    int rc = validate(c, N, means3D, scales, rots, opacity, shs, cam, W, H, o);
    if (rc) return rc;
    cudaSetDevice(c->device);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    gs::launch_preprocess(c->ws, st, N, means3D, scales, rots, opacity, shs, o->sh_degree, o->sh_stride,
                          o->scale_modifier, *cam, W, H, gs::intersect_mode(o->flags), true, 0,
                          gs::ceil_div_i(H, GS_TILE));
    c->last_counters = c->ws.counters;
    c->last_sticky = c->sticky;
    if (N > 0) {
        cudaMemsetAsync(depth, 0, sizeof(float) * N, st);
        cudaMemsetAsync(xy, 0, sizeof(float) * 2 * N, st);
        cudaMemsetAsync(conic, 0, sizeof(float) * 3 * N, st);
        cudaMemsetAsync(rgb, 0, sizeof(float) * 3 * N, st);
        cudaMemsetAsync(rect, 0, sizeof(int32_t) * 4 * N, st);
        cudaMemsetAsync(radius, 0, sizeof(int32_t) * N, st);
        cudaMemsetAsync(touched, 0, sizeof(uint32_t) * N, st);
        k_unpack_pre<<<gs::ceil_div_i(N, 256), 256, 0, st>>>(N, c->ws, depth, xy, conic, rgb, rect, radius, touched);
    }
    return finish(c, st, *o, N);
}

int gs_debug_binning(gs_ctx *c, void *stream, int N, const float *means3D, const float *scales, const float *rots,
                     const float *opacity, const float *shs, const gs_camera *cam, int W, int H, const gs_opts *o,
                     uint64_t *keys, uint32_t *vals, uint32_t *ranges, int64_t capacity, int64_t *n_keys) {
    int rc = validate(c, N, means3D, scales, rots, opacity, shs, cam, W, H, o);
    if (rc) return rc;
    if (!n_keys || !ranges) return GS_ERR_INVALID_ARG;
    cudaSetDevice(c->device);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    enqueue_front(c, st, N, means3D, scales, rots, opacity, shs, *cam, W, H, *o, true);   // + debug outputs
    c->last_stream = st;
    gs_stats s;
    rc = gs_last_stats(c, &s);
    if (rc) return rc;
    *n_keys = s.n_keys;
    if (s.status) return s.status;
    if (s.n_keys > capacity) return GS_ERR_CAPACITY;
    const int gx = gs::ceil_div_i(W, GS_TILE);
    const int ntiles = gx * gs::ceil_div_i(H, GS_TILE);
    if (c->ws.list_sgx) {
        // supertile lists: per-tile counts, their scan on the host (test path), ordered fill
        const gs::TileLists l = lists_of(c->ws);
        k_st_tile_count<<<ntiles, 256, 0, st>>>(l, gx, c->ws.tile_cnt);
        std::vector<uint32_t> cnt(ntiles), rg(2 * (size_t)ntiles);
        if (check_cuda(cudaMemcpyAsync(cnt.data(), c->ws.tile_cnt, 4 * (size_t)ntiles, cudaMemcpyDeviceToHost, st)) ||
            check_cuda(cudaStreamSynchronize(st)))
            return GS_ERR_CUDA;
        uint64_t acc = 0;
        for (int t = 0; t < ntiles; t++) {
            rg[2 * t] = cnt[t] ? (uint32_t)acc : 0u;
            rg[2 * t + 1] = cnt[t] ? (uint32_t)(acc + cnt[t]) : 0u;
            acc += cnt[t];
        }
        if (acc != (uint64_t)s.n_keys) {
            fprintf(stderr, "gs_debug_binning: supertile lists hold %llu pairs, K = %lld\n",
                    (unsigned long long)acc, (long long)s.n_keys);
            return GS_ERR_CUDA;
        }
        cudaMemcpyAsync(ranges, rg.data(), 8 * (size_t)ntiles, cudaMemcpyHostToDevice, st);
        k_st_tile_fill<<<ntiles, 32, 0, st>>>(l, gx, reinterpret_cast<const uint2 *>(ranges), c->ws.depth_bits,
                                               c->ws.orig, keys, vals);
    } else {
        if (s.n_keys > 0)
            k_keys_out<<<ntiles, 256, 0, st>>>(c->ws.ranges, c->ws.kv[0], c->ws.depth_bits, c->ws.orig, keys, vals);
        cudaMemcpyAsync(ranges, c->ws.ranges, sizeof(uint2) * ntiles, cudaMemcpyDeviceToDevice, st);
    }
    if (check_cuda(cudaStreamSynchronize(st))) return GS_ERR_CUDA;
    return GS_OK;
}

static int debug_blend_common(gs_ctx *c, void *stream, int N, const float *xy, const float *conic,
                              const float *opacity, const float *rgb, const uint32_t *vals, int64_t K,
                              const uint32_t *ranges, int W, int H, const gs_opts *o, float *out_rgb, float *out_T,
                              float *dump) {
    if (!c || !o || N < 0 || N > c->max_points || W <= 0 || H <= 0 || W > c->max_w || H > c->max_h || K < 0)
        return GS_ERR_INVALID_ARG;
    if (!ranges || (N > 0 && (!xy || !conic || !opacity))) return GS_ERR_INVALID_ARG;
    cudaSetDevice(c->device);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    cudaMemsetAsync(c->ws.counters, 0, sizeof(gs::Counters), st);
    c->last_sticky = c->sticky;
    if (N > 0) {
        k_pack_splats<<<gs::ceil_div_i(N, 256), 256, 0, st>>>(N, xy, conic, opacity, rgb, c->ws.splat);
        c->launches++;
    }
    c->last_counters = c->ws.counters;
    enqueue_blend(c, c->ws, st, c->ws.splat, gs::TileLists{vals, nullptr, reinterpret_cast<const uint2 *>(ranges), 0}, W, H,
                  *o, out_rgb, out_T, dump);
    return finish(c, st, *o, N);
}

int gs_debug_blend(gs_ctx *c, void *stream, int N, const float *xy, const float *conic, const float *opacity,
                   const float *rgb, const uint32_t *vals, int64_t K, const uint32_t *ranges, int W, int H,
                   const gs_opts *o, float *out_rgb, float *out_T) {
    if (!out_rgb || !out_T || (N > 0 && !rgb)) return GS_ERR_INVALID_ARG;
    return debug_blend_common(c, stream, N, xy, conic, opacity, rgb, vals, K, ranges, W, H, o, out_rgb, out_T,
                              nullptr);
}

int gs_debug_set_trace(gs_ctx *c, long long *trace) {
    if (!c) return GS_ERR_INVALID_ARG;
    gs::g_blend_trace = trace;
    return GS_OK;
}

int gs_debug_exponents(gs_ctx *c, void *stream, int N, const float *xy, const float *conic, const float *opacity,
                       const uint32_t *vals, int64_t K, const uint32_t *ranges, int W, int H, float *out_m) {
    if (!out_m) return GS_ERR_INVALID_ARG;
    gs_opts o{};
    o.blend = GS_BLEND_TC;
    o.flags = GS_FLAG_SYNC;
    return debug_blend_common(c, stream, N, xy, conic, opacity, nullptr, vals, K, ranges, W, H, &o, nullptr, nullptr,
                              out_m);
}

}  // extern "C"
