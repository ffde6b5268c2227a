// preprocess.cu -- stage (a) "Preprocessing": per
// Gaussian projection to a 2D ellipse (EWA), tile rectangle, depth and SH colour.
//
// The operation order is written once in docs/preprocess_order.md; this file
// implements it independently of the oracle. Every expression is one IEEE
// binary32 operation in the documented order: this translation unit is built
// with -fmad=false (no FMA contraction), -prec-div=true -prec-sqrt=true and
// no FTZ, so depth / mean / conic / radius / rect / tiles_touched / rgb are
// bit-identical to the oracle.
//
// HBM-bound: reads 12 B (culled) .. 248 B (SH3, visible) per Gaussian and
// writes 64 B. One thread per Gaussian, SoA outputs, float4 SH loads.
#include "gs_common.cuh"

namespace gs {

__device__ __forceinline__ int rect_bound(float v, int g) {
    float c = fminf((float)g, fmaxf(0.0f, v));   // step 10: trunc(min(g, max(0, v)))
    return (int)c;
}

#ifndef GS_PRE_THREADS
#define GS_PRE_THREADS 256
#endif
constexpr int PRE_THREADS = GS_PRE_THREADS;

// Tile-exact intersection (GS_FLAG_TIGHT). A pixel p can keep the Gaussian only if
// ln(o) - q/2 >= ln(1/255) - margin (Eq. 3 power, q = d^T Q d, d = p - mu up to sign),
// i.e. p - mu lies in the ellipse E = {d : d^T Q d <= lim}, lim = 2 (ln(255 o) + margin),
// margin 5e-3 in ln(alpha) (25x the documented exponent error delta_a). With
// Sigma = Q^-1 = (a, b; b, c) the dilated 2-D covariance:
//   - E's bounding box is |dx| <= sqrt(lim a), |dy| <= sqrt(lim c): the rect shrinks to it;
//   - E cut by a band of pixel rows v in [v0, v1] spans dx in [L, R] with
//     R = max_v (-B v + sqrt(A lim - det_Q v^2)) / A, a concave function whose
//     maximiser is v* = b sqrt(lim / a); L is its mirror image (v -> -v).
// Each row of tiles therefore keeps a contiguous run of columns; for boxes of <= 64
// tiles bit (ty-y0)*w + (tx-x0) of the mask marks the kept tiles. The column test
// uses the half-open [16 tx, 16 tx + 16) so it is a superset of the exact pixel set.
// Not part of the bit-exact set: explicit FMAs / approximate reciprocals are fine.
__device__ __forceinline__ bool tight_rect(float mx, float my, float A, float B, float a, float b, float c, float op,
                                           int gx, int gy, int &xmin, int &ymin, int &xmax, int &ymax,
                                           unsigned long long &mask, uint32_t &count) {
    const float lim = 2.0f * (__logf(255.0f * op) + 5e-3f);
    if (!(lim > 0.f)) return false;
    const float ex = __fsqrt_rn(lim * a), ey = __fsqrt_rn(lim * c);
    xmin = max(xmin, (int)fminf((float)gx, fmaxf(0.0f, floorf((mx - ex) * 0.0625f))));
    xmax = min(xmax, (int)fminf((float)gx, fmaxf(0.0f, floorf((mx + ex) * 0.0625f) + 1.0f)));
    ymin = max(ymin, (int)fminf((float)gy, fmaxf(0.0f, floorf((my - ey) * 0.0625f))));
    ymax = min(ymax, (int)fminf((float)gy, fmaxf(0.0f, floorf((my + ey) * 0.0625f) + 1.0f)));
    const int w = xmax - xmin, h = ymax - ymin;
    if (w <= 0 || h <= 0) return false;
    if (w == 1 || h == 1 || w * h > 64) {   // a 1-wide box is covered by convexity; > 64 keeps all
        mask = w * h >= 64 ? ~0ull : (1ull << (w * h)) - 1ull;
        count = (uint32_t)(w * h);
        return true;
    }
    const float iA = __frcp_rn(A), detQ = __frcp_rn(a * c - b * b);
    const float vstar = b * __fsqrt_rn(lim * __frcp_rn(a));
    unsigned long long m = 0ull;
    uint32_t n = 0;
    for (int r = 0; r < h; r++) {
        const float by0 = (float)(GS_TILE * (ymin + r));
        const float v0 = fmaxf(by0 - my, -ey), v1 = fminf(by0 + 15.0f - my, ey);
        if (v0 > v1) continue;
        const float vr = fminf(fmaxf(vstar, v0), v1), vl = fminf(fmaxf(-vstar, v0), v1);
        const float R = (-B * vr + __fsqrt_rn(fmaxf(A * lim - detQ * vr * vr, 0.f))) * iA;
        const float L = (-B * vl - __fsqrt_rn(fmaxf(A * lim - detQ * vl * vl, 0.f))) * iA;
        const int c0 = max(xmin, (int)floorf((mx + L) * 0.0625f)) - xmin;
        const int c1 = min(xmax - 1, (int)floorf((mx + R) * 0.0625f)) - xmin;
        if (c0 > c1) continue;
        m |= (((1ull << (c1 - c0 + 1)) - 1ull) << c0) << (r * w);
        n += (uint32_t)(c1 - c0 + 1);
    }
    mask = m;
    count = n;
    return n != 0;
}

// Steps 2-4 (view-independent): quaternion normalisation, rotation matrix, 3D covariance.
__device__ __forceinline__ void cov3d(const float4 &q, float s0, float s1, float s2, float scale_mod, float (&S)[3][3]) {
    // 2. quaternion normalisation
    const float n2 = __fmaf_rn(q.w, q.w, __fmaf_rn(q.z, q.z, __fmaf_rn(q.y, q.y, q.x * q.x)));
    const float nr = sqrtf(n2);
    const float inr = 1.0f / nr;
    const float w = q.x * inr, x = q.y * inr, y = q.z * inr, z = q.w * inr;
    // 3. rotation matrix
    const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, xz = x * z, yz = y * z;
    const float wx = w * x, wy = w * y, wz = w * z;
    float M[3][3];
    M[0][0] = 1.0f - 2.0f * (yy + zz); M[0][1] = 2.0f * (xy - wz); M[0][2] = 2.0f * (xz + wy);
    M[1][0] = 2.0f * (xy + wz); M[1][1] = 1.0f - 2.0f * (xx + zz); M[1][2] = 2.0f * (yz - wx);
    M[2][0] = 2.0f * (xz - wy); M[2][1] = 2.0f * (yz + wx); M[2][2] = 1.0f - 2.0f * (xx + yy);
    // 4. 3D covariance
    float v[3];
    const float sc[3] = {s0, s1, s2};
#pragma unroll
    for (int k = 0; k < 3; k++) {
        const float g = scale_mod * sc[k];
        v[k] = g * g;
    }
    float u[3][3];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
        for (int k = 0; k < 3; k++) u[a][k] = M[a][k] * v[k];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
        for (int b = a; b < 3; b++) {
            S[a][b] = __fmaf_rn(u[a][2], M[b][2], __fmaf_rn(u[a][1], M[b][1], u[a][0] * M[b][0]));
            S[b][a] = S[a][b];
        }
}

// Step 11: SH colour for the view direction normalize(p - campos).
template <class KF>
__device__ __forceinline__ void sh_colour(KF k, int sh_degree, float px, float py, float pz,
                                          const gs_camera &cam, float (&res3)[3]) {
    const float dx = px - cam.campos[0], dy = py - cam.campos[1], dz = pz - cam.campos[2];
    const float len = sqrtf(__fmaf_rn(dz, dz, __fmaf_rn(dy, dy, dx * dx)));
    const float il = 1.0f / len;
    const float X = dx * il, Y = dy * il, Z = dz * il;
    const float C0 = 0.28209479177387814f, C1 = 0.4886025119029199f;
    const float C20 = 1.0925484305920792f, C21 = -1.0925484305920792f, C22 = 0.31539156525252005f,
                C23 = -1.0925484305920792f, C24 = 0.5462742152960396f;
    const float C30 = -0.5900435899266435f, C31 = 2.890611442640554f, C32 = -0.4570457994644658f,
                C33 = 0.3731763325901154f, C34 = -0.4570457994644658f, C35 = 1.445305721320277f,
                C36 = -0.5900435899266435f;
#pragma unroll
    for (int ch = 0; ch < 3; ch++) {
#define SHK(j) k((j) * 3 + ch)
        float res = C0 * SHK(0);
        if (sh_degree >= 1) {
            res = __fmaf_rn(-(C1 * Y), SHK(1), res);
            res = __fmaf_rn(C1 * Z, SHK(2), res);
            res = __fmaf_rn(-(C1 * X), SHK(3), res);
        }
        if (sh_degree >= 2) {
            const float XX = X * X, YY = Y * Y, ZZ = Z * Z, XY = X * Y, YZ = Y * Z, XZ = X * Z;
            res = __fmaf_rn((C20 * XY), SHK(4), res);
            res = __fmaf_rn((C21 * YZ), SHK(5), res);
            res = __fmaf_rn((C22 * (((2.0f * ZZ) - XX) - YY)), SHK(6), res);
            res = __fmaf_rn((C23 * XZ), SHK(7), res);
            res = __fmaf_rn((C24 * (XX - YY)), SHK(8), res);
            if (sh_degree >= 3) {
                res = __fmaf_rn(((C30 * Y) * ((3.0f * XX) - YY)), SHK(9), res);
                res = __fmaf_rn(((C31 * XY) * Z), SHK(10), res);
                res = __fmaf_rn(((C32 * Y) * (((4.0f * ZZ) - XX) - YY)), SHK(11), res);
                res = __fmaf_rn(((C33 * Z) * (((2.0f * ZZ) - (3.0f * XX)) - (3.0f * YY))), SHK(12), res);
                res = __fmaf_rn(((C34 * X) * (((4.0f * ZZ) - XX) - YY)), SHK(13), res);
                res = __fmaf_rn(((C35 * Z) * (XX - YY)), SHK(14), res);
                res = __fmaf_rn(((C36 * X) * (XX - (3.0f * YY))), SHK(15), res);
            }
        }
#undef SHK
        res3[ch] = fmaxf(res + 0.5f, 0.0f);
    }
}

// One thread per Gaussian, pv.n views (1..MAX_VIEW_GROUP) of the same scene: the scene
// record (means, scales, rotation, opacity and the SH coefficients, up to 236 B) is read
// from HBM once and projected for every view of the group, so an orbit's dominant
// preprocess traffic is paid once per group instead of once per view. Per view the
// operation order is the one of docs/preprocess_order.md (outputs bit-identical to a
// single-view launch: the view-independent steps 2-4 are the same operations).
// ln(t) for t >= 1 by a fixed sequence of IEEE +, -, *, / (bit-reproducible by the
// oracle, unlike logf): t = 2^e m, m in [1, 2), ln t = e ln 2 + 2 atanh(s), s = (m-1)/(m+1)
// in [0, 1/3), series to s^9 (truncation < 2e-6). docs/preprocess_order.md step 10b.
__device__ __forceinline__ float ln_repro(float t) {
    const uint32_t bits = __float_as_uint(t);
    const float e = (float)((int)((bits >> 23) & 0xFFu) - 127);
    const float m = __uint_as_float((bits & 0x7FFFFFu) | 0x3F800000u);
    const float sn = (m - 1.0f) / (m + 1.0f);
    const float s2 = sn * sn;
    const float p = (((s2 * 0.11111111f + 0.14285715f) * s2 + 0.2f) * s2 + 0.33333334f) * s2 + 1.0f;
    return e * 0.6931472f + 2.0f * (sn * p);
}

// Opacity-aware box (GS_FLAG_OBOX): a pixel p can have alpha >= 1/255 only
// if d^T Q d <= lim = 2 (ln(255 o) + 5e-3) (Eq. 3 power, margin 5e-3 in ln alpha, 25x the
// documented exponent error delta_a), i.e. inside the ellipse whose bounding box is
// |dx| <= sqrt(lim a), |dy| <= sqrt(lim c) (a, c: the dilated 2-D covariance). The rect
// becomes its intersection with that box (tiles whose pixel centres are all outside are
// dropped): every dropped pair is alpha-skipped by the blend anyway, so frames are
// bit-identical to the vanilla rect's. 255 o < 1.0 culls (alpha < 1/255 everywhere).
// lim depends on the Gaussian only: obox_lim() once per Gaussian, opacity_box() per view
// (the same operations as evaluating both per view; negative = culled, 255 o < 1)
__device__ __forceinline__ float obox_lim(float op) {
    const float t = 255.0f * op;
    if (!(t >= 1.0f)) return -1.0f;
    return 2.0f * (ln_repro(t) + 5e-3f);
}
__device__ __forceinline__ bool opacity_box(float mx, float my, float a, float c, float lim, int gx, int gy, int &xmin,
                                            int &ymin, int &xmax, int &ymax) {
    if (!(lim >= 0.0f)) return false;
    const float ex = sqrtf(lim * a), ey = sqrtf(lim * c);
    xmin = max(xmin, rect_bound(floorf((mx - ex) * 0.0625f), gx));
    xmax = min(xmax, rect_bound(floorf((mx + ex) * 0.0625f) + 1.0f, gx));
    ymin = max(ymin, rect_bound(floorf((my - ey) * 0.0625f), gy));
    ymax = min(ymax, rect_bound(floorf((my + ey) * 0.0625f) + 1.0f, gy));
    return xmax > xmin && ymax > ymin;
}

// Steps 5-10 (+ 10b, the row band and the tile-exact mask) of one (Gaussian, view) pair whose
// view-space point (step 1) passed vz > znear; S: the Gaussian's 3D covariance (steps 2-4).
struct ViewProj {
    float mx, my, cA, cB, cC;
    int r, xmin, ymin, xmax, ymax;
    uint32_t n_tiles;
    unsigned long long tm;
    bool vis;
};
__device__ __forceinline__ void project_view(const gs_camera &cam, float vx, float vy, float vz, const float (&S)[3][3],
                                             float op, float lim, int gx, int gy, int imode, int band_y0,
                                             int band_y1, ViewProj &o) {
    const float *R = cam.R;
    o.vis = false;
    o.mx = o.my = o.cA = o.cB = o.cC = 0.f;
    o.r = o.xmin = o.xmax = o.ymin = o.ymax = 0;
    float sxx = 0.f, sxy = 0.f, syy = 0.f;
    {
        // 5. clamped Jacobian
        const float lx = 1.3f * cam.tan_fovx, ly = 1.3f * cam.tan_fovy;
        const float iz = 1.0f / vz;
        const float ux = vx * iz, uy = vy * iz;
        const float cxz = fminf(lx, fmaxf(-lx, ux));
        const float cyz = fminf(ly, fmaxf(-ly, uy));
        const float j00 = cam.fx * iz, j02 = -((cam.fx * cxz) * iz);
        const float j11 = cam.fy * iz, j12 = -((cam.fy * cyz) * iz);
        // 6. EWA 2D covariance, T = J R
        float T[2][3], U[2][3];
#pragma unroll
        for (int kk = 0; kk < 3; kk++) {
            T[0][kk] = __fmaf_rn(j02, R[6 + kk], j00 * R[0 + kk]);
            T[1][kk] = __fmaf_rn(j12, R[6 + kk], j11 * R[3 + kk]);
        }
#pragma unroll
        for (int a = 0; a < 2; a++)
#pragma unroll
            for (int kk = 0; kk < 3; kk++)
                U[a][kk] = __fmaf_rn(T[a][2], S[2][kk], __fmaf_rn(T[a][1], S[1][kk], T[a][0] * S[0][kk]));
        const float c00 = __fmaf_rn(U[0][2], T[0][2], __fmaf_rn(U[0][1], T[0][1], U[0][0] * T[0][0]));
        const float c01 = __fmaf_rn(U[0][2], T[1][2], __fmaf_rn(U[0][1], T[1][1], U[0][0] * T[1][0]));
        const float c11 = __fmaf_rn(U[1][2], T[1][2], __fmaf_rn(U[1][1], T[1][1], U[1][0] * T[1][0]));
        const float a = c00 + 0.3f, b = c01, c = c11 + 0.3f;
        // 7. conic
        const float det = __fmaf_rn(a, c, -(b * b));
        if (det > 0.0f) {
            const float id = 1.0f / det;
            o.cA = c * id; o.cB = -(b * id); o.cC = a * id;
            sxx = a; sxy = b; syy = c;
            // 8. radius
            const float mid = 0.5f * (a + c);
            const float lam = mid + sqrtf(fmaxf(0.1f, __fmaf_rn(mid, mid, -det)));
            o.r = (int)ceilf(3.0f * sqrtf(lam));
            // 9. projected mean
            o.mx = __fmaf_rn(cam.fx, ux, cam.cx);
            o.my = __fmaf_rn(cam.fy, uy, cam.cy);
            // 10. tile rectangle
            const float rf = (float)o.r;
            o.xmin = rect_bound((o.mx - rf) / 16.0f, gx);
            o.xmax = rect_bound(((o.mx + rf) + 15.0f) / 16.0f, gx);
            o.ymin = rect_bound((o.my - rf) / 16.0f, gy);
            o.ymax = rect_bound(((o.my + rf) + 15.0f) / 16.0f, gy);
            o.vis = (o.xmax - o.xmin) * (o.ymax - o.ymin) != 0;
        }
    }
    if (imode == 2 && o.vis) o.vis = opacity_box(o.mx, o.my, sxx, syy, lim, gx, gy, o.xmin, o.ymin, o.xmax, o.ymax);
    if (o.vis && (band_y0 > 0 || band_y1 < gy)) {   // row band of a split frame: its rows only
        o.ymin = max(o.ymin, band_y0);
        o.ymax = min(o.ymax, band_y1);
        o.vis = o.ymax > o.ymin;
    }
    o.n_tiles = (uint32_t)((o.xmax - o.xmin) * (o.ymax - o.ymin));
    o.tm = ~0ull;
    if (imode == 1 && o.vis)   // the stored rect becomes the opacity-aware box, the mask its kept tiles
        o.vis = tight_rect(o.mx, o.my, o.cA, o.cB, sxx, sxy, syy, op, gx, gy, o.xmin, o.ymin, o.xmax, o.ymax, o.tm,
                           o.n_tiles);
}

// 12. outputs of a visible pair at its slot
__device__ __forceinline__ void store_view(const PreOut &out, int slot, uint32_t i, float vz, const ViewProj &o,
                                           float op, const float (&col)[3], bool tight) {
    if (tight) out.tmask[slot] = o.tm;
    if (out.orig) out.orig[slot] = i;   // debug outputs only
    out.depth_bits[slot] = __float_as_uint(vz);
    {   // the blend's 48-B record: three 16-B stores
        float4 *d = reinterpret_cast<float4 *>(out.splat + slot);
        d[0] = make_float4(o.mx, o.my, 0.f, 0.f);
        d[1] = make_float4(o.cA, o.cB, o.cC, op);
        d[2] = make_float4(col[0], col[1], col[2], 0.f);
    }
    out.rect[slot] = make_ushort4((unsigned short)o.xmin, (unsigned short)o.ymin, (unsigned short)o.xmax,
                                  (unsigned short)o.ymax);
    out.touched[slot] = o.n_tiles;
    if (out.radius) out.radius[slot] = o.r;
}

#ifndef GS_PRE_MINB
#define GS_PRE_MINB 4   // 64 registers, 4 x 48 KB SH staging per SM (3: 0.138 ms, 4: 0.128 ms per view)
#endif
// Single-view launches (and view groups with GS_PRE_CV=0): one thread per Gaussian, the
// group's views in a loop.
__global__ void __launch_bounds__(PRE_THREADS, GS_PRE_MINB) k_preprocess(int N, const float *__restrict__ means,
                                                               const float *__restrict__ scales,
                                                               const float4 *__restrict__ rots,
                                                               const float *__restrict__ opacity,
                                                               const float *__restrict__ shs, int sh_degree,
                                                               int sh_stride, float scale_mod, int W, int H,
                                                               const PreViews pv, int imode) {
    pdl_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0)   // the frames' device counters (no memset node: keeps PDL chained)
        for (int v = 0; v < pv.n; v++) *pv.out[v].counters = Counters{};
    if ((i & ~31) >= N) return;   // whole warps only: the slot packing below votes per warp
    const bool in = i < N;
    const uint32_t lane = threadIdx.x & 31u;
    const int gx = (W + GS_TILE - 1) / GS_TILE, gy = (H + GS_TILE - 1) / GS_TILE;

    const int ii = in ? i : N - 1;   // tail lanes read a valid record and are culled below
    const float px = __ldcs(means + 3 * ii), py = __ldcs(means + 3 * ii + 1), pz = __ldcs(means + 3 * ii + 2);
    const float4 q = __ldcs(rots + ii);
    const float s0 = __ldcs(scales + 3 * ii), s1 = __ldcs(scales + 3 * ii + 1), s2 = __ldcs(scales + 3 * ii + 2);
    const float op = __ldcs(opacity + ii);
    float S[3][3];
    float lim = 0.f;
    bool have_cov = false, have_sh = false;
    // the SH record, once loaded, lives in shared memory (coefficient-major: conflict-free)
    // rather than in 48 registers, so the kernel keeps 3 blocks per SM
    __shared__ float s_sh[48][PRE_THREADS];
    auto K = [&](int j) { return s_sh[j][threadIdx.x]; };

#pragma unroll 1
    for (int view = 0; view < pv.n; view++) {
        const gs_camera &cam = pv.cam[view];
        const PreOut &out = pv.out[view];
        const float *R = cam.R;
        // 1. view-space point
        const float vx = __fmaf_rn(R[2], pz, __fmaf_rn(R[1], py, __fmaf_rn(R[0], px, cam.t[0])));
        const float vy = __fmaf_rn(R[5], pz, __fmaf_rn(R[4], py, __fmaf_rn(R[3], px, cam.t[1])));
        const float vz = __fmaf_rn(R[8], pz, __fmaf_rn(R[7], py, __fmaf_rn(R[6], px, cam.t[2])));
        ViewProj o;
        o.vis = false;
        if (in && vz > cam.znear) {
            if (!have_cov) {   // 2-4 (and 10b's lim), once per Gaussian
                cov3d(q, s0, s1, s2, scale_mod, S);
                if (imode == 2) lim = obox_lim(op);
                have_cov = true;
            }
            project_view(cam, vx, vy, vz, S, op, lim, gx, gy, imode, pv.band_y0, pv.band_y1, o);
        }
        // slot packing: the warp's visible Gaussians (index order) take slots warp*32 + 0, 1, ...;
        // culled ones write nothing (dense writes, no partial-sector fills but one per warp)
        const uint32_t bal = __ballot_sync(0xffffffffu, o.vis);
        if (lane == 0) out.wcount[i >> 5] = __popc(bal);
        if (!o.vis) continue;
        const int slot = (i & ~31) + __popc(bal & ((1u << lane) - 1u));
        // 11. colour
        float col[3];
        if (sh_degree < 0) {
            col[0] = shs[3 * (size_t)i]; col[1] = shs[3 * (size_t)i + 1]; col[2] = shs[3 * (size_t)i + 2];
        } else {
            if (!have_sh) {   // the SH record is read once per Gaussian, by its first visible view
                const int ncoef = (sh_degree + 1) * (sh_degree + 1);
                const float *sh = shs + (size_t)i * (size_t)sh_stride * 3;
                if ((sh_stride & 3) == 0 && ((reinterpret_cast<uintptr_t>(shs) & 15) == 0)) {
                    const float4 *sh4 = reinterpret_cast<const float4 *>(sh);
#pragma unroll
                    for (int j = 0; j < 12; j++) {
                        if (4 * j < ncoef * 3) {
                            const float4 t4 = __ldcs(sh4 + j);
                            s_sh[4 * j][threadIdx.x] = t4.x; s_sh[4 * j + 1][threadIdx.x] = t4.y;
                            s_sh[4 * j + 2][threadIdx.x] = t4.z; s_sh[4 * j + 3][threadIdx.x] = t4.w;
                        }
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 48; j++)
                        if (j < ncoef * 3) s_sh[j][threadIdx.x] = __ldg(sh + j);
                }
                have_sh = true;
            }
            sh_colour(K, sh_degree, px, py, pz, cam, col);
        }
        store_view(out, slot, (uint32_t)i, vz, o, op, col, imode == 1);
    }
}

// ---------------------------------------------------------------------------
// View groups (pv.n >= 2): (Gaussian, view) pairs compacted per warp.
// Thread-per-Gaussian leaves the lanes of culled pairs idle through the whole
// projection (about half of an orbit's pairs are culled), so each warp first
// tests its 32 x n pairs with a cheap conservative bound, lists the candidates
// in (view, Gaussian) order, and then projects them 32 at a time, every lane
// busy. A candidate's Gaussian is another lane's: its mean, opacity and 3D
// covariance (steps 2-4, computed once by its own lane) and its SH record sit in
// shared memory, the group's cameras and output descriptors too. The per-pair
// arithmetic is project_view / sh_colour / store_view above, the same operations
// as k_preprocess, so the outputs are bit-identical; the per-view slot of a
// visible pair is its rank among the warp's visible Gaussians of that view, as in
// k_preprocess (candidates of one view are consecutive and in index order, so
// the rank is a running count plus a ballot over the round's segment of that view).
// ---------------------------------------------------------------------------
#ifndef GS_PRE_CV
#define GS_PRE_CV 0   // 1: view groups use the compacted kernel. Measured slower (profiles/r2_sweep_n.txt,
                      // r2_ncu_pre16_cv.txt): 0.1345 vs 0.1228 ms per view at group 16. It issues 19 % fewer
                      // instructions (9.2 rounds of 32 pairs per warp instead of 16 views) but the conservative
                      // bound costs 80 instructions per (warp, view), every round reloads the camera and the
                      // pair's Gaussian from shared memory, and 72 KB of shared memory per block leave 24 warps
                      // per SM (issue 61 % vs 82 %).
#endif
#ifndef GS_PRE_CV_MINB
#define GS_PRE_CV_MINB 3
#endif
constexpr int CV_THREADS = 256, CV_WARPS = CV_THREADS / 32;
struct __align__(16) CvGauss {
    float4 p_op;    // mean, opacity
    float4 s_a;     // S00, S01, S02, S11
    float4 s_b;     // S12, S22, -, -
};
struct CvSmem {
    float sh[48][CV_THREADS];                         // SH records, coefficient-major
    CvGauss g[CV_THREADS];
    uint16_t pairs[CV_WARPS][MAX_VIEW_GROUP * 32];    // candidates: view << 5 | lane, (view, lane) order
    uint32_t cnt[CV_WARPS][MAX_VIEW_GROUP];           // visible pairs of each view so far (per warp)
    gs_camera cam[MAX_VIEW_GROUP];
    PreOut out[MAX_VIEW_GROUP];
};

// Conservative candidate test of a pair with vz > znear (steps 5-10 cannot keep a pair it
// rejects): the rect of step 10 is empty unless mx + r >= 1, mx - r < 16 gx (same for y),
// with r <= 3 sqrt(lam) + 1 and lam <= |J|_F^2 smax^2 + 0.3 + sqrt(0.1) (the dilated
// covariance's largest eigenvalue plus step 8's max(0.1, .) slack; smax = the largest
// scaled axis, |J|_F the clamped Jacobian's Frobenius norm). Margins cover the rounding of
// this approximate evaluation. NaN inputs fail it, as they fail the exact path.
__device__ __forceinline__ bool cv_candidate(const gs_camera &cam, float px, float py, float pz, float vz,
                                             float smax, int gx, int gy) {
    const float *R = cam.R;
    const float vx = fmaf(R[2], pz, fmaf(R[1], py, fmaf(R[0], px, cam.t[0])));
    const float vy = fmaf(R[5], pz, fmaf(R[4], py, fmaf(R[3], px, cam.t[1])));
    const float iz = __frcp_rn(vz);
    const float ux = vx * iz, uy = vy * iz;
    const float lx = 1.3f * cam.tan_fovx, ly = 1.3f * cam.tan_fovy;
    const float cxz = fminf(lx, fmaxf(-lx, ux)), cyz = fminf(ly, fmaxf(-ly, uy));
    const float f2 = fmaxf(cam.fx * cam.fx, cam.fy * cam.fy) * (iz * iz);
    const float lam = fmaf(f2 * (2.0f + fmaf(cxz, cxz, cyz * cyz)), smax * smax, 0.62f);
    const float mx = fmaf(cam.fx, ux, cam.cx), my = fmaf(cam.fy, uy, cam.cy);
    const float rb = fmaf(3.003f, __fsqrt_rn(lam), 3.0f) + 1e-4f * fmaxf(fabsf(mx), fabsf(my));
    return mx + rb > 0.0f && mx - rb < (float)(GS_TILE * gx) && my + rb > 0.0f && my - rb < (float)(GS_TILE * gy);
}

__global__ void __launch_bounds__(CV_THREADS, GS_PRE_CV_MINB)
    k_preprocess_cv(int N, const float *__restrict__ means, const float *__restrict__ scales,
                    const float4 *__restrict__ rots, const float *__restrict__ opacity, const float *__restrict__ shs,
                    int sh_degree, int sh_stride, float scale_mod, int W, int H, const PreViews pv, int imode) {
    extern __shared__ __align__(16) uint8_t cv_raw[];
    CvSmem &sm = *reinterpret_cast<CvSmem *>(cv_raw);
    pdl_wait();
    const int nv = pv.n;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    if (threadIdx.x < (uint32_t)nv) {
        sm.cam[threadIdx.x] = pv.cam[threadIdx.x];
        sm.out[threadIdx.x] = pv.out[threadIdx.x];
    }
    const int i = blockIdx.x * CV_THREADS + threadIdx.x;
    if (i == 0)   // the frames' device counters (no memset node: keeps PDL chained)
        for (int v = 0; v < nv; v++) *pv.out[v].counters = Counters{};
    __syncthreads();
    if ((i & ~31) >= N) return;   // whole warps only
    const bool in = i < N;
    const int gx = (W + GS_TILE - 1) / GS_TILE, gy = (H + GS_TILE - 1) / GS_TILE;

    // ---- own Gaussian: candidate views, then (if any) covariance and SH into shared memory
    const int ii = in ? i : N - 1;
    const float px = __ldcs(means + 3 * ii), py = __ldcs(means + 3 * ii + 1), pz = __ldcs(means + 3 * ii + 2);
    const float s0 = __ldcs(scales + 3 * ii), s1 = __ldcs(scales + 3 * ii + 1), s2 = __ldcs(scales + 3 * ii + 2);
    const float smax = scale_mod * fmaxf(s0, fmaxf(s1, s2));
    uint32_t cbits = 0;
    if (in) {
#pragma unroll 1
        for (int v = 0; v < nv; v++) {
            const gs_camera &cam = sm.cam[v];
            const float *R = cam.R;
            // step 1's vz exactly (the exact path's cull decision)
            const float vz = __fmaf_rn(R[8], pz, __fmaf_rn(R[7], py, __fmaf_rn(R[6], px, cam.t[2])));
            if (vz > cam.znear && cv_candidate(cam, px, py, pz, vz, smax, gx, gy)) cbits |= 1u << v;
        }
    }
    if (cbits) {
        const float4 q = __ldcs(rots + ii);
        const float op = __ldcs(opacity + ii);
        float S[3][3];
        cov3d(q, s0, s1, s2, scale_mod, S);
        CvGauss &g = sm.g[threadIdx.x];
        g.p_op = make_float4(px, py, pz, op);
        g.s_a = make_float4(S[0][0], S[0][1], S[0][2], S[1][1]);
        g.s_b = make_float4(S[1][2], S[2][2], 0.f, 0.f);
        if (sh_degree >= 0) {
            const int ncoef = (sh_degree + 1) * (sh_degree + 1);
            const float *sh = shs + (size_t)i * (size_t)sh_stride * 3;
            if ((sh_stride & 3) == 0 && ((reinterpret_cast<uintptr_t>(shs) & 15) == 0)) {
                const float4 *sh4 = reinterpret_cast<const float4 *>(sh);
#pragma unroll
                for (int j = 0; j < 12; j++) {
                    if (4 * j < ncoef * 3) {
                        const float4 t4 = __ldcs(sh4 + j);
                        sm.sh[4 * j][threadIdx.x] = t4.x; sm.sh[4 * j + 1][threadIdx.x] = t4.y;
                        sm.sh[4 * j + 2][threadIdx.x] = t4.z; sm.sh[4 * j + 3][threadIdx.x] = t4.w;
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < 48; j++)
                    if (j < ncoef * 3) sm.sh[j][threadIdx.x] = __ldg(sh + j);
            }
        }
    }
    // ---- the warp's candidate list, (view, lane) order
    uint32_t P = 0;
    for (int v = 0; v < nv; v++) {
        const bool c = (cbits >> v) & 1u;
        const uint32_t b = __ballot_sync(0xffffffffu, c);
        if (c) sm.pairs[warp][P + __popc(b & lanemask_lt_u32())] = (uint16_t)((v << 5) | lane);
        P += __popc(b);
    }
    if (lane < (uint32_t)nv) sm.cnt[warp][lane] = 0;
    __syncwarp();
    const int wbase = (i & ~31);   // the warp's first Gaussian = its slot base in every view
    // ---- the candidates, 32 per round
    for (uint32_t base = 0; base < P; base += 32) {
        const uint32_t k = base + lane;
        const bool act = k < P;
        const uint32_t e = sm.pairs[warp][act ? k : P - 1];
        const int v = (int)(e >> 5), gl = (int)(e & 31u);
        const int gt = (int)warp * 32 + gl;          // the Gaussian's thread in the block
        const uint32_t gi = (uint32_t)(wbase + gl);   // its index
        const gs_camera &cam = sm.cam[v];
        const float4 p_op = sm.g[gt].p_op, sa = sm.g[gt].s_a, sb = sm.g[gt].s_b;
        const float S[3][3] = {{sa.x, sa.y, sa.z}, {sa.y, sa.w, sb.x}, {sa.z, sb.x, sb.y}};
        const float *R = cam.R;
        // 1. view-space point (again: the pair's own arithmetic, as in k_preprocess)
        const float gpx = p_op.x, gpy = p_op.y, gpz = p_op.z;
        const float vx = __fmaf_rn(R[2], gpz, __fmaf_rn(R[1], gpy, __fmaf_rn(R[0], gpx, cam.t[0])));
        const float vy = __fmaf_rn(R[5], gpz, __fmaf_rn(R[4], gpy, __fmaf_rn(R[3], gpx, cam.t[1])));
        const float vz = __fmaf_rn(R[8], gpz, __fmaf_rn(R[7], gpy, __fmaf_rn(R[6], gpx, cam.t[2])));
        ViewProj o;
        o.vis = false;
        if (act) project_view(cam, vx, vy, vz, S, p_op.w, imode == 2 ? obox_lim(p_op.w) : 0.f, gx, gy, imode,
                              pv.band_y0, pv.band_y1, o);
        // slot: running count of the view + rank in this round's segment of the view
        const uint32_t vb = __ballot_sync(0xffffffffu, o.vis);
        const int vprev = __shfl_up_sync(0xffffffffu, v, 1);
        const uint32_t starts = __ballot_sync(0xffffffffu, lane == 0 || v != vprev);
        const uint32_t le = lanemask_lt_u32() | (1u << lane);
        const uint32_t seg0 = 31u - __clz(starts & le);                  // first lane of my segment
        const uint32_t nxt = starts & ~((2u << lane) - 1u);                // starts after me
        const uint32_t seg_end = nxt ? (uint32_t)__ffs(nxt) - 1u : 32u;    // one past my segment
        const uint32_t segmask = (seg_end >= 32u ? 0xffffffffu : ((1u << seg_end) - 1u)) & ~((1u << seg0) - 1u);
        const uint32_t c0 = sm.cnt[warp][v];
        __syncwarp();
        if (lane + 1u == seg_end || lane == 31u) sm.cnt[warp][v] = c0 + __popc(vb & segmask);
        if (o.vis) {
            const int slot = wbase + (int)(c0 + __popc(vb & segmask & lanemask_lt_u32()));
            float col[3];
            if (sh_degree < 0) {
                col[0] = shs[3 * (size_t)gi]; col[1] = shs[3 * (size_t)gi + 1]; col[2] = shs[3 * (size_t)gi + 2];
            } else {
                auto K = [&](int j) { return sm.sh[j][gt]; };
                sh_colour(K, sh_degree, gpx, gpy, gpz, cam, col);
            }
            store_view(sm.out[v], slot, gi, vz, o, p_op.w, col, imode == 1);
        }
        __syncwarp();
    }
    if (lane < (uint32_t)nv) sm.out[lane].wcount[i >> 5] = sm.cnt[warp][lane];
}

PreOut pre_out_of(const Workspace &ws, bool with_radius) {
    return PreOut{ws.wcount, with_radius ? ws.orig : nullptr, ws.depth_bits, ws.splat, ws.rect, ws.touched, ws.tmask,
                  with_radius ? ws.radius : nullptr, ws.counters};
}

void launch_preprocess_views(const PreViews &pv, cudaStream_t st, int N, const float *means, const float *scales,
                             const float *rots, const float *opacity, const float *shs, int sh_degree,
                             int sh_stride, float scale_mod, int W, int H, int imode) {
    if (N <= 0) return;
    if (GS_PRE_CV && pv.n >= 2) {
        cudaFuncSetAttribute(k_preprocess_cv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(CvSmem));
        launch_pdl(k_preprocess_cv, ceil_div_i(N, CV_THREADS), CV_THREADS, sizeof(CvSmem), st, N, means, scales,
                   reinterpret_cast<const float4 *>(rots), opacity, shs, sh_degree, sh_stride, scale_mod, W, H, pv,
                   imode);
        return;
    }
    launch_pdl(k_preprocess, ceil_div_i(N, PRE_THREADS), PRE_THREADS, 0, st,
        N, means, scales, reinterpret_cast<const float4 *>(rots), opacity, shs, sh_degree, sh_stride, scale_mod, W,
        H, pv, imode);
}

void launch_preprocess(const Workspace &ws, cudaStream_t st, int N, const float *means, const float *scales,
                       const float *rots, const float *opacity, const float *shs, int sh_degree,
                       int sh_stride, float scale_mod, const gs_camera &cam, int W, int H, int imode,
                       bool with_radius, int band_y0, int band_y1) {
    PreViews pv{};
    pv.n = 1;
    pv.band_y0 = band_y0;
    pv.band_y1 = band_y1;
    pv.cam[0] = cam;
    pv.out[0] = pre_out_of(ws, with_radius);
    launch_preprocess_views(pv, st, N, means, scales, rots, opacity, shs, sh_degree, sh_stride, scale_mod, W, H,
                            imode);
}

}  // namespace gs
