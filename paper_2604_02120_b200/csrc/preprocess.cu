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
__device__ __forceinline__ bool opacity_box(float mx, float my, float a, float c, float op, int gx, int gy, int &xmin,
                                            int &ymin, int &xmax, int &ymax) {
    const float t = 255.0f * op;
    if (!(t >= 1.0f)) return false;
    const float lim = 2.0f * (ln_repro(t) + 5e-3f);
    const float ex = sqrtf(lim * a), ey = sqrtf(lim * c);
    xmin = max(xmin, rect_bound(floorf((mx - ex) * 0.0625f), gx));
    xmax = min(xmax, rect_bound(floorf((mx + ex) * 0.0625f) + 1.0f, gx));
    ymin = max(ymin, rect_bound(floorf((my - ey) * 0.0625f), gy));
    ymax = min(ymax, rect_bound(floorf((my + ey) * 0.0625f) + 1.0f, gy));
    return xmax > xmin && ymax > ymin;
}

#ifndef GS_PRE_MINB
#define GS_PRE_MINB 4   // 64 registers, 4 x 48 KB SH staging per SM (3: 0.138 ms, 4: 0.128 ms per view)
#endif
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
        bool vis = false;
        float mx = 0.f, my = 0.f, cA = 0.f, cB = 0.f, cC = 0.f, sxx = 0.f, sxy = 0.f, syy = 0.f;
        int r = 0, xmin = 0, xmax = 0, ymin = 0, ymax = 0;
        // 1. view-space point
        const float vx = __fmaf_rn(R[2], pz, __fmaf_rn(R[1], py, __fmaf_rn(R[0], px, cam.t[0])));
        const float vy = __fmaf_rn(R[5], pz, __fmaf_rn(R[4], py, __fmaf_rn(R[3], px, cam.t[1])));
        const float vz = __fmaf_rn(R[8], pz, __fmaf_rn(R[7], py, __fmaf_rn(R[6], px, cam.t[2])));
        if (in && vz > cam.znear) {
            if (!have_cov) {   // 2-4, once per Gaussian
                cov3d(q, s0, s1, s2, scale_mod, S);
                have_cov = true;
            }
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
                cA = c * id; cB = -(b * id); cC = a * id;
                sxx = a; sxy = b; syy = c;
                // 8. radius
                const float mid = 0.5f * (a + c);
                const float lam = mid + sqrtf(fmaxf(0.1f, __fmaf_rn(mid, mid, -det)));
                r = (int)ceilf(3.0f * sqrtf(lam));
                // 9. projected mean
                mx = __fmaf_rn(cam.fx, ux, cam.cx);
                my = __fmaf_rn(cam.fy, uy, cam.cy);
                // 10. tile rectangle
                const float rf = (float)r;
                xmin = rect_bound((mx - rf) / 16.0f, gx);
                xmax = rect_bound(((mx + rf) + 15.0f) / 16.0f, gx);
                ymin = rect_bound((my - rf) / 16.0f, gy);
                ymax = rect_bound(((my + rf) + 15.0f) / 16.0f, gy);
                vis = (xmax - xmin) * (ymax - ymin) != 0;
            }
        }
        const bool tight = imode == 1;
        if (imode == 2 && vis) vis = opacity_box(mx, my, sxx, syy, op, gx, gy, xmin, ymin, xmax, ymax);
        if (vis && (pv.band_y0 > 0 || pv.band_y1 < gy)) {   // row band of a split frame: its rows only
            ymin = max(ymin, pv.band_y0);
            ymax = min(ymax, pv.band_y1);
            vis = ymax > ymin;
        }
        uint32_t n_tiles = (uint32_t)((xmax - xmin) * (ymax - ymin));
        unsigned long long tm = ~0ull;
        if (tight && vis)   // the stored rect becomes the opacity-aware box, the mask its kept tiles
            vis = tight_rect(mx, my, cA, cB, sxx, sxy, syy, op, gx, gy, xmin, ymin, xmax, ymax, tm, n_tiles);
        // slot packing: the warp's visible Gaussians (index order) take slots warp*32 + 0, 1, ...;
        // culled ones write nothing (dense writes, no partial-sector fills but one per warp)
        const uint32_t bal = __ballot_sync(0xffffffffu, vis);
        if (lane == 0) out.wcount[i >> 5] = __popc(bal);
        if (!vis) continue;
        const int slot = (i & ~31) + __popc(bal & ((1u << lane) - 1u));
        if (tight) out.tmask[slot] = tm;
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
        // 12. outputs (slot-addressed)
        if (out.orig) out.orig[slot] = (uint32_t)i;   // debug outputs only
        out.depth_bits[slot] = __float_as_uint(vz);
        {   // the blend's 48-B record: three 16-B stores
            float4 *d = reinterpret_cast<float4 *>(out.splat + slot);
            d[0] = make_float4(mx, my, 0.f, 0.f);
            d[1] = make_float4(cA, cB, cC, op);
            d[2] = make_float4(col[0], col[1], col[2], 0.f);
        }
        out.rect[slot] = make_ushort4((unsigned short)xmin, (unsigned short)ymin, (unsigned short)xmax,
                                      (unsigned short)ymax);
        out.touched[slot] = n_tiles;
        if (out.radius) out.radius[slot] = r;
    }
}

PreOut pre_out_of(const Workspace &ws, bool with_radius) {
    return PreOut{ws.wcount, with_radius ? ws.orig : nullptr, ws.depth_bits, ws.splat, ws.rect, ws.touched, ws.tmask,
                  with_radius ? ws.radius : nullptr, ws.counters};
}

void launch_preprocess_views(const PreViews &pv, cudaStream_t st, int N, const float *means, const float *scales,
                             const float *rots, const float *opacity, const float *shs, int sh_degree,
                             int sh_stride, float scale_mod, int W, int H, int imode) {
    if (N <= 0) return;
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
