/*
 * oracle.c -- plain, slow, obviously-correct CPU reference of the forward
 * 3DGS render path of GEMM-GS (arXiv 2604.02120).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.  The
 * product path (paper_2604_02120_b200/) never imports, links or executes it,
 * and shares no code, header, table or constant generator with it.
 *
 * What it computes (citations: P:n = /root/reference/PAPER.md line n):
 *   orc_preprocess  -- stage (a) "Preprocessing", fp32 in the
 *                      operation order written once in docs/preprocess_order.md
 *                      (vanilla formulas, readings R-14..R-16).
 *   orc_binning     -- stages (b) "Duplication" + (c) "Sorting":
 *                      the plain definition -- per tile, the Gaussians whose
 *                      rectangle contains it, ordered by (depth bits, index)
 *                      (R-12, R-13); key = tile << 32 | depth bits.
 *   orc_blend       -- stage (d) "Blending", Eq. (1), Eq. (2)-(3)
 *                       and Algorithm 1 with the
 *                      readings R-1..R-5, in float64.  GEMM-GS reaches this
 *                      result exactly in real arithmetic (Eq. 6 is an identity,
 *                      P:269-301), so the oracle is the plain definition.
 *                      It also emits the decision-margin mask (R-21), a test
 *                      device: which decisions lie within the documented GPU error.
 *   orc_vg / orc_vp -- Eq. (6) coefficient and monomial vectors,
 *                      float64, used only by the algebra pins.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared -pthread
 * (no implicit FMA contraction -- fmaf() only where docs/preprocess_order.md writes fma --,
 * no FTZ/DAZ: the fp32 preprocess must be bit-reproducible).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define TILE 16

typedef struct {
    float R[9], t[3];
    float fx, fy, cx, cy;
    float znear, tan_fovx, tan_fovy;
    float campos[3];
} orc_camera;

/* ------------------------------------------------------------------------ */
/* Stage (a): preprocessing, one Gaussian at a time, fp32, fixed order.       */
/* ------------------------------------------------------------------------ */

static const float SH_C0 = 0.28209479177387814f;
static const float SH_C1 = 0.4886025119029199f;
static const float SH_C2[5] = {1.0925484305920792f, -1.0925484305920792f, 0.31539156525252005f,
                               -1.0925484305920792f, 0.5462742152960396f};
static const float SH_C3[7] = {-0.5900435899266435f, 2.890611442640554f, -0.4570457994644658f,
                               0.3731763325901154f, -0.4570457994644658f, 1.445305721320277f,
                               -0.5900435899266435f};

static int ceil_div(int a, int b) { return (a + b - 1) / b; }

static int rect_bound(float v, int g) {
    /* step 10: trunc(min(g, max(0, v))) */
    float c = fminf((float)g, fmaxf(0.0f, v));
    return (int)c;
}

/* Step 10b of docs/preprocess_order.md: natural log of t >= 1 by a fixed sequence
 * of binary32 operations. t = 2^e * m with m in [1, 2);
 * ln t = e * ln2 + 2 * atanh(s), s = (m - 1) / (m + 1), atanh(s) = s (1 + s^2/3 +
 * s^4/5 + s^6/7 + s^8/9 + ...), the polynomial evaluated by Horner's rule. */
static float ln_step10b(float t) {
    uint32_t u;
    memcpy(&u, &t, 4);
    const int e = (int)((u >> 23) & 0xFFu) - 127;
    const uint32_t mu = (u & 0x7FFFFFu) | 0x3F800000u;
    float m;
    memcpy(&m, &mu, 4);
    const float s = (m - 1.0f) / (m + 1.0f);
    const float s2 = s * s;
    float h = s2 * 0.11111111f;           /* 1/9 */
    h = (h + 0.14285715f) * s2;           /* 1/7 */
    h = (h + 0.2f) * s2;                  /* 1/5 */
    h = (h + 0.33333334f) * s2;           /* 1/3 */
    h = h + 1.0f;
    return (float)e * 0.6931472f + 2.0f * (s * h);
}

float orc_ln_step10b(float t) { return ln_step10b(t); }   /* exported for the pins */

/* Returns number of visible Gaussians. Outputs are zero for culled ones.
 * obox != 0: step 10b (GS_FLAG_OBOX), the rect clipped to the opacity-aware box. */
int orc_preprocess_mode(int N, const float *means, const float *scales, const float *rots,
                        const float *opacity, const float *shs, int sh_degree, int sh_stride,
                        float scale_modifier, const orc_camera *cam, int W, int H,
                        float *depth, float *xy, float *conic, float *rgb, int32_t *rect,
                        int32_t *radius, uint32_t *touched, int obox) {
    const float *R = cam->R;
    const int gx = ceil_div(W, TILE), gy = ceil_div(H, TILE);
    int visible = 0;
    for (int i = 0; i < N; i++) {
        depth[i] = 0.0f; xy[2 * i] = xy[2 * i + 1] = 0.0f;
        conic[3 * i] = conic[3 * i + 1] = conic[3 * i + 2] = 0.0f;
        rgb[3 * i] = rgb[3 * i + 1] = rgb[3 * i + 2] = 0.0f;
        rect[4 * i] = rect[4 * i + 1] = rect[4 * i + 2] = rect[4 * i + 3] = 0;
        radius[i] = 0; touched[i] = 0;

        const float px = means[3 * i], py = means[3 * i + 1], pz = means[3 * i + 2];
        /* 1. view-space point */
        float vx = fmaf(R[2], pz, fmaf(R[1], py, fmaf(R[0], px, cam->t[0])));
        float vy = fmaf(R[5], pz, fmaf(R[4], py, fmaf(R[3], px, cam->t[1])));
        float vz = fmaf(R[8], pz, fmaf(R[7], py, fmaf(R[6], px, cam->t[2])));
        if (!(vz > cam->znear)) continue;

        /* 2. quaternion normalisation */
        float qw = rots[4 * i], qx = rots[4 * i + 1], qy = rots[4 * i + 2], qz = rots[4 * i + 3];
        float n2 = fmaf(qz, qz, fmaf(qy, qy, fmaf(qx, qx, qw * qw)));
        float nr = sqrtf(n2);
        float inr = 1.0f / nr;
        float w = qw * inr, x = qx * inr, y = qy * inr, z = qz * inr;

        /* 3. rotation matrix */
        float xx = x * x, yy = y * y, zz = z * z, xy_ = x * y, xz = x * z, yz = y * z;
        float wx = w * x, wy = w * y, wz = w * z;
        float M[3][3];
        M[0][0] = 1.0f - 2.0f * (yy + zz); M[0][1] = 2.0f * (xy_ - wz); M[0][2] = 2.0f * (xz + wy);
        M[1][0] = 2.0f * (xy_ + wz); M[1][1] = 1.0f - 2.0f * (xx + zz); M[1][2] = 2.0f * (yz - wx);
        M[2][0] = 2.0f * (xz - wy); M[2][1] = 2.0f * (yz + wx); M[2][2] = 1.0f - 2.0f * (xx + yy);

        /* 4. 3D covariance */
        float v[3];
        for (int k = 0; k < 3; k++) {
            float g = scale_modifier * scales[3 * i + k];
            v[k] = g * g;
        }
        float u[3][3];
        for (int a = 0; a < 3; a++)
            for (int k = 0; k < 3; k++) u[a][k] = M[a][k] * v[k];
        float S[3][3];
        for (int a = 0; a < 3; a++)
            for (int b = a; b < 3; b++) {
                S[a][b] = fmaf(u[a][2], M[b][2], fmaf(u[a][1], M[b][1], u[a][0] * M[b][0]));
                S[b][a] = S[a][b];
            }

        /* 5. clamped Jacobian */
        float lx = 1.3f * cam->tan_fovx, ly = 1.3f * cam->tan_fovy;
        float iz = 1.0f / vz;
        float ux = vx * iz, uy = vy * iz;
        float cxz = fminf(lx, fmaxf(-lx, ux));
        float cyz = fminf(ly, fmaxf(-ly, uy));
        float j00 = cam->fx * iz, j02 = -((cam->fx * cxz) * iz);
        float j11 = cam->fy * iz, j12 = -((cam->fy * cyz) * iz);

        /* 6. EWA 2D covariance, T = J R (2x3) */
        float T[2][3];
        for (int k = 0; k < 3; k++) {
            T[0][k] = fmaf(j02, R[6 + k], j00 * R[0 + k]);
            T[1][k] = fmaf(j12, R[6 + k], j11 * R[3 + k]);
        }
        float U[2][3];
        for (int a = 0; a < 2; a++)
            for (int k = 0; k < 3; k++)
                U[a][k] = fmaf(T[a][2], S[2][k], fmaf(T[a][1], S[1][k], T[a][0] * S[0][k]));
        float c00 = fmaf(U[0][2], T[0][2], fmaf(U[0][1], T[0][1], U[0][0] * T[0][0]));
        float c01 = fmaf(U[0][2], T[1][2], fmaf(U[0][1], T[1][1], U[0][0] * T[1][0]));
        float c11 = fmaf(U[1][2], T[1][2], fmaf(U[1][1], T[1][1], U[1][0] * T[1][0]));
        float a = c00 + 0.3f, b = c01, c = c11 + 0.3f;

        /* 7. conic */
        float det = fmaf(a, c, -(b * b));
        if (!(det > 0.0f)) continue;
        float id = 1.0f / det;
        float cA = c * id, cB = -(b * id), cC = a * id;

        /* 8. radius */
        float mid = 0.5f * (a + c);
        float lam = mid + sqrtf(fmaxf(0.1f, fmaf(mid, mid, -det)));
        float rr = ceilf(3.0f * sqrtf(lam));
        int r = (int)rr;

        /* 9. projected mean */
        float mx = fmaf(cam->fx, ux, cam->cx);
        float my = fmaf(cam->fy, uy, cam->cy);

        /* 10. tile rectangle */
        float rf = (float)r;
        int xmin = rect_bound((mx - rf) / 16.0f, gx);
        int xmax = rect_bound(((mx + rf) + 15.0f) / 16.0f, gx);
        int ymin = rect_bound((my - rf) / 16.0f, gy);
        int ymax = rect_bound(((my + rf) + 15.0f) / 16.0f, gy);
        int area = (xmax - xmin) * (ymax - ymin);
        if (area == 0) continue;

        /* 10b. opacity-aware box (GS_FLAG_OBOX): alpha >= 1/255 needs
         * d^T Sigma^-1 d <= lim = 2 (ln(255 o) + 0.005); that ellipse lies inside
         * |dx| <= sqrt(lim a), |dy| <= sqrt(lim c). Tiles outside are dropped; 255 o < 1 culls. */
        if (obox) {
            const float t = 255.0f * opacity[i];
            if (!(t >= 1.0f)) continue;
            const float lim = 2.0f * (ln_step10b(t) + 0.005f);
            const float ex = sqrtf(lim * a), ey = sqrtf(lim * c);
            const int bx0 = rect_bound(floorf((mx - ex) * 0.0625f), gx);
            const int bx1 = rect_bound(floorf((mx + ex) * 0.0625f) + 1.0f, gx);
            const int by0 = rect_bound(floorf((my - ey) * 0.0625f), gy);
            const int by1 = rect_bound(floorf((my + ey) * 0.0625f) + 1.0f, gy);
            if (bx0 > xmin) xmin = bx0;
            if (bx1 < xmax) xmax = bx1;
            if (by0 > ymin) ymin = by0;
            if (by1 < ymax) ymax = by1;
            if (!(xmax > xmin && ymax > ymin)) continue;
            area = (xmax - xmin) * (ymax - ymin);
        }

        /* 11. colour */
        float col[3];
        if (sh_degree < 0) {
            for (int ch = 0; ch < 3; ch++) col[ch] = shs[3 * (size_t)i + ch];
        } else {
            float dx = px - cam->campos[0], dy = py - cam->campos[1], dz = pz - cam->campos[2];
            float len = sqrtf(fmaf(dz, dz, fmaf(dy, dy, dx * dx)));
            float il = 1.0f / len;
            float X = dx * il, Y = dy * il, Z = dz * il;
            const float *sh = shs + (size_t)i * (size_t)sh_stride * 3;
            for (int ch = 0; ch < 3; ch++) {
#define SH(k) sh[(k) * 3 + ch]
                float res = SH_C0 * SH(0);
                if (sh_degree >= 1) {
                    res = fmaf(-(SH_C1 * Y), SH(1), res);
                    res = fmaf(SH_C1 * Z, SH(2), res);
                    res = fmaf(-(SH_C1 * X), SH(3), res);
                }
                if (sh_degree >= 2) {
                    float XX = X * X, YY = Y * Y, ZZ = Z * Z, XY = X * Y, YZ = Y * Z, XZ = X * Z;
                    res = fmaf((SH_C2[0] * XY), SH(4), res);
                    res = fmaf((SH_C2[1] * YZ), SH(5), res);
                    res = fmaf((SH_C2[2] * (((2.0f * ZZ) - XX) - YY)), SH(6), res);
                    res = fmaf((SH_C2[3] * XZ), SH(7), res);
                    res = fmaf((SH_C2[4] * (XX - YY)), SH(8), res);
                    if (sh_degree >= 3) {
                        res = fmaf(((SH_C3[0] * Y) * ((3.0f * XX) - YY)), SH(9), res);
                        res = fmaf(((SH_C3[1] * XY) * Z), SH(10), res);
                        res = fmaf(((SH_C3[2] * Y) * (((4.0f * ZZ) - XX) - YY)), SH(11), res);
                        res = fmaf(((SH_C3[3] * Z) * (((2.0f * ZZ) - (3.0f * XX)) - (3.0f * YY))), SH(12), res);
                        res = fmaf(((SH_C3[4] * X) * (((4.0f * ZZ) - XX) - YY)), SH(13), res);
                        res = fmaf(((SH_C3[5] * Z) * (XX - YY)), SH(14), res);
                        res = fmaf(((SH_C3[6] * X) * (XX - (3.0f * YY))), SH(15), res);
                    }
                }
#undef SH
                col[ch] = fmaxf(res + 0.5f, 0.0f);
            }
        }

        depth[i] = vz;
        xy[2 * i] = mx; xy[2 * i + 1] = my;
        conic[3 * i] = cA; conic[3 * i + 1] = cB; conic[3 * i + 2] = cC;
        rgb[3 * i] = col[0]; rgb[3 * i + 1] = col[1]; rgb[3 * i + 2] = col[2];
        rect[4 * i] = xmin; rect[4 * i + 1] = ymin; rect[4 * i + 2] = xmax; rect[4 * i + 3] = ymax;
        radius[i] = r;
        touched[i] = (uint32_t)area;
        visible++;
    }
    return visible;
}

int orc_preprocess(int N, const float *means, const float *scales, const float *rots,
                   const float *opacity, const float *shs, int sh_degree, int sh_stride,
                   float scale_modifier, const orc_camera *cam, int W, int H,
                   float *depth, float *xy, float *conic, float *rgb, int32_t *rect,
                   int32_t *radius, uint32_t *touched) {
    return orc_preprocess_mode(N, means, scales, rots, opacity, shs, sh_degree, sh_stride, scale_modifier, cam,
                               W, H, depth, xy, conic, rgb, rect, radius, touched, 0);
}

/* ------------------------------------------------------------------------ */
/* Stages (b)+(c): duplication and sorting, as a plain definition.            */
/* ------------------------------------------------------------------------ */

typedef struct { uint32_t dbits, idx; } entry;

static int cmp_entry(const void *pa, const void *pb) {
    const entry *a = (const entry *)pa, *b = (const entry *)pb;
    if (a->dbits != b->dbits) return a->dbits < b->dbits ? -1 : 1;
    if (a->idx != b->idx) return a->idx < b->idx ? -1 : 1;
    return 0;
}

/* Returns K (number of (Gaussian, tile) pairs). If K > capacity, nothing is
 * written to keys/vals (the caller re-calls with enough room) -- never truncated.
 * ranges: [tiles][2] = [start, end) into the sorted arrays; empty tiles (0,0). */
int64_t orc_binning(int N, const float *depth, const int32_t *rect, const uint32_t *touched,
                    int W, int H, uint64_t *keys, uint32_t *vals, uint32_t *ranges,
                    int64_t capacity) {
    const int gx = ceil_div(W, TILE), gy = ceil_div(H, TILE), ntiles = gx * gy;
    int64_t *count = (int64_t *)calloc((size_t)ntiles, sizeof(int64_t));
    int64_t K = 0;
    for (int i = 0; i < N; i++) {
        if (touched[i] == 0) continue;
        for (int ty = rect[4 * i + 1]; ty < rect[4 * i + 3]; ty++)
            for (int tx = rect[4 * i]; tx < rect[4 * i + 2]; tx++) { count[ty * gx + tx]++; K++; }
    }
    if (K > capacity) { free(count); return K; }
    entry **lists = (entry **)calloc((size_t)ntiles, sizeof(entry *));
    int64_t *fill = (int64_t *)calloc((size_t)ntiles, sizeof(int64_t));
    for (int t = 0; t < ntiles; t++) lists[t] = (entry *)malloc(sizeof(entry) * (size_t)(count[t] + 1));
    for (int i = 0; i < N; i++) {      /* ascending Gaussian index */
        if (touched[i] == 0) continue;
        uint32_t db;
        memcpy(&db, &depth[i], 4);
        for (int ty = rect[4 * i + 1]; ty < rect[4 * i + 3]; ty++)
            for (int tx = rect[4 * i]; tx < rect[4 * i + 2]; tx++) {
                int t = ty * gx + tx;
                lists[t][fill[t]].dbits = db;
                lists[t][fill[t]].idx = (uint32_t)i;
                fill[t]++;
            }
    }
    int64_t pos = 0;
    for (int t = 0; t < ntiles; t++) {
        qsort(lists[t], (size_t)count[t], sizeof(entry), cmp_entry);
        ranges[2 * t] = (uint32_t)(count[t] ? pos : 0);
        for (int64_t j = 0; j < count[t]; j++) {
            keys[pos] = ((uint64_t)(uint32_t)t << 32) | lists[t][j].dbits;
            vals[pos] = lists[t][j].idx;
            pos++;
        }
        ranges[2 * t + 1] = (uint32_t)(count[t] ? pos : 0);
        free(lists[t]);
    }
    free(lists); free(fill); free(count);
    return K;
}

/* ------------------------------------------------------------------------ */
/* Stage (d): blending, float64, per pixel, serial over the sorted list.     */
/* ------------------------------------------------------------------------ */

typedef struct {
    /* inputs */
    const float *xy, *conic, *opacity, *rgb;
    const uint32_t *vals, *ranges;
    int W, H, gx, gy;
    double bg[3];
    double delta0;       /* documented GPU bound on |d ln alpha| (R-21):       */
    double eps_rel;      /*   delta = delta0 + eps_rel * S per pair, S below    */
    double budget;       /* flag a pixel when its summed flip impacts exceed it */
    double cmax;         /* max |colour| over the scene, and bg               */
    /* outputs */
    double *out_rgb, *out_T, *flip_bound;
    uint8_t *flag;
    /* work split */
    int nthreads, tid;
    /* per-thread counters */
    int64_t evaluated, live;
} blend_job;

static void blend_tile(blend_job *J, int t) {
    const double a_min = (double)(1.0f / 255.0f);
    const double ln_amin = log(a_min);
    const double t_min = 1e-4, ln_tmin = log(1e-4);
    const int tx = t % J->gx, ty = t / J->gx;
    /* tile reference pixel of the GEMM form (Eq. 4; reading R-6), for the mask only */
    const double xc = TILE * tx + 7.5, yc = TILE * ty + 7.5;
    const uint32_t start = J->ranges[2 * t], end = J->ranges[2 * t + 1];
    for (int py = ty * TILE; py < ty * TILE + TILE; py++) {
        for (int px = tx * TILE; px < tx * TILE + TILE; px++) {
            if (px >= J->W || py >= J->H) continue;     /* R-19: in-frame pixels only */
            double T = 1.0, C[3] = {0.0, 0.0, 0.0};
            double Serr = 0.0;       /* sum of delta alpha/(1-alpha) over composited steps */
            double bound = 0.0;
            const double xb = xc - (double)px, yb = yc - (double)py;
            for (uint32_t e = start; e < end; e++) {
                const uint32_t i = J->vals[e];
                /* Eq. (2)-(3): x_g = [x_g - x_p, y_g - y_p], power = -1/2 x^T Sigma^-1 x */
                const double dx = (double)J->xy[2 * i] - (double)px;
                const double dy = (double)J->xy[2 * i + 1] - (double)py;
                const double A = J->conic[3 * i], B = J->conic[3 * i + 1], Cc = J->conic[3 * i + 2];
                const double power = -0.5 * (A * dx * dx + Cc * dy * dy) - B * dx * dy;
                const double o = J->opacity[i];
                const double a_raw = o * exp(power);
                const double alpha = a_raw < 0.99 ? a_raw : 0.99;           /* R-4 */
                J->evaluated++;
                /* decision margin (R-21): the GPU sums the Eq. (6) terms v_k p_k about the tile
                 * centre in fp32 / TF32 hi-lo, so its |d ln alpha| scales with their magnitude S */
                const double xh = (double)J->xy[2 * i] - xc, yh = (double)J->xy[2 * i + 1] - yc;
                const double Smag = 0.5 * fabs(A) * xb * xb + 0.5 * fabs(Cc) * yb * yb + fabs(B * xb * yb) +
                                    fabs(A * xh + B * yh) * fabs(xb) + fabs(Cc * yh + B * xh) * fabs(yb) +
                                    0.5 * fabs(A) * xh * xh + 0.5 * fabs(Cc) * yh * yh + fabs(B * xh * yh) +
                                    fabs(log(o));
                const double delta = J->delta0 + J->eps_rel * Smag;
                /* margin mask (i): the alpha-skip decision */
                const double ln_a = log(o) + power;
                if (fabs(ln_a - ln_amin) < 2.0 * delta)
                    bound += T * a_min * (1.0 + 2.0 * J->cmax) * exp(2.0 * delta);
                if (alpha < a_min) continue;                                /* R-1 */
                J->live++;
                const double tT = T * (1.0 - alpha);
                /* margin mask (ii): the early-termination decision */
                const double clamped_both = (a_raw * exp(-2.0 * delta) >= 0.99);
                const double err = Serr + (clamped_both ? 0.0 : delta * alpha / (1.0 - alpha)) +
                                   1e-6 * (double)(e - start + 1);
                if (fabs(log(tT) - ln_tmin) < 2.0 * err) bound += T * (1.0 + 2.0 * J->cmax);
                if (tT < t_min) break;                                      /* R-2 */
                for (int ch = 0; ch < 3; ch++) C[ch] += (double)J->rgb[3 * i + ch] * alpha * T; /* R-3 */
                T = tT;
                if (!clamped_both) Serr += delta * alpha / (1.0 - alpha);
            }
            const int flagged = bound > J->budget;
            const size_t pix = (size_t)py * (size_t)J->W + (size_t)px;
            const size_t plane = (size_t)J->W * (size_t)J->H;
            for (int ch = 0; ch < 3; ch++) J->out_rgb[ch * plane + pix] = C[ch] + T * J->bg[ch];
            J->out_T[pix] = T;
            if (J->flag) J->flag[pix] = (uint8_t)flagged;
            if (J->flip_bound) J->flip_bound[pix] = bound;
        }
    }
}

static void *blend_worker(void *arg) {
    blend_job *J = (blend_job *)arg;
    const int ntiles = J->gx * J->gy;
    for (int t = J->tid; t < ntiles; t += J->nthreads) blend_tile(J, t);
    return NULL;
}

/* out_rgb: [3][H][W] planar, out_T: [H][W]; flag / flip_bound may be NULL.
 * Decision-margin mask (R-21, test device): a decision is ambiguous when it lies within
 * 2 delta of its threshold, delta = delta0 + eps_rel * S the documented bound on the GPU's
 * |d ln alpha| for that pair; flip_bound = the summed first-order impacts of a pixel's
 * ambiguous decisions, flag = flip_bound > budget.
 * stats[0] = evaluated pairs, stats[1] = pairs with alpha >= 1/255. */
void orc_blend(const float *xy, const float *conic, const float *opacity, const float *rgb,
               const uint32_t *vals, const uint32_t *ranges, int W, int H, const float *bg,
               double delta0, double eps_rel, double budget, double cmax, int nthreads,
               double *out_rgb, double *out_T, uint8_t *flag, double *flip_bound,
               int64_t *stats) {
    if (nthreads < 1) nthreads = 1;
    blend_job *jobs = (blend_job *)calloc((size_t)nthreads, sizeof(blend_job));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int k = 0; k < nthreads; k++) {
        blend_job *J = &jobs[k];
        J->xy = xy; J->conic = conic; J->opacity = opacity; J->rgb = rgb;
        J->vals = vals; J->ranges = ranges; J->W = W; J->H = H;
        J->gx = ceil_div(W, TILE); J->gy = ceil_div(H, TILE);
        for (int ch = 0; ch < 3; ch++) J->bg[ch] = bg[ch];
        J->delta0 = delta0; J->eps_rel = eps_rel; J->budget = budget; J->cmax = cmax;
        J->out_rgb = out_rgb; J->out_T = out_T; J->flag = flag; J->flip_bound = flip_bound;
        J->nthreads = nthreads; J->tid = k;
        if (nthreads > 1) pthread_create(&th[k], NULL, blend_worker, J);
    }
    if (nthreads == 1) blend_worker(&jobs[0]);
    else for (int k = 0; k < nthreads; k++) pthread_join(th[k], NULL);
    if (stats) {
        stats[0] = stats[1] = 0;
        for (int k = 0; k < nthreads; k++) { stats[0] += jobs[k].evaluated; stats[1] += jobs[k].live; }
    }
    free(jobs); free(th);
}

/* Single pixel blend over an explicit Gaussian list (in the given order), for
 * the brute-force "unsorted then sorted" pin. Same arithmetic as blend_tile. */
void orc_blend_pixel(int n, const uint32_t *order, const float *xy, const float *conic,
                     const float *opacity, const float *rgb, double px, double py,
                     const float *bg, double *out3, double *outT) {
    double T = 1.0, C[3] = {0, 0, 0};
    for (int e = 0; e < n; e++) {
        const uint32_t i = order[e];
        const double dx = (double)xy[2 * i] - px, dy = (double)xy[2 * i + 1] - py;
        const double A = conic[3 * i], B = conic[3 * i + 1], Cc = conic[3 * i + 2];
        const double power = -0.5 * (A * dx * dx + Cc * dy * dy) - B * dx * dy;
        double alpha = (double)opacity[i] * exp(power);
        if (alpha > 0.99) alpha = 0.99;
        if (alpha < (double)(1.0f / 255.0f)) continue;
        const double tT = T * (1.0 - alpha);
        if (tT < 1e-4) break;
        for (int ch = 0; ch < 3; ch++) C[ch] += (double)rgb[3 * i + ch] * alpha * T;
        T = tT;
    }
    for (int ch = 0; ch < 3; ch++) out3[ch] = C[ch] + T * (double)bg[ch];
    *outT = T;
}

/* ------------------------------------------------------------------------ */
/* Eq. (6): v_g and v_p, float64 (algebra pins only).                        */
/* ------------------------------------------------------------------------ */

/* v_g = [-A/2, -C/2, -B, -A xh - B yh, -C yh - B xh, -A xh^2/2 - C yh^2/2 - B xh yh]
 * with xh = x_g - x_c, yh = y_g - y_c. */
void orc_vg(double A, double B, double C, double xh, double yh, double *v) {
    v[0] = -0.5 * A;
    v[1] = -0.5 * C;
    v[2] = -B;
    v[3] = -A * xh - B * yh;
    v[4] = -C * yh - B * xh;
    v[5] = -0.5 * A * xh * xh - 0.5 * C * yh * yh - B * xh * yh;
}

/* v_p = [xb^2, yb^2, xb yb, xb, yb, 1] with (x_p, y_p) = (x_c - xb, y_c - yb). */
void orc_vp(double xb, double yb, double *v) {
    v[0] = xb * xb; v[1] = yb * yb; v[2] = xb * yb; v[3] = xb; v[4] = yb; v[5] = 1.0;
}
