/*
 * nolf_oracle.c -- CPU restatement of the reference i-NOLF render path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker the CUDA path is compared
 * against (and the CPU baseline bench.py times); it is never linked into the
 * product library.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs load it.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against the
 * golden vectors tests/golden/*.npz produced by running the reference itself
 * (tests/golden/make_golden.py).
 *
 * It follows the reference semantics one ray at a time (the reference runs
 * the same per-ray arithmetic vectorised in numpy, lockstep over rays):
 *
 *   camera_dirs          core.py:162-170
 *   transform_points     core.py:301-304   (numpy dgemm == sequential FMA chain)
 *   aabb_intersect_batch core.py:206-223
 *   march_rays           lightfield.py:129-186  (fixed step, NO empty skipping:
 *                                                every step is evaluated, as in
 *                                                the reference)
 *   query_atlas          atlas.py:158-185
 *   AtlasSource.sample   atlas.py:210-217
 *   _base_weights        encoding.py:346-365
 *   corner_slots         encoding.py:130-140
 *   psh_encode           encoding.py:390-394
 *   HashGridEncoder      encoding.py:438-478
 *   sh_encode_batch      core.py:239-261
 *   mlp_forward          neural.py:89-108, _apply_heads neural.py:74-86
 *   shade_batch          lightfield.py:267-336
 *   render_rays          lightfield.py:400-456
 *   compose              farm.py:129-172
 *
 * Floating point: compiled with -ffp-contract=off so every product and sum
 * rounds separately, as numpy's elementwise ufuncs do; fma() is written out
 * exactly where numpy's OpenBLAS dgemm fuses (measured: 100% of elements).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define MAXL 4
#define MAXW 128

typedef struct {
    int n_layers;              /* weight matrices */
    int widths[MAXL + 1];      /* widths[0] = input */
    const float *w[MAXL];      /* (out, in) row-major */
    const float *b[MAXL];
    int n_heads;
    int head_act[8];           /* 0 identity, 1 sigmoid, 2 exponential */
    int head_w[8];
} OMlp;

typedef struct {
    int b, r, channels;
    const int32_t *index;      /* b^3 */
    const float *cubes;        /* n, r+1, r+1, r+1, channels */
} OAtlas;

typedef struct {
    OAtlas density;
    int has_diffuse_atlas;
    OAtlas diffuse;
    /* PSH (encoding.py:109-140) */
    int psh_n;
    uint64_t psh_m, psh_mphi;
    const int64_t *psh_offsets;
    uint64_t p0[3], p1[3];
    const float *psh_features;
    int psh_f;
    /* live diffuse: hash grid + diffuse MLP (encoding.py:405-478) */
    int hg_levels, hg_f;
    uint64_t hg_table;
    int hg_res[16];
    int hg_dense[16];
    const float *hg_feat[16];
    OMlp fs, fd;
    double step, t_stop, alpha_floor;
    double pmin[3], pmax[3];
    int use_hit_point, use_opacity, refine_opacity, use_tint, use_diffuse_color;
    /* triangle-mesh proxy (no reference counterpart): 9 doubles per triangle */
    int64_t n_tri;
    const double *tri;
} OAsset;

/* optional per-ray debug outputs (NULL to skip) */
typedef struct {
    uint8_t *boxhit, *hit;
    double *t_near, *t_far, *t_hit, *alpha_c, *p_h, *o_obj, *d_obj;
    int64_t *samples, *istar, *slots;
    float *es, *fs_out, *diffuse;
} ODebug;

/* ------------------------------------------------------------------ */
static inline double dmin(double a, double b) { return (isnan(a) || a < b) ? a : (isnan(b) ? b : b); }
/* numpy minimum/maximum propagate NaN */
static inline double np_min(double a, double b) { if (isnan(a) || isnan(b)) return NAN; return a < b ? a : b; }
static inline double np_max(double a, double b) { if (isnan(a) || isnan(b)) return NAN; return a > b ? a : b; }
static inline int64_t clampi(int64_t v, int64_t lo, int64_t hi) { return v < lo ? lo : (v > hi ? hi : v); }
static inline double clampd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* row of (N,3) @ M.T : out[j] = fma(a2, M[j][2], fma(a1, M[j][1], a0*M[j][0])) */
static inline void mat3_apply(const double *M, int ld, const double *a, double *out) {
    for (int j = 0; j < 3; ++j) {
        const double *row = M + j * ld;
        out[j] = fma(a[2], row[2], fma(a[1], row[1], a[0] * row[0]));
    }
}

static inline void normalize3(double *v) {
    double n = sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
    v[0] /= n; v[1] /= n; v[2] /= n;
}

/* core.py:162-170 */
void oracle_camera_dirs(const double *pose /*4x4*/, double fx, double fy, double cx, double cy,
                        const double *px, const double *py, int64_t n, double *out) {
    for (int64_t i = 0; i < n; ++i) {
        double u = ((px[i] + 0.5) - cx) / fx;
        double v = -((py[i] + 0.5) - cy) / fy;
        double d[3] = {u, v, -1.0};
        mat3_apply(pose, 4, d, out + 3 * i);
        normalize3(out + 3 * i);
    }
}

/* atlas.py:158-185 (one point). out[channels] */
static void query_atlas1(const OAtlas *a, const double *x, float *out) {
    int b = a->b, r = a->r, C = a->channels;
    double scaled[3];
    int64_t cell[3];
    for (int k = 0; k < 3; ++k) {
        scaled[k] = x[k] * b;
        cell[k] = clampi((int64_t)floor(scaled[k]), 0, b - 1);
    }
    int32_t cid = a->index[(cell[0] * b + cell[1]) * b + cell[2]];
    if (cid == -1) { for (int c = 0; c < C; ++c) out[c] = 0.f; return; }
    double frac[3];
    int64_t base[3];
    for (int k = 0; k < 3; ++k) {
        double local = (scaled[k] - (double)cell[k]) * r;
        base[k] = clampi((int64_t)floor(local), 0, r - 1);
        frac[k] = local - (double)base[k];
    }
    int s = r + 1;
    const float *cube = a->cubes + (int64_t)cid * s * s * s * C;
    double acc[4] = {0, 0, 0, 0};
    for (int c = 0; c < 8; ++c) {
        int dx = c & 1, dy = (c >> 1) & 1, dz = (c >> 2) & 1;
        double w = ((dx ? frac[0] : 1.0 - frac[0]) * (dy ? frac[1] : 1.0 - frac[1])) *
                   (dz ? frac[2] : 1.0 - frac[2]);
        const float *v = cube + (((base[0] + dx) * s + (base[1] + dy)) * s + (base[2] + dz)) * C;
        for (int ch = 0; ch < C; ++ch) acc[ch] += w * (double)v[ch];
    }
    for (int ch = 0; ch < C; ++ch) out[ch] = (float)acc[ch];
}

/* encoding.py:346-365 */
static void base_weights(const double *x, int res, int64_t *base, double *w) {
    double f[3], g[3];
    for (int k = 0; k < 3; ++k) {
        double scaled = x[k] * res;
        int64_t bb = (int64_t)floor(scaled);
        if (bb > res - 1) bb = res - 1;
        if (bb < 0) bb = 0;
        base[k] = bb;
        f[k] = scaled - (double)bb;
        g[k] = 1.0 - f[k];
    }
    double gygz = g[1] * g[2], fygz = f[1] * g[2], gyfz = g[1] * f[2], fyfz = f[1] * f[2];
    w[0] = g[0] * gygz; w[1] = f[0] * gygz; w[2] = g[0] * fygz; w[3] = f[0] * fygz;
    w[4] = g[0] * gyfz; w[5] = f[0] * gyfz; w[6] = g[0] * fyfz; w[7] = f[0] * fyfz;
}

/* encoding.py:130-140 */
static void psh_corner_slots(const OAsset *A, const int64_t *base, int64_t *slots) {
    uint64_t m = A->psh_m, mp = A->psh_mphi;
    uint64_t p[3] = {(uint64_t)base[0], (uint64_t)base[1], (uint64_t)base[2]};
    uint64_t h0b = (p[0] * A->p0[0] + p[1] * A->p0[1] + p[2] * A->p0[2]) % m;
    uint64_t h1b = (p[0] * A->p1[0] + p[1] * A->p1[1] + p[2] * A->p1[2]) % mp;
    for (int c = 0; c < 8; ++c) {
        uint64_t cx = c & 1, cy = (c >> 1) & 1, cz = (c >> 2) & 1;
        uint64_t ch0 = (cx * A->p0[0] + cy * A->p0[1] + cz * A->p0[2]) % m;
        uint64_t ch1 = (cx * A->p1[0] + cy * A->p1[1] + cz * A->p1[2]) % mp;
        uint64_t h0 = h0b + ch0;
        uint64_t h1 = (h1b + ch1) % mp;
        slots[c] = (int64_t)((h0 + (uint64_t)A->psh_offsets[h1]) % m);
    }
}

/* core.py:239-261 */
static void sh_encode(const double *d, double *o) {
    const double C0 = 0.28209479177387814, C1 = 0.4886025119029199;
    const double C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                          -1.0925484305920792, 0.5462742152960396};
    const double C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                          0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                          -0.5900435899266435};
    double x = d[0], y = d[1], z = d[2];
    double xx = x * x, yy = y * y, zz = z * z;
    o[0] = C0;
    o[1] = -C1 * y;
    o[2] = C1 * z;
    o[3] = -C1 * x;
    o[4] = C2[0] * x * y;
    o[5] = C2[1] * y * z;
    o[6] = C2[2] * (2.0 * zz - xx - yy);
    o[7] = C2[3] * x * z;
    o[8] = C2[4] * (xx - yy);
    o[9] = C3[0] * y * (3.0 * xx - yy);
    o[10] = C3[1] * x * y * z;
    o[11] = C3[2] * y * (4.0 * zz - xx - yy);
    o[12] = C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    o[13] = C3[4] * x * (4.0 * zz - xx - yy);
    o[14] = C3[5] * z * (xx - yy);
    o[15] = C3[6] * x * (xx - 3.0 * yy);
}

static inline float sigmoidf_np(float z) {
    if (z >= 0.f) return 1.0f / (1.0f + expf(-z));
    float ez = expf(z);
    return ez / (1.0f + ez);
}
static inline double sigmoid_np(double z) {
    if (z >= 0.0) return 1.0 / (1.0 + exp(-z));
    double ez = exp(z);
    return ez / (1.0 + ez);
}

/* neural.py:89-108 + _apply_heads neural.py:74-86 ; f32, sequential-FMA dot */
static void mlp_forward1(const OMlp *M, const float *x, float *out) {
    float a[MAXW], h[MAXW];
    int win = M->widths[0];
    memcpy(a, x, sizeof(float) * win);
    for (int l = 0; l < M->n_layers; ++l) {
        int wo = M->widths[l + 1], wi = M->widths[l];
        const float *W = M->w[l], *B = M->b[l];
        for (int o = 0; o < wo; ++o) {
            float acc = 0.f;
            for (int i = 0; i < wi; ++i) acc = fmaf(a[i], W[o * wi + i], acc);
            float z = acc + B[o];
            h[o] = (l < M->n_layers - 1) ? (z > 0.f ? z : 0.f) : z;
        }
        memcpy(a, h, sizeof(float) * wo);
    }
    int i = 0;
    for (int hd = 0; hd < M->n_heads; ++hd) {
        for (int k = 0; k < M->head_w[hd]; ++k, ++i) {
            float z = a[i];
            out[i] = M->head_act[hd] == 0 ? z : (M->head_act[hd] == 1 ? sigmoidf_np(z) : expf(z));
        }
    }
}

/* encoding.py:438-478 ; out (levels*F) f32 */
static void hashgrid_encode1(const OAsset *A, const double *x, float *out) {
    static const uint64_t P0[3] = {1ull, 2654435761ull, 805459861ull};
    int F = A->hg_f;
    for (int l = 0; l < A->hg_levels; ++l) {
        int n = A->hg_res[l];
        int64_t base[3];
        double w[8];
        base_weights(x, n, base, w);
        double acc[8] = {0};
        for (int c = 0; c < 8; ++c) {
            int64_t cx = c & 1, cy = (c >> 1) & 1, cz = (c >> 2) & 1;
            int64_t idx;
            if (A->hg_dense[l]) {
                int64_t side = n + 1;
                idx = ((base[0] * side + base[1]) * side + base[2]) + ((cx * side + cy) * side + cz);
            } else {
                uint64_t h = ((uint64_t)(base[0] + cx) * P0[0]) ^ ((uint64_t)(base[1] + cy) * P0[1]) ^
                             ((uint64_t)(base[2] + cz) * P0[2]);
                idx = (int64_t)(h % A->hg_table);
            }
            const float *row = A->hg_feat[l] + idx * F;
            for (int f = 0; f < F; ++f) acc[f] += (double)row[f] * w[c];
        }
        for (int f = 0; f < F; ++f) out[l * F + f] = (float)acc[f];
    }
}

/* Moller-Trumbore in f64, same operation order as the CUDA kernel
 * (csrc/nolf_mesh.cuh mt_hit); -1 on miss. */
static double mt_hit(const double *T, const double *o, const double *d) {
    double e1x = T[3] - T[0], e1y = T[4] - T[1], e1z = T[5] - T[2];
    double e2x = T[6] - T[0], e2y = T[7] - T[1], e2z = T[8] - T[2];
    double px = d[1] * e2z - d[2] * e2y;
    double py = d[2] * e2x - d[0] * e2z;
    double pz = d[0] * e2y - d[1] * e2x;
    double det = (e1x * px + e1y * py) + e1z * pz;
    if (fabs(det) < 1e-300) return -1.0;
    double inv = 1.0 / det;
    double sx = o[0] - T[0], sy = o[1] - T[1], sz = o[2] - T[2];
    double u = ((sx * px + sy * py) + sz * pz) * inv;
    if (u < 0.0 || u > 1.0) return -1.0;
    double qx = sy * e1z - sz * e1y;
    double qy = sz * e1x - sx * e1z;
    double qz = sx * e1y - sy * e1x;
    double v = ((d[0] * qx + d[1] * qy) + d[2] * qz) * inv;
    if (v < 0.0 || u + v > 1.0) return -1.0;
    double t = ((e2x * qx + e2y * qy) + e2z * qz) * inv;
    return t >= 0.0 ? t : -1.0;
}

/* brute-force first hit over every triangle */
double oracle_mesh_hit(const double *tri, int64_t n_tri, const double *o, const double *d) {
    double best = -1.0;
    for (int64_t i = 0; i < n_tri; ++i) {
        double t = mt_hit(tri + 9 * i, o, d);
        if (t >= 0.0 && (best < 0.0 || t < best)) best = t;
    }
    return best;
}

/* lightfield.py:400-456 for one world ray */
static void render_one(const OAsset *A, const double *w2o, double scale, const double *o_w,
                       const double *d_w, float *rgba, float *depth, int64_t *cnt, ODebug *dbg,
                       int64_t ri) {
    double o[3], d[3];
    mat3_apply(w2o, 4, o_w, o);
    for (int k = 0; k < 3; ++k) o[k] = o[k] + w2o[k * 4 + 3];
    mat3_apply(w2o, 4, d_w, d);
    normalize3(d);
    rgba[0] = rgba[1] = rgba[2] = rgba[3] = 0.f;
    *depth = INFINITY;
    if (dbg && dbg->o_obj) memcpy(dbg->o_obj + 3 * ri, o, 24);
    if (dbg && dbg->d_obj) memcpy(dbg->d_obj + 3 * ri, d, 24);

    /* core.py:206-223 slab */
    double lo_max = -INFINITY, hi_min = INFINITY;
    int first = 1;
    for (int k = 0; k < 3; ++k) {
        double lo, hi;
        if (d[k] == 0.0) {
            int inside = (o[k] >= A->pmin[k]) && (o[k] <= A->pmax[k]);
            lo = inside ? -INFINITY : INFINITY;
            hi = inside ? INFINITY : -INFINITY;
        } else {
            double inv = 1.0 / d[k];
            double t0 = (A->pmin[k] - o[k]) * inv;
            double t1 = (A->pmax[k] - o[k]) * inv;
            lo = np_min(t0, t1);
            hi = np_max(t0, t1);
        }
        if (first) { lo_max = lo; hi_min = hi; first = 0; }
        else { lo_max = np_max(lo_max, lo); hi_min = np_min(hi_min, hi); }
    }
    double t_near = np_max(lo_max, 0.0);
    double t_far = np_min(hi_min, INFINITY);
    int boxhit = t_near <= t_far;
    if (dbg && dbg->boxhit) dbg->boxhit[ri] = (uint8_t)boxhit;
    if (dbg && dbg->t_near) { dbg->t_near[ri] = t_near; dbg->t_far[ri] = t_far; }
    if (boxhit && A->n_tri > 0) {   /* mesh proxy: march from its first hit */
        double tm = oracle_mesh_hit(A->tri, A->n_tri, o, d);
        if (tm < 0.0) boxhit = 0;
        else t_near = tm;
    }
    if (!boxhit) return;

    /* lightfield.py:129-186 march, every fixed step evaluated */
    double alpha_c = 0.0, best_w = 0.0, t_hit = INFINITY, trans = 1.0;
    int64_t samples = 0, istar = -1;
    const double delta = A->step;
    if (t_near < t_far) {
        const OAtlas *at = &A->density;
        int b = at->b;
        for (int64_t i = 0;; ++i) {
            double t_mid = t_near + ((double)i + 0.5) * delta;
            if (!(t_mid < t_far)) break;
            double pos[3];
            for (int k = 0; k < 3; ++k) pos[k] = clampd(o[k] + t_mid * d[k], 0.0, 1.0);
            int64_t c0 = clampi((int64_t)floor(pos[0] * b), 0, b - 1);
            int64_t c1 = clampi((int64_t)floor(pos[1] * b), 0, b - 1);
            int64_t c2 = clampi((int64_t)floor(pos[2] * b), 0, b - 1);
            int active = at->index[(c0 * b + c1) * b + c2] != -1;
            double sigma = 0.0;
            if (active) {
                float s;
                query_atlas1(at, pos, &s);
                sigma = (double)s;
            }
            samples += active;
            double absorb = exp(-sigma * delta);
            double w = trans * (1.0 - absorb);
            if (w > best_w) { best_w = w; t_hit = t_mid; istar = i; }
            alpha_c += w;
            trans *= absorb;
            if (!(trans > A->t_stop)) break;
        }
    }
    int hit = alpha_c > A->alpha_floor;
    if (!hit) { t_hit = INFINITY; istar = -1; }
    double p_h[3] = {0, 0, 0};
    if (hit)
        for (int k = 0; k < 3; ++k) p_h[k] = clampd(o[k] + t_hit * d[k], 0.0, 1.0);
    cnt[3] += samples;
    if (dbg) {
        if (dbg->hit) dbg->hit[ri] = (uint8_t)hit;
        if (dbg->t_hit) dbg->t_hit[ri] = t_hit;
        if (dbg->alpha_c) dbg->alpha_c[ri] = alpha_c;
        if (dbg->samples) dbg->samples[ri] = samples;
        if (dbg->istar) dbg->istar[ri] = istar;
        if (dbg->p_h) memcpy(dbg->p_h + 3 * ri, p_h, 24);
    }
    if (!hit) return;

    double t_obj = t_hit;
    double ps[3] = {p_h[0], p_h[1], p_h[2]};
    if (!A->use_hit_point) {
        t_obj = t_near;
        for (int k = 0; k < 3; ++k) ps[k] = clampd(o[k] + t_near * d[k], 0.0, 1.0);
    }

    /* shade_batch lightfield.py:267-336 */
    int64_t base[3], slots[8];
    double w8[8];
    base_weights(ps, A->psh_n, base, w8);
    psh_corner_slots(A, base, slots);
    int F = A->psh_f;
    float es[8];
    {
        double acc[8] = {0};
        for (int c = 0; c < 8; ++c)
            for (int f = 0; f < F; ++f) acc[f] += (double)A->psh_features[slots[c] * F + f] * w8[c];
        for (int f = 0; f < F; ++f) es[f] = (float)acc[f];
    }
    double sh[16];
    sh_encode(d, sh);
    double ac = clampd(alpha_c, 1e-4, 1.0 - 1e-4);
    float fs_in[MAXW], fs_out[8];
    int nin = 0;
    for (int f = 0; f < F; ++f) fs_in[nin++] = es[f];
    for (int k = 0; k < 16; ++k) fs_in[nin++] = (float)sh[k];
    if (A->refine_opacity) fs_in[nin++] = (float)ac;
    mlp_forward1(&A->fs, fs_in, fs_out);
    cnt[0] += 1;
    cnt[2] += 1;
    double c_s[3] = {fs_out[0], fs_out[1], fs_out[2]};
    double z = fs_out[3];
    double alpha;
    if (!A->use_opacity) alpha = clampd(alpha_c, 0.0, 1.0);
    else if (A->refine_opacity) alpha = sigmoid_np(z + log(ac / (1.0 - ac)));
    else alpha = sigmoid_np(z);

    double c_d[3], t;
    float dv[4] = {0, 0, 0, 0};
    if (!A->use_diffuse_color) {
        c_d[0] = c_d[1] = c_d[2] = 0.0;
        t = 1.0;
    } else if (A->has_diffuse_atlas) {
        query_atlas1(&A->diffuse, ps, dv);
        c_d[0] = dv[0]; c_d[1] = dv[1]; c_d[2] = dv[2];
        t = dv[3];
    } else {
        float ed[64];
        hashgrid_encode1(A, ps, ed);
        mlp_forward1(&A->fd, ed, dv);
        cnt[1] += 1;
        c_d[0] = dv[0]; c_d[1] = dv[1]; c_d[2] = dv[2];
        t = dv[3];
    }
    if (!A->use_tint) t = 0.5;
    for (int k = 0; k < 3; ++k) rgba[k] = (float)clampd(c_d[k] + t * c_s[k], 0.0, 1.0);
    rgba[3] = (float)alpha;
    *depth = (float)(t_obj / scale);
    if (dbg) {
        if (dbg->slots) memcpy(dbg->slots + 8 * ri, slots, 64);
        if (dbg->es) for (int f = 0; f < F; ++f) dbg->es[2 * ri + f] = es[f];
        if (dbg->fs_out) memcpy(dbg->fs_out + 4 * ri, fs_out, 16);
        if (dbg->diffuse) memcpy(dbg->diffuse + 4 * ri, dv, 16);
    }
    if (rgba[3] <= 0.f) {  /* lightfield.py:453-455 */
        rgba[0] = rgba[1] = rgba[2] = rgba[3] = 0.f;
        *depth = INFINITY;
    }
}

/* lightfield.py:400-456 batched; origins stride 0 => one shared origin.
 * counters: [fs_evals, fd_evals, hit_pixels, march_samples] (lightfield.py:113-126) */
int oracle_render_rays(const OAsset *A, const double *w2o, double scale, const double *origins,
                       int origin_stride, const double *dirs, int64_t n, float *rgba, float *depth,
                       int64_t *counters, ODebug *dbg, int nthreads) {
    int64_t c0 = 0, c1 = 0, c2 = 0, c3 = 0;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 256) reduction(+ : c0, c1, c2, c3)
#endif
    for (int64_t i = 0; i < n; ++i) {
        int64_t cnt[4] = {0, 0, 0, 0};
        render_one(A, w2o, scale, origins + (origin_stride ? 3 * i : 0), dirs + 3 * i,
                   rgba + 4 * i, depth + i, cnt, dbg, i);
        c0 += cnt[0]; c1 += cnt[1]; c2 += cnt[2]; c3 += cnt[3];
    }
    counters[0] += c0; counters[1] += c1; counters[2] += c2; counters[3] += c3;
    return 0;
}

/* renderer.render_range (renderer.py:63-93) fused with camera_dirs: rect of
 * one camera, rows y0..y1, columns x0..x1, outputs row-major over the rect. */
int oracle_render_rect(const OAsset *A, const double *w2o, double scale, const double *pose,
                       double fx, double fy, double cx, double cy, int x0, int y0, int x1, int y1,
                       float *rgba, float *depth, int64_t *counters, int nthreads) {
    int64_t w = x1 - x0, h = y1 - y0, n = w * h;
    int64_t c0 = 0, c1 = 0, c2 = 0, c3 = 0;
    const double o[3] = {pose[3], pose[7], pose[11]};
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 64) reduction(+ : c0, c1, c2, c3)
#endif
    for (int64_t i = 0; i < n; ++i) {
        double px = (double)(x0 + i % w), py = (double)(y0 + i / w), d[3];
        oracle_camera_dirs(pose, fx, fy, cx, cy, &px, &py, 1, d);
        int64_t cnt[4] = {0, 0, 0, 0};
        render_one(A, w2o, scale, o, d, rgba + 4 * i, depth + i, cnt, NULL, i);
        c0 += cnt[0]; c1 += cnt[1]; c2 += cnt[2]; c3 += cnt[3];
    }
    counters[0] += c0; counters[1] += c1; counters[2] += c2; counters[3] += c3;
    return 0;
}

/* farm.py:129-172 ; frames (K, P, 4) f32 + (K, P) f32 */
int oracle_compose(int K, int64_t P, const float *rgba, const float *depth, double alpha_vis,
                   float *out_rgba, float *out_depth, int nthreads) {
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for num_threads(nthreads) schedule(static)
#endif
    for (int64_t p = 0; p < P; ++p) {
        int order_small[64];
        int *order = K <= 64 ? order_small : (int *)malloc(sizeof(int) * (size_t)K);
        /* stable argsort by depth (NaN never produced upstream) */
        for (int k = 0; k < K; ++k) {
            int j = k;
            float dk = depth[(int64_t)k * P + p];
            while (j > 0 && depth[(int64_t)order[j - 1] * P + p] > dk) { order[j] = order[j - 1]; --j; }
            order[j] = k;
        }
        double oc[3] = {0, 0, 0}, trans = 1.0;
        float od = INFINITY;
        int set = 0;
        for (int r = 0; r < K; ++r) {
            int k = order[r];
            const float *c = rgba + ((int64_t)k * P + p) * 4;
            float a = c[3];
            for (int ch = 0; ch < 3; ++ch) oc[ch] += trans * (double)c[ch];
            if (!set && a > (float)alpha_vis) { /* f32 compare: numpy 2 weak scalar */ od = depth[(int64_t)k * P + p]; set = 1; }
            trans *= (double)(1.0f - a); /* numpy 2: python float - f32 array stays f32 */
        }
        float *o = out_rgba + p * 4;
        for (int ch = 0; ch < 3; ++ch) o[ch] = (float)clampd(oc[ch], 0.0, 1.0);
        o[3] = (float)clampd(1.0 - trans, 0.0, 1.0);
        out_depth[p] = od;
        if (o[3] <= 0.f) { o[0] = o[1] = o[2] = o[3] = 0.f; out_depth[p] = INFINITY; }
        if (order != order_small) free(order);
    }
    return 0;
}

int oracle_abi_version(void) { return 1; }
