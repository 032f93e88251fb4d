// nolf_device.cuh -- device-side data layout and bit-exact fp64 helpers for
// the i-NOLF render path.  Every routine cites the reference (radfarm) line it
// restates; fp64 arithmetic uses explicit *_rn intrinsics so nvcc cannot
// contract products and sums into FMAs that numpy does not perform, and
// __fma_rn exactly where numpy's OpenBLAS dgemm fuses (core.py:169,304).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#include "nolf_mesh.cuh"

namespace nolf {

constexpr int kHid = 64;       // MLP hidden width (lightfield.py:594 hidden=64)
constexpr int kInp = 24;       // padded MLP input width (fs: 19, fd: 12)
constexpr int kMaxLevels = 16;

struct DevAtlas {              // CubeAtlas (atlas.py:25-51)
  int b, r, C, s;              // s = r + 1
  const int32_t *index;        // b^3, -1 empty
  const float *cubes;          // n * s^3 * C
  const uint8_t *dist;         // b^3: Chebyshev distance (cells) to the nearest
                               // occupied cell, 0 = occupied, capped at 255
  const uint2 *cubes16;        // C == 4 atlases: the cubes again as fp16 (4 halves per corner) for the
                               // bf16 shading path's diffuse term (null: use cubes)
  const uint8_t *odist;        // 8 x b^3 (octant-major): edge (cells) of the largest empty cube
                               // anchored at the cell and extending in the octant's direction
                               // (octant bit k set: axis k negative); 0 = occupied, capped at 255
  const uint32_t *zmask;       // per cube, r^3 bits: sub-voxel whose 8 corners are all 0
  int zwords;                  // 32-bit words per cube
  int lr;                      // log2(r) when b and r are both powers of two, else -1
};


// Fully fused MLP parameter block (neural.py:29-108), fp32, padded:
//   w0t [kInp][kHid]  (layer-0 weights TRANSPOSED: in-major)
//   b0  [kHid]
//   w1  [kHid][kHid]  (out-major, only when n_layers == 3)
//   b1  [kHid]
//   wl  [4][kHid]     (last layer, out-major)
//   bl  [4]
struct MlpOff {
  static constexpr int w0t = 0;
  static constexpr int b0 = w0t + kInp * kHid;
  static constexpr int w1 = b0 + kHid;
  static constexpr int b1 = w1 + kHid * kHid;
  static constexpr int wl = b1 + kHid;
  static constexpr int bl = wl + 4 * kHid;
  static constexpr int total = bl + 4;
};

struct DevMlp {
  int n_layers;                // 2 or 3
  int in;                      // input width <= kInp
  int act[4];                  // head activation per output (NOLF_HEAD_*)
  const float *params;         // MlpOff::total floats
};

struct DevAsset {              // LightFieldAsset (lightfield.py:217-248)
  DevAtlas den, dif;
  int has_dif;
  // PSH (encoding.py:109-140); Phi narrowed to u32 (values < m)
  int N;
  uint32_t m, mphi;
  const uint32_t *phi;
  const float *feat;           // m * F
  int F;
  const uint32_t *tab;         // 6 * (N+1): (x*P0[a]) % m, a=0..2 ; (x*P1[a]) % mphi
  // live diffuse hash grid (encoding.py:405-459)
  int hg_levels, hg_F;
  unsigned long long hg_table;
  int hg_res[kMaxLevels];
  int hg_dense[kMaxLevels];
  const float *hg_feat[kMaxLevels];
  DevMlp fs, fd;
  double step, t_stop, alpha_floor;
  double inv_step;             // 1 / step: only for conservative sample-index bounds (margins absorb its rounding)
  float inv_step_f, inv_b_f;   // fp32 1/step and 1/b: the march's jump estimates (verified exactly)
  double pmin[3], pmax[3];
  int use_hit_point, use_opacity, refine_opacity, use_tint, use_diffuse_color;
  int mlp_mode;
  // tensor-core shading tables (NOLF_MLP_BF16)
  const uint8_t *tc_w;         // bf16 W0 [64 x 32] then W1 [64 x 64], UMMA K-major layout
                               // then the fp32 block (b0, b1, W2 [o][4], b2) and the PSH
                               // residue tables: the shader's smem image, one bulk copy
  uint32_t tc_w_bytes;
  const uint16_t *phi16;       // Phi narrowed to u16 (m <= 65536), else null
  uint32_t phi16_bytes;        // padded to 16 B for the TMA bulk copy
  DevMesh mesh;                // triangle-mesh proxy (nodes == null: slab only)
  // host-side culling box: AABB of the occupied density cells grown by one
  // cell (faces reaching the unit-cube boundary extended to the proxy, where
  // clipped sample positions land), clipped to the proxy box
  double cull_lo[3], cull_hi[3];
  int cull_empty;              // no occupied cell: no ray can ever sample density
};

// One placed asset for a launch (NolfInstance minus the host handle).
struct DevInst {
  const DevAsset *a;           // device pointer
  double w2o[12];              // rows of [R | t]
  double scale;
};

// Hit record written by the march (80 B, 16-B aligned).
struct __align__(16) HitRec {
  double p[3];                 // shading point (p_h or proxy entry), object space
  double alpha_c;              // coarse opacity (lightfield.py:175)
  double t_obj;                // object-space depth of the shading point
  double d[3];                 // object-space unit direction (SH input, lightfield.py:447)
  uint32_t out_idx;            // output row / packed pixel
  uint32_t ordinal;            // layer index of this hit within its pixel
};

// ---------------------------------------------------------------- fp64 helpers
__device__ __forceinline__ double np_min(double a, double b) {   // np.minimum
  return (a != a || b != b) ? __longlong_as_double(0x7ff8000000000000ll) : (a < b ? a : b);
}
__device__ __forceinline__ double np_max(double a, double b) {   // np.maximum
  return (a != a || b != b) ? __longlong_as_double(0x7ff8000000000000ll) : (a > b ? a : b);
}
__device__ __forceinline__ double clamp01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }
__device__ __forceinline__ double clampd(double v, double lo, double hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}
__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// (N,3) @ M.T row for a 3x3 block with leading dim ld:
// numpy/OpenBLAS dgemm == fma(a2, m2, fma(a1, m1, a0*m0)) (measured 100%).
__device__ __forceinline__ void mat3_apply(const double *M, int ld, const double a[3], double out[3]) {
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const double *row = M + j * ld;
    out[j] = __fma_rn(a[2], row[2], __fma_rn(a[1], row[1], __dmul_rn(a[0], row[0])));
  }
}
// d / np.linalg.norm(d): sqrt((x*x + y*y) + z*z), then 3 divisions
__device__ __forceinline__ void normalize3(double v[3]) {
  double n = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(v[0], v[0]), __dmul_rn(v[1], v[1])),
                                  __dmul_rn(v[2], v[2])));
  v[0] = __ddiv_rn(v[0], n);
  v[1] = __ddiv_rn(v[1], n);
  v[2] = __ddiv_rn(v[2], n);
}

// camera_dirs (core.py:162-170) for one pixel; pose row-major 4x4.
__device__ __forceinline__ void camera_dir(const double *pose, double fx, double fy, double cx,
                                           double cy, double px, double py, double out[3]) {
  double u = __ddiv_rn(__dsub_rn(__dadd_rn(px, 0.5), cx), fx);
  double v = -__ddiv_rn(__dsub_rn(__dadd_rn(py, 0.5), cy), fy);
  double d[3] = {u, v, -1.0};
  mat3_apply(pose, 4, d, out);
  normalize3(out);
}

// render_rays world->object (lightfield.py:408-412): o@R.T + t ; normalize(d@R.T)
__device__ __forceinline__ void to_object(const double *w2o12, const double ow[3], const double dw[3],
                                          double o[3], double d[3]) {
  mat3_apply(w2o12, 4, ow, o);
#pragma unroll
  for (int k = 0; k < 3; ++k) o[k] = __dadd_rn(o[k], w2o12[k * 4 + 3]);
  mat3_apply(w2o12, 4, dw, d);
  normalize3(d);
}

// aabb_intersect_batch (core.py:206-223), t_min = 0, t_max = inf.
// numpy's minimum/maximum propagate NaN; a NaN slab value can only come from
// 0*inf (d subnormal, o on a face) and makes t_near/t_far NaN, i.e. a miss.
// Tracking it with one flag instead of NaN-aware selects is observably
// identical (every non-NaN value is computed with the same comparisons).
// inv[] returns 1/d (inf for d == 0) for reuse by the march.
// HAVE_INV: inv[] already holds 1/d from an earlier slab of the same ray.
template <bool HAVE_INV = false>
__device__ __forceinline__ bool slab(const double pmin[3], const double pmax[3], const double o[3],
                                     const double d[3], double &t_near, double &t_far, double inv[3]) {
  const double INF = __longlong_as_double(0x7ff0000000000000ll);
  double lo_max = 0, hi_min = 0;
  bool nan = false;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double lo, hi;
    if (d[k] == 0.0) {
      const bool inside = (o[k] >= pmin[k]) && (o[k] <= pmax[k]);
      lo = inside ? -INF : INF;
      hi = inside ? INF : -INF;
      if (!HAVE_INV) inv[k] = INF;
    } else {
      if (!HAVE_INV) inv[k] = __drcp_rn(d[k]);   // IEEE 1/d, == __ddiv_rn(1.0, d)
      const double t0 = __dmul_rn(__dsub_rn(pmin[k], o[k]), inv[k]);
      const double t1 = __dmul_rn(__dsub_rn(pmax[k], o[k]), inv[k]);
      nan |= (t0 != t0) | (t1 != t1);
      lo = t0 < t1 ? t0 : t1;
      hi = t0 > t1 ? t0 : t1;
    }
    if (k == 0) { lo_max = lo; hi_min = hi; }
    else { lo_max = lo_max > lo ? lo_max : lo; hi_min = hi_min < hi ? hi_min : hi; }
  }
  t_near = lo_max > 0.0 ? lo_max : 0.0;
  t_far = hi_min < INF ? hi_min : INF;
  if (nan) t_near = t_far = __longlong_as_double(0x7ff8000000000000ll);
  return t_near <= t_far;
}

// Sub-voxel of x inside its cube and the trilinear fractions (atlas.py:162-172).
__device__ __forceinline__ void atlas_subvoxel(const DevAtlas &at, const double x[3], int base[3], double frac[3]) {
  const double bd = (double)at.b, rd = (double)at.r;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double scaled = __dmul_rn(x[k], bd);
    int cell = clampi((int)floor(scaled), 0, at.b - 1);
    double local = __dmul_rn(__dsub_rn(scaled, (double)cell), rd);
    base[k] = clampi((int)floor(local), 0, at.r - 1);
    frac[k] = __dsub_rn(local, (double)base[k]);
  }
}

// atlas_subvoxel with the index cell already known (sample_cell computed it
// from the same pos with the same ops).
__device__ __forceinline__ void atlas_subvoxel_in(const DevAtlas &at, const double x[3], const int cell[3], int base[3],
                                                  double frac[3]) {
  const double bd = (double)at.b, rd = (double)at.r;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double local = __dmul_rn(__dsub_rn(__dmul_rn(x[k], bd), (double)cell[k]), rd);
    base[k] = clampi(__double2int_rd(local), 0, at.r - 1);
    frac[k] = __dsub_rn(local, (double)base[k]);
  }
}

template <int C>
__device__ __forceinline__ void atlas_trilinear_at(const DevAtlas &at, int cid, const int base[3], const double frac[3],
                                                   float out[C]);

// query_atlas (atlas.py:158-185) inside a known non-empty cube; C <= 4.
template <int C>
__device__ __forceinline__ void atlas_trilinear(const DevAtlas &at, int cid, const double x[3], float out[C]) {
  int base[3];
  double frac[3];
  atlas_subvoxel(at, x, base, frac);
  atlas_trilinear_at<C>(at, cid, base, frac, out);
}

template <int C>
__device__ __forceinline__ void atlas_trilinear_at(const DevAtlas &at, int cid, const int base[3], const double frac[3],
                                                   float out[C]) {
  const int s = at.s;
  const float *cube = at.cubes + (size_t)cid * (size_t)(s * s * s * C);
  double acc[C];
#pragma unroll
  for (int ch = 0; ch < C; ++ch) acc[ch] = 0.0;
  double g[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) g[k] = __dsub_rn(1.0, frac[k]);
  if constexpr (C == 4) {      // 8 corner loads in flight, then the ordered f64 sum
    float4 q[8];
#pragma unroll
    for (int c = 0; c < 8; ++c)
      q[c] = __ldg(reinterpret_cast<const float4 *>(
          cube + (((base[0] + (c & 1)) * s + (base[1] + ((c >> 1) & 1))) * s + (base[2] + ((c >> 2) & 1))) * C));
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int dx = c & 1, dy = (c >> 1) & 1, dz = (c >> 2) & 1;
      const double w = __dmul_rn(__dmul_rn(dx ? frac[0] : g[0], dy ? frac[1] : g[1]), dz ? frac[2] : g[2]);
      const float qq[4] = {q[c].x, q[c].y, q[c].z, q[c].w};
#pragma unroll
      for (int ch = 0; ch < C; ++ch) acc[ch] = __dadd_rn(acc[ch], __dmul_rn(w, (double)qq[ch]));
    }
#pragma unroll
    for (int ch = 0; ch < C; ++ch) out[ch] = (float)acc[ch];
  } else {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int dx = c & 1, dy = (c >> 1) & 1, dz = (c >> 2) & 1;
      const double w = __dmul_rn(__dmul_rn(dx ? frac[0] : g[0], dy ? frac[1] : g[1]), dz ? frac[2] : g[2]);
      const float *v = cube + (((base[0] + dx) * s + (base[1] + dy)) * s + (base[2] + dz)) * C;
#pragma unroll
      for (int ch = 0; ch < C; ++ch) acc[ch] = __dadd_rn(acc[ch], __dmul_rn(w, (double)__ldg(v + ch)));
    }
#pragma unroll
    for (int ch = 0; ch < C; ++ch) out[ch] = (float)acc[ch];
  }
}

// query_atlas at an arbitrary point (empty cell -> zeros).
// Cube id of x's index cell (-1 empty): issued early, the load overlaps other work.
__device__ __forceinline__ int atlas_cell_id(const DevAtlas &at, const double x[3]) {
  const double bd = (double)at.b;
  int cell[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) cell[k] = clampi((int)floor(__dmul_rn(x[k], bd)), 0, at.b - 1);
  return __ldg(at.index + (cell[0] * at.b + cell[1]) * at.b + cell[2]);
}

template <int C>
__device__ __forceinline__ void atlas_query_cid(const DevAtlas &at, int cid, const double x[3], float out[C]) {
  if (cid < 0) {
#pragma unroll
    for (int ch = 0; ch < C; ++ch) out[ch] = 0.f;
    return;
  }
  atlas_trilinear<C>(at, cid, x, out);
}

// query_atlas with the trilinear weights and sums in fp32 (the bf16 shading
// path's diffuse term: 2/255 budget); cell / sub-voxel selection as above.
__device__ __forceinline__ void atlas_query4_f(const DevAtlas &at, int cid, const double x[3], float out[4]) {
  if (cid < 0) {
    out[0] = out[1] = out[2] = out[3] = 0.f;
    return;
  }
  int base[3];
  double frac[3];
  atlas_subvoxel(at, x, base, frac);
  const int s = at.s;
  float4 q[8];
  if (at.cubes16) {            // fp16 corners: half the bytes per gather (|err| <= 2^-11 relative)
    const uint2 *cube = at.cubes16 + (size_t)cid * (size_t)(s * s * s);
    uint2 h[8];
#pragma unroll
    for (int c = 0; c < 8; ++c)
      h[c] = __ldg(cube + (((base[0] + (c & 1)) * s + (base[1] + ((c >> 1) & 1))) * s + (base[2] + ((c >> 2) & 1))));
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float2 lo = __half22float2(*reinterpret_cast<const __half2 *>(&h[c].x));
      const float2 hi = __half22float2(*reinterpret_cast<const __half2 *>(&h[c].y));
      q[c] = make_float4(lo.x, lo.y, hi.x, hi.y);
    }
  } else {
    const float *cube = at.cubes + (size_t)cid * (size_t)(s * s * s * 4);
#pragma unroll
    for (int c = 0; c < 8; ++c)
      q[c] = __ldg(reinterpret_cast<const float4 *>(
          cube + (((base[0] + (c & 1)) * s + (base[1] + ((c >> 1) & 1))) * s + (base[2] + ((c >> 2) & 1))) * 4));
  }
  const float f0 = (float)frac[0], f1 = (float)frac[1], f2 = (float)frac[2];
  const float g0 = 1.0f - f0, g1 = 1.0f - f1, g2 = 1.0f - f2;
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const float w = ((c & 1) ? f0 : g0) * (((c >> 1) & 1) ? f1 : g1) * (((c >> 2) & 1) ? f2 : g2);
    a0 = fmaf(w, q[c].x, a0);
    a1 = fmaf(w, q[c].y, a1);
    a2 = fmaf(w, q[c].z, a2);
    a3 = fmaf(w, q[c].w, a3);
  }
  out[0] = a0; out[1] = a1; out[2] = a2; out[3] = a3;
}

// L2 prefetch of the 8 corners atlas_query4_f(at, ., x) will read (4-channel atlas).
__device__ __forceinline__ void atlas_prefetch4(const DevAtlas &at, const double x[3]) {
  const int cid = atlas_cell_id(at, x);
  if (cid < 0) return;
  int base[3];
  double frac[3];
  atlas_subvoxel(at, x, base, frac);
  const int s = at.s;
  const float *cube = at.cubes + (size_t)cid * (size_t)(s * s * s * 4);
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const float *p = cube + (((base[0] + (c & 1)) * s + (base[1] + ((c >> 1) & 1))) * s + (base[2] + ((c >> 2) & 1))) * 4;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
  }
}

template <int C>
__device__ __forceinline__ void atlas_query(const DevAtlas &at, const double x[3], float out[C]) {
  const int cid = atlas_cell_id(at, x);
  if (cid < 0) {
#pragma unroll
    for (int ch = 0; ch < C; ++ch) out[ch] = 0.f;
    return;
  }
  atlas_trilinear<C>(at, cid, x, out);
}

// _base_weights (encoding.py:346-365)
__device__ __forceinline__ void base_weights(const double x[3], int res, int base[3], double w[8]) {
  double f[3], g[3];
  const double rd = (double)res;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double scaled = __dmul_rn(x[k], rd);
    double fl = floor(scaled);
    int bb = fl > (double)(res - 1) ? res - 1 : (int)fl;
    if (bb < 0) bb = 0;
    base[k] = bb;
    f[k] = __dsub_rn(scaled, (double)bb);
    g[k] = __dsub_rn(1.0, f[k]);
  }
  double gygz = __dmul_rn(g[1], g[2]), fygz = __dmul_rn(f[1], g[2]);
  double gyfz = __dmul_rn(g[1], f[2]), fyfz = __dmul_rn(f[1], f[2]);
  w[0] = __dmul_rn(g[0], gygz); w[1] = __dmul_rn(f[0], gygz);
  w[2] = __dmul_rn(g[0], fygz); w[3] = __dmul_rn(f[0], fygz);
  w[4] = __dmul_rn(g[0], gyfz); w[5] = __dmul_rn(f[0], gyfz);
  w[6] = __dmul_rn(g[0], fyfz); w[7] = __dmul_rn(f[0], fyfz);
}

// PshTable.corner_slots (encoding.py:130-140) via per-axis residue tables:
// ((p+c).P0 mod m + Phi[((p+c).P1) mod mphi]) mod m, identical integers.
__device__ __forceinline__ uint32_t psh_slot(const uint32_t *tab, const uint32_t *phi, int N, uint32_t m,
                                             uint32_t mphi, int x, int y, int z) {
  const int s = N + 1;
  uint32_t h0 = tab[x] + tab[s + y];
  h0 = h0 >= m ? h0 - m : h0;
  h0 += tab[2 * s + z];
  h0 = h0 >= m ? h0 - m : h0;
  uint32_t h1 = tab[3 * s + x] + tab[4 * s + y];
  h1 = h1 >= mphi ? h1 - mphi : h1;
  h1 += tab[5 * s + z];
  h1 = h1 >= mphi ? h1 - mphi : h1;
  uint32_t slot = h0 + phi[h1];
  return slot >= m ? slot - m : slot;
}

// sh_encode_batch (core.py:239-261), product order as written in numpy.
__device__ __forceinline__ void sh_encode(const double d[3], double o[16]) {
  const double C0 = 0.28209479177387814, C1 = 0.4886025119029199;
  const double C20 = 1.0925484305920792, C21 = -1.0925484305920792, C22 = 0.31539156525252005,
               C23 = -1.0925484305920792, C24 = 0.5462742152960396;
  const double C30 = -0.5900435899266435, C31 = 2.890611442640554, C32 = -0.4570457994644658,
               C33 = 0.3731763325901154, C34 = -0.4570457994644658, C35 = 1.445305721320277,
               C36 = -0.5900435899266435;
  const double x = d[0], y = d[1], z = d[2];
  const double xx = __dmul_rn(x, x), yy = __dmul_rn(y, y), zz = __dmul_rn(z, z);
#define M_ __dmul_rn
#define S_ __dsub_rn
  o[0] = C0;
  o[1] = M_(-C1, y);
  o[2] = M_(C1, z);
  o[3] = M_(-C1, x);
  o[4] = M_(M_(C20, x), y);
  o[5] = M_(M_(C21, y), z);
  o[6] = M_(C22, S_(S_(M_(2.0, zz), xx), yy));
  o[7] = M_(M_(C23, x), z);
  o[8] = M_(C24, S_(xx, yy));
  o[9] = M_(M_(C30, y), S_(M_(3.0, xx), yy));
  o[10] = M_(M_(M_(C31, x), y), z);
  o[11] = M_(M_(C32, y), S_(S_(M_(4.0, zz), xx), yy));
  o[12] = M_(M_(C33, z), S_(S_(M_(2.0, zz), M_(3.0, xx)), M_(3.0, yy)));
  o[13] = M_(M_(C34, x), S_(S_(M_(4.0, zz), xx), yy));
  o[14] = M_(M_(C35, z), S_(xx, yy));
  o[15] = M_(M_(C36, x), S_(xx, M_(3.0, yy)));
#undef M_
#undef S_
}

// sh_encode's polynomial in fp32 (inputs of the bf16 MLP path only).
__device__ __forceinline__ void sh_encode_f(const double dd[3], float o[16]) {
  const float x = (float)dd[0], y = (float)dd[1], z = (float)dd[2];
  const float xx = x * x, yy = y * y, zz = z * z;
  o[0] = 0.28209479177387814f;
  o[1] = -0.4886025119029199f * y;
  o[2] = 0.4886025119029199f * z;
  o[3] = -0.4886025119029199f * x;
  o[4] = 1.0925484305920792f * x * y;
  o[5] = -1.0925484305920792f * y * z;
  o[6] = 0.31539156525252005f * (2.0f * zz - xx - yy);
  o[7] = -1.0925484305920792f * x * z;
  o[8] = 0.5462742152960396f * (xx - yy);
  o[9] = -0.5900435899266435f * y * (3.0f * xx - yy);
  o[10] = 2.890611442640554f * x * y * z;
  o[11] = -0.4570457994644658f * y * (4.0f * zz - xx - yy);
  o[12] = 0.3731763325901154f * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
  o[13] = -0.4570457994644658f * x * (4.0f * zz - xx - yy);
  o[14] = 1.445305721320277f * z * (xx - yy);
  o[15] = -0.5900435899266435f * x * (xx - 3.0f * yy);
}

__device__ __forceinline__ float sigmoidf_np(float z) {   // neural._sigmoid in f32
  if (z >= 0.f) return 1.0f / (1.0f + expf(-z));
  float ez = expf(z);
  return ez / (1.0f + ez);
}
__device__ __forceinline__ double sigmoid_np(double z) {  // lightfield._sigmoid in f64
  if (z >= 0.0) return 1.0 / (1.0 + exp(-z));
  double ez = exp(z);
  return ez / (1.0 + ez);
}

}  // namespace nolf
