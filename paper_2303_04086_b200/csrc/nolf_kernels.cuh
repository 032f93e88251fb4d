// nolf_kernels.cuh -- the i-NOLF hot path as three sm_100a kernels:
//
//   k_march    per ray (x placed asset): proxy slab test + fixed-step
//              transmittance march with EXACT empty-space skipping; emits one
//              HitRec per hit into a per-instance queue (lightfield.py:400-445,
//              129-186).
//   k_shade    per hit record: PSH slots + trilinear features, SH(d_obj),
//              fused fp32 MLP (weights staged in shared memory), diffuse atlas
//              or live hash-grid diffuse, combine (lightfield.py:267-336,
//              446-455).
//   k_compose  per pixel: stable depth sort of its hit layers + front-to-back
//              over in f64 + encode_frame RAW quantisation (farm.py:129-172,
//              protocol.py:256-266).
#pragma once
#include <climits>

#include "nolf_device.cuh"

namespace nolf {

enum RayMode { kModeRays = 0, kModeRect = 1, kModeScene = 2 };

struct CamParams {             // NolfCamera with pose rows
  double pose[16];
  double fx, fy, cx, cy;
  int width, height;
  long long pix_base;          // frame-layout output offset of this camera
};

// Conservative screen rectangle (inclusive pixel indices) outside which a
// pixel's ray cannot meet an instance's proxy box: the box lies in front of
// the camera, so its image is the convex hull of its projected corners.
struct ScreenBox { int x0, y0, x1, y1; };

struct TileParams { int cam, x0, y0, x1, y1; };

struct MarchArgs {
  const DevInst *inst;         // n_inst instances (device)
  int n_inst;
  // ray source
  const double *origins;       // kModeRays
  int origin_stride;           // 0 => shared origin
  const double *dirs;          // kModeRays
  long long n_rays;            // total ray slots
  const CamParams *cams;       // kModeRect / kModeScene (device)
  const TileParams *tiles;     // kModeScene (device) ; kModeRect: tiles[0] is the rect
  long long tile_stride;       // kModeScene: pixel slots per tile
  const ScreenBox *cull;       // [n_inst * n_cams] (NULL: no culling)
  int n_cams;
  // outputs
  HitRec *queue;               // per-instance queues at qoff[k] .. qoff[k+1]
  const long long *qoff;
  unsigned int *counts;        // n_inst
  float *rgba;                 // kModeRays/kModeRect: miss init (n, 4)
  float *depth;
  uint8_t *nhit;               // kModeScene: per pixel layer count
  unsigned long long *counters;
  // march_rays mode (lightfield.py:129-186 outputs per ray, no queue)
  int raw_rays;                // 1: rays are already in object space (no w2o, no renormalise)
  int use_zmask;               // skip zero-corner sub-voxels (always on; 0 for A/B checks)
  uint8_t *out_hit;
  double *out_t_hit, *out_alpha_c, *out_p_h;
  long long *out_samples;
  // scene mode with 128-slot-aligned tiles: compacted list of the chunks
  // (128 consecutive slots of one tile) some screen box meets, and the
  // persistent marcher's work counter
  const unsigned *chunks;      // live chunks bucketed by candidate count: bucket b at chunks + b * list_stride
  const unsigned *n_chunks;    // [0] all live chunks, [2 + b] bucket b's count (b = 1..kChunkBuckets-1)
  unsigned *fetch;
  long long list_stride;
  int heavy_first;             // walk the buckets (most candidates first) instead of the spatial list
  unsigned *chunk_cost;        // per chunk: the CTA's duration (clock cycles) in the last frame that marched
                               // it, or 0 -- the heavy-first buckets of the next frame (null: candidate counts)
  int max_layers;              // scene mode: compose layers per pixel slot in the workspace
  unsigned *errors;            // sticky device error counters (kErr*), never NULL
};

// Device error counters (nolf_capi.cu reads them back and fails loudly):
// a hit record that did not fit its instance's queue, a hit beyond the
// pixel's compose layers, a scene tile outside its camera's frame (or larger
// than tile_stride, or naming a missing camera), a BVH traversal deeper than
// its stack.  Each is impossible for valid inputs (the host sizes queues and
// layers from the screen boxes); they guard against invalid ones, and the
// offending work is dropped instead of writing out of bounds.
enum { kErrQueue = 0, kErrLayers = 1, kErrTile = 2, kErrBvh = 3, kNumErr = 4 };

// A scene tile the kernels may address: a rect inside its camera's frame
// with no more pixels than a tile slot holds (empty rects are the padding of
// uneven shards: valid, no pixels).
__device__ __forceinline__ bool tile_valid(const TileParams &tp, const CamParams *cams, int n_cams,
                                           long long stride) {
  if (tp.cam < 0 || tp.cam >= n_cams) return false;
  const CamParams &c = cams[tp.cam];
  return tp.x0 >= 0 && tp.y0 >= 0 && tp.x1 >= tp.x0 && tp.y1 >= tp.y0 && tp.x1 <= c.width && tp.y1 <= c.height &&
         (long long)(tp.x1 - tp.x0) * (tp.y1 - tp.y0) <= stride;
}

#ifndef NOLF_CHUNK_BUCKETS
#define NOLF_CHUNK_BUCKETS 8
#endif
// heavy-first buckets of live chunks (1 .. kChunkBuckets-1; the list keeps one
// region per bucket): the previous frame's CTA duration class, else the
// candidate-instance count (the last bucket: >= kChunkBuckets-1 instances)
constexpr int kChunkBuckets = NOLF_CHUNK_BUCKETS;

// it-th live chunk: spatial order (list region 0, best cache locality) or
// heavy-first (most candidate instances first, so the longest CTAs start
// early and light ones fill the tail -- for launches of only a few waves).
__device__ __forceinline__ unsigned chunk_at(const unsigned *list, const unsigned *counts, long long stride,
                                             unsigned it, int heavy_first) {
  if (!heavy_first) return list[it];
#pragma unroll
  for (int b = kChunkBuckets - 1; b >= 1; --b) {
    const unsigned c = counts[2 + b];
    if (it < c) return list[(long long)b * stride + it];
    it -= c;
  }
  return 0u;
}

__device__ __forceinline__ double t_stop_of(const DevAsset &A) { return A.t_stop; }

// Sample i's clipped position and index cell, exactly as march_rays computes
// them (t_mid = t_near + (i+0.5)*step ; pos = clip(o + t_mid*d, 0, 1)).
// CLIP = false when the caller proved every position it will ask for lies in
// [0,1] already (then clip() is the identity and is skipped).
template <bool CLIP = true>
__device__ __forceinline__ double sample_cell(const double o[3], const double d[3], double t_near, double delta,
                                              int i, int b, double pos[3], int cell[3]) {
  double t_mid = __dadd_rn(t_near, __dmul_rn((double)i + 0.5, delta));
  const double bd = (double)b;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double v = __dadd_rn(o[k], __dmul_rn(t_mid, d[k]));
    pos[k] = CLIP ? clamp01(v) : v;
    cell[k] = min(__double2int_rd(__dmul_rn(pos[k], bd)), b - 1);   // pos in [0,1]: floor >= 0
  }
  return t_mid;
}

// Power-of-two grids (b = 2^lb, r = 2^lr, the reference defaults 32 / 8):
// multiplying by b, r or G = b*r is exact, and so is (x*b - cell) (Sterbenz:
// cell <= x*b < cell+1 <= 2*cell, or cell = 0), hence local = x*G - cell*r
// EXACTLY.  So with gi = floor(x*G): cell = min(gi >> lr, b-1),
// base = min(gi - cell*r, r-1), frac = x*G - (cell*r + base), bit-identical
// to atlas.py:162-172's floor/clip/subtract sequence, in integer ops.
template <bool CLIP = true>
__device__ __forceinline__ double sample_grid(const double o[3], const double d[3], double t_near, double delta,
                                              int i, double G, int lr, int b, double pos[3], int gi[3],
                                              int cell[3]) {
  double t_mid = __dadd_rn(t_near, __dmul_rn((double)i + 0.5, delta));
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double v = __dadd_rn(o[k], __dmul_rn(t_mid, d[k]));
    pos[k] = CLIP ? clamp01(v) : v;
    gi[k] = __double2int_rd(__dmul_rn(pos[k], G));
    cell[k] = min(gi[k] >> lr, b - 1);
  }
  return t_mid;
}

__device__ __forceinline__ void subvoxel_grid(const double pos[3], const int gi[3], const int cell[3], double G,
                                              int lr, int r, int base[3], double frac[3]) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int c0 = cell[k] << lr;
    base[k] = min(gi[k] - c0, r - 1);
    frac[k] = __dsub_rn(__dmul_rn(pos[k], G), (double)(c0 + base[k]));
  }
}

// True when the unclipped positions of samples lo and hi are inside [0,1]^3:
// each coordinate fl(o + fl(t_mid*d)) is monotone in the sample index, so all
// samples between them are inside too and clip() is exactly the identity.
__device__ __forceinline__ bool samples_inside_unit(const double o[3], const double d[3], double t_near,
                                                    double delta, int lo, int hi) {
  const double ta = __dadd_rn(t_near, __dmul_rn((double)lo + 0.5, delta));
  const double tb = __dadd_rn(t_near, __dmul_rn((double)hi + 0.5, delta));
  bool in = true;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double a = __dadd_rn(o[k], __dmul_rn(ta, d[k])), c = __dadd_rn(o[k], __dmul_rn(tb, d[k]));
    in = in && a >= 0.0 && a <= 1.0 && c >= 0.0 && c <= 1.0;
  }
  return in;
}

#ifdef NOLF_STATS   // diagnostic build only: march work counters (-DNOLF_STATS_CTR) / CTA spans
__device__ unsigned long long g_stats[16];
__device__ unsigned long long g_cta_start[1 << 20], g_cta_end[1 << 20];
__device__ unsigned g_cta_work[1 << 20][4];   // per CTA: warp-instance passes, max lane iterations
                                               // of one march, max lane iterations over all, max instances
#define NOLF_ITER(x) (x)
#else
#define NOLF_ITER(x) ((void)0)
#endif
#if defined(NOLF_STATS) && defined(NOLF_STATS_CTR)
#define NOLF_STAT(k, v) atomicAdd(&g_stats[k], (unsigned long long)(v))
#else
#define NOLF_STAT(k, v) ((void)0)
#endif

// Pixel of packed slot `local` inside a w x h tile.  Tiles whose sides are
// multiples of 8 x 4 are stored in 8x4 blocks of 32 slots (one warp marches a
// compact 8x4 pixel patch -> coherent rays, less divergence); other tiles are
// row-major.  render.py:unpack_index mirrors this.
__device__ __forceinline__ void slot_xy(long long local, int w, int h, int &x, int &y) {
  const unsigned lo = (unsigned)local;         // local < w*h < 2^31
  if ((w & 7) == 0 && (h & 3) == 0) {
    const unsigned blk = lo >> 5, l = lo & 31u, bx = (unsigned)w >> 3;
    unsigned by, bxi;
    if ((bx & (bx - 1u)) == 0u) {               // power-of-two blocks per row (32-wide tiles)
      const int sh = __ffs(bx) - 1;
      by = blk >> sh;
      bxi = blk & (bx - 1u);
    } else {
      by = blk / bx;
      bxi = blk - by * bx;
    }
    x = (int)(bxi * 8u + (l & 7u));
    y = (int)(by * 4u + (l >> 3));
  } else {
    const unsigned uy = lo / (unsigned)w;
    x = (int)(lo - uy * (unsigned)w);
    y = (int)uy;
  }
}

// (tile, local slot) of packed index p; 32-bit divide when it fits.
__device__ __forceinline__ void split_slot(long long p, long long stride, long long &t, long long &local) {
  if ((stride & (stride - 1)) == 0) {          // power-of-two tiles (32x32 = 1024 slots): shift
    const int sh = __ffsll(stride) - 1;
    t = p >> sh;
    local = p & (stride - 1);
  } else if (p < 0xffffffffll && stride < 0xffffffffll) {
    const unsigned p32 = (unsigned)p, s32 = (unsigned)stride, t32 = p32 / s32;
    t = t32;
    local = p32 - t32 * s32;
  } else {
    t = p / stride;
    local = p % stride;
  }
}

// march_rays (lightfield.py:129-186) for one ray.
//
// Exact empty-space skipping: an empty sample has sigma = 0, so absorb = 1,
// w = 0 (never "better", best_w starts at 0), alpha_c and T are unchanged and
// it is not counted; skipping it is bitwise neutral.  From an empty sample
// i in an empty box B (a macro cell, else an index cell) we jump to a guess j
// (the last sample before B's analytic exit) and VERIFY sample j's cell is in
// B.  Each computed cell coordinate is a monotone function of i (fl() is
// monotone, t_mid is monotone in i, clip/floor are monotone), so cells of all
// samples between i and j lie between cell(i) and cell(j), i.e. inside B:
// every skipped sample is provably empty, whatever the rounding.
struct MarchOut {
  double alpha_c, t_hit;
  long long samples;
  bool hit;
#ifdef NOLF_STATS
  unsigned iters;
#endif
};

template <bool CLIP, bool POW2>
__device__ __forceinline__ MarchOut march_ray(const DevAsset &A, const double o[3], const double d[3],
                                              const float invf[3], double t_near, double t_far, bool use_zmask,
                                              int i_start, double t_end) {
  MarchOut r;
  r.alpha_c = 0.0;
  r.t_hit = __longlong_as_double(0x7ff0000000000000ll);
  r.samples = 0;
  r.hit = false;
  if (!(t_near < t_far)) return r;
  const DevAtlas &at = A.den;
  const double delta = A.step;
  const int b = at.b;
  const float inv_bf = A.inv_b_f;
  const float inv_delta_f = A.inv_step_f;
  const float t_near_f = (float)t_near;
  double best_w = 0.0, trans = 1.0, alpha_c = 0.0, t_hit = r.t_hit;
  int samples = 0;
  // samples before i_start and from t_end on are empty: march [i_start, t_lim)
  const double t_lim = fmin(t_far, t_end);
  const float t_lim_f = (float)t_lim;
  const double t_stop = A.t_stop;
  int i = i_start;
  const int lr = at.lr;
  const double G = (double)(b * at.r);
#if defined(NOLF_STATS) && defined(NOLF_STATS_CTR)
  unsigned iters_dbg = 0;
#endif
  for (;;) {
    double pos[3];
    int cell[3], gi[3];
    const double t_mid = POW2 ? sample_grid<CLIP>(o, d, t_near, delta, i, G, lr, b, pos, gi, cell)
                              : sample_cell<CLIP>(o, d, t_near, delta, i, b, pos, cell);
    if (!(t_mid < t_lim)) break;
    NOLF_STAT(7, 1);
#if defined(NOLF_STATS) && defined(NOLF_STATS_CTR)
    ++iters_dbg;
#endif
#if defined(NOLF_STATS) && defined(NOLF_STATS_CTR)
    {
      const unsigned am = __activemask();
      if ((threadIdx.x & 31) == (unsigned)(__ffs(am) - 1)) { NOLF_STAT(9, 1); NOLF_STAT(10, __popc(am)); }
    }
#endif
    int lo_c[3], hi_c[3];
    bool empty = false;
    int cid = -1;
    const int ci = (cell[0] * b + cell[1]) * b + cell[2];
    const int dist = __ldg(at.dist + ci);
    if (dist > 0) {            // every cell within Chebyshev radius dist-1 is empty
      empty = true;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        lo_c[k] = max(cell[k] - (dist - 1), 0);
        hi_c[k] = min(cell[k] + (dist - 1), b - 1);
      }
    } else {
      cid = __ldg(at.index + ci);
    }
    if (empty) {
      NOLF_STAT(3, 1);
      // the jump target is an estimate (verified below), so it is computed
      // in fp32 relative to t_near: box faces, exit and sample index
      float te = __int_as_float(0x7f800000);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const float ok = (float)o[k];
        if (invf[k] > 0.f && hi_c[k] < b - 1) te = fminf(te, ((float)(hi_c[k] + 1) * inv_bf - ok) * invf[k]);
        else if (invf[k] < 0.f && lo_c[k] > 0) te = fminf(te, ((float)lo_c[k] * inv_bf - ok) * invf[k]);
      }
      const float jf = floorf((fminf(te, t_lim_f) - t_near_f) * inv_delta_f - 0.5f);
      int j = jf > 2.0e9f ? 2000000000 : (int)jf;
      int next = i + 1;
      for (int attempt = 0; attempt < 2 && j > i; ++attempt, --j) {
        double pj[3];
        int cj[3];
        int gj[3];
        double tj = POW2 ? sample_grid<CLIP>(o, d, t_near, delta, j, G, lr, b, pj, gj, cj)
                         : sample_cell<CLIP>(o, d, t_near, delta, j, b, pj, cj);
        bool inside = tj < t_lim;
#pragma unroll
        for (int k = 0; k < 3; ++k) inside = inside && cj[k] >= lo_c[k] && cj[k] <= hi_c[k];
        if (inside) { next = j + 1; break; }
      }
      i = next;
      continue;
    }
    // sub-voxel whose 8 corner densities are all 0: sigma = +0 exactly, so
    // absorb = exp(-0) = 1, w = 0 -- only the active-sample count changes
    int base[3];
    double frac[3];
    if (POW2) subvoxel_grid(pos, gi, cell, G, lr, at.r, base, frac);
    else atlas_subvoxel_in(at, pos, cell, base, frac);
    const int bit = POW2 ? (((base[0] << lr) + base[1]) << lr) + base[2] : (base[0] * at.r + base[1]) * at.r + base[2];
    ++samples;
    if (use_zmask && ((__ldg(at.zmask + (unsigned)(cid * at.zwords + (bit >> 5))) >> (bit & 31)) & 1u)) {
      NOLF_STAT(5, 1);
      ++i;
      continue;
    }
    float s;
    NOLF_STAT(6, 1);
    atlas_trilinear_at<1>(at, cid, base, frac, &s);
    const double sigma = (double)s;
    const double absorb = exp(__dmul_rn(-sigma, delta));
    const double w = __dmul_rn(trans, __dsub_rn(1.0, absorb));
    if (w > best_w) { best_w = w; t_hit = t_mid; }
    alpha_c = __dadd_rn(alpha_c, w);
    trans = __dmul_rn(trans, absorb);
    if (!(trans > t_stop)) break;
    ++i;
  }
#if defined(NOLF_STATS) && defined(NOLF_STATS_CTR)
  atomicMax(&g_stats[11], (unsigned long long)iters_dbg);
  atomicMax(&g_stats[12], (unsigned long long)samples);
  atomicMax(&g_stats[13], (unsigned long long)((t_lim - t_near) / delta));
#endif
  r.alpha_c = alpha_c;
  r.samples = samples;
  r.hit = alpha_c > A.alpha_floor;
  r.t_hit = r.hit ? t_hit : __longlong_as_double(0x7ff0000000000000ll);
  return r;
}

// ---------------------------------------------------------------- power-of-two grids
// The reference defaults (b = 32, r = 8) make the sub-voxel grid G = b*r a
// power of two, so the march runs in GRID UNITS: with oG = o*G and dG = d*G
// (exact: scaling by a power of two), every sample position
//   xg = clip(fl(oG + fl(t_mid * dG)), 0, G) == clip(fl(o + fl(t_mid * d)), 0, 1) * G
// bit for bit (rounding commutes with power-of-two scaling; no sub-normals or
// overflow at these magnitudes).  Then
//   gi   = floor(xg)            = low word of fl_rd(xg + 2^52)   (0 <= xg < 2^52)
//   cell = min(gi >> lr, b - 1) , base = gi - (cell << lr), frac = xg - floor(xg)
// except at xg == G (pos == 1.0: cell b-1, base r-1, frac 1.0), which is
// exactly atlas.py:162-172's floor / clip / subtract sequence without a single
// fp64 <-> int conversion.  t_mid = t_near + (i + 0.5) * step with (i + 0.5)
// carried as a double (exact for i < 2^52).
__device__ __forceinline__ int floor_grid(double xg) {    // 0 <= xg < 2^52
  return __double2loint(__dadd_rd(xg, 4503599627370496.0));
}
__device__ __forceinline__ double frac_grid(double xg) {  // xg - floor(xg), exact
  return __dsub_rn(xg, __dsub_rn(__dadd_rd(xg, 4503599627370496.0), 4503599627370496.0));
}

template <bool CLIP>
__device__ __forceinline__ double grid_pos(const double oG[3], const double dG[3], double t_mid, double G, int k) {
  const double v = __dadd_rn(oG[k], __dmul_rn(t_mid, dG[k]));
  return CLIP ? (v < 0.0 ? 0.0 : (v > G ? G : v)) : v;
}

template <bool CLIP>
__device__ __forceinline__ MarchOut march_p2(const DevAsset &A, const double oG[3], const double dG[3],
                                             const float invG[3], double t_near, double t_far, bool use_zmask,
                                             int i_start, double t_end) {
  MarchOut r;
  r.alpha_c = 0.0;
  r.t_hit = __longlong_as_double(0x7ff0000000000000ll);
  r.samples = 0;
  r.hit = false;
  if (!(t_near < t_far)) return r;
  const DevAtlas &at = A.den;
  const double delta = A.step;
  const int b = at.b, lr = at.lr;
  const int Gi = b << lr;
  const double G = (double)Gi;
  const double t_lim = fmin(t_far, t_end);
  double best_w = 0.0, trans = 1.0, alpha_c = 0.0, t_hit = r.t_hit;
  int samples = 0;
  int i = i_start;
  double ti = (double)i_start + 0.5;          // i + 0.5, exact
#ifdef NOLF_CHEB_DIST
  const uint8_t *dfield = at.dist;           // symmetric (Chebyshev) empty boxes
#else
  // empty cubes anchored at the cell in the ray's direction of travel: the
  // samples between here and the box exit only move forward, so they stay
  // inside it (no room is spent behind the ray)
  const int oct = (dG[0] < 0.0 ? 1 : 0) | (dG[1] < 0.0 ? 2 : 0) | (dG[2] < 0.0 ? 4 : 0);
  const uint8_t *dfield = at.odist + (size_t)oct * (size_t)(b * b * b);
#endif
#ifdef NOLF_STATS
  unsigned iters_cta = 0;
#endif
  for (;;) {
    NOLF_ITER(++iters_cta);
    const double t_mid = __dadd_rn(t_near, __dmul_rn(ti, delta));
    if (!(t_mid < t_lim)) break;
    NOLF_STAT(7, 1);
#if defined(NOLF_STATS) && defined(NOLF_STATS_CTR)
    {
      const unsigned am = __activemask();
      if ((threadIdx.x & 31) == (unsigned)(__ffs(am) - 1)) { NOLF_STAT(9, 1); NOLF_STAT(10, __popc(am)); }
    }
#endif
    int gi[3], cell[3];
#ifdef NOLF_KEEP_XG
    double xg[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      xg[k] = grid_pos<CLIP>(oG, dG, t_mid, G, k);
      gi[k] = floor_grid(xg[k]);
      cell[k] = min(gi[k] >> lr, b - 1);
    }
#else
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      gi[k] = floor_grid(grid_pos<CLIP>(oG, dG, t_mid, G, k));
      cell[k] = min(gi[k] >> lr, b - 1);
    }
#endif
    const int ci = (cell[0] * b + cell[1]) * b + cell[2];
    const int dist = __ldg(dfield + ci);
    if (dist > 0) {            // every cell of the empty box around / ahead of this one: jump (verified)
      NOLF_STAT(3, 1);
      int lo_c[3], hi_c[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
#ifdef NOLF_CHEB_DIST
        lo_c[k] = max(cell[k] - (dist - 1), 0);
        hi_c[k] = min(cell[k] + (dist - 1), b - 1);
#else
        const bool neg = (oct >> k) & 1;
        lo_c[k] = neg ? max(cell[k] - (dist - 1), 0) : cell[k];
        hi_c[k] = neg ? cell[k] : min(cell[k] + (dist - 1), b - 1);
#endif
      }
      // fp32 estimate of the last sample before the empty box's exit
      float te = __int_as_float(0x7f800000);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const float ok = (float)oG[k];
#ifdef NOLF_INVG_REG
        const float ig = invG[k];
#else
        // an estimate only (the jump is verified): 1/dG from the MUFU instead
        // of three floats held across the whole march
        float ig;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(ig) : "f"((float)dG[k]));
#endif
        if (ig > 0.f && hi_c[k] < b - 1) te = fminf(te, ((float)((hi_c[k] + 1) << lr) - ok) * ig);
        else if (ig < 0.f && lo_c[k] > 0) te = fminf(te, ((float)(lo_c[k] << lr) - ok) * ig);
      }
      const float jf = floorf((fminf(te, (float)t_lim) - (float)t_near) * A.inv_step_f - 0.5f);
      int j = jf > 2.0e9f ? 2000000000 : (int)jf;
      int next = i + 1;
      for (int attempt = 0; attempt < 2 && j > i; ++attempt, --j) {
        const double tj = __dadd_rn(t_near, __dmul_rn((double)j + 0.5, delta));
        bool inside = tj < t_lim;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const int cj = min(floor_grid(grid_pos<CLIP>(oG, dG, tj, G, k)) >> lr, b - 1);
          inside = inside && cj >= lo_c[k] && cj <= hi_c[k];
        }
        if (inside) { next = j + 1; break; }
      }
      ti = next == i + 1 ? ti + 1.0 : (double)next + 0.5;
      i = next;
      continue;
    }
    const int cid = __ldg(at.index + ci);
    int base[3];
    double frac[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      base[k] = gi[k] - (cell[k] << lr);
#ifdef NOLF_KEEP_XG
      frac[k] = frac_grid(xg[k]);
#else
      // the position again (cheaper than keeping three doubles live across
      // the distance-field load: they were spilled every iteration); the
      // volatile asm keeps the compiler from merging it with the first one
      double v;
      asm volatile("{\n\t.reg .f64 m;\n\tmul.rn.f64 m, %1, %2;\n\tadd.rn.f64 %0, %3, m;\n\t}"
                   : "=d"(v) : "d"(t_mid), "d"(dG[k]), "d"(oG[k]));
      if (CLIP) v = v < 0.0 ? 0.0 : (v > G ? G : v);
      frac[k] = frac_grid(v);
#endif
      if (gi[k] >= Gi) { base[k] = (1 << lr) - 1; frac[k] = 1.0; }   // pos == 1.0 (clipped to the far face)
    }
    ++samples;
    const int bit = (((base[0] << lr) + base[1]) << lr) + base[2];
    // sub-voxel whose 8 corner densities are all 0: sigma = +0 exactly, so
    // absorb = exp(-0) = 1, w = 0 -- only the active-sample count changes
    // (every uploaded atlas has its zero mask: use_zmask only matters for the general-grid march)
    if (!((__ldg(at.zmask + (unsigned)(cid * at.zwords + (bit >> 5))) >> (bit & 31)) & 1u)) {
      NOLF_STAT(6, 1);
      float s;
      atlas_trilinear_at<1>(at, cid, base, frac, &s);
      const double sigma = (double)s;
      const double absorb = exp(__dmul_rn(-sigma, delta));
      const double w = __dmul_rn(trans, __dsub_rn(1.0, absorb));
      if (w > best_w) { best_w = w; t_hit = t_mid; }
      alpha_c = __dadd_rn(alpha_c, w);
      trans = __dmul_rn(trans, absorb);
      if (!(trans > t_stop_of(A))) break;
    }
    ++i;
    ti += 1.0;
  }
#ifdef NOLF_STATS
  atomicMax(&g_cta_work[blockIdx.x & ((1 << 20) - 1)][1], iters_cta);
  r.iters = iters_cta;
#endif
  r.alpha_c = alpha_c;
  r.samples = samples;
  r.hit = alpha_c > A.alpha_floor;
  r.t_hit = r.hit ? t_hit : __longlong_as_double(0x7ff0000000000000ll);
  return r;
}

#ifndef NOLF_MARCH_MINB
#define NOLF_MARCH_MINB 8  // latency-bound: 50% occupancy beats the spills it costs (measured 4..8)
#endif

#ifdef NOLF_STATS
__device__ __forceinline__ void stat_cta_start() {
  if (threadIdx.x == 0 && blockIdx.x < (1u << 20)) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    g_cta_start[blockIdx.x] = now;
  }
}
__device__ __forceinline__ void stat_cta_end() {   // global ns timer at the last warp's end
  unsigned long long now;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
  if ((threadIdx.x & 31) == 0 && blockIdx.x < (1u << 20)) atomicMax(&g_cta_end[blockIdx.x], now);
}
#else
__device__ __forceinline__ void stat_cta_start() {}
__device__ __forceinline__ void stat_cta_end() {}
#endif

constexpr int kMarchThreads = 128;   // k_march CTA size (launch uses the same)

// CTA-level pre-cull (scene mode): all of the CTA's slots lie in one tile;
// when no instance's screen box meets the tile every pixel is a miss.  Returns
// true when the CTA is done (nhit = 0 written).
__device__ __forceinline__ bool cta_precull(const MarchArgs &args, long long gid) {
  if (!args.cull || args.tile_stride % kMarchThreads != 0) return false;
  long long t, local0;
  split_slot((long long)blockIdx.x * kMarchThreads, args.tile_stride, t, local0);
  const TileParams tp = args.tiles[t];
  bool meets = false;
  for (int k = threadIdx.x; k < args.n_inst; k += kMarchThreads) {
    const ScreenBox bb = args.cull[k * args.n_cams + tp.cam];
    meets = meets || (bb.x0 <= bb.x1 && bb.x0 < tp.x1 && bb.x1 >= tp.x0 && bb.y0 < tp.y1 && bb.y1 >= tp.y0);
  }
  if (__syncthreads_or(meets)) return false;
  if (gid < args.n_rays) args.nhit[gid] = 0;
  return true;
}

// Pixel (and camera) of ray slot gid; false for tile padding.
template <int MODE>
__device__ __forceinline__ bool slot_pixel(const MarchArgs &args, long long gid, int &pix_x, int &pix_y, int &cam) {
  long long t = 0, local = gid;
  if (MODE != kModeRect) split_slot(gid, args.tile_stride, t, local);
  const TileParams tp = args.tiles[t];
  if (MODE == kModeScene && !tile_valid(tp, args.cams, args.n_cams, args.tile_stride)) {
    if (local == 0) atomicAdd(args.errors + kErrTile, 1u);
    return false;
  }
  const int w = tp.x1 - tp.x0, h = tp.y1 - tp.y0;
  if (local >= (long long)w * h) return false;
  cam = tp.cam;
  if (MODE == kModeScene) {
    slot_xy(local, w, h, pix_x, pix_y);
    pix_x += tp.x0;
    pix_y += tp.y0;
  } else {
    pix_x = tp.x0 + (int)(local % w);
    pix_y = tp.y0 + (int)(local / w);
  }
  return true;
}

// Instances whose conservative screen box covers this lane's pixel (all
// instances without culling).  Warp-collective.
// Instances g0 .. g0+63 (bit k - g0).
template <int MODE>
__device__ __forceinline__ unsigned long long candidate_mask(const MarchArgs &args, bool valid, int pix_x, int pix_y,
                                                             int cam, unsigned lane, int g0) {
  unsigned long long lane_mask = 0;
  const int g1 = min(args.n_inst, g0 + 64);
  if (MODE == kModeRays || !args.cull) {
    if (valid) lane_mask = g1 - g0 >= 64 ? ~0ull : ((1ull << (g1 - g0)) - 1ull);
    return lane_mask;
  }
  const int cmin = __reduce_min_sync(0xffffffffu, valid ? cam : INT_MAX);
  const int cmax = __reduce_max_sync(0xffffffffu, valid ? cam : -1);
  if (cmin == cmax) {
    // one camera for the whole warp: lane k tests instance k's box against
    // the warp's pixel rectangle, then only the candidates are tested per pixel
    const int xmin = __reduce_min_sync(0xffffffffu, valid ? pix_x : INT_MAX);
    const int xmax = __reduce_max_sync(0xffffffffu, valid ? pix_x : INT_MIN);
    const int ymin = __reduce_min_sync(0xffffffffu, valid ? pix_y : INT_MAX);
    const int ymax = __reduce_max_sync(0xffffffffu, valid ? pix_y : INT_MIN);
    for (int base = g0; base < g1; base += 32) {
      const int k = base + (int)lane;
      ScreenBox bb{1, 1, 0, 0};
      if (k < g1) bb = args.cull[k * args.n_cams + cmin];
      unsigned cand = __ballot_sync(0xffffffffu, bb.x0 <= xmax && bb.x1 >= xmin && bb.y0 <= ymax && bb.y1 >= ymin &&
                                                     bb.x0 <= bb.x1);
      while (cand) {
        const int j = __ffs(cand) - 1;
        cand &= cand - 1;
        const int x0 = __shfl_sync(0xffffffffu, bb.x0, j), x1 = __shfl_sync(0xffffffffu, bb.x1, j);
        const int y0 = __shfl_sync(0xffffffffu, bb.y0, j), y1 = __shfl_sync(0xffffffffu, bb.y1, j);
        if (valid && pix_x >= x0 && pix_x <= x1 && pix_y >= y0 && pix_y <= y1) lane_mask |= 1ull << (base - g0 + j);
      }
    }
  } else if (valid) {
    for (int k = g0; k < g1; ++k) {
      const ScreenBox bb = args.cull[k * args.n_cams + cam];
      if (pix_x >= bb.x0 && pix_x <= bb.x1 && pix_y >= bb.y0 && pix_y <= bb.y1) lane_mask |= 1ull << (k - g0);
    }
  }
  return lane_mask;
}

// World ray of a slot: camera ray (core.py:162-170) or the caller's ray.
template <int MODE>
__device__ __forceinline__ void world_ray(const MarchArgs &args, long long gid, int cam, int pix_x, int pix_y,
                                          double ow[3], double dw[3]) {
  if (MODE == kModeRays) {
    const double *op = args.origins + (args.origin_stride ? 3 * gid : 0);
    ow[0] = op[0]; ow[1] = op[1]; ow[2] = op[2];
    dw[0] = args.dirs[3 * gid]; dw[1] = args.dirs[3 * gid + 1]; dw[2] = args.dirs[3 * gid + 2];
  } else {
    const CamParams &cp = args.cams[cam];
    camera_dir(cp.pose, cp.fx, cp.fy, cp.cx, cp.cy, (double)pix_x, (double)pix_y, dw);
    ow[0] = cp.pose[3]; ow[1] = cp.pose[7]; ow[2] = cp.pose[11];
  }
}

// Everything march_rays does before its first sample (lightfield.py:129-150):
// object-space ray, proxy entry/exit (box slab or mesh first hit), then the
// exact clip of the sample range to the grown occupied-cell box.  False:
// the ray never samples an occupied cell (exact miss, no samples).
struct MarchSpan {
  double t_near, t_far, t_end;
  int i_start;
  bool noclip;
};

// (1) per lane: object-space ray and proxy-box slab
__device__ __forceinline__ bool prepare_slab(const DevInst &I, const DevAsset &A, bool raw_rays, const double ow[3],
                                             const double dw[3], double o[3], double d[3], double inv[3],
                                             MarchSpan &sp) {
  if (raw_rays) {
#pragma unroll
    for (int q = 0; q < 3; ++q) { o[q] = ow[q]; d[q] = dw[q]; }
  } else {
    to_object(I.w2o, ow, dw, o, d);
  }
  sp.t_near = 0.0;
  sp.t_far = 0.0;
  sp.i_start = 0;
  sp.noclip = false;
  return slab(A.pmin, A.pmax, o, d, sp.t_near, sp.t_far, inv);
}

// (2) per lane, after the (warp-cooperative) mesh first hit
__device__ __forceinline__ bool prepare_clip(const DevAsset &A, const double o[3], const double d[3],
                                             const double inv[3], MarchSpan &sp) {
  bool boxhit = true;
  sp.t_end = sp.t_far;
  NOLF_STAT(1, 1);
  // Clip the march to the ray's span in the culling box (occupied cells
  // grown by one cell): every sample outside it lies in an empty cell, so
  // starting 2 samples before the entry and stopping 2 after the exit
  // leaves the result bit-identical (empty samples change nothing).
  if (sp.t_near < sp.t_far) {
    double ca, cb;
    double inv_c[3] = {inv[0], inv[1], inv[2]};
    if (!slab<true>(A.cull_lo, A.cull_hi, o, d, ca, cb, inv_c) || A.cull_empty) {
      boxhit = false;                     // never meets an occupied cell: exact miss
    } else {
      const double f = floor((ca - sp.t_near) * A.inv_step - 2.5);   // 2-sample margins absorb the rounding
      sp.i_start = f > 0.0 ? (f < 2.0e9 ? (int)f : 2000000000) : 0;
      sp.t_end = cb + 2.0 * A.step;
    }
  }
  if (boxhit) {
    // every sample the march can visit has index in [i_start, i_hi]
    const double lim = fmin(sp.t_far, sp.t_end);
    const double hf = floor((lim - sp.t_near) * A.inv_step) + 2.0;
    sp.noclip = sp.t_near < lim && hf < 2.0e9 && samples_inside_unit(o, d, sp.t_near, A.step, sp.i_start, (int)hf);
  }
  return boxhit;
}

// o, d: the object-space ray; power-of-two grids march in grid units, so
// there o and d arrive already scaled by G (prepare_for_march) and invf is
// 1/(d*G) -- see march_p2.
__device__ __forceinline__ MarchOut run_march(const DevAsset &A, const double o[3], const double d[3],
                                              const float invf[3], const MarchSpan &sp, bool use_zmask) {
  if (A.den.lr >= 0) {
    if (sp.noclip) return march_p2<false>(A, o, d, invf, sp.t_near, sp.t_far, use_zmask, sp.i_start, sp.t_end);
    return march_p2<true>(A, o, d, invf, sp.t_near, sp.t_far, use_zmask, sp.i_start, sp.t_end);
  }
  if (sp.noclip) return march_ray<false, false>(A, o, d, invf, sp.t_near, sp.t_far, use_zmask, sp.i_start, sp.t_end);
  return march_ray<true, false>(A, o, d, invf, sp.t_near, sp.t_far, use_zmask, sp.i_start, sp.t_end);
}

// Grid units for power-of-two atlases (exact scaling, see march_p2): o, d and
// 1/d are multiplied / divided by G in place; returns the factor that maps
// positions back to object space (1/G, or 1 for the general path).
__device__ __forceinline__ double to_grid_units(const DevAsset &A, double o[3], double d[3], float invf[3]) {
  if (A.den.lr < 0) return 1.0;
  const double G = (double)(A.den.b << A.den.lr);
  const float igf = 1.0f / (float)G;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    o[k] = __dmul_rn(o[k], G);
    d[k] = __dmul_rn(d[k], G);
    invf[k] *= igf;
  }
  return 1.0 / G;
}

// Hit record for the shading pass (lightfield.py:433-445).  o, d in units
// scaled by 1/unit (to_grid_units): positions and the direction are mapped
// back exactly (power-of-two factors).
__device__ __forceinline__ HitRec hit_record(const DevAsset &A, const double o[3], const double d[3], double unit,
                                             double t_near, const MarchOut &mr, uint32_t out_idx, uint32_t ordinal) {
  HitRec rec;
  double t_obj = mr.t_hit;
  if (!A.use_hit_point) t_obj = t_near;   // ablation: shade at the proxy entry (lightfield.py:438-445)
#pragma unroll
  for (int q = 0; q < 3; ++q) rec.p[q] = clamp01(__dmul_rn(__dadd_rn(o[q], __dmul_rn(t_obj, d[q])), unit));
  rec.alpha_c = mr.alpha_c;
  rec.t_obj = t_obj;
  rec.d[0] = __dmul_rn(d[0], unit); rec.d[1] = __dmul_rn(d[1], unit); rec.d[2] = __dmul_rn(d[2], unit);
  rec.out_idx = out_idx;
  rec.ordinal = ordinal;
  return rec;
}

// One thread per ray, every candidate instance marched in scene order by
// that thread (kModeRays / kModeRect, and the march_rays entry point).
// GROUPS: more than 64 instances (candidate masks per group of 64); the
// common case compiles without the group loop.
template <int MODE, bool GROUPS = false>
__device__ __forceinline__ void march_chunk(const MarchArgs &args, unsigned chunk, bool precull, int sub = 0) {
  const long long gid = (long long)chunk * kMarchThreads + (long long)sub * blockDim.x + threadIdx.x;
  const unsigned lane = threadIdx.x & 31;
  if (MODE == kModeScene && precull && cta_precull(args, gid)) return;
  bool valid = gid < args.n_rays;
  int pix_x = 0, pix_y = 0, cam = 0;
  if (valid) {
    if (MODE != kModeRays) valid = slot_pixel<MODE>(args, gid, pix_x, pix_y, cam);
    if (MODE != kModeScene && valid && args.rgba) {   // miss defaults (lightfield.py:415-416)
      reinterpret_cast<float4 *>(args.rgba)[gid] = make_float4(0.f, 0.f, 0.f, 0.f);
      args.depth[gid] = __int_as_float(0x7f800000);
    }
  }
  unsigned samples_total = 0;  // per lane (< 2^32: at most n_inst * samples per ray)
  unsigned ordinal = 0;
#ifdef NOLF_STATS
  unsigned st_iters = 0, st_inst = 0, st_pass = 0;
#endif
  // candidates OR-ed over the warp so the instance loop below is
  // warp-uniform (ascending = scene order, so layer ordinals match); in
  // groups of 64 instances
  for (int g0 = 0; g0 < (GROUPS ? args.n_inst : 1); g0 += 64) {
  const unsigned long long lane_mask = candidate_mask<MODE>(args, valid, pix_x, pix_y, cam, lane, g0);
  unsigned long long wmask = ((unsigned long long)__reduce_or_sync(0xffffffffu, (unsigned)(lane_mask >> 32)) << 32) |
                             __reduce_or_sync(0xffffffffu, (unsigned)lane_mask);
  while (wmask) {
    const int kb = __ffsll((long long)wmask) - 1;
    const int k = g0 + kb;
    wmask &= wmask - 1;
    const DevInst &I = args.inst[k];
    const DevAsset &A = *I.a;
    bool hit = false;
    double o[3], d[3], inv[3];
    double unit = 1.0;
    MarchSpan sp{0.0, 0.0, 0.0, 0, false};
    MarchOut mr{0.0, __longlong_as_double(0x7ff0000000000000ll), 0, false};
    const bool live = (lane_mask >> kb) & 1ull;
    if (lane == 0) NOLF_STAT(8, 1);
    NOLF_ITER(++st_pass);
    bool boxhit = false;
    if (live) {
      NOLF_STAT(0, 1);
      double ow[3], dw[3];     // rebuilt per candidate instead of held across the march
      world_ray<MODE>(args, gid, cam, pix_x, pix_y, ow, dw);
      boxhit = prepare_slab(I, A, args.raw_rays, ow, dw, o, d, inv, sp);
    }
    if (A.mesh.nodes) {        // mesh proxy (warp-uniform: k is): march from its first hit
#if defined(NOLF_MESH_TIMING_ONLY)   // diagnostic (wrong results): the march from the slab entry
      const double tm = sp.t_near;
#elif defined(NOLF_MESH_PER_THREAD)
      const double tm = boxhit ? mesh_first_hit(A.mesh, o, d, args.errors + kErrBvh) : -1.0;
#elif defined(NOLF_MESH_BINARY)
      const double tm = mesh_first_hit_warp(A.mesh, o, d, boxhit, args.errors + kErrBvh);
#else
      const double tm = mesh_first_hit_warp4(A.mesh, o, d, boxhit, args.errors + kErrBvh);
#endif
      if (boxhit) {
        if (tm < 0.0) boxhit = false;
        else sp.t_near = tm;
      }
    }
    if (boxhit && prepare_clip(A, o, d, inv, sp)) {
      NOLF_STAT(2, 1);
      float invf[3] = {(float)inv[0], (float)inv[1], (float)inv[2]};
      unit = to_grid_units(A, o, d, invf);
      mr = run_march(A, o, d, invf, sp, args.use_zmask);
      samples_total += (unsigned)mr.samples;
#ifdef NOLF_STATS
      st_iters += mr.iters;
      ++st_inst;
#endif
      hit = mr.hit;
    }
    if (args.out_hit) {        // march_rays outputs (MarchResult, lightfield.py:101-110)
      if (live) {
        args.out_hit[gid] = hit ? 1 : 0;
        args.out_t_hit[gid] = mr.t_hit;
        args.out_alpha_c[gid] = mr.alpha_c;
        args.out_samples[gid] = mr.samples;
#pragma unroll
        for (int q = 0; q < 3; ++q)
          args.out_p_h[3 * gid + q] = hit ? clamp01(__dmul_rn(__dadd_rn(o[q], __dmul_rn(mr.t_hit, d[q])), unit)) : 0.0;
      }
      continue;
    }
    // a pixel never has more hits than compose layers (the host bounds the
    // layers by the screen-box overlap); a violation is counted and dropped
    if (MODE == kModeScene && hit && (int)ordinal >= args.max_layers) {
      atomicAdd(args.errors + kErrLayers, 1u);
      hit = false;
    }
    // warp-aggregated queue append (one atomic per warp per instance)
    const unsigned ballot = __ballot_sync(0xffffffffu, hit);
    if (ballot) {
      unsigned base = 0;
      if (lane == __ffs(ballot) - 1) base = atomicAdd(args.counts + k, (unsigned)__popc(ballot));
      base = __shfl_sync(0xffffffffu, base, __ffs(ballot) - 1);
      if (hit) {
        const unsigned pos = base + __popc(ballot & ((1u << lane) - 1u));
        if ((long long)pos < args.qoff[k + 1] - args.qoff[k]) {
          args.queue[args.qoff[k] + pos] = hit_record(A, o, d, unit, sp.t_near, mr, (uint32_t)gid, ordinal);
          ++ordinal;           // the layer exists only if its record does
        } else {
          atomicAdd(args.errors + kErrQueue, 1u);
        }
      }
    }
  }
  }  // instance groups
  if (MODE == kModeScene && valid) args.nhit[gid] = (uint8_t)ordinal;
#ifdef NOLF_STATS
  {
    unsigned *w = g_cta_work[blockIdx.x & ((1 << 20) - 1)];
    if (lane == 0) atomicAdd(w + 0, st_pass);
    atomicMax(w + 2, st_iters);
    atomicMax(w + 3, st_inst);
  }
#endif
  // march_samples counter (lightfield.py:430-431)
  const unsigned warp_samples = __reduce_add_sync(0xffffffffu, samples_total);
  if (lane == 0 && warp_samples && args.counters) atomicAdd(args.counters + 3, (unsigned long long)warp_samples);
}

// One CTA per 128 slots (rays / rect mode, and scene tiles that are not
// 128-slot aligned: those pre-cull per CTA).
template <int MODE, bool GROUPS = false>
__global__ void __launch_bounds__(kMarchThreads, NOLF_MARCH_MINB) k_march(MarchArgs args) {
  stat_cta_start();
  march_chunk<MODE, GROUPS>(args, blockIdx.x, true);
  stat_cta_end();
}

// Scene chunks (128 slots of one tile) that some instance's screen box
// meets, compacted into a work list; every other chunk is a miss and is
// never launched (k_compose reads chunk_live instead of its layer counts).
__global__ void __launch_bounds__(128) k_cull_chunks(MarchArgs args, long long n_chunks, uint8_t *chunk_live,
                                                     unsigned *list, unsigned *count) {
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  bool live = false;
  int ncand = 0;
  // the previous frame's duration of this chunk: when known it is the bucket,
  // and any one candidate instance makes the chunk live
  const unsigned prev_cost = (c < n_chunks && args.chunk_cost) ? args.chunk_cost[c] : 0u;
  const bool count_all = args.heavy_first && !prev_cost;
  if (c < n_chunks) {
    long long t, local0;
    split_slot(c * kMarchThreads, args.tile_stride, t, local0);
    const TileParams tp = args.tiles[t];
    const int w = tp.x1 - tp.x0, h = tp.y1 - tp.y0;
    const bool tv = tile_valid(tp, args.cams, args.n_cams, args.tile_stride);
    if (!tv && local0 == 0) atomicAdd(args.errors + kErrTile, 1u);
    if (tv && local0 < (long long)w * h) {
      // pixel rectangle of the chunk's valid slots: the bbox of the slot
      // positions at every 8x4-block start/end (row-major tiles: the rows)
      const long long l1 = min(local0 + kMarchThreads, (long long)w * h) - 1;
      int xa = INT_MAX, xb = INT_MIN, ya = INT_MAX, yb = INT_MIN;
      const int nb = w >> 3;                    // 8x4 blocks per block row
      const long long blk0 = local0 >> 5;
      if ((w & 7) == 0 && (h & 3) == 0 && l1 == local0 + kMarchThreads - 1 && (blk0 % nb) + 3 < nb) {
        // 4 whole blocks in one block row (32-wide tiles: every chunk)
        xa = (int)(blk0 % nb) * 8;
        xb = xa + 31;
        ya = (int)(blk0 / nb) * 4;
        yb = ya + 3;
      } else
      for (long long l = local0; l <= l1; l += 32) {
        int x, y;
        slot_xy(min(l, l1), w, h, x, y);
        xa = min(xa, x); xb = max(xb, x); ya = min(ya, y); yb = max(yb, y);
        slot_xy(min((l | 31), l1), w, h, x, y);
        xa = min(xa, x); xb = max(xb, x); ya = min(ya, y); yb = max(yb, y);
      }
      if (yb > ya && !((w & 7) == 0 && (h & 3) == 0)) { xa = 0; xb = w - 1; }   // row-major: rows span the width
      xa += tp.x0; xb += tp.x0; ya += tp.y0; yb += tp.y0;
      for (int k = 0; k < args.n_inst; ++k) {   // count them only when the buckets are used
        const ScreenBox bb = args.cull[k * args.n_cams + tp.cam];
        ncand += (bb.x0 <= bb.x1 && bb.x0 <= xb && bb.x1 >= xa && bb.y0 <= yb && bb.y1 >= ya) ? 1 : 0;
        if (ncand && !count_all) break;
      }
      live = ncand > 0;
    }
    chunk_live[c] = live ? 1 : 0;
  }
  const unsigned lane = threadIdx.x & 31;
  const unsigned ballot = __ballot_sync(0xffffffffu, live);
  if (ballot) {
    unsigned sbase = 0;        // spatial list (region 0) and the total
    if (lane == __ffs(ballot) - 1) sbase = atomicAdd(count, (unsigned)__popc(ballot));
    sbase = __shfl_sync(0xffffffffu, sbase, __ffs(ballot) - 1);
    if (live) list[sbase + __popc(ballot & ((1u << lane) - 1u))] = (unsigned)c;
    if (live && args.heavy_first) {   // and this chunk's bucket (regions 1..): heaviest last frame first
      int b = min(ncand, kChunkBuckets - 1);
      if (args.chunk_cost) {
        const unsigned cyc = prev_cost;
        // CTA duration classes (0: never marched -> candidate count): octaves
        // [2^12, 2^13) -> 1 ... with 8 buckets, half octaves from 2^12 with 16
        if (cyc) {
          const int msb = 31 - __clz((int)min(cyc, 0x7fffffffu));
          const int cls = kChunkBuckets >= 16 ? 2 * msb + (int)((cyc >> max(msb - 1, 0)) & 1u) - 23 : msb - 11;
          b = min(max(cls, 1), kChunkBuckets - 1);
        }
      }
      const unsigned peers = __match_any_sync(ballot, b);
      const int leader = __ffs(peers) - 1;
      unsigned base = 0;
      if ((int)lane == leader) base = atomicAdd(count + 2 + b, (unsigned)__popc(peers));
      base = __shfl_sync(peers, base, leader);
      list[(long long)b * n_chunks + base + __popc(peers & ((1u << lane) - 1u))] = (unsigned)c;
    }
  }
  if (prev_cost) args.chunk_cost[c] = 0u;   // this frame's marcher records afresh
}

// Scene marcher over the compacted live chunks: one CTA per list entry.  The
// host sizes the grid from the live count of an earlier frame (read back
// asynchronously, never waited for) plus headroom; a grid-stride loop keeps
// any size correct, and CTAs past the list exit after one load.
template <bool GROUPS = false>
__global__ void __launch_bounds__(kMarchThreads, NOLF_MARCH_MINB) k_march_chunks(MarchArgs args) {
  const unsigned n = *args.n_chunks;
  stat_cta_start();
  for (unsigned it = blockIdx.x; it < n; it += gridDim.x) {  // normally one pass: the grid is sized
    const long long t0 = clock64();
    const unsigned chunk = chunk_at(args.chunks, args.n_chunks, args.list_stride, it, args.heavy_first);
    march_chunk<kModeScene, GROUPS>(args, chunk, false);
    if (args.chunk_cost && (threadIdx.x & 31) == 0)         // the CTA's duration = its slowest warp's
      atomicMax(args.chunk_cost + chunk, (unsigned)min(clock64() - t0, 0x7fffffffll) | 1u);
  }
  stat_cta_end();
}

// Each live chunk marched by two 64-thread CTAs (half the work per CTA: a
// shorter tail for launches of few waves -- multi-GPU shards).
template <bool GROUPS = false>
__global__ void __launch_bounds__(kMarchThreads / 2, 2 * NOLF_MARCH_MINB) k_march_chunks_half(MarchArgs args) {
  const unsigned n = *args.n_chunks;
  for (unsigned it = blockIdx.x; it < 2 * n; it += gridDim.x) {
    const long long t0 = clock64();
    const unsigned chunk = chunk_at(args.chunks, args.n_chunks, args.list_stride, it >> 1, args.heavy_first);
    march_chunk<kModeScene, GROUPS>(args, chunk, false, (int)(it & 1));
    if (args.chunk_cost && (threadIdx.x & 31) == 0)         // the chunk's duration = its slowest half's
      atomicMax(args.chunk_cost + chunk, (unsigned)min(clock64() - t0, 0x7fffffffll) | 1u);
  }
}

// ---------------------------------------------------------------- shading
struct ShadeArgs {
  const DevInst *inst;
  int n_inst;
  const HitRec *queue;
  const long long *qoff;
  const unsigned int *counts;
  int mode;                    // RayMode
  float *rgba;                 // rays/rect: (n,4); scene: layers (L, P, 4)
  float *depth;                // rays/rect: (n,);  scene: layers (L, P)
  long long layer_stride;      // scene: P
  int tile_order;              // 0 round-robin tiles over CTAs, 1 blocked ranges
  unsigned long long *counters;
  uint32_t *dbg_slots;         // debug (nolf_debug_psh_slots): 8 PSH slots per output row, or NULL
  long long dbg_rows;          // rows dbg_slots holds
  uint32_t tab_bytes;          // bf16 shader: largest staged residue table of the launch's assets
};

constexpr int kShadeThreads = 128;

// Fully fused MLP forward for one row (neural.py:89-108), fp32 with
// sequential FMA accumulation.  Layer 0 is computed input-major from a
// per-thread input column in shared memory so every weight read is a
// warp-uniform broadcast; layers 1 and 2 are fused output-by-output so only
// one hidden vector lives in registers.
__device__ __forceinline__ void mlp_row(const float *__restrict__ P, int n_layers, int in, const int act[4],
                                        const float *xcol, float out[4]) {
  float h[kHid];
#pragma unroll
  for (int o = 0; o < kHid; ++o) h[o] = 0.f;
  for (int i = 0; i < in; ++i) {
    const float xi = xcol[i * kShadeThreads];
    const float4 *wr = reinterpret_cast<const float4 *>(P + MlpOff::w0t + i * kHid);
#pragma unroll
    for (int q = 0; q < kHid / 4; ++q) {
      const float4 wv = wr[q];
      h[4 * q + 0] = fmaf(xi, wv.x, h[4 * q + 0]);
      h[4 * q + 1] = fmaf(xi, wv.y, h[4 * q + 1]);
      h[4 * q + 2] = fmaf(xi, wv.z, h[4 * q + 2]);
      h[4 * q + 3] = fmaf(xi, wv.w, h[4 * q + 3]);
    }
  }
#pragma unroll
  for (int o = 0; o < kHid; ++o) {
    const float z = h[o] + P[MlpOff::b0 + o];
    h[o] = z > 0.f ? z : 0.f;
  }
  float acc4[4] = {0.f, 0.f, 0.f, 0.f};
  if (n_layers == 3) {
    for (int o = 0; o < kHid; ++o) {
      const float4 *wr = reinterpret_cast<const float4 *>(P + MlpOff::w1 + o * kHid);
      float acc = 0.f;
#pragma unroll
      for (int q = 0; q < kHid / 4; ++q) {
        const float4 wv = wr[q];
        acc = fmaf(h[4 * q + 0], wv.x, acc);
        acc = fmaf(h[4 * q + 1], wv.y, acc);
        acc = fmaf(h[4 * q + 2], wv.z, acc);
        acc = fmaf(h[4 * q + 3], wv.w, acc);
      }
      float z = acc + P[MlpOff::b1 + o];
      z = z > 0.f ? z : 0.f;
      // last layer accumulates this hidden unit (index o) into all 4 outputs
      // -- sequential in o, matching a row-major dot product
#pragma unroll
      for (int j = 0; j < 4; ++j) acc4[j] = fmaf(z, P[MlpOff::wl + j * kHid + o], acc4[j]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float acc = 0.f;
#pragma unroll
      for (int o = 0; o < kHid; ++o) acc = fmaf(h[o], P[MlpOff::wl + j * kHid + o], acc);
      acc4[j] = acc;
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float z = acc4[j] + P[MlpOff::bl + j];
    out[j] = act[j] == 0 ? z : (act[j] == 1 ? sigmoidf_np(z) : expf(z));
  }
}

__device__ __forceinline__ int hashgrid_encode_col(const DevAsset &A, const double p[3], float *xcol);

__global__ void __launch_bounds__(kShadeThreads) k_shade(ShadeArgs args) {
  extern __shared__ __align__(16) float smem[];
  float *s_fs = smem;                               // MlpOff::total
  float *s_fd = smem + MlpOff::total;               // MlpOff::total
  float *s_x = smem + 2 * MlpOff::total;            // kInp * kShadeThreads
  const int tid = threadIdx.x;
  int cur = -1;
  unsigned long long n_fs = 0, n_fd = 0;
  // blocked tile ranges: consecutive tiles (mostly one instance) per CTA, so
  // each CTA reloads few assets' weights
  long long total_tiles = 0;
  for (int q = 0; q < args.n_inst; ++q)
    total_tiles += (min((long long)args.counts[q], args.qoff[q + 1] - args.qoff[q]) + kShadeThreads - 1) / kShadeThreads;
  const long long tile_lo = total_tiles * blockIdx.x / gridDim.x;
  const long long tile_hi = total_tiles * (blockIdx.x + 1) / gridDim.x;
  for (long long tile = tile_lo; tile < tile_hi; ++tile) {
    // map the global tile id onto (instance, first record)
    int k = 0;
    long long t = tile;
    unsigned cnt = 0;
    for (; k < args.n_inst; ++k) {
      cnt = min((long long)args.counts[k], args.qoff[k + 1] - args.qoff[k]);
      long long nt = (cnt + kShadeThreads - 1) / kShadeThreads;
      if (t < nt) break;
      t -= nt;
    }
    if (k >= args.n_inst) break;
    const DevInst &I = args.inst[k];
    const DevAsset &A = *I.a;
    if (k != cur) {
      __syncthreads();
      for (int q = tid; q < MlpOff::total; q += kShadeThreads) {
        s_fs[q] = A.fs.params[q];
        s_fd[q] = A.fd.params ? A.fd.params[q] : 0.f;
      }
      __syncthreads();
      cur = k;
    }
    const long long r = t * kShadeThreads + tid;
    if (r >= cnt) continue;
    const HitRec rec = args.queue[args.qoff[k] + r];
    float *xcol = s_x + tid;
    // PSH encode (encoding.py:390-394)
    int base[3];
    double w8[8];
    base_weights(rec.p, A.N, base, w8);
    double es0 = 0.0, es1 = 0.0, es_rest[2] = {0.0, 0.0};
    const long long orow = args.mode == kModeScene ? (long long)rec.ordinal * args.layer_stride + rec.out_idx
                                                   : (long long)rec.out_idx;
    uint32_t *dbg = (args.dbg_slots && orow < args.dbg_rows) ? args.dbg_slots + 8 * orow : nullptr;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint32_t slot = psh_slot(A.tab, A.phi, A.N, A.m, A.mphi, base[0] + (c & 1),
                                     base[1] + ((c >> 1) & 1), base[2] + ((c >> 2) & 1));
      if (dbg) dbg[c] = slot;
      if (A.F == 2) {
        const float2 f = __ldg(reinterpret_cast<const float2 *>(A.feat) + slot);
        es0 = __dadd_rn(es0, __dmul_rn((double)f.x, w8[c]));
        es1 = __dadd_rn(es1, __dmul_rn((double)f.y, w8[c]));
      } else {
        const float *f = A.feat + (size_t)slot * A.F;
        es0 = __dadd_rn(es0, __dmul_rn((double)__ldg(f), w8[c]));
        if (A.F > 1) es1 = __dadd_rn(es1, __dmul_rn((double)__ldg(f + 1), w8[c]));
        if (A.F > 2) es_rest[0] = __dadd_rn(es_rest[0], __dmul_rn((double)__ldg(f + 2), w8[c]));
        if (A.F > 3) es_rest[1] = __dadd_rn(es_rest[1], __dmul_rn((double)__ldg(f + 3), w8[c]));
      }
    }
    int nin = 0;
    xcol[(nin++) * kShadeThreads] = (float)es0;
    if (A.F > 1) xcol[(nin++) * kShadeThreads] = (float)es1;
    if (A.F > 2) xcol[(nin++) * kShadeThreads] = (float)es_rest[0];
    if (A.F > 3) xcol[(nin++) * kShadeThreads] = (float)es_rest[1];
    double sh[16];
    sh_encode(rec.d, sh);
#pragma unroll
    for (int q = 0; q < 16; ++q) xcol[(nin + q) * kShadeThreads] = (float)sh[q];
    nin += 16;
    const double ac = clampd(rec.alpha_c, 1e-4, 1.0 - 1e-4);
    if (A.refine_opacity) xcol[(nin++) * kShadeThreads] = (float)ac;
    float fs_out[4];
    mlp_row(s_fs, A.fs.n_layers, A.fs.in, A.fs.act, xcol, fs_out);
    ++n_fs;
    double alpha;
    const double z = (double)fs_out[3];
    if (!A.use_opacity) alpha = clampd(rec.alpha_c, 0.0, 1.0);
    else if (A.refine_opacity) alpha = sigmoid_np(z + log(ac / (1.0 - ac)));
    else alpha = sigmoid_np(z);
    double cd[3], tint;
    if (!A.use_diffuse_color) {
      cd[0] = cd[1] = cd[2] = 0.0;
      tint = 1.0;
    } else if (A.has_dif) {
      float dv[4];
      atlas_query<4>(A.dif, rec.p, dv);
      cd[0] = dv[0]; cd[1] = dv[1]; cd[2] = dv[2];
      tint = dv[3];
    } else {
      // live diffuse: hash grid (encoding.py:467-478) + diffuse MLP
      hashgrid_encode_col(A, rec.p, xcol);
      float dv[4];
      mlp_row(s_fd, A.fd.n_layers, A.fd.in, A.fd.act, xcol, dv);
      ++n_fd;
      cd[0] = dv[0]; cd[1] = dv[1]; cd[2] = dv[2];
      tint = dv[3];
    }
    if (!A.use_tint) tint = 0.5;
    float4 out;
    out.x = (float)clampd(__dadd_rn(cd[0], __dmul_rn(tint, (double)fs_out[0])), 0.0, 1.0);
    out.y = (float)clampd(__dadd_rn(cd[1], __dmul_rn(tint, (double)fs_out[1])), 0.0, 1.0);
    out.z = (float)clampd(__dadd_rn(cd[2], __dmul_rn(tint, (double)fs_out[2])), 0.0, 1.0);
    out.w = (float)alpha;
    float dep = (float)__ddiv_rn(rec.t_obj, I.scale);
    if (out.w <= 0.f) {        // lightfield.py:453-455
      out = make_float4(0.f, 0.f, 0.f, 0.f);
      dep = __int_as_float(0x7f800000);
    }
    reinterpret_cast<float4 *>(args.rgba)[orow] = out;
    args.depth[orow] = dep;
  }
  // fs_evals, fd_evals, hit_pixels (lightfield.py:299-301, 324-325)
  const unsigned lane = tid & 31;
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    n_fs += __shfl_xor_sync(0xffffffffu, n_fs, off);
    n_fd += __shfl_xor_sync(0xffffffffu, n_fd, off);
  }
  if (lane == 0) {
    if (n_fs) { atomicAdd(args.counters + 0, n_fs); atomicAdd(args.counters + 2, n_fs); }
    if (n_fd) atomicAdd(args.counters + 1, n_fd);
  }
}

// ---------------------------------------------------------------- live diffuse
// Hash-grid encode (encoding.py:467-478) of one point into a per-thread smem
// column; returns the encoded width.
__device__ __forceinline__ int hashgrid_encode_col(const DevAsset &A, const double p[3], float *xcol) {
  int ni = 0;
  for (int l = 0; l < A.hg_levels; ++l) {
    const int n = A.hg_res[l];
    int bl[3];
    double wl[8];
    base_weights(p, n, bl, wl);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int c = 0; c < 8; ++c) {
      const int cx = c & 1, cy = (c >> 1) & 1, cz = (c >> 2) & 1;
      long long idx;
      if (A.hg_dense[l]) {     // dense levels (encoding.py:449-453)
        const long long side = n + 1;
        idx = ((bl[0] * side + bl[1]) * side + bl[2]) + ((cx * side + cy) * side + cz);
      } else {                 // xor-prime hashed levels (encoding.py:454-459)
        unsigned long long h = ((unsigned long long)(bl[0] + cx) * 1ull) ^
                               ((unsigned long long)(bl[1] + cy) * 2654435761ull) ^
                               ((unsigned long long)(bl[2] + cz) * 805459861ull);
        idx = (long long)(h % A.hg_table);
      }
      const float *row = A.hg_feat[l] + idx * A.hg_F;
      for (int f = 0; f < A.hg_F && f < 4; ++f)
        acc[f] = __dadd_rn(acc[f], __dmul_rn((double)__ldg(row + f), wl[c]));
    }
    for (int f = 0; f < A.hg_F && f < 4; ++f) xcol[(ni++) * kShadeThreads] = (float)acc[f];
  }
  return ni;
}

// Diffuse network at arbitrary points: (c_d, t) post-activation, i.e. what
// bake_diffuse_cubes caches (lightfield.py:547-576) and what the live path
// returns (lightfield.py:319-327).
__global__ void __launch_bounds__(kShadeThreads) k_eval_diffuse(const DevAsset *Ap, const double *pts, long long n,
                                                                float *out) {
  extern __shared__ __align__(16) float smem[];
  float *s_fd = smem;
  float *s_x = smem + MlpOff::total;
  const DevAsset &A = *Ap;
  for (int q = threadIdx.x; q < MlpOff::total; q += kShadeThreads) s_fd[q] = A.fd.params[q];
  __syncthreads();
  for (long long i = (long long)blockIdx.x * kShadeThreads + threadIdx.x; i < n;
       i += (long long)gridDim.x * kShadeThreads) {
    const double p[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    float *xcol = s_x + threadIdx.x;
    hashgrid_encode_col(A, p, xcol);
    float dv[4];
    mlp_row(s_fd, A.fd.n_layers, A.fd.in, A.fd.act, xcol, dv);
    reinterpret_cast<float4 *>(out)[i] = make_float4(dv[0], dv[1], dv[2], dv[3]);
  }
}

// ---------------------------------------------------------------- compose
struct ComposeArgs {
  long long n_pix;             // total pixel slots
  const uint8_t *nhit;         // scene mode: per-pixel layer count (NULL => K layers)
  int K;                       // layers when nhit == NULL
  const float *rgba;           // (L, P, 4)
  const float *depth;          // (L, P)
  long long layer_stride;      // P
  const TileParams *tiles;     // scene mode: skip padding slots (NULL => none)
  long long tile_stride;
  const CamParams *cams;       // scene mode: camera sizes / output bases (tile validation, frame layout)
  int n_cams;
  int frame_layout;            // 0: outputs tile-packed at p ; 1: row-major frame per camera
  int peer;                    // outputs are a peer GPU's memory: fence system-wide at the end
  float alpha_vis;             // compared in f32 (numpy 2 weak scalar)
  float *out_rgba;
  float *out_depth;
  uint8_t *out_rgba8;
  uint16_t *out_depth16;
  float depth_far;
  int four;                    // slots per thread: 0 -> 1, 1 -> 4, 2 -> 8 (tiles && nhit && stride % 4 / 8 == 0)
  const uint8_t *chunk_live;   // scene: per 128-slot chunk, 0 = never marched (all misses)
  int prefilled;               // outputs already hold the miss encoding: dead chunks are not written
  uint16_t *chunk_state;       // prefilled buffers re-used across frames: per chunk, bit r = 8-pixel
                               // run r holds non-miss bytes from an earlier frame (NULL: freshly cleared)
  uint8_t *pack;               // sparse frame (NolfSceneOut.pack): 48 B per non-miss 8-pixel run, or NULL
  uint32_t *pack_ids;          // per live chunk: {chunk id, run mask, first run in pack}
  uint32_t *pack_count;        // [0] live chunks, [1] runs in pack
  unsigned *errors;            // device error counters (kErrTile for tiles the pack cannot hold)
};

constexpr int kMaxLayers = 64;

// farm.compose (farm.py:129-172) of slot p's n hit layers; frames whose
// pixel is a miss (rgba 0, depth inf) sort last and leave out_c and T
// unchanged, so compositing only the hit layers is bitwise equal to
// compositing all K.  n == 0 -> the miss sentinel (farm.py:169-171).
__device__ __forceinline__ void compose_px(const ComposeArgs &a, const long long p, const int n, float4 &o,
                                           float &od) {
  o = make_float4(0.f, 0.f, 0.f, 0.f);
  od = __int_as_float(0x7f800000);
  if (n == 0) return;
  if (n == 1) {                // one layer: no sort; the same f64 arithmetic as below
    const float d0 = a.depth[p];
    if (a.nhit && !(d0 < __int_as_float(0x7f800000))) return;   // missed / alpha <= 0: nothing
    const float4 c = reinterpret_cast<const float4 *>(a.rgba)[p];
    const double oc0 = __dadd_rn(0.0, __dmul_rn(1.0, (double)c.x));
    const double oc1 = __dadd_rn(0.0, __dmul_rn(1.0, (double)c.y));
    const double oc2 = __dadd_rn(0.0, __dmul_rn(1.0, (double)c.z));
    const double trans = __dmul_rn(1.0, (double)(1.0f - c.w));
    if (c.w > a.alpha_vis) od = d0;
    o.x = (float)clampd(oc0, 0.0, 1.0);
    o.y = (float)clampd(oc1, 0.0, 1.0);
    o.z = (float)clampd(oc2, 0.0, 1.0);
    o.w = (float)clampd(__dsub_rn(1.0, trans), 0.0, 1.0);
    if (o.w <= 0.f) {
      o = make_float4(0.f, 0.f, 0.f, 0.f);
      od = __int_as_float(0x7f800000);
    }
    return;
  }
  if (n <= 4) {                // few layers: the same stable sort and f64 over, in registers
    float dk4[4];
    int ord4[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      dk4[k] = __int_as_float(0x7f800000);
      ord4[k] = k;
      if (k < n) dk4[k] = a.depth[(long long)k * a.layer_stride + p];
    }
    // stable: insertion by strict '>' (np.argsort kind="stable")
#pragma unroll
    for (int k = 1; k < 4; ++k)
#pragma unroll
      for (int j = k; j > 0; --j)
        if (j <= k && k < n && dk4[j - 1] > dk4[j]) {
          const float td = dk4[j - 1]; dk4[j - 1] = dk4[j]; dk4[j] = td;
          const int to = ord4[j - 1]; ord4[j - 1] = ord4[j]; ord4[j] = to;
        }
    double oc0 = 0.0, oc1 = 0.0, oc2 = 0.0, trans = 1.0;
    bool set = false;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (r >= n) break;
      if (a.nhit && !(dk4[r] < __int_as_float(0x7f800000))) break;
      const float4 c = reinterpret_cast<const float4 *>(a.rgba)[(long long)ord4[r] * a.layer_stride + p];
      oc0 = __dadd_rn(oc0, __dmul_rn(trans, (double)c.x));
      oc1 = __dadd_rn(oc1, __dmul_rn(trans, (double)c.y));
      oc2 = __dadd_rn(oc2, __dmul_rn(trans, (double)c.z));
      if (!set && c.w > a.alpha_vis) { od = dk4[r]; set = true; }
      trans = __dmul_rn(trans, (double)(1.0f - c.w));
    }
    o.x = (float)clampd(oc0, 0.0, 1.0);
    o.y = (float)clampd(oc1, 0.0, 1.0);
    o.z = (float)clampd(oc2, 0.0, 1.0);
    o.w = (float)clampd(__dsub_rn(1.0, trans), 0.0, 1.0);
    if (o.w <= 0.f) {
      o = make_float4(0.f, 0.f, 0.f, 0.f);
      od = __int_as_float(0x7f800000);
    }
    return;
  }
  if (n > kMaxLayers) {        // many layers: stable order by repeated selection, no per-thread arrays
    double oc0 = 0.0, oc1 = 0.0, oc2 = 0.0, trans = 1.0;
    bool set = false;
    float last_d = -__int_as_float(0x7f800000);
    int last_k = -1;
    for (int r = 0; r < n; ++r) {
      // next (depth, index) in lexicographic order after (last_d, last_k)
      float bd = 0.f;
      int bk = -1;
      for (int k = 0; k < n; ++k) {
        const float dv = a.depth[(long long)k * a.layer_stride + p];
        const bool after = dv > last_d || (dv == last_d && k > last_k);
        if (after && (bk < 0 || dv < bd)) { bd = dv; bk = k; }
      }
      if (bk < 0) break;
      last_d = bd;
      last_k = bk;
      if (a.nhit && !(bd < __int_as_float(0x7f800000))) break;
      const float4 c = reinterpret_cast<const float4 *>(a.rgba)[(long long)bk * a.layer_stride + p];
      oc0 = __dadd_rn(oc0, __dmul_rn(trans, (double)c.x));
      oc1 = __dadd_rn(oc1, __dmul_rn(trans, (double)c.y));
      oc2 = __dadd_rn(oc2, __dmul_rn(trans, (double)c.z));
      if (!set && c.w > a.alpha_vis) { od = bd; set = true; }
      trans = __dmul_rn(trans, (double)(1.0f - c.w));
    }
    o.x = (float)clampd(oc0, 0.0, 1.0);
    o.y = (float)clampd(oc1, 0.0, 1.0);
    o.z = (float)clampd(oc2, 0.0, 1.0);
    o.w = (float)clampd(__dsub_rn(1.0, trans), 0.0, 1.0);
    if (o.w <= 0.f) {
      o = make_float4(0.f, 0.f, 0.f, 0.f);
      od = __int_as_float(0x7f800000);
    }
    return;
  }
  float dk[kMaxLayers];
  unsigned char ord[kMaxLayers];
  // stable insertion sort by depth (np.argsort kind="stable")
  for (int k = 0; k < n; ++k) {
    const float dv = a.depth[(long long)k * a.layer_stride + p];
    int j = k;
    while (j > 0 && dk[j - 1] > dv) { dk[j] = dk[j - 1]; ord[j] = ord[j - 1]; --j; }
    dk[j] = dv;
    ord[j] = (unsigned char)k;
  }
  double oc0 = 0.0, oc1 = 0.0, oc2 = 0.0, trans = 1.0;
  bool set = false;
  for (int r = 0; r < n; ++r) {
    // scene layers: depth inf = a candidate that missed (rgba never written)
    // or a hit with alpha <= 0 (rgba 0); both sort last and change nothing
    if (a.nhit && !(dk[r] < __int_as_float(0x7f800000))) break;
    const int k = ord[r];
    const float4 c = reinterpret_cast<const float4 *>(a.rgba)[(long long)k * a.layer_stride + p];
    oc0 = __dadd_rn(oc0, __dmul_rn(trans, (double)c.x));
    oc1 = __dadd_rn(oc1, __dmul_rn(trans, (double)c.y));
    oc2 = __dadd_rn(oc2, __dmul_rn(trans, (double)c.z));
    if (!set && c.w > a.alpha_vis) { od = dk[r]; set = true; }
    trans = __dmul_rn(trans, (double)(1.0f - c.w));
  }
  o.x = (float)clampd(oc0, 0.0, 1.0);
  o.y = (float)clampd(oc1, 0.0, 1.0);
  o.z = (float)clampd(oc2, 0.0, 1.0);
  o.w = (float)clampd(__dsub_rn(1.0, trans), 0.0, 1.0);
  if (o.w <= 0.f) {
    o = make_float4(0.f, 0.f, 0.f, 0.f);
    od = __int_as_float(0x7f800000);
  }
}

// encode_frame (protocol.py:256-266): clip(round(x*255)) and the u16 depth
__device__ __forceinline__ uchar4 encode_rgba8(const float4 o) {
  const float qv[4] = {o.x, o.y, o.z, o.w};
  unsigned char uu[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    float v = rintf(qv[c] * 255.0f);
    v = v < 0.f ? 0.f : (v > 255.f ? 255.f : v);
    uu[c] = (unsigned char)v;
  }
  return make_uchar4(uu[0], uu[1], uu[2], uu[3]);
}
__device__ __forceinline__ uint16_t encode_depth16(const float od, const float far) {
  return isfinite(od) ? (uint16_t)rintf(fminf(od, far) / far * 65534.0f) : (uint16_t)65535;
}

// protocol.encode_frame (protocol.py:256-266) of a whole f32 frame.
__global__ void __launch_bounds__(256) k_encode_frame(const float4 *rgba, const float *depth, long long n,
                                                      float far, uchar4 *rgba8, uint16_t *depth16) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    rgba8[i] = encode_rgba8(rgba[i]);
    depth16[i] = encode_depth16(depth[i], far);
  }
}

// Output index of slot p (-1 for tile padding).
__device__ __forceinline__ long long compose_dst(const ComposeArgs &a, const TileParams &tp, long long local,
                                                 long long p) {
  const int w = tp.x1 - tp.x0, h = tp.y1 - tp.y0;
  if (local >= (long long)w * h) return -1;
  if (!tile_valid(tp, a.cams, a.n_cams, a.tile_stride)) return -1;   // never marched (kErrTile)
  if (!a.frame_layout) return p;
  const CamParams &cp = a.cams[tp.cam];
  int x, y;
  slot_xy(local, w, h, x, y);
  return cp.pix_base + (long long)(tp.y0 + y) * cp.width + (tp.x0 + x);
}

__device__ __forceinline__ void compose_store(const ComposeArgs &a, long long q, const float4 o, const float od) {
  if (a.out_rgba) reinterpret_cast<float4 *>(a.out_rgba)[q] = o;
  if (a.out_depth) a.out_depth[q] = od;
  if (a.out_rgba8) reinterpret_cast<uchar4 *>(a.out_rgba8)[q] = encode_rgba8(o);
  if (a.out_depth16) a.out_depth16[q] = encode_depth16(od, a.depth_far);
}

__device__ __forceinline__ void compose_one(const ComposeArgs &a, const long long p) {
  long long q = p;             // output index
  if (a.tiles) {
    long long t, local;
    split_slot(p, a.tile_stride, t, local);
    q = compose_dst(a, a.tiles[t], local, p);
    if (q < 0) return;
  }
  float4 o;
  float od;
  const bool skip = a.chunk_live && !a.chunk_live[p >> 7];
  if (skip && a.prefilled) return;
  compose_px(a, p, skip ? 0 : (a.nhit ? (int)a.nhit[p] : a.K), o, od);
  compose_store(a, q, o, od);
}

// Four consecutive slots of one tile per thread (scene mode, tile_stride % 4
// == 0): one tile/camera lookup and one 4-byte layer-count load per thread,
// and 16 B rgba8 / 8 B depth16 stores when the 4 pixels are one aligned run
// (8x4-block layout: slots 4k..4k+3 are 4 adjacent pixels of one row).
__device__ __forceinline__ void compose_four(const ComposeArgs &a, const long long p0) {
  long long t, local0;
  split_slot(p0, a.tile_stride, t, local0);
  const TileParams tp = a.tiles[t];
  const bool dead4 = a.chunk_live && !a.chunk_live[p0 >> 7];
  if (dead4 && a.prefilled) return;
  const uchar4 nh = dead4 ? make_uchar4(0, 0, 0, 0) : *reinterpret_cast<const uchar4 *>(a.nhit + p0);
  const int ns[4] = {nh.x, nh.y, nh.z, nh.w};
  long long q[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) q[j] = compose_dst(a, tp, local0 + j, p0 + j);
  const bool run = q[0] >= 0 && (q[0] & 3) == 0 && q[1] == q[0] + 1 && q[2] == q[0] + 2 && q[3] == q[0] + 3 &&
                   !a.out_rgba && !a.out_depth;
  if (run && (ns[0] | ns[1] | ns[2] | ns[3]) == 0) {     // common case: four misses
    if (a.prefilled) return;                              // the miss encoding is already there
    if (a.out_rgba8) reinterpret_cast<uint4 *>(a.out_rgba8)[q[0] >> 2] = make_uint4(0u, 0u, 0u, 0u);
    if (a.out_depth16) reinterpret_cast<uint2 *>(a.out_depth16)[q[0] >> 2] = make_uint2(0xffffffffu, 0xffffffffu);
    return;
  }
  if (run) {
    unsigned c8[4], d16[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float4 o;
      float od;
      compose_px(a, p0 + j, ns[j], o, od);
      const uchar4 u = encode_rgba8(o);
      c8[j] = (unsigned)u.x | ((unsigned)u.y << 8) | ((unsigned)u.z << 16) | ((unsigned)u.w << 24);
      d16[j] = encode_depth16(od, a.depth_far);
    }
    if (a.out_rgba8) reinterpret_cast<uint4 *>(a.out_rgba8)[q[0] >> 2] = make_uint4(c8[0], c8[1], c8[2], c8[3]);
    if (a.out_depth16)
      reinterpret_cast<uint2 *>(a.out_depth16)[q[0] >> 2] = make_uint2(d16[0] | (d16[1] << 16), d16[2] | (d16[3] << 16));
    return;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (q[j] < 0) continue;
    float4 o;
    float od;
    compose_px(a, p0 + j, ns[j], o, od);
    compose_store(a, q[j], o, od);
  }
}

// Eight consecutive slots per thread (tile_stride % 8 == 0): in an 8x4-block
// tile they are one 8-pixel row of a block, i.e. 32 contiguous rgba8 bytes
// and 16 depth16 bytes of the frame -> two 16 B + one 16 B stores, one 8 B
// layer-count load; anything else goes through the 4-slot path twice.
// known_live: the caller walks the live-chunk list (no chunk_live loads);
// the layer counts are then loaded before the tile record, not after it
template <bool known_live = false>
__device__ __forceinline__ void compose_eight(const ComposeArgs &a, const long long p0) {
  if (!known_live && a.prefilled && a.chunk_live && !a.chunk_live[p0 >> 7]) return;   // misses already in place
  uint2 nh_early = make_uint2(0u, 0u);
  if (known_live) nh_early = *reinterpret_cast<const uint2 *>(a.nhit + p0);
  long long t, local0;
  split_slot(p0, a.tile_stride, t, local0);
  const TileParams tp = a.tiles[t];
  const int w = tp.x1 - tp.x0, h = tp.y1 - tp.y0;
  if (a.frame_layout && (w & 7) == 0 && (h & 3) == 0 && local0 < (long long)w * h && !a.out_rgba && !a.out_depth &&
      tile_valid(tp, a.cams, a.n_cams, a.tile_stride)) {
    const CamParams &cp = a.cams[tp.cam];
    int x, y;
    slot_xy(local0, w, h, x, y);
    const long long q0 = cp.pix_base + (long long)(tp.y0 + y) * cp.width + (tp.x0 + x);
    if ((q0 & 7) == 0) {
      uint2 nh = nh_early;
      if (!known_live) {
        const bool live = !a.chunk_live || a.chunk_live[p0 >> 7];
        nh = live ? *reinterpret_cast<const uint2 *>(a.nhit + p0) : make_uint2(0u, 0u);
      }
      uint4 *r8 = reinterpret_cast<uint4 *>(a.out_rgba8 + q0 * 4);
      uint4 *d16 = reinterpret_cast<uint4 *>(a.out_depth16 + q0);
      if ((nh.x | nh.y) == 0) {                 // eight misses
        if (a.prefilled) return;                // the miss encoding is already there
        if (a.out_rgba8) { r8[0] = make_uint4(0u, 0u, 0u, 0u); r8[1] = make_uint4(0u, 0u, 0u, 0u); }
        if (a.out_depth16) d16[0] = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
        return;
      }
      unsigned c8[8], dd[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int n = (int)(((j < 4 ? nh.x : nh.y) >> (8 * (j & 3))) & 0xffu);
        float4 o;
        float od;
        compose_px(a, p0 + j, n, o, od);
        const uchar4 u = encode_rgba8(o);
        c8[j] = (unsigned)u.x | ((unsigned)u.y << 8) | ((unsigned)u.z << 16) | ((unsigned)u.w << 24);
        dd[j] = encode_depth16(od, a.depth_far);
      }
      if (a.out_rgba8) {
        r8[0] = make_uint4(c8[0], c8[1], c8[2], c8[3]);
        r8[1] = make_uint4(c8[4], c8[5], c8[6], c8[7]);
      }
      if (a.out_depth16)
        d16[0] = make_uint4(dd[0] | (dd[1] << 16), dd[2] | (dd[3] << 16), dd[4] | (dd[5] << 16), dd[6] | (dd[7] << 16));
      return;
    }
  }
  compose_four(a, p0);
  compose_four(a, p0 + 4);
}

__global__ void __launch_bounds__(256) k_compose(ComposeArgs a) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (a.four == 2) {
    if (8 * gid < a.n_pix) compose_eight(a, 8 * gid);
  } else if (a.four) {
    if (4 * gid < a.n_pix) compose_four(a, 4 * gid);
  } else if (gid < a.n_pix) {
    compose_one(a, gid);
  }
  if (a.peer) {                // outputs in another GPU's memory: the barrier
    __syncthreads();           // orders the CTA's stores before one system-scope
    if (threadIdx.x == 0) __threadfence_system();   // fence (cumulative), ahead of
  }                            // the completion collective that follows
}

// Sparse frame: 8 consecutive slots (one 8-pixel run of an 8x4 block) of
// live chunk `idx` (16 consecutive lanes hold the chunk's 16 runs).  Runs
// that encode to anything but the miss encoding are packed (32 B rgba8 +
// 16 B depth16, run order within the chunk, chunks in allocation order); the
// chunk's header is {chunk id, mask of packed runs, index of its first run}.
// The frame itself is written as compose_eight does (when given).
__device__ __forceinline__ void compose_pack8(const ComposeArgs &a, const long long p0, const unsigned idx,
                                              const unsigned chunk_id, const unsigned lane) {
  long long t, local0;
  split_slot(p0, a.tile_stride, t, local0);
  const TileParams tp = a.tiles[t];
  const int w = tp.x1 - tp.x0, h = tp.y1 - tp.y0;
  const bool blocks = !(w & 7) && !(h & 3);
  if (!blocks && (local0 & 127) == 0) atomicAdd(a.errors + kErrTile, 1u);   // no 8-pixel runs: cannot be packed
  unsigned c8[8], dd[8];
  bool nonmiss = false;
#pragma unroll
  for (int j = 0; j < 8; ++j) { c8[j] = 0u; dd[j] = 0xffffu; }
  if (blocks) {
    const uint2 nh = *reinterpret_cast<const uint2 *>(a.nhit + p0);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int n = local0 + j < (long long)w * h ? (int)(((j < 4 ? nh.x : nh.y) >> (8 * (j & 3))) & 0xffu) : 0;
      if (n == 0) continue;
      float4 o;
      float od;
      compose_px(a, p0 + j, n, o, od);
      const uchar4 u = encode_rgba8(o);
      c8[j] = (unsigned)u.x | ((unsigned)u.y << 8) | ((unsigned)u.z << 16) | ((unsigned)u.w << 24);
      dd[j] = encode_depth16(od, a.depth_far);
      nonmiss = nonmiss || c8[j] != 0u || dd[j] != 0xffffu;
    }
  }
  // run allocation for the chunk: one atomic per chunk (lane of run 0)
  const unsigned half = 0xffffu << (lane & 16u);
  const unsigned mask = (__ballot_sync(half, nonmiss) >> (lane & 16u)) & 0xffffu;
  const int run = (int)((p0 & 127) >> 3);
  unsigned first = 0;
  if (run == 0) {
    first = mask ? atomicAdd(a.pack_count + 1, (unsigned)__popc(mask)) : 0u;
    a.pack_ids[3 * idx + 0] = chunk_id;
    a.pack_ids[3 * idx + 1] = mask;
    a.pack_ids[3 * idx + 2] = first;
  }
  first = __shfl_sync(half, first, (int)(lane & 16u));
  if (nonmiss) {
    uint8_t *e = a.pack + 48ull * (first + (unsigned)__popc(mask & ((1u << run) - 1u)));
    reinterpret_cast<uint4 *>(e)[0] = make_uint4(c8[0], c8[1], c8[2], c8[3]);
    reinterpret_cast<uint4 *>(e)[1] = make_uint4(c8[4], c8[5], c8[6], c8[7]);
    reinterpret_cast<uint4 *>(e)[2] =
        make_uint4(dd[0] | (dd[1] << 16), dd[2] | (dd[3] << 16), dd[4] | (dd[5] << 16), dd[6] | (dd[7] << 16));
  }
  if (a.out_rgba8 && blocks && local0 < (long long)w * h && tile_valid(tp, a.cams, a.n_cams, a.tile_stride) &&
      (nonmiss || !a.prefilled)) {
    const CamParams &cp = a.cams[tp.cam];
    int x, y;
    slot_xy(local0, w, h, x, y);
    const long long q0 = cp.pix_base + (long long)(tp.y0 + y) * cp.width + (tp.x0 + x);
    uint4 *r8 = reinterpret_cast<uint4 *>(a.out_rgba8 + q0 * 4);
    r8[0] = make_uint4(c8[0], c8[1], c8[2], c8[3]);
    r8[1] = make_uint4(c8[4], c8[5], c8[6], c8[7]);
    if (a.out_depth16)
      *reinterpret_cast<uint4 *>(a.out_depth16 + q0) =
          make_uint4(dd[0] | (dd[1] << 16), dd[2] | (dd[3] << 16), dd[4] | (dd[5] << 16), dd[6] | (dd[7] << 16));
  }
}

// Frame buffers re-used across frames (NolfSceneOut.chunk_state): every
// 8-pixel run of a chunk has a dirty bit (non-miss bytes written by an
// earlier frame).  A live chunk's all-miss run is written only if dirty, a
// run with hits always (and becomes dirty); a dead chunk's dirty runs are
// reset (k_clear_stale).  The buffer therefore never needs a full clear and
// only changed runs cross NVLink.  8 slots (one run) per thread; the 16 runs
// of a chunk are 16 consecutive lanes (their dirty mask is one ballot).
__device__ __forceinline__ void compose_eight_state(const ComposeArgs &a, const long long p0, unsigned lane) {
  const long long c = p0 >> 7;
  const int run = (int)((p0 & 127) >> 3);
  const unsigned half = 0xffffu << (lane & 16u);
  const bool was = (a.chunk_state[c] >> run) & 1u;
  bool dirty = false;
  long long t, local0;
  split_slot(p0, a.tile_stride, t, local0);
  const TileParams tp = a.tiles[t];
  const int w = tp.x1 - tp.x0, h = tp.y1 - tp.y0;
  if (!(w & 7) && !(h & 3) && local0 < (long long)w * h && tile_valid(tp, a.cams, a.n_cams, a.tile_stride)) {
    const CamParams &cp = a.cams[tp.cam];
    int x, y;
    slot_xy(local0, w, h, x, y);
    const long long q0 = cp.pix_base + (long long)(tp.y0 + y) * cp.width + (tp.x0 + x);
    const uint2 nh = *reinterpret_cast<const uint2 *>(a.nhit + p0);
    uint4 r0 = make_uint4(0u, 0u, 0u, 0u), r1 = r0, dv = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
    if (nh.x | nh.y) {
      unsigned c8[8], dd[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int n = (int)(((j < 4 ? nh.x : nh.y) >> (8 * (j & 3))) & 0xffu);
        float4 o;
        float od;
        compose_px(a, p0 + j, n, o, od);
        const uchar4 u = encode_rgba8(o);
        c8[j] = (unsigned)u.x | ((unsigned)u.y << 8) | ((unsigned)u.z << 16) | ((unsigned)u.w << 24);
        dd[j] = encode_depth16(od, a.depth_far);
      }
      r0 = make_uint4(c8[0], c8[1], c8[2], c8[3]);
      r1 = make_uint4(c8[4], c8[5], c8[6], c8[7]);
      dv = make_uint4(dd[0] | (dd[1] << 16), dd[2] | (dd[3] << 16), dd[4] | (dd[5] << 16), dd[6] | (dd[7] << 16));
      dirty = true;
    }
    if (dirty || was) {
      uint4 *r8 = reinterpret_cast<uint4 *>(a.out_rgba8 + q0 * 4);
      r8[0] = r0;
      r8[1] = r1;
      *reinterpret_cast<uint4 *>(a.out_depth16 + q0) = dv;
    }
  }
  const unsigned mask = (__ballot_sync(half, dirty) >> (lane & 16u)) & 0xffffu;
  if (run == 0) a.chunk_state[c] = (uint16_t)mask;
}

// Dead chunks (no screen box reaches them now): reset their dirty runs.
__global__ void __launch_bounds__(256) k_clear_stale(ComposeArgs a, long long n_chunks) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long c = g >> 4;
  const int run = (int)(g & 15);
  const bool in = c < n_chunks && !a.chunk_live[c];
  const unsigned st = in ? a.chunk_state[c] : 0u;
  __syncwarp();                                  // every run read the state before it is reset
  if (in && st) {
    if (run == 0) a.chunk_state[c] = 0;
    if ((st >> run) & 1u) {
      const long long p0 = c * 128 + run * 8;
      long long t, local0;
      split_slot(p0, a.tile_stride, t, local0);
      const TileParams tp = a.tiles[t];
      const int w = tp.x1 - tp.x0, h = tp.y1 - tp.y0;
      if (!(w & 7) && !(h & 3) && local0 < (long long)w * h && tile_valid(tp, a.cams, a.n_cams, a.tile_stride)) {
        const CamParams &cp = a.cams[tp.cam];
        int x, y;
        slot_xy(local0, w, h, x, y);
        const long long q0 = cp.pix_base + (long long)(tp.y0 + y) * cp.width + (tp.x0 + x);
        uint4 *r8 = reinterpret_cast<uint4 *>(a.out_rgba8 + q0 * 4);
        r8[0] = make_uint4(0u, 0u, 0u, 0u);
        r8[1] = make_uint4(0u, 0u, 0u, 0u);
        *reinterpret_cast<uint4 *>(a.out_depth16 + q0) = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
      }
    }
  }
  if (a.peer) {                // stores into another GPU's frame: fenced before the completion flag
    __syncthreads();
    if (threadIdx.x == 0) __threadfence_system();
  }
}

// Prefilled outputs: compose only the live chunks, from the compacted list
// (16 threads x 8 slots per chunk, grid-stride over the list's length).
// G slots per thread (8 or 4): a launch over few live chunks (a multi-GPU
// shard) uses 4 so twice the threads hide the layer-read latency.
template <int G>
__global__ void __launch_bounds__(256) k_compose_live(ComposeArgs a, const unsigned *live_list, const unsigned *count,
                                                      long long list_stride) {
  constexpr int per_chunk = 128 / G;
  const long long total = (long long)count[0] * per_chunk;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (long long)gridDim.x * blockDim.x) {
    const long long p0 = (long long)live_list[g / per_chunk] * 128 + (g % per_chunk) * G;   // spatial list
    if (G == 8 && a.pack) {
      compose_pack8(a, p0, (unsigned)(g / per_chunk), live_list[g / per_chunk], threadIdx.x & 31u);
    } else if (G == 8 && a.chunk_state) {
      compose_eight_state(a, p0, threadIdx.x & 31u);
    } else if (G == 8) {
      compose_eight<true>(a, p0);
    } else {
      compose_four(a, p0);
    }
  }
  if (a.pack_count && blockIdx.x == 0 && threadIdx.x == 0) a.pack_count[0] = count[0];
  if (a.peer) {
    __syncthreads();
    if (threadIdx.x == 0) __threadfence_system();
  }
}

// Frame assembly after an all-rank gather: rank r's buffer holds n_per_rank
// tile slots of rgba8 (stride*4 B each) followed by their depth16; slot_tiles
// lists the tile of every (rank, slot) in rank-major order.
__global__ void __launch_bounds__(256) k_unpack(const uint8_t *gathered, long long rank_bytes, int n_per_rank,
                                                long long tile_stride, const TileParams *slot_tiles,
                                                long long n_slots, int width, int height, uchar4 *rgba8,
                                                uint16_t *depth16) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long s, local;
  split_slot(i, tile_stride, s, local);
  if (s >= n_slots) return;
  const TileParams tp = slot_tiles[s];
  const int w = tp.x1 - tp.x0, h = tp.y1 - tp.y0;
  if (local >= (long long)w * h) return;
  const long long r = s / n_per_rank, j = s % n_per_rank;
  const uint8_t *base = gathered + r * rank_bytes;
  const long long src = j * tile_stride + local;
  int x, y;
  slot_xy(local, w, h, x, y);
  const long long dst = (long long)tp.cam * width * height + (long long)(tp.y0 + y) * width + (tp.x0 + x);
  rgba8[dst] = reinterpret_cast<const uchar4 *>(base)[src];
  depth16[dst] = reinterpret_cast<const uint16_t *>(base + (long long)n_per_rank * tile_stride * 4)[src];
}

// n words from device memory to (typically host-mapped) memory by plain
// stores: no copy-engine operation in the stream.
__global__ void k_store_u32(uint32_t *dst, const uint32_t *src, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
  __threadfence_system();
}

// ---------------------------------------------------------------- cross-GPU flags
__global__ void k_flag_set(uint32_t *flag, uint32_t value) {
  __threadfence_system();      // the stream's earlier (peer) stores become visible first
  *reinterpret_cast<volatile uint32_t *>(flag) = value;
  __threadfence_system();
}

__global__ void k_flag_wait(const uint32_t *flags, int n, uint32_t value, uint32_t *timed_out) {
  const int i = threadIdx.x;
  bool ok = i >= n;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (!__all_sync(0xffffffffu, ok)) {
    if (!ok) ok = *reinterpret_cast<const volatile uint32_t *>(flags + i) >= value;
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (now - t0 > 4000000000ull) {          // bounded: never hang the device
      if (i == 0 && timed_out) *timed_out = 1u;
      break;
    }
    __nanosleep(200);
  }
  __threadfence_system();      // order the peers' data before what follows on this stream
}

}  // namespace nolf
