// nolf_mesh.cuh -- triangle-mesh proxy first hit (BVH traversal).
//
// The reference's proxy is an AABB (lightfield.py:229, slab test core.py:206);
// BASELINE config 2 / the north star add a mesh proxy with no reference
// counterpart.  Semantics here: the march starts at the mesh's first hit
// t_mesh >= 0 (instead of the slab's t_near) and ends at the slab's t_far of
// the proxy box; a ray that misses every triangle is a miss.  Triangle
// tests are fp64 Moller-Trumbore written with explicit *_rn operations so
// the brute-force oracle (oracle/nolf_oracle.c, oracle_mesh_hit) reproduces
// t_mesh bit for bit; the BVH only prunes (fp32 boxes padded outward).
#pragma once
#include <cstdint>

namespace nolf {

struct BvhNode {              // 32 B
  float lo[3], hi[3];
  int first;                  // leaf: first triangle ; inner: left child (right = first + 1)
  int count;                  // > 0 leaf
};

// 4-wide node (one 128 B line): the boxes of up to 4 children (structure of
// arrays, fp32, padded outward like BvhNode) and what they are: count > 0 a
// leaf of `count` triangles from `child`, count == 0 an inner 4-wide node
// `child`, count < 0 an empty slot (box empty too).
struct Bvh4Node {
  float lo[3][4], hi[3][4];
  int child[4];
  int count[4];
};
static_assert(sizeof(Bvh4Node) == 128, "one cache line");

struct DevMesh {
  const BvhNode *nodes;       // null: no mesh proxy (binary tree: the per-thread walk)
  const double *tri;          // 9 doubles per triangle (v0, v1, v2), BVH leaf order
  int n_tri;
  const Bvh4Node *nodes4;     // the same tree collapsed 4-wide (the warp walk); root = 0
};

#ifdef NOLF_MT_FP32_TIMING   // diagnostic (approximate results): the triangle test in fp32
__device__ __forceinline__ double mt_hit(const double *T, const double o[3], const double d[3]) {
  float v[9];
  for (int i = 0; i < 9; ++i) v[i] = (float)T[i];
  const float e1x = v[3] - v[0], e1y = v[4] - v[1], e1z = v[5] - v[2];
  const float e2x = v[6] - v[0], e2y = v[7] - v[1], e2z = v[8] - v[2];
  const float dx = (float)d[0], dy = (float)d[1], dz = (float)d[2];
  const float px = dy * e2z - dz * e2y, py = dz * e2x - dx * e2z, pz = dx * e2y - dy * e2x;
  const float det = e1x * px + e1y * py + e1z * pz;
  if (fabsf(det) < 1e-30f) return -1.0;
  const float inv = 1.f / det;
  const float sx = (float)o[0] - v[0], sy = (float)o[1] - v[1], sz = (float)o[2] - v[2];
  const float u = (sx * px + sy * py + sz * pz) * inv;
  if (u < 0.f || u > 1.f) return -1.0;
  const float qx = sy * e1z - sz * e1y, qy = sz * e1x - sx * e1z, qz = sx * e1y - sy * e1x;
  const float w = (dx * qx + dy * qy + dz * qz) * inv;
  if (w < 0.f || u + w > 1.f) return -1.0;
  const float t = (e2x * qx + e2y * qy + e2z * qz) * inv;
  return t >= 0.f ? (double)t : -1.0;
}
#else
// Moller-Trumbore (fp64, explicit rounding) -> t or -1.
__device__ __forceinline__ double mt_hit(const double *T, const double o[3], const double d[3]) {
  const double e1x = __dsub_rn(T[3], T[0]), e1y = __dsub_rn(T[4], T[1]), e1z = __dsub_rn(T[5], T[2]);
  const double e2x = __dsub_rn(T[6], T[0]), e2y = __dsub_rn(T[7], T[1]), e2z = __dsub_rn(T[8], T[2]);
  const double px = __dsub_rn(__dmul_rn(d[1], e2z), __dmul_rn(d[2], e2y));
  const double py = __dsub_rn(__dmul_rn(d[2], e2x), __dmul_rn(d[0], e2z));
  const double pz = __dsub_rn(__dmul_rn(d[0], e2y), __dmul_rn(d[1], e2x));
  const double det = __dadd_rn(__dadd_rn(__dmul_rn(e1x, px), __dmul_rn(e1y, py)), __dmul_rn(e1z, pz));
  if (fabs(det) < 1e-300) return -1.0;
  const double inv = __drcp_rn(det);          // IEEE 1/det (== __ddiv_rn(1.0, det))
  const double sx = __dsub_rn(o[0], T[0]), sy = __dsub_rn(o[1], T[1]), sz = __dsub_rn(o[2], T[2]);
  const double u = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(sx, px), __dmul_rn(sy, py)), __dmul_rn(sz, pz)), inv);
  if (u < 0.0 || u > 1.0) return -1.0;
  const double qx = __dsub_rn(__dmul_rn(sy, e1z), __dmul_rn(sz, e1y));
  const double qy = __dsub_rn(__dmul_rn(sz, e1x), __dmul_rn(sx, e1z));
  const double qz = __dsub_rn(__dmul_rn(sx, e1y), __dmul_rn(sy, e1x));
  const double v = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(d[0], qx), __dmul_rn(d[1], qy)), __dmul_rn(d[2], qz)), inv);
  if (v < 0.0 || __dadd_rn(u, v) > 1.0) return -1.0;
  const double t = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(e2x, qx), __dmul_rn(e2y, qy)), __dmul_rn(e2z, qz)), inv);
  return t >= 0.0 ? t : -1.0;
}
#endif

// Conservative fp32 slab of a node (boxes padded at build time; +-2% in t):
// entry distance, or +inf when the ray cannot reach a triangle inside
// before the best hit so far.
__device__ __forceinline__ float node_entry(const BvhNode &n, float ox, float oy, float oz, float ix, float iy,
                                            float iz, float best_f) {
  float t0 = (n.lo[0] - ox) * ix, t1 = (n.hi[0] - ox) * ix;
  float tmin = fminf(t0, t1), tmax = fmaxf(t0, t1);
  t0 = (n.lo[1] - oy) * iy; t1 = (n.hi[1] - oy) * iy;
  tmin = fmaxf(tmin, fminf(t0, t1)); tmax = fminf(tmax, fmaxf(t0, t1));
  t0 = (n.lo[2] - oz) * iz; t1 = (n.hi[2] - oz) * iz;
  tmin = fmaxf(tmin, fminf(t0, t1)); tmax = fminf(tmax, fmaxf(t0, t1));
  if (tmax < 0.0f || tmin > tmax * 1.02f + 1e-6f || tmin > best_f * 1.02f + 1e-6f) return __int_as_float(0x7f800000);
  return tmin;
}

// Closest hit over the mesh: t_mesh >= 0, or -1 when the ray misses it.
// Children are visited near-first (both boxes tested at the parent, the far
// one pushed with its entry distance and dropped on pop if a closer hit was
// found meanwhile); pruning only, the fp64 triangle tests decide t.
// The host builds median-split trees of depth <= 28 (nolf_capi.cu
// upload_mesh), so the stack (one far child per level) never fills; a deeper
// tree would be counted in *err_overflow and its nodes dropped.
__device__ __forceinline__ double mesh_first_hit(const DevMesh &M, const double o[3], const double d[3],
                                                 unsigned *err_overflow) {
  const float ox = (float)o[0], oy = (float)o[1], oz = (float)o[2];
  // finite reciprocals: a zero component gets +-1e30 so (lo - o) * inv is never 0*inf
  auto rcp = [](double x) { const float f = (float)x; return 1.0f / copysignf(fmaxf(fabsf(f), 1e-30f), f); };
  const float ix = rcp(d[0]), iy = rcp(d[1]), iz = rcp(d[2]);
  double best = -1.0;
  float best_f = __int_as_float(0x7f800000);
  int stack[32];
  float stack_t[32];
  int sp = 0;
  {
    const float te = node_entry(M.nodes[0], ox, oy, oz, ix, iy, iz, best_f);
    if (te == __int_as_float(0x7f800000)) return -1.0;
    stack[0] = 0;
    stack_t[0] = te;
    sp = 1;
  }
  while (sp) {
    --sp;
    if (stack_t[sp] > best_f * 1.02f + 1e-6f) continue;   // a closer hit appeared after the push
    const BvhNode n = M.nodes[stack[sp]];
    if (n.count > 0) {
      for (int i = 0; i < n.count; ++i) {
        const double t = mt_hit(M.tri + 9ll * (n.first + i), o, d);
        if (t >= 0.0 && (best < 0.0 || t < best)) {
          best = t;
          best_f = (float)t;
        }
      }
    } else if (sp >= 30) {
      atomicAdd(err_overflow, 1u);
    } else {
      const BvhNode L = M.nodes[n.first], R = M.nodes[n.first + 1];
      const float tl = node_entry(L, ox, oy, oz, ix, iy, iz, best_f);
      const float tr = node_entry(R, ox, oy, oz, ix, iy, iz, best_f);
      const bool hl = tl != __int_as_float(0x7f800000), hr = tr != __int_as_float(0x7f800000);
      if (hl && hr) {
        const bool lfirst = tl <= tr;
        stack[sp] = lfirst ? n.first + 1 : n.first;      // far
        stack_t[sp++] = lfirst ? tr : tl;
        stack[sp] = lfirst ? n.first : n.first + 1;      // near on top
        stack_t[sp++] = lfirst ? tl : tr;
      } else if (hl || hr) {
        stack[sp] = hl ? n.first : n.first + 1;
        stack_t[sp++] = hl ? tl : tr;
      }
    }
  }
  return best;
}

// Warp-cooperative variant (all 32 lanes call it; `active` lanes have a ray
// to test): the warp walks ONE node stack (in shared memory, uniform), each
// node is fetched once per warp and tested against every lane's ray, a
// subtree is entered when any lane's ray can reach it, and a leaf's
// triangles are tested by the lanes that reach it, each against its own ray
// with the same fp64 Moller-Trumbore.  Every lane ends with the minimum t
// over all triangles its ray hits -- the same value as mesh_first_hit, since
// pruning only ever skips boxes that cannot hold a closer hit for that lane.
// Children are pushed in the order most lanes would visit them (near first).
constexpr int kMeshWarps = 4;          // warps per CTA of the marcher (kMarchThreads / 32)

__device__ __forceinline__ double mesh_first_hit_warp(const DevMesh &M, const double o[3], const double d[3],
                                                      bool active, unsigned *err_overflow) {
  __shared__ int s_stack[kMeshWarps][32];
  const unsigned lane = threadIdx.x & 31;
  int *stack = s_stack[(threadIdx.x >> 5) & (kMeshWarps - 1)];
  const float ox = active ? (float)o[0] : 0.f, oy = active ? (float)o[1] : 0.f, oz = active ? (float)o[2] : 0.f;
  auto rcp = [](double x) { const float f = (float)x; return 1.0f / copysignf(fmaxf(fabsf(f), 1e-30f), f); };
  const float ix = active ? rcp(d[0]) : 1.f, iy = active ? rcp(d[1]) : 1.f, iz = active ? rcp(d[2]) : 1.f;
  const float INFF = __int_as_float(0x7f800000);
  double best = -1.0;
  float best_f = INFF;
  if (!__any_sync(0xffffffffu, active && node_entry(M.nodes[0], ox, oy, oz, ix, iy, iz, best_f) != INFF)) return -1.0;
  if (lane == 0) stack[0] = 0;
  int sp = 1;                              // warp-uniform
  __syncwarp();
  while (sp) {
    --sp;
    const int ni = stack[sp];
    __syncwarp();                          // read before any push below overwrites the slot
    const BvhNode n = M.nodes[ni];
    const bool in = active && node_entry(n, ox, oy, oz, ix, iy, iz, best_f) != INFF;
    if (!__any_sync(0xffffffffu, in)) continue;
    if (n.count > 0) {
      if (in) {
        for (int i = 0; i < n.count; ++i) {
          const double t = mt_hit(M.tri + 9ll * (n.first + i), o, d);
          if (t >= 0.0 && (best < 0.0 || t < best)) {
            best = t;
            best_f = (float)t;
          }
        }
      }
    } else if (sp >= 30) {
      if (lane == 0) atomicAdd(err_overflow, 1u);
    } else {
      const BvhNode L = M.nodes[n.first], R = M.nodes[n.first + 1];
      const float tl = in ? node_entry(L, ox, oy, oz, ix, iy, iz, best_f) : INFF;
      const float tr = in ? node_entry(R, ox, oy, oz, ix, iy, iz, best_f) : INFF;
      const bool hl = tl != INFF, hr = tr != INFF;
      const unsigned bl = __ballot_sync(0xffffffffu, hl), br = __ballot_sync(0xffffffffu, hr);
      const int votes_l = __popc(__ballot_sync(0xffffffffu, hl && (!hr || tl <= tr)));
      const int votes_r = __popc(__ballot_sync(0xffffffffu, hr && (!hl || tr < tl)));
      const int nearc = votes_l >= votes_r ? n.first : n.first + 1, farc = nearc == n.first ? n.first + 1 : n.first;
      const bool near_hit = nearc == n.first ? bl != 0u : br != 0u;
      const bool far_hit = farc == n.first ? bl != 0u : br != 0u;
      if (lane == 0) {
        if (far_hit) stack[sp] = farc;
        if (near_hit) stack[sp + (far_hit ? 1 : 0)] = nearc;
      }
      sp += (far_hit ? 1 : 0) + (near_hit ? 1 : 0);
      __syncwarp();
    }
  }
  return best;
}

// Box slot j of a 4-wide node against one ray (node_entry's conservative
// test): entry distance or +inf.
__device__ __forceinline__ float node4_entry(const Bvh4Node &n, int j, float ox, float oy, float oz, float ix,
                                             float iy, float iz, float best_f) {
  float t0 = (n.lo[0][j] - ox) * ix, t1 = (n.hi[0][j] - ox) * ix;
  float tmin = fminf(t0, t1), tmax = fmaxf(t0, t1);
  t0 = (n.lo[1][j] - oy) * iy; t1 = (n.hi[1][j] - oy) * iy;
  tmin = fmaxf(tmin, fminf(t0, t1)); tmax = fminf(tmax, fmaxf(t0, t1));
  t0 = (n.lo[2][j] - oz) * iz; t1 = (n.hi[2][j] - oz) * iz;
  tmin = fmaxf(tmin, fminf(t0, t1)); tmax = fminf(tmax, fmaxf(t0, t1));
  if (tmax < 0.0f || tmin > tmax * 1.02f + 1e-6f || tmin > best_f * 1.02f + 1e-6f) return __int_as_float(0x7f800000);
  return tmin;
}

// Warp-cooperative walk of the 4-wide tree: half the levels of the binary
// tree, so half the dependent node loads per warp.  A popped inner node's
// (one 128 B line) 4 child boxes are tested by every active lane against its
// own ray with its current closest hit; the children some lane reaches are
// pushed farthest first (ordered by the warp's nearest entry distance, so
// the nearest is walked next).  A leaf is pushed as (node, slot) and its box
// re-tested on pop with the lane's closest hit by then; its triangles are
// tested with the same fp64 Moller-Trumbore.  Every lane ends with the
// minimum t over all triangles its ray hits, as mesh_first_hit.
constexpr int kMesh4Stack = 96;      // >= 3 x (4-wide depth) + 1, checked at upload

__device__ __forceinline__ double mesh_first_hit_warp4(const DevMesh &M, const double o[3], const double d[3],
                                                       bool active, unsigned *err_overflow) {
  __shared__ int s_stack4[kMeshWarps][kMesh4Stack];
  const unsigned lane = threadIdx.x & 31;
  int *stack = s_stack4[(threadIdx.x >> 5) & (kMeshWarps - 1)];
  const float ox = active ? (float)o[0] : 0.f, oy = active ? (float)o[1] : 0.f, oz = active ? (float)o[2] : 0.f;
  auto rcp = [](double x) { const float f = (float)x; return 1.0f / copysignf(fmaxf(fabsf(f), 1e-30f), f); };
  const float ix = active ? rcp(d[0]) : 1.f, iy = active ? rcp(d[1]) : 1.f, iz = active ? rcp(d[2]) : 1.f;
  const float INFF = __int_as_float(0x7f800000);
  double best = -1.0;
  float best_f = INFF;
  if (!__any_sync(0xffffffffu, active)) return -1.0;
  if (lane == 0) stack[0] = 0;             // entries: inner node n >= 0, leaf (node, slot) as -(4 n + slot) - 1
  int sp = 1;                              // warp-uniform
  __syncwarp();
  while (sp) {
    --sp;
    const int e = stack[sp];
    __syncwarp();                          // read before any push below overwrites the slot
    if (e < 0) {                           // a leaf: re-test its box, then its triangles
      const int ni = (-e - 1) >> 2, j = (-e - 1) & 3;
      const Bvh4Node &n = M.nodes4[ni];
      const bool in = active && node4_entry(n, j, ox, oy, oz, ix, iy, iz, best_f) != INFF;
      if (in) {
        const int first = n.child[j], cnt = n.count[j];
        for (int i = 0; i < cnt; ++i) {
          const double t = mt_hit(M.tri + 9ll * (first + i), o, d);
          if (t >= 0.0 && (best < 0.0 || t < best)) {
            best = t;
            best_f = (float)t;
          }
        }
      }
      continue;
    }
    const Bvh4Node &n = M.nodes4[e];
    // per child: the warp's nearest entry (as an orderable key; +inf: nobody)
    unsigned key[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float t = active && n.count[j] >= 0 ? node4_entry(n, j, ox, oy, oz, ix, iy, iz, best_f) : INFF;
      const unsigned u = __float_as_uint(t);
      key[j] = __reduce_min_sync(0xffffffffu, (u & 0x80000000u) ? ~u : (u | 0x80000000u));
    }
    const unsigned none = 0xff800000u;     // key of +inf
    if (sp + 4 > kMesh4Stack) {
      if (lane == 0) atomicAdd(err_overflow, 1u);
      continue;
    }
    // push the reached children farthest first: a 5-exchange sorting network
    // on (key, slot), descending (warp-uniform), then the entries in order
    int slot[4] = {0, 1, 2, 3};
    auto cx = [&](int p, int q) {
      if (key[p] < key[q]) {
        const unsigned tk = key[p]; key[p] = key[q]; key[q] = tk;
        const int ts = slot[p]; slot[p] = slot[q]; slot[q] = ts;
      }
    };
    cx(0, 1); cx(2, 3); cx(0, 2); cx(1, 3); cx(1, 2);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (key[q] == none) continue;          // +inf sorts first: nobody reaches it
      const int jm = slot[q];
      if (lane == 0) stack[sp] = n.count[jm] > 0 ? -(4 * e + jm) - 1 : n.child[jm];
      ++sp;
    }
    __syncwarp();
  }
  return best;
}

}  // namespace nolf
