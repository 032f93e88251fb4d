// nolf_capi.cu -- C ABI (include/nolf.h): asset upload, workspace layout and
// the launch sequence of the i-NOLF hot path on sm_100a.
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstring>
#include <string>
#include <vector>
#include <functional>

#include "../../include/nolf.h"
#include "nolf_kernels.cuh"
#include "nolf_load.h"
#include "nolf_shade_tc.cuh"
#include "nolf_host.h"
#include "nolf_train.cuh"

using namespace nolf;

namespace {

thread_local std::string g_err;

// Restores the caller's current device when it goes out of scope.
struct DeviceRestore {
  int dev;
  ~DeviceRestore() { cudaSetDevice(dev); }
};

int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(x)                                                                     \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) return fail(NOLF_ECUDA, "%s: %s", #x, cudaGetErrorString(e_)); \
  } while (0)

constexpr int kMaxInst = 255;    // compose layers per pixel are counted in a u8
constexpr int kMaxCams = 4096;

}  // namespace

struct NolfAsset {
  int device = 0;
  DevAsset host{};             // host copy with device pointers
  DevAsset *dev = nullptr;     // device copy
  std::vector<void *> allocs;
  int64_t bytes = 0;

  template <class T>
  int upload(const T *src, size_t count, T **dst) {
    *dst = nullptr;
    if (count == 0) return 0;
    void *p = nullptr;
    cudaError_t e = cudaMalloc(&p, count * sizeof(T));
    if (e != cudaSuccess) return fail(NOLF_ENOMEM, "cudaMalloc(%zu): %s", count * sizeof(T), cudaGetErrorString(e));
    allocs.push_back(p);
    bytes += (int64_t)(count * sizeof(T));
    e = cudaMemcpy(p, src, count * sizeof(T), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return fail(NOLF_ECUDA, "cudaMemcpy: %s", cudaGetErrorString(e));
    *dst = static_cast<T *>(p);
    return 0;
  }
  ~NolfAsset() {
    for (void *p : allocs) cudaFree(p);
    if (dev) cudaFree(dev);
  }
};

namespace {

int upload_atlas(NolfAsset *A, const NolfAtlasDesc &d, int channels, DevAtlas *out, const char *what) {
  if (d.b < 1 || d.r < 1 || d.channels != channels || !d.index)
    return fail(NOLF_EINVAL, "%s atlas: bad shape (b=%d r=%d C=%d)", what, d.b, d.r, d.channels);
  const int b = d.b, s = d.r + 1;
  const int64_t ncell = (int64_t)b * b * b;
  for (int64_t i = 0; i < ncell; ++i)
    if (d.index[i] < -1 || d.index[i] >= d.n_cubes)
      return fail(NOLF_EINVAL, "%s atlas: index entries must reference valid cubes", what);
  out->b = b;
  out->r = d.r;
  out->C = channels;
  out->s = s;
  // Chebyshev (L-inf) distance transform of the occupancy, separable:
  // f1 = 1-D distance along x; f2 = min_y' max(|y-y'|, f1); f3 likewise in z.
  const int INF = 1 << 20;
  std::vector<int> f((size_t)ncell), g((size_t)ncell);
  auto at3 = [b](int x, int y, int z) { return ((size_t)x * b + y) * b + z; };
  for (int y = 0; y < b; ++y)
    for (int z = 0; z < b; ++z) {
      int last = -INF;
      for (int x = 0; x < b; ++x) {
        if (d.index[at3(x, y, z)] != -1) last = x;
        f[at3(x, y, z)] = last == -INF ? INF : x - last;
      }
      last = INF;
      for (int x = b - 1; x >= 0; --x) {
        if (d.index[at3(x, y, z)] != -1) last = x;
        if (last != INF) f[at3(x, y, z)] = std::min(f[at3(x, y, z)], last - x);
      }
    }
  for (int pass = 0; pass < 2; ++pass) {      // pass 0: along y, pass 1: along z
    for (int x = 0; x < b; ++x)
      for (int u = 0; u < b; ++u)
        for (int v = 0; v < b; ++v) {
          int best = INF;
          for (int w = 0; w < b; ++w) {
            const size_t src = pass == 0 ? at3(x, w, u) : at3(x, u, w);
            const int dv = std::max(std::abs(v - w), f[src]);
            best = std::min(best, dv);
          }
          g[pass == 0 ? at3(x, v, u) : at3(x, u, v)] = best;
        }
    f.swap(g);
  }
  std::vector<uint8_t> dist((size_t)ncell);
  for (int64_t i = 0; i < ncell; ++i) dist[(size_t)i] = (uint8_t)std::min(f[(size_t)i], 255);
  // octant fields: r_o(c) = 0 when c is occupied, else 1 + the minimum of r_o
  // over the 7 neighbours c + e_S (S a nonempty subset of the axes, stepping
  // in the octant's direction; outside the grid counts as unbounded): the
  // cube of r_o(c) cells per axis anchored at c in that direction is empty
  std::vector<uint8_t> odist(8 * (size_t)ncell);
  for (int o = 0; o < 8; ++o) {
    const int sx = (o & 1) ? -1 : 1, sy = (o & 2) ? -1 : 1, sz = (o & 4) ? -1 : 1;
    uint8_t *r8 = odist.data() + (size_t)o * ncell;
    for (int ix = 0; ix < b; ++ix)
      for (int iy = 0; iy < b; ++iy)
        for (int iz = 0; iz < b; ++iz) {
          const int x = sx > 0 ? b - 1 - ix : ix, y = sy > 0 ? b - 1 - iy : iy, z = sz > 0 ? b - 1 - iz : iz;
          int m = 255;
          if (d.index[at3(x, y, z)] != -1) {
            m = -1;
          } else {
            for (int S = 1; S < 8; ++S) {
              const int nx = x + ((S & 1) ? sx : 0), ny = y + ((S & 2) ? sy : 0), nz = z + ((S & 4) ? sz : 0);
              if (nx < 0 || ny < 0 || nz < 0 || nx >= b || ny >= b || nz >= b) continue;
              m = std::min(m, (int)r8[at3(nx, ny, nz)]);
            }
          }
          r8[at3(x, y, z)] = (uint8_t)std::min(m + 1, 255);
        }
  }
  int32_t *idx;
  uint8_t *mac;
  float *cubes;
  int rc;
  if ((rc = A->upload(d.index, (size_t)ncell, &idx))) return rc;
  if ((rc = A->upload(dist.data(), dist.size(), &mac))) return rc;
  uint8_t *omac;
  if ((rc = A->upload(odist.data(), odist.size(), &omac))) return rc;
  out->odist = omac;
  const size_t nc = (size_t)d.n_cubes * s * s * s * channels;
  if (nc == 0) {               // keep a valid pointer for empty atlases
    float z4[4] = {0, 0, 0, 0};
    if ((rc = A->upload(z4, 4, &cubes))) return rc;
  } else if ((rc = A->upload(d.cubes, nc, &cubes))) {
    return rc;
  }
  // per-cube sub-voxel zero mask (8 corners exactly 0 -> trilinear value +0)
  const int r = d.r, words = (r * r * r + 31) / 32;
  std::vector<uint32_t> zm((size_t)std::max<int64_t>(d.n_cubes, 1) * words, 0u);
  for (int64_t c = 0; c < d.n_cubes; ++c) {
    const float *cube = d.cubes + (size_t)c * s * s * s * channels;
    for (int x = 0; x < r; ++x)
      for (int y = 0; y < r; ++y)
        for (int z = 0; z < r; ++z) {
          bool zero = true;
          for (int q = 0; q < 8 && zero; ++q) {
            const float *v = cube + ((size_t)((x + (q & 1)) * s + (y + ((q >> 1) & 1))) * s + (z + ((q >> 2) & 1))) * channels;
            for (int ch = 0; ch < channels; ++ch) zero = zero && v[ch] == 0.0f;
          }
          if (zero) {
            const int bit = (x * r + y) * r + z;
            zm[(size_t)c * words + (bit >> 5)] |= 1u << (bit & 31);
          }
        }
  }
  uint32_t *zmp;
  if ((rc = A->upload(zm.data(), zm.size(), &zmp))) return rc;
  out->index = idx;
  out->dist = mac;
  out->cubes = cubes;
  out->cubes16 = nullptr;
  if (channels == 4 && nc > 0) {   // fp16 copy for the bf16 shading path (round to nearest)
    std::vector<uint16_t> h(nc);
    for (size_t i = 0; i < nc; ++i) h[i] = __half_as_ushort(__float2half_rn(d.cubes[i]));
    uint16_t *hp;
    if ((rc = A->upload(h.data(), h.size(), &hp))) return rc;
    out->cubes16 = reinterpret_cast<const uint2 *>(hp);
  }
  out->zmask = zmp;
  out->zwords = words;
  auto pow2 = [](int v) { return v > 0 && (v & (v - 1)) == 0; };
  out->lr = -1;
  if (pow2(b) && pow2(r) && (int64_t)b * r < (1 << 30)) {
    out->lr = 0;
    while ((1 << out->lr) < r) ++out->lr;
  }
  return 0;
}

// Median-split BVH over triangle centroids (longest centroid axis, leaves of
// <= 4 triangles); node boxes rounded outward to fp32 and padded so the fp32
// traversal test only ever over-approximates.
struct BvhBuilder {
  const double *V;
  const int32_t *T;
  std::vector<int> order;
  std::vector<BvhNode> nodes;
  std::vector<double> cen;
  void bounds(int first, int count, double lo[3], double hi[3]) const {
    for (int k = 0; k < 3; ++k) { lo[k] = 1e300; hi[k] = -1e300; }
    for (int i = first; i < first + count; ++i)
      for (int c = 0; c < 3; ++c) {
        const double *v = V + 3ll * T[3ll * order[(size_t)i] + c];
        for (int k = 0; k < 3; ++k) { lo[k] = std::min(lo[k], v[k]); hi[k] = std::max(hi[k], v[k]); }
      }
  }
  // writes the subtree over order[first, first+count) into nodes[slot]
#ifndef NOLF_BVH_LEAF
#define NOLF_BVH_LEAF 4
#endif
  static constexpr int kBvhLeaf = NOLF_BVH_LEAF;   // triangles per leaf at most
  void build(int slot, int first, int count) {
    double lo[3], hi[3];
    bounds(first, count, lo, hi);
    BvhNode n{};
    for (int k = 0; k < 3; ++k) {
      const double pad = 1e-6 * (hi[k] - lo[k]) + 1e-6;
      n.lo[k] = nextafterf((float)(lo[k] - pad), -INFINITY);
      n.hi[k] = nextafterf((float)(hi[k] + pad), INFINITY);
    }
    if (count <= kBvhLeaf) {
      n.first = first;
      n.count = count;
      nodes[(size_t)slot] = n;
      return;
    }
    double clo[3] = {1e300, 1e300, 1e300}, chi[3] = {-1e300, -1e300, -1e300};
    for (int i = first; i < first + count; ++i)
      for (int k = 0; k < 3; ++k) {
        const double c = cen[3ull * order[(size_t)i] + k];
        clo[k] = std::min(clo[k], c);
        chi[k] = std::max(chi[k], c);
      }
    int ax = 0;
    for (int k = 1; k < 3; ++k)
      if (chi[k] - clo[k] > chi[ax] - clo[ax]) ax = k;
    const int mid = first + count / 2;
    std::nth_element(order.begin() + first, order.begin() + mid, order.begin() + first + count, [&](int a, int b) {
      const double ca = cen[3ull * a + ax], cb = cen[3ull * b + ax];
      return ca < cb || (ca == cb && a < b);
    });
    const int left = (int)nodes.size();
    nodes.push_back(BvhNode{});
    nodes.push_back(BvhNode{});
    build(left, first, mid - first);
    build(left + 1, mid, first + count - mid);
    n.first = left;
    n.count = 0;
    nodes[(size_t)slot] = n;
  }
};

int upload_mesh(NolfAsset *A, const NolfAssetDesc &d, DevMesh *out) {
  out->nodes = nullptr;
  out->tri = nullptr;
  out->n_tri = 0;
  out->nodes4 = nullptr;
  if (d.mesh_n_triangles <= 0) return 0;
  if (!d.mesh_vertices || !d.mesh_triangles || d.mesh_n_vertices <= 0)
    return fail(NOLF_EINVAL, "mesh proxy: missing arrays");
  if (d.mesh_n_triangles >= (1ll << 30)) return fail(NOLF_EINVAL, "mesh proxy: too many triangles");
  for (int64_t i = 0; i < 3 * d.mesh_n_triangles; ++i)
    if (d.mesh_triangles[i] < 0 || d.mesh_triangles[i] >= d.mesh_n_vertices)
      return fail(NOLF_EINVAL, "mesh proxy: triangle index out of range");
  for (int64_t i = 0; i < d.mesh_n_vertices; ++i)
    for (int k = 0; k < 3; ++k) {
      const double v = d.mesh_vertices[3 * i + k];
      if (!(v >= d.proxy_min[k] && v <= d.proxy_max[k]))
        return fail(NOLF_EINVAL, "mesh proxy: vertices must lie inside the proxy box");
    }
  BvhBuilder B;
  B.V = d.mesh_vertices;
  B.T = d.mesh_triangles;
  const int nt = (int)d.mesh_n_triangles;
  B.order.resize((size_t)nt);
  B.cen.resize(3ull * nt);
  for (int i = 0; i < nt; ++i) {
    B.order[(size_t)i] = i;
    for (int k = 0; k < 3; ++k) {
      double c = 0;
      for (int v = 0; v < 3; ++v) c += d.mesh_vertices[3ll * d.mesh_triangles[3ll * i + v] + k];
      B.cen[3ull * i + k] = c / 3.0;
    }
  }
  B.nodes.push_back(BvhNode{});
  B.build(0, 0, nt);
  // traversal keeps one far child per level on a 32-entry stack
  // (nolf_mesh.cuh): median splits give depth ceil(log2(nt / 4)) <= 28
  {
    std::vector<std::pair<int, int>> st{{0, 0}};
    int depth = 0;
    while (!st.empty()) {
      const auto [nd, dd] = st.back();
      st.pop_back();
      depth = std::max(depth, dd);
      if (B.nodes[(size_t)nd].count == 0) {
        st.push_back({B.nodes[(size_t)nd].first, dd + 1});
        st.push_back({B.nodes[(size_t)nd].first + 1, dd + 1});
      }
    }
    if (depth > 28) return fail(NOLF_EINVAL, "mesh proxy: BVH depth %d exceeds the traversal stack", depth);
  }
  // the same tree collapsed 4-wide for the warp walk: each 4-wide node takes
  // the binary node's children, then repeatedly the children of its largest
  // inner child, up to 4 slots (leaves stay leaves)
  std::vector<Bvh4Node> n4;
  int depth4 = 0;
  std::function<int(int, int)> collapse = [&](int b, int lvl) -> int {
    depth4 = std::max(depth4, lvl);
    const int idx = (int)n4.size();
    n4.push_back(Bvh4Node{});
    std::vector<int> kids;
    if (B.nodes[(size_t)b].count > 0) kids.push_back(b);    // a leaf root
    else kids = {B.nodes[(size_t)b].first, B.nodes[(size_t)b].first + 1};
    auto area = [&](int k) {
      const BvhNode &c = B.nodes[(size_t)k];
      const double ex = c.hi[0] - c.lo[0], ey = c.hi[1] - c.lo[1], ez = c.hi[2] - c.lo[2];
      return ex * ey + ey * ez + ez * ex;
    };
    while (kids.size() < 4) {
      int bi = -1;
      for (int i = 0; i < (int)kids.size(); ++i)
        if (B.nodes[(size_t)kids[i]].count == 0 && (bi < 0 || area(kids[i]) > area(kids[bi]))) bi = i;
      if (bi < 0) break;
      const int k = kids[(size_t)bi];
      kids.erase(kids.begin() + bi);
      kids.push_back(B.nodes[(size_t)k].first);
      kids.push_back(B.nodes[(size_t)k].first + 1);
    }
    Bvh4Node nn{};
    for (int j = 0; j < 4; ++j) {
      for (int a = 0; a < 3; ++a) nn.lo[a][j] = nn.hi[a][j] = 0.f;
      nn.child[j] = -1;
      nn.count[j] = -1;
    }
    for (int j = 0; j < (int)kids.size(); ++j) {
      const BvhNode c = B.nodes[(size_t)kids[(size_t)j]];
      for (int a = 0; a < 3; ++a) { nn.lo[a][j] = c.lo[a]; nn.hi[a][j] = c.hi[a]; }
      if (c.count > 0) {
        nn.child[j] = c.first;
        nn.count[j] = c.count;
      } else {
        nn.child[j] = collapse(kids[(size_t)j], lvl + 1);
        nn.count[j] = 0;
      }
    }
    n4[(size_t)idx] = nn;
    return idx;
  };
  collapse(0, 0);
  if (3 * (depth4 + 1) + 1 > kMesh4Stack)
    return fail(NOLF_EINVAL, "mesh proxy: 4-wide BVH depth %d exceeds the traversal stack", depth4);
  std::vector<double> tri(9ull * nt);
  for (int i = 0; i < nt; ++i)
    for (int v = 0; v < 3; ++v)
      for (int k = 0; k < 3; ++k)
        tri[9ull * i + 3 * v + k] = d.mesh_vertices[3ll * d.mesh_triangles[3ll * B.order[(size_t)i] + v] + k];
  BvhNode *nd;
  double *tp;
  int rc;
  if ((rc = A->upload(B.nodes.data(), B.nodes.size(), &nd))) return rc;
  if ((rc = A->upload(tri.data(), tri.size(), &tp))) return rc;
  Bvh4Node *nd4;
  if ((rc = A->upload(n4.data(), n4.size(), &nd4))) return rc;
  out->nodes4 = nd4;
  out->nodes = nd;
  out->tri = tp;
  out->n_tri = nt;
  return 0;
}

int pack_mlp(NolfAsset *A, const NolfMlpDesc &m, DevMlp *out, const char *what) {
  if (m.n_layers != 2 && m.n_layers != 3)
    return fail(NOLF_EINVAL, "%s MLP: %d layers unsupported (need 2 or 3)", what, m.n_layers);
  if (m.widths[0] < 1 || m.widths[0] > kInp)
    return fail(NOLF_EINVAL, "%s MLP: input width %d > %d", what, m.widths[0], kInp);
  for (int l = 1; l < m.n_layers; ++l)
    if (m.widths[l] != kHid) return fail(NOLF_EINVAL, "%s MLP: hidden width %d != %d", what, m.widths[l], kHid);
  if (m.widths[m.n_layers] != 4) return fail(NOLF_EINVAL, "%s MLP: output width must be 4", what);
  std::vector<float> P(MlpOff::total, 0.f);
  const int in = m.widths[0];
  for (int o = 0; o < kHid; ++o) {
    for (int i = 0; i < in; ++i) P[MlpOff::w0t + i * kHid + o] = m.w[0][o * in + i];
    P[MlpOff::b0 + o] = m.b[0][o];
  }
  if (m.n_layers == 3) {
    for (int o = 0; o < kHid; ++o) {
      for (int i = 0; i < kHid; ++i) P[MlpOff::w1 + o * kHid + i] = m.w[1][o * kHid + i];
      P[MlpOff::b1 + o] = m.b[1][o];
    }
  }
  const int L = m.n_layers - 1;
  for (int j = 0; j < 4; ++j) {
    for (int i = 0; i < kHid; ++i) P[MlpOff::wl + j * kHid + i] = m.w[L][j * kHid + i];
    P[MlpOff::bl + j] = m.b[L][j];
  }
  int j = 0;
  for (int h = 0; h < m.n_heads; ++h)
    for (int k = 0; k < m.head_w[h]; ++k, ++j) {
      if (j >= 4) return fail(NOLF_EINVAL, "%s MLP: head widths exceed output width", what);
      out->act[j] = m.head_act[h];
    }
  if (j != 4) return fail(NOLF_EINVAL, "%s MLP: head widths must sum to the output width", what);
  out->n_layers = m.n_layers;
  out->in = in;
  float *p;
  int rc = A->upload(P.data(), P.size(), &p);
  out->params = p;
  return rc;
}

int num_sms() {                 // per device (a process may drive several)
  static int sms[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!sms[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    sms[dev] = v > 0 ? v : 148;
  }
  return sms[dev];
}

constexpr size_t kShadeSmem = (size_t)(2 * MlpOff::total + kInp * kShadeThreads) * sizeof(float);

int ensure_attrs() {            // function attributes are per device
  static bool done_dev[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  bool &done = done_dev[dev >= 0 && dev < 64 ? dev : 0];
  if (!done) {
    CUDA_TRY(cudaFuncSetAttribute(k_shade, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kShadeSmem));
    CUDA_TRY(cudaFuncSetAttribute(k_eval_diffuse, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kShadeSmem));
    CUDA_TRY(cudaFuncSetAttribute(k_shade_tc<kShadeTG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)tc_smem_bytes(kShadeTG, kTcPhiMax, kTcTabMax * 4)));
    CUDA_TRY(cudaFuncSetAttribute(k_mlp_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTcSmem));
    CUDA_TRY(cudaFuncSetAttribute(k_mlp_fp32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kShadeSmem));
    done = true;
  }
  return 0;
}

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct Workspace {
  unsigned int *counts;        // per-instance hit counts, then [n_inst]: live chunks, [n_inst+1]: fetch
  unsigned int *chunk_list;    // scene: live 128-slot chunks
  uint8_t *chunk_live;
  unsigned *chunk_cost;        // last frame's per-chunk CTA durations (fixed offset: persists across frames)
  HitRec *queue;
  uint8_t *nhit;
  float *lrgba, *ldepth;
  long long P;                 // pixel slots (layer stride)
};

// queue_recs: total hit-record capacity over instances; layers: compose
// layers per pixel slot (scene mode), P: pixel slots.
size_t ws_layout(int n_inst, long long queue_recs, int layers, long long P, char *base, Workspace *w) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes, 256);
    return base ? base + o : nullptr;
  };
  const size_t n = (size_t)(P > 0 ? P : 1);
  char *counts = take(sizeof(unsigned) * (size_t)((n_inst > 0 ? n_inst : 1) + 2 + kChunkBuckets));
  const size_t n_chunks = (size_t)((P > 0 ? P : 1) + 127) / 128;
  char *chunk_list = take(sizeof(unsigned) * n_chunks * kChunkBuckets);
  char *chunk_live = take(n_chunks);
  char *chunk_cost = take(sizeof(unsigned) * n_chunks);
  char *queue = take(sizeof(HitRec) * (size_t)(queue_recs > 0 ? queue_recs : 1));
  char *nhit = take(layers > 0 ? n : 1);
  char *lrgba = take(sizeof(float) * 4 * n * (size_t)layers);
  char *ldepth = take(sizeof(float) * n * (size_t)layers);
  if (w) {
    w->counts = reinterpret_cast<unsigned *>(counts);
    w->chunk_list = reinterpret_cast<unsigned *>(chunk_list);
    w->chunk_live = reinterpret_cast<uint8_t *>(chunk_live);
    w->chunk_cost = reinterpret_cast<unsigned *>(chunk_cost);
    w->queue = reinterpret_cast<HitRec *>(queue);
    w->nhit = reinterpret_cast<uint8_t *>(nhit);
    w->lrgba = reinterpret_cast<float *>(lrgba);
    w->ldepth = reinterpret_cast<float *>(ldepth);
    w->P = (long long)n;
  }
  return off;
}

int fill_inst(const NolfInstance *in, DevInst *out) {
  if (!in || !in->asset) return fail(NOLF_EINVAL, "null asset instance");
  if (!(in->scale > 0.0)) return fail(NOLF_EINVAL, "instance scale must be positive");
  out->a = in->asset->dev;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 4; ++c) out->w2o[r * 4 + c] = in->w2o[r * 4 + c];
  out->scale = in->scale;
  return 0;
}

int run_shade(const DevInst *inst, const long long *qoff, int n_inst, const Workspace &w, int mode, float *rgba,
              float *depth, long long layer_stride, unsigned long long *counters, cudaStream_t st, bool use_tc,
              uint32_t phi_smem_bytes, uint32_t tab_smem_bytes, long long max_recs = -1);

}  // namespace

// Per-launch instance / camera tables live in a device-side parameter block.
namespace {
// Packed per launch (only what the launch uses crosses PCIe):
//   inst[n_inst] | cams[n_cams] | rect | qoff[n_inst + 1] | cull[n_inst * n_cams]
struct ParamBlock {
  DevInst *inst;
  CamParams *cams;
  TileParams *rect;
  long long *qoff;                       // hit-queue offset of every instance
  ScreenBox *cull;
};

struct ParamLayout {
  size_t inst, cams, rect, qoff, cull, total;
};

ParamLayout param_layout(int n_inst, int n_cams) {
  ParamLayout L;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = (off + bytes + 15) / 16 * 16;
    return o;
  };
  const size_t nc = (size_t)(n_cams > 0 ? n_cams : 1);
  L.inst = take(sizeof(DevInst) * (size_t)n_inst);
  L.cams = take(sizeof(CamParams) * nc);
  L.rect = take(sizeof(TileParams));
  L.qoff = take(sizeof(long long) * (size_t)(n_inst + 1));
  L.cull = take(sizeof(ScreenBox) * (size_t)n_inst * nc);
  L.total = off;
  return L;
}

ParamBlock param_view(void *base, const ParamLayout &L) {
  char *b = static_cast<char *>(base);
  return ParamBlock{reinterpret_cast<DevInst *>(b + L.inst), reinterpret_cast<CamParams *>(b + L.cams),
                    reinterpret_cast<TileParams *>(b + L.rect), reinterpret_cast<long long *>(b + L.qoff),
                    reinterpret_cast<ScreenBox *>(b + L.cull)};
}

size_t param_bytes(int n_inst, int n_cams) { return param_layout(n_inst, n_cams).total; }

// Conservative image rectangle of an instance's culling box (occupied cells,
// see nolf_asset_create) for one camera.
// All 8 world corners strictly in front of the camera: the projection of the
// (convex) box is the hull of the projected corners, so pixels outside their
// bounding rectangle (plus a 2-pixel margin for rounding) cannot hit it.
// Corners behind/on the camera plane: no culling (or none visible when all
// are behind, since every pixel ray goes forward from the camera).
ScreenBox screen_box(const NolfInstance &in, const DevAsset &H, const CamParams &c) {
  const ScreenBox full{-(1 << 29), -(1 << 29), 1 << 29, 1 << 29};
  const double *w = in.w2o;
  const double a00 = w[0], a01 = w[1], a02 = w[2], a10 = w[4], a11 = w[5], a12 = w[6], a20 = w[8], a21 = w[9],
               a22 = w[10];
  const double det = a00 * (a11 * a22 - a12 * a21) - a01 * (a10 * a22 - a12 * a20) + a02 * (a10 * a21 - a11 * a20);
  if (!(det != 0.0) || det != det) return full;
  const double id = 1.0 / det;
  const double Ai[9] = {(a11 * a22 - a12 * a21) * id, (a02 * a21 - a01 * a22) * id, (a01 * a12 - a02 * a11) * id,
                        (a12 * a20 - a10 * a22) * id, (a00 * a22 - a02 * a20) * id, (a02 * a10 - a00 * a12) * id,
                        (a10 * a21 - a11 * a20) * id, (a01 * a20 - a00 * a21) * id, (a00 * a11 - a01 * a10) * id};
  if (H.cull_empty) return ScreenBox{1, 1, 0, 0};
  double xmin = 1e300, xmax = -1e300, ymin = 1e300, ymax = -1e300;
  int behind = 0, near = 0;
  for (int cnr = 0; cnr < 8; ++cnr) {
    const double po[3] = {(cnr & 1) ? H.cull_hi[0] : H.cull_lo[0], (cnr & 2) ? H.cull_hi[1] : H.cull_lo[1],
                          (cnr & 4) ? H.cull_hi[2] : H.cull_lo[2]};
    const double q[3] = {po[0] - w[3], po[1] - w[7], po[2] - w[11]};
    double pw[3];
    for (int r = 0; r < 3; ++r) pw[r] = Ai[3 * r] * q[0] + Ai[3 * r + 1] * q[1] + Ai[3 * r + 2] * q[2];
    const double v[3] = {pw[0] - c.pose[3], pw[1] - c.pose[7], pw[2] - c.pose[11]};
    double cc[3];
    for (int j = 0; j < 3; ++j) cc[j] = c.pose[j] * v[0] + c.pose[4 + j] * v[1] + c.pose[8 + j] * v[2];
    const double depth = -cc[2];
    const double vn = fabs(v[0]) + fabs(v[1]) + fabs(v[2]);
    if (depth <= 1e-7 * (1.0 + vn)) {
      ++near;
      if (depth < 0.0) ++behind;
      continue;
    }
    const double px = cc[0] / depth * c.fx + c.cx - 0.5;
    const double py = -cc[1] / depth * c.fy + c.cy - 0.5;
    xmin = fmin(xmin, px); xmax = fmax(xmax, px);
    ymin = fmin(ymin, py); ymax = fmax(ymax, py);
  }
  if (behind == 8) return ScreenBox{1, 1, 0, 0};
  if (near) return full;
  auto clampi64 = [](double v) { return v < -(1 << 29) ? -(1 << 29) : (v > (1 << 29) ? (1 << 29) : (int)v); };
  return ScreenBox{clampi64(floor(xmin) - 2), clampi64(floor(ymin) - 2), clampi64(ceil(xmax) + 2),
                   clampi64(ceil(ymax) + 2)};
}
// Per-launch memory plan.  A pixel yields at most one hit per instance and
// only inside the instance's screen box, so the box area (clipped to the
// frame, or to the rect) bounds the instance's hit queue; the number of
// boxes overlapping any pixel bounds its compose layers.
struct Plan {
  std::vector<ScreenBox> cull;   // [n_inst * n_cams]
  std::vector<long long> qoff;   // n_inst + 1
  int layers = 0;
  size_t bytes = 0;
};

long long box_area(const ScreenBox &b, int x0, int y0, int x1, int y1) {   // [x0,x1) x [y0,y1)
  const long long w = (long long)std::min(b.x1 + 1, x1) - std::max(b.x0, x0);
  const long long h = (long long)std::min(b.y1 + 1, y1) - std::max(b.y0, y0);
  return (w > 0 && h > 0) ? w * h : 0;
}

void make_plan(int mode, const NolfInstance *ins, int n_inst, const CamParams *cams, int n_cams, TileParams rect,
               long long n_rays, Plan &pl) {
  pl.qoff.assign((size_t)n_inst + 1, 0);
  pl.cull.clear();
  if (mode == kModeRays || n_cams == 0) {
    for (int k = 0; k < n_inst; ++k) pl.qoff[(size_t)k + 1] = pl.qoff[(size_t)k] + n_rays;
    pl.layers = mode == kModeScene ? n_inst : 0;
  } else {
    pl.cull.resize((size_t)n_inst * n_cams);
    for (int k = 0; k < n_inst; ++k)
      for (int c = 0; c < n_cams; ++c) pl.cull[(size_t)k * n_cams + c] = screen_box(ins[k], ins[k].asset->host, cams[c]);
    for (int k = 0; k < n_inst; ++k) {
      long long cap = 0;
      for (int c = 0; c < n_cams; ++c) {
        const ScreenBox &b = pl.cull[(size_t)k * n_cams + c];
        cap += mode == kModeRect ? box_area(b, rect.x0, rect.y0, rect.x1, rect.y1)
                                 : box_area(b, 0, 0, cams[c].width, cams[c].height);
      }
      pl.qoff[(size_t)k + 1] = pl.qoff[(size_t)k] + std::min(cap, n_rays);
    }
    int L = 1;
    if (mode == kModeScene) {
      for (int c = 0; c < n_cams; ++c)
        for (int i = 0; i < n_inst; ++i)
          for (int j = 0; j < n_inst; ++j) {
            const ScreenBox &bi = pl.cull[(size_t)i * n_cams + c], &bj = pl.cull[(size_t)j * n_cams + c];
            const int px = std::max(bi.x0, 0), py = std::max(bj.y0, 0);
            if (px >= cams[c].width || py >= cams[c].height) continue;
            int cnt = 0;
            for (int k = 0; k < n_inst; ++k) {
              const ScreenBox &b = pl.cull[(size_t)k * n_cams + c];
              cnt += px >= b.x0 && px <= b.x1 && py >= b.y0 && py <= b.y1;
            }
            L = std::max(L, cnt);
          }
    }
    pl.layers = mode == kModeScene ? L : 0;
  }
  pl.bytes = ws_layout(n_inst, pl.qoff[(size_t)n_inst], pl.layers, n_rays, nullptr, nullptr);
}

void fill_cams(const NolfCamera *cams, int n_cams, CamParams *out) {
  long long pix_base = 0;
  for (int c = 0; c < n_cams; ++c) {
    const NolfCamera &C = cams[c];
    for (int q = 0; q < 16; ++q) out[c].pose[q] = C.pose[q];
    out[c].fx = C.fx;
    out[c].fy = C.fy;
    out[c].cx = C.cx;
    out[c].cy = C.cy;
    out[c].width = C.width;
    out[c].height = C.height;
    out[c].pix_base = pix_base;
    pix_base += (long long)C.width * C.height;
  }
}

}  // namespace

extern "C" {

int nolf_abi_version(void) { return NOLF_ABI_VERSION; }
const char *nolf_last_error(void) { return g_err.c_str(); }

int nolf_asset_create(const NolfAssetDesc *d, int device, nolf_asset_t *out) {
  if (!d || !out) return fail(NOLF_EINVAL, "null argument");
  *out = nullptr;
  int prev_dev = 0;
  CUDA_TRY(cudaGetDevice(&prev_dev));
  CUDA_TRY(cudaSetDevice(device));
  DeviceRestore restore_{prev_dev};   // the caller's current device on every exit
  NolfAsset *A = new NolfAsset();
  A->device = device;
  DevAsset &H = A->host;
  int rc = 0;
  auto bail = [&](int code) { delete A; return code; };
  if ((rc = upload_atlas(A, d->density, 1, &H.den, "density"))) return bail(rc);
  H.has_dif = d->has_diffuse_atlas ? 1 : 0;
  if (H.has_dif && (rc = upload_atlas(A, d->diffuse, 4, &H.dif, "diffuse"))) return bail(rc);
  // PSH
  if (d->psh_resolution < 1 || d->psh_table_size < 1 || d->psh_offset_size < 1 || !d->psh_offsets ||
      !d->psh_features)
    return bail(fail(NOLF_EINVAL, "psh: missing table"));
  if (d->psh_table_size >= (1ll << 30) || d->psh_offset_size >= (1ll << 30))
    return bail(fail(NOLF_EINVAL, "psh: table too large for u32 slot arithmetic"));
  if (d->psh_features_dim < 1 || d->psh_features_dim > 4)
    return bail(fail(NOLF_EINVAL, "psh: feature dim %d unsupported (1..4)", d->psh_features_dim));
  H.N = d->psh_resolution;
  H.m = (uint32_t)d->psh_table_size;
  H.mphi = (uint32_t)d->psh_offset_size;
  H.F = d->psh_features_dim;
  {
    std::vector<uint32_t> phi((size_t)d->psh_offset_size);
    for (int64_t i = 0; i < d->psh_offset_size; ++i) {
      int64_t v = d->psh_offsets[i];
      if (v < 0 || v >= d->psh_table_size) return bail(fail(NOLF_EINVAL, "psh: offset out of range"));
      phi[(size_t)i] = (uint32_t)v;
    }
    const int s = H.N + 1;
    std::vector<uint32_t> tab((size_t)6 * s);
    for (int a = 0; a < 3; ++a)
      for (int x = 0; x < s; ++x) {
        tab[(size_t)a * s + x] = (uint32_t)(((uint64_t)x * d->primes_h0[a]) % (uint64_t)H.m);
        tab[(size_t)(3 + a) * s + x] = (uint32_t)(((uint64_t)x * d->primes_h1[a]) % (uint64_t)H.mphi);
      }
    uint32_t *pp, *tp;
    float *fp;
    if ((rc = A->upload(phi.data(), phi.size(), &pp))) return bail(rc);
    if ((rc = A->upload(tab.data(), tab.size(), &tp))) return bail(rc);
    if ((rc = A->upload(d->psh_features, (size_t)d->psh_table_size * H.F, &fp))) return bail(rc);
    H.phi = pp;
    H.tab = tp;
    H.feat = fp;
  }
  // hash grid (live diffuse)
  H.hg_levels = d->hg_levels;
  H.hg_F = d->hg_features;
  H.hg_table = (unsigned long long)d->hg_table_size;
  if (H.hg_levels < 0 || H.hg_levels > kMaxLevels) return bail(fail(NOLF_EINVAL, "hash grid: bad level count"));
  for (int l = 0; l < H.hg_levels; ++l) {
    H.hg_res[l] = d->hg_resolution[l];
    H.hg_dense[l] = d->hg_dense[l];
    float *fp;
    if ((rc = A->upload(d->hg_feat[l], (size_t)d->hg_rows[l] * H.hg_F, &fp))) return bail(rc);
    H.hg_feat[l] = fp;
  }
  if ((rc = pack_mlp(A, d->specular, &H.fs, "specular"))) return bail(rc);
  if (d->diffuse_mlp.n_layers) {
    if ((rc = pack_mlp(A, d->diffuse_mlp, &H.fd, "diffuse"))) return bail(rc);
  } else {
    H.fd.params = nullptr;
  }
  // tensor-core tables: bf16 specular weights in the UMMA K-major layout
  // (core matrix (row group g, K chunk c) at c*(rows/8)*128 + g*128) + u16 Phi
  if (d->specular.n_layers == 3 && d->specular.widths[0] <= kTcIn) {
    std::vector<uint16_t> wt(kTcWBytes / 2, 0);
    auto bf16 = [](float f) {
      uint32_t u;
      memcpy(&u, &f, 4);
      u += 0x7FFFu + ((u >> 16) & 1u);            // round to nearest even
      return (uint16_t)(u >> 16);
    };
    auto bf16_f = [](uint16_t h) {
      const uint32_t u = (uint32_t)h << 16;
      float f;
      memcpy(&f, &u, 4);
      return f;
    };
    // element (row, k) of a K-major operand with `rows` rows at base_elems
    auto put = [&](size_t base_elems, int rows, int row, int k, uint16_t v) {
      const size_t off = (size_t)(k >> 3) * (rows / 8) * 128 + (size_t)(row >> 3) * 128 + (row & 7) * 16 + (k & 7) * 2;
      wt[base_elems + off / 2] = v;
    };
    // an fp32 bias as bf16 hi + lo in K columns (k, k+1)
    auto put_bias = [&](size_t base_elems, int rows, int row, int k, float b) {
      const uint16_t hi = bf16(b);
      put(base_elems, rows, row, k, hi);
      put(base_elems, rows, row, k + 1, bf16(b - bf16_f(hi)));
    };
    const int in = d->specular.widths[0];
    const size_t e_w1 = kOffW1 / 2, e_w2 = kOffW2 / 2, e_w1b = kOffW1b / 2, e_w2b = kOffW2b / 2,
                 e_one = kOffOne / 2;
    for (int o = 0; o < 64; ++o) {
      for (int i = 0; i < in; ++i) put(0, 64, o, i, bf16(d->specular.w[0][o * in + i]));
      put_bias(0, 64, o, kTcIn, d->specular.b[0][o]);
      for (int i = 0; i < 64; ++i) put(e_w1, 64, o, i, bf16(d->specular.w[1][o * 64 + i]));
      put_bias(e_w1b, 64, o, 0, d->specular.b[1][o]);
    }
    // W2 (4 x 64) as a 16-row operand (rows 4..15 zero)
    for (int o = 0; o < 4; ++o) {
      for (int i = 0; i < 64; ++i) put(e_w2, 16, o, i, bf16(d->specular.w[2][o * 64 + i]));
      put_bias(e_w2b, 16, o, 0, d->specular.b[2][o]);
    }
    // the broadcast ones operand: one core matrix of rows {1, 1, 0 ...}
    for (int r = 0; r < 8; ++r) wt[e_one + r * 8] = wt[e_one + r * 8 + 1] = bf16(1.0f);
    // the shader's shared-memory image after the bf16 weights: [the fp32
    // block (W2 hidden-major [o][4], b2) for -DNOLF_SHADE_L2_FP32 builds] and
    // the PSH residue tables when they fit, so one TMA bulk copy stages all of it
    const int nt = 6 * (H.N + 1);
    const size_t tab_bytes = tc_tab_bytes(H.N);
    std::vector<uint8_t> img(kTcWBytes + kTcF32 * 4 + tab_bytes, 0);
    memcpy(img.data(), wt.data(), kTcWBytes);
    if (kTcF32) {
      std::vector<float> fpb((size_t)std::max(kTcF32, 1), 0.f);
      for (int q = 128; q < kTcF32; ++q)
        fpb[q] = q < 128 + 256 ? d->specular.w[2][((q - 128) & 3) * 64 + ((q - 128) >> 2)] : d->specular.b[2][q - 384];
      memcpy(img.data() + kTcWBytes, fpb.data(), (size_t)kTcF32 * 4);
    }
    if (tab_bytes) {
      std::vector<uint32_t> tab((size_t)nt);
      const int s1 = H.N + 1;
      for (int a = 0; a < 3; ++a)
        for (int x = 0; x < s1; ++x) {
          tab[(size_t)a * s1 + x] = (uint32_t)(((uint64_t)x * d->primes_h0[a]) % (uint64_t)H.m);
          tab[(size_t)(3 + a) * s1 + x] = (uint32_t)(((uint64_t)x * d->primes_h1[a]) % (uint64_t)H.mphi);
        }
      memcpy(img.data() + kTcWBytes + kTcF32 * 4, tab.data(), (size_t)nt * 4);
    }
    uint8_t *tw;
    if ((rc = A->upload(img.data(), img.size(), &tw))) return bail(rc);
    H.tc_w = tw;
    H.tc_w_bytes = (uint32_t)img.size();
  }
  if (d->psh_table_size <= 65536) {
    const size_t n16 = ((size_t)d->psh_offset_size + 7) / 8 * 8;
    std::vector<uint16_t> p16(n16, 0);
    for (int64_t i = 0; i < d->psh_offset_size; ++i) p16[(size_t)i] = (uint16_t)d->psh_offsets[i];
    uint16_t *pp16;
    if ((rc = A->upload(p16.data(), p16.size(), &pp16))) return bail(rc);
    H.phi16 = pp16;
    H.phi16_bytes = (uint32_t)(n16 * 2);
  }
  const int expect_in = H.F + 16 + (d->refine_opacity ? 1 : 0);
  if (H.fs.in != expect_in)
    return bail(fail(NOLF_EINVAL, "specular MLP input %d != F+16+refine %d", H.fs.in, expect_in));
  if (!H.has_dif && d->use_diffuse_color) {
    if (!H.fd.params) return bail(fail(NOLF_EINVAL, "no diffuse atlas and no diffuse MLP"));
    if (H.fd.in != H.hg_levels * H.hg_F || H.hg_F > 4)
      return bail(fail(NOLF_EINVAL, "diffuse MLP input %d != levels*F %d", H.fd.in, H.hg_levels * H.hg_F));
  }
  H.step = d->step;
  H.t_stop = d->t_stop;
  H.alpha_floor = d->alpha_floor;
  if (!(H.step > 0.0)) return bail(fail(NOLF_EINVAL, "march step must be positive"));
  H.inv_step = 1.0 / H.step;
  H.inv_step_f = (float)(1.0 / H.step);
  H.inv_b_f = 1.0f / (float)H.den.b;
  for (int k = 0; k < 3; ++k) {
    H.pmin[k] = d->proxy_min[k];
    H.pmax[k] = d->proxy_max[k];
  }
  if ((rc = upload_mesh(A, *d, &H.mesh))) return bail(rc);
  {
    // Rays that never enter an occupied cell sample only empty cells: sigma = 0
    // everywhere, so the march returns "miss, 0 samples" exactly.  A pixel whose
    // ray misses the occupied-cell AABB (grown by a full cell, far beyond any
    // rounding of sample positions) can therefore skip the asset entirely.
    const int b = d->density.b;
    int lo[3] = {b, b, b}, hi[3] = {-1, -1, -1};
    for (int x = 0; x < b; ++x)
      for (int y = 0; y < b; ++y)
        for (int z = 0; z < b; ++z)
          if (d->density.index[((int64_t)x * b + y) * b + z] != -1) {
            const int c[3] = {x, y, z};
            for (int k = 0; k < 3; ++k) {
              lo[k] = std::min(lo[k], c[k]);
              hi[k] = std::max(hi[k], c[k]);
            }
          }
    H.cull_empty = hi[0] < 0 ? 1 : 0;
    for (int k = 0; k < 3; ++k) {
      double l = (lo[k] - 1) / (double)b, h = (hi[k] + 2) / (double)b;
      if (l <= 0.0) l = std::min(0.0, d->proxy_min[k]);   // clipped positions reach face cells
      if (h >= 1.0) h = std::max(1.0, d->proxy_max[k]);
      H.cull_lo[k] = std::max(l, d->proxy_min[k]);
      H.cull_hi[k] = std::min(h, d->proxy_max[k]);
    }
  }
  H.use_hit_point = d->use_hit_point;
  H.use_opacity = d->use_opacity;
  H.refine_opacity = d->refine_opacity;
  H.use_tint = d->use_tint;
  H.use_diffuse_color = d->use_diffuse_color;
  H.mlp_mode = NOLF_MLP_FP32;
  cudaError_t e = cudaMalloc(&A->dev, sizeof(DevAsset));
  if (e != cudaSuccess) return bail(fail(NOLF_ENOMEM, "cudaMalloc asset: %s", cudaGetErrorString(e)));
  e = cudaMemcpy(A->dev, &H, sizeof(DevAsset), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return bail(fail(NOLF_ECUDA, "cudaMemcpy asset: %s", cudaGetErrorString(e)));
  A->bytes += sizeof(DevAsset);
  *out = A;
  return 0;
}

int nolf_asset_destroy(nolf_asset_t a) {
  if (!a) return 0;
  int prev_dev = 0;
  cudaGetDevice(&prev_dev);
  cudaSetDevice(a->device);
  DeviceRestore restore_{prev_dev};
  delete a;
  return 0;
}

int nolf_asset_set_mlp_mode(nolf_asset_t a, int mode) {
  if (!a) return fail(NOLF_EINVAL, "null asset");
  if (mode != NOLF_MLP_FP32 && mode != NOLF_MLP_BF16) return fail(NOLF_EINVAL, "unknown MLP mode %d", mode);
  if (mode == NOLF_MLP_BF16) {
    if (!a->host.tc_w) return fail(NOLF_EINVAL, "bf16 tensor-core MLP needs a 3-layer specular net with <= 30 inputs");
    if (a->host.use_diffuse_color && !a->host.has_dif)
      return fail(NOLF_EINVAL, "bf16 tensor-core shading needs a baked diffuse atlas (live diffuse runs in fp32)");
  }
  a->host.mlp_mode = mode;
  CUDA_TRY(cudaMemcpy(a->dev, &a->host, sizeof(DevAsset), cudaMemcpyHostToDevice));
  return 0;
}

int64_t nolf_asset_device_bytes(nolf_asset_t a) { return a ? a->bytes : 0; }

size_t nolf_workspace_bytes(int32_t n_inst, int64_t n_rays) {
  return ws_layout(n_inst, (long long)n_inst * n_rays, n_inst, n_rays, nullptr, nullptr);
}

size_t nolf_scene_workspace_bytes(const NolfInstance *inst, int32_t n_inst, const NolfCamera *cams, int32_t n_cams,
                                  int64_t n_rays) {
  if (!inst || !cams || n_inst < 1 || n_inst > kMaxInst || n_cams < 1 || n_cams > kMaxCams) return 0;
  for (int k = 0; k < n_inst; ++k)
    if (!inst[k].asset) return 0;
  std::vector<CamParams> cp((size_t)n_cams);
  fill_cams(cams, n_cams, cp.data());
  Plan pl;
  make_plan(kModeScene, inst, n_inst, cp.data(), n_cams, TileParams{0, 0, 0, 0, 0}, n_rays, pl);
  return pl.bytes;
}

}  // extern "C"

namespace {

// Launch-variant knobs (nolf_set_option), per thread; defaults from the
// environment (NOLF_HEAVY_WAVES, NOLF_COMPOSE_G) at first use.
struct Options {
  long long heavy_waves = 3;   // marcher launches below this many CTA waves go heaviest-chunk-first
  int march_order = 0;         // 0 auto, 1 spatial list, 2 heavy-first buckets
  int compose_slots = 0;       // live-chunk compose slots per thread: 0 auto, 4, 8
  int march_split = 1;         // CTAs per live chunk in the chunked marcher: 1 or 2
  int chunk_cost = 1;          // heavy-first buckets: 1 last frame's CTA durations, 0 candidate counts
  long long cost_waves = 96;   // auto order: duration-ordered heaviest-first below this many CTA waves
  bool init = false;
};
thread_local Options g_opt;

Options &options() {
  if (!g_opt.init) {
    if (const char *e = getenv("NOLF_HEAVY_WAVES")) g_opt.heavy_waves = atoll(e);
    if (const char *e = getenv("NOLF_COMPOSE_G")) g_opt.compose_slots = atoi(e);
    if (const char *e = getenv("NOLF_MARCH_SPLIT")) g_opt.march_split = atoi(e) == 2 ? 2 : 1;
    if (const char *e = getenv("NOLF_CHUNK_COST")) g_opt.chunk_cost = atoi(e) ? 1 : 0;
    if (const char *e = getenv("NOLF_COST_WAVES")) g_opt.cost_waves = atoll(e);
    g_opt.init = true;
  }
  return g_opt;
}

// Sticky device error counters (kErr*, nolf_kernels.cuh) per device, read
// back asynchronously after every render call on a side stream; an increase
// fails the next call on this thread (or nolf_check_errors) with
// NOLF_ECAPACITY -- the dropped work is never silently blended.
struct ErrState {
  unsigned *dev = nullptr;     // [kNumErr] device counters (monotone)
  unsigned *host = nullptr;    // pinned mirror
  cudaEvent_t ev = nullptr, ev_done = nullptr;
  bool pending = false;
  unsigned seen[kNumErr] = {0, 0, 0, 0};
};
constexpr int kMaxDevices = 64;
thread_local ErrState g_errs[kMaxDevices];

int cur_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev >= 0 && dev < kMaxDevices ? dev : 0;
}

int err_state(ErrState **out) {
  ErrState &E = g_errs[cur_device()];
  if (!E.dev) {
    CUDA_TRY(cudaMalloc(&E.dev, sizeof(unsigned) * kNumErr));
    CUDA_TRY(cudaMemset(E.dev, 0, sizeof(unsigned) * kNumErr));
    CUDA_TRY(cudaMallocHost(&E.host, sizeof(unsigned) * kNumErr));
    memset(E.host, 0, sizeof(unsigned) * kNumErr);
    CUDA_TRY(cudaEventCreateWithFlags(&E.ev, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&E.ev_done, cudaEventDisableTiming));
  }
  *out = &E;
  return 0;
}

int report_errors(ErrState &E) {
  const char *what[kNumErr] = {"hit records dropped: an instance's hit queue overflowed",
                               "hits dropped: more hits than compose layers at a pixel",
                               "scene tiles skipped: outside their camera's frame, larger than tile_stride or "
                               "naming a missing camera",
                               "BVH nodes dropped: traversal stack overflow"};
  for (int i = 0; i < kNumErr; ++i)
    if (E.host[i] != E.seen[i]) {
      const unsigned n = E.host[i] - E.seen[i];
      for (int j = 0; j < kNumErr; ++j) E.seen[j] = E.host[j];
      return fail(NOLF_ECAPACITY, "%u %s (device error counter %d)", n, what[i], i);
    }
  return 0;
}

// Non-blocking: fold in the last read-back if it has landed.
int poll_errors() {
  ErrState *E;
  int rc;
  if ((rc = err_state(&E))) return rc;
  if (E->pending && cudaEventQuery(E->ev_done) == cudaSuccess) {
    E->pending = false;
    return report_errors(*E);
  }
  return 0;
}

// Queue a read-back of the counters after the work on st (side stream aux).
int post_errors(cudaStream_t st, cudaStream_t aux) {
  ErrState *E;
  int rc;
  if ((rc = err_state(&E))) return rc;
  if (E->pending) return 0;
  CUDA_TRY(cudaEventRecord(E->ev, st));
  CUDA_TRY(cudaStreamWaitEvent(aux, E->ev, 0));
  CUDA_TRY(cudaMemcpyAsync(E->host, E->dev, sizeof(unsigned) * kNumErr, cudaMemcpyDeviceToHost, aux));
  CUDA_TRY(cudaEventRecord(E->ev_done, aux));
  E->pending = true;
  return 0;
}

// nolf_last_launch: the variants the calling thread's last scene launch ran
// {chunked live-chunk march, heavy_first, compose slots per thread (0 = k_compose), mlp bf16}
thread_local int32_t g_last_launch[4] = {0, 0, 0, 0};

// nolf_debug_psh_slots: PSH-slot read-back buffer of the calling thread
thread_local uint32_t *g_dbg_slots = nullptr;
thread_local long long g_dbg_rows = 0;

int run_shade(const DevInst *inst, const long long *qoff, int n_inst, const Workspace &w, int mode, float *rgba,
              float *depth, long long layer_stride, unsigned long long *counters, cudaStream_t st, bool use_tc,
              uint32_t phi_smem_bytes, uint32_t tab_smem_bytes, long long max_recs) {
  ShadeArgs sa{};
  sa.dbg_slots = g_dbg_slots;
  sa.dbg_rows = g_dbg_rows;
  sa.inst = inst;
  sa.n_inst = n_inst;
  sa.queue = w.queue;
  sa.qoff = qoff;
  sa.counts = w.counts;
  sa.mode = mode;
  sa.rgba = rgba;
  sa.depth = depth;
  sa.layer_stride = layer_stride;
  sa.counters = counters;
  if (use_tc) {
    sa.tab_bytes = tab_smem_bytes;
    // dynamic smem sized to the largest Phi the launch stages (not the 64 KB
    // worst case) so more CTAs fit per SM
    sa.tile_order = 1;               // blocked tile ranges per CTA
    const size_t smem = tc_smem_bytes(kShadeTG, phi_smem_bytes, sa.tab_bytes);
    // resident CTAs per SM from registers and shared memory (TMEM: 64
    // columns per tile group, never the limit here)
    static int regs = 0;
    static size_t static_smem = 0;
    if (!regs) {
      cudaFuncAttributes fa{};
      CUDA_TRY(cudaFuncGetAttributes(&fa, k_shade_tc<kShadeTG>));
      regs = fa.numRegs > 0 ? fa.numRegs : 168;
      static_smem = fa.sharedSizeBytes;
    }
    const int threads = 128 * kShadeTG;
    const int by_regs = 65536 / (((regs + 7) / 8 * 8) * threads);
    const int by_smem = (int)((227u * 1024u) / (smem + static_smem + 1024u));
    const int by_tmem = 512 / (kTcCols * kShadeTG);
    const int per_sm = std::max(1, std::min(std::min(by_regs, by_smem), by_tmem));
    g_last_launch[3] = per_sm;
    // no more CTAs than 128-hit tiles the queues can hold (small launches:
    // a farm worker's 32x32 tile needs at most 8 per instance)
    long long grid = (long long)num_sms() * per_sm;
    if (max_recs >= 0) grid = std::max(1ll, std::min(grid, (max_recs + 127) / 128 + n_inst));
    k_shade_tc<kShadeTG><<<(unsigned)grid, threads, smem, st>>>(sa);
  } else {
    long long grid = (long long)num_sms() * 3;
    if (max_recs >= 0) grid = std::max(1ll, std::min(grid, (max_recs + kShadeThreads - 1) / kShadeThreads));
    k_shade<<<(unsigned)grid, kShadeThreads, kShadeSmem, st>>>(sa);
  }
  CUDA_TRY(cudaGetLastError());
  return 0;
}

// Device-resident copies of the per-launch instance / camera tables.  They
// are written with cudaMemcpyAsync from pinned staging on the caller's
// stream, so consecutive launches on one stream never race.
struct ParamRing {
  char *host = nullptr;
  char *dev = nullptr;
  size_t slot_bytes = 0;
  int slots = 0, next = 0;
  cudaEvent_t *done = nullptr;
};
thread_local ParamRing g_rings[kMaxDevices];   // per device: kernels read their own GPU's copy

// A staging slot of at least `bytes` (the ring grows -- after draining --
// when a launch needs more than any before).
int ring_acquire(size_t bytes, char **h, char **d, int *slot) {
  ParamRing &R = g_rings[cur_device()];
  if (!R.host || bytes > R.slot_bytes) {
    if (R.host) {
      for (int i = 0; i < R.slots; ++i) CUDA_TRY(cudaEventSynchronize(R.done[i]));
      cudaFreeHost(R.host);
      cudaFree(R.dev);
    } else {
      R.slots = 8;
      R.done = new cudaEvent_t[R.slots];
      for (int i = 0; i < R.slots; ++i) CUDA_TRY(cudaEventCreateWithFlags(&R.done[i], cudaEventDisableTiming));
    }
    R.slot_bytes = std::max<size_t>((bytes + 255) / 256 * 256, 16384);
    CUDA_TRY(cudaMallocHost(&R.host, R.slot_bytes * R.slots));
    CUDA_TRY(cudaMalloc(&R.dev, R.slot_bytes * R.slots));
    for (int i = 0; i < R.slots; ++i) CUDA_TRY(cudaEventRecord(R.done[i], 0));
    R.next = 0;
  }
  int s = R.next;
  R.next = (R.next + 1) % R.slots;
  CUDA_TRY(cudaEventSynchronize(R.done[s]));   // host staging slot free again
  *h = R.host + (size_t)s * R.slot_bytes;
  *d = R.dev + (size_t)s * R.slot_bytes;
  *slot = s;
  return 0;
}

int ring_release(int slot, cudaStream_t st) {
  CUDA_TRY(cudaEventRecord(g_rings[cur_device()].done[slot], st));
  return 0;
}

// Optional per-kernel timing: CUDA events recorded on the launching stream
// around k_march / k_shade / k_compose of every render call, kept in a ring
// so a whole timed region can be read back after it ends.
constexpr int kProfRing = 4096;
struct Prof {
  bool on = false;
  bool created = false;
  int calls = 0;               // render calls recorded since nolf_profile(1)
  cudaEvent_t ev[kProfRing][4];
};
thread_local Prof *g_prof = nullptr;

int prof_mark(int i, cudaStream_t st) {
  if (!g_prof || !g_prof->on) return 0;
  if (g_prof->calls >= kProfRing) return 0;
  CUDA_TRY(cudaEventRecord(g_prof->ev[g_prof->calls][i], st));
  if (i == 3) ++g_prof->calls;
  return 0;
}

// A side stream per launching stream (thread-local cache of one): the
// parameter upload and the live-count read-back run there so the launch
// stream's kernels never queue behind a PCIe round trip.
struct Aux {
  cudaStream_t for_st = nullptr, s = nullptr;
  cudaEvent_t ev_param = nullptr, ev_cull = nullptr;
  int device = -1;
};
thread_local Aux g_aux;

Aux &aux_for(cudaStream_t st) {
  Aux &a = g_aux;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!a.s || a.device != dev) {
    if (a.s) {
      cudaStreamSynchronize(a.s);
      cudaStreamDestroy(a.s);
      cudaEventDestroy(a.ev_param);
      cudaEventDestroy(a.ev_cull);
      a.s = nullptr;
    }
    cudaError_t e = cudaStreamCreateWithFlags(&a.s, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&a.ev_param, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&a.ev_cull, cudaEventDisableTiming);
    if (e != cudaSuccess) {
      g_err = cudaGetErrorString(e);
      a.s = nullptr;
      return a;
    }
    a.device = dev;
  }
  a.for_st = st;
  return a;
}

// Live-chunk count of an earlier frame per (workspace, stream): sizes the
// marcher's grid without a host wait.
struct LiveEstimate {
  void *ws = nullptr;
  long long n_chunks = 0;
  cudaStream_t st = nullptr;
  unsigned *host = nullptr;
  cudaEvent_t ev = nullptr;
  bool pending = false;
  long long last = 0;
};
thread_local LiveEstimate g_live;

int launch_march_shade(int mode, const NolfInstance *ins, int n_inst, const NolfCamera *cams, int n_cams,
                       const NolfTile *tiles_dev, int n_tiles, TileParams rect, long long n_rays,
                       long long tile_stride, const double *origins, int origin_stride, const double *dirs,
                       float *rgba, float *depth, const NolfSceneOut *sout, double alpha_vis,
                       unsigned long long *counters, void *workspace, size_t ws_bytes, cudaStream_t st) {
  if (n_inst < 1 || n_inst > kMaxInst) return fail(NOLF_EINVAL, "instance count %d outside 1..%d", n_inst, kMaxInst);
  if (n_cams > kMaxCams) return fail(NOLF_EINVAL, "camera count %d > %d", n_cams, kMaxCams);
  if (!counters) return fail(NOLF_EINVAL, "counters pointer required");
  if (mode == kModeScene && n_inst > 255) return fail(NOLF_EINVAL, "too many layers");
  const int dev_now = cur_device();
  for (int k = 0; k < n_inst; ++k) {
    if (!ins[k].asset) return fail(NOLF_EINVAL, "null asset instance");
    if (ins[k].asset->device != dev_now)
      return fail(NOLF_EINVAL, "instance %d: asset lives on device %d, the current device is %d", k,
                  ins[k].asset->device, dev_now);
  }
  int rc0;
  if ((rc0 = poll_errors())) return rc0;    // an earlier launch dropped work: fail loudly
  ErrState *errs;
  if ((rc0 = err_state(&errs))) return rc0;
  std::vector<CamParams> hcams((size_t)std::max(n_cams, 1));
  fill_cams(cams, n_cams, hcams.data());
  thread_local Plan pl;
  make_plan(mode, ins, n_inst, hcams.data(), n_cams, rect, n_rays, pl);
  if (!workspace || ws_bytes < pl.bytes) return fail(NOLF_EINVAL, "workspace too small: %zu < %zu", ws_bytes, pl.bytes);
  int rc;
  if ((rc = ensure_attrs())) return rc;
  Workspace w;
  ws_layout(n_inst, pl.qoff[(size_t)n_inst], pl.layers, n_rays, static_cast<char *>(workspace), &w);
  const ParamLayout PL = param_layout(n_inst, n_cams);
  char *hraw, *draw;
  int slot;
  if ((rc = ring_acquire(PL.total, &hraw, &draw, &slot))) return rc;
  ParamBlock hb = param_view(hraw, PL), db = param_view(draw, PL);
  ParamBlock *hp = &hb, *dp = &db;
  bool use_tc = true;
  uint32_t phi_smem = 0, tab_smem = 0;
  for (int k = 0; k < n_inst; ++k) {
    if ((rc = fill_inst(ins + k, hp->inst + k))) return rc;
    const DevAsset &H = ins[k].asset->host;
    use_tc = use_tc && H.mlp_mode == NOLF_MLP_BF16;
    if (H.phi16 && H.phi16_bytes <= kTcPhiMax) phi_smem = std::max(phi_smem, H.phi16_bytes);
    tab_smem = std::max(tab_smem, tc_tab_bytes(H.N));
  }
  for (int c = 0; c < n_cams; ++c) hp->cams[c] = hcams[(size_t)c];
  *hp->rect = rect;
  for (int k = 0; k <= n_inst; ++k) hp->qoff[k] = pl.qoff[(size_t)k];
  for (size_t i = 0; i < pl.cull.size(); ++i) hp->cull[i] = pl.cull[i];
  // the parameter block goes up on a side stream (the copy overlaps the
  // previous frame's kernels); the launch stream waits for it
  Aux &ax = aux_for(st);
  if (!ax.s) return fail(NOLF_ECUDA, "aux stream: %s", g_err.c_str());
  CUDA_TRY(cudaMemcpyAsync(draw, hraw, PL.total, cudaMemcpyHostToDevice, ax.s));
  CUDA_TRY(cudaEventRecord(ax.ev_param, ax.s));
  CUDA_TRY(cudaStreamWaitEvent(st, ax.ev_param, 0));
  if (n_rays == 0) return ring_release(slot, st);
  CUDA_TRY(cudaMemsetAsync(w.counts, 0, sizeof(unsigned) * (n_inst + 2 + kChunkBuckets), st));

  g_last_launch[0] = g_last_launch[1] = g_last_launch[2] = 0;
  g_last_launch[3] = use_tc ? 1 : 0;
  MarchArgs ma{};
  ma.inst = dp->inst;
  ma.n_inst = n_inst;
  ma.origins = origins;
  ma.origin_stride = origin_stride;
  ma.dirs = dirs;
  ma.n_rays = n_rays;
  ma.cams = dp->cams;
  ma.tiles = mode == kModeScene ? reinterpret_cast<const TileParams *>(tiles_dev) : dp->rect;
  ma.tile_stride = tile_stride;
  ma.cull = n_cams > 0 ? dp->cull : nullptr;
  ma.use_zmask = 1;
  ma.n_cams = n_cams > 0 ? n_cams : 1;
  ma.queue = w.queue;
  ma.qoff = dp->qoff;
  ma.counts = w.counts;
  ma.rgba = rgba;
  ma.depth = depth;
  ma.nhit = w.nhit;
  ma.counters = counters;
  ma.max_layers = pl.layers;
  ma.errors = errs->dev;
  const unsigned grid = (unsigned)((n_rays + kMarchThreads - 1) / kMarchThreads);
  const bool chunked = mode == kModeScene && n_cams > 0 && tile_stride % kMarchThreads == 0;
  g_last_launch[0] = chunked ? 1 : 0;
  if ((rc = prof_mark(0, st))) return rc;
  if (mode == kModeRays) k_march<kModeRays><<<grid, kMarchThreads, 0, st>>>(ma);
  else if (mode == kModeRect) k_march<kModeRect><<<grid, kMarchThreads, 0, st>>>(ma);
  else if (!chunked && n_inst > 64) k_march<kModeScene, true><<<grid, kMarchThreads, 0, st>>>(ma);
  else if (!chunked) k_march<kModeScene><<<grid, kMarchThreads, 0, st>>>(ma);
  else {                       // compact the live chunks, then a persistent marcher drains them
    const long long n_chunks = n_rays / kMarchThreads;
    ma.chunks = w.chunk_list;
    ma.n_chunks = w.counts + n_inst;
    ma.list_stride = n_chunks;
    ma.fetch = w.counts + n_inst + 1;
    // grid from the last live count that has landed on the host (async
    // read-back of an earlier frame on this workspace; worst case at first)
    LiveEstimate &le = g_live;
    if (le.ws != workspace || le.n_chunks != n_chunks || le.st != st) {
      if (!le.host) {
        CUDA_TRY(cudaMallocHost(&le.host, sizeof(unsigned)));
        CUDA_TRY(cudaEventCreateWithFlags(&le.ev, cudaEventDisableTiming));
      }
      if (le.pending) CUDA_TRY(cudaEventSynchronize(le.ev));
      le.ws = workspace;
      le.n_chunks = n_chunks;
      le.st = st;
      le.last = n_chunks;
      le.pending = false;
    } else if (le.pending && cudaEventQuery(le.ev) == cudaSuccess) {
      le.last = *le.host;
      le.pending = false;
    }
    const long long want = (long long)le.last + (long long)le.last / 8 + 2ll * num_sms();
    // a launch of only a few waves is bounded by its heaviest CTAs: start them
    // first (NOLF_OPT_MARCH_ORDER forces either order)
    const Options &opt = options();
    // auto: heaviest first by the previous frame's measured chunk durations
    // below cost_waves CTA waves (longer launches keep the spatial order's
    // cache locality: measured on 16 single-asset 4K views), or by candidate
    // counts below heavy_waves
    const long long wave = (long long)NOLF_MARCH_MINB * num_sms();
    ma.heavy_first = opt.march_order == 1 ? 0 : opt.march_order == 2 ? 1
                   : ((opt.chunk_cost && le.last < opt.cost_waves * wave) || le.last < opt.heavy_waves * wave ? 1 : 0);
    g_last_launch[1] = ma.heavy_first;
    // heavy-first buckets from the previous frame's measured CTA durations
    // (frames of a session are coherent; the first one uses candidate counts)
    ma.chunk_cost = ma.heavy_first && opt.chunk_cost ? w.chunk_cost : nullptr;
    k_cull_chunks<<<(unsigned)((n_chunks + 127) / 128), 128, 0, st>>>(ma, n_chunks, w.chunk_live, w.chunk_list,
                                                                      w.counts + n_inst);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventRecord(ax.ev_cull, st));   // the live count is final here
    const unsigned mgrid = (unsigned)std::max<long long>(1, std::min(n_chunks, want));
    if (opt.march_split == 2) {           // two 64-thread CTAs per chunk
      if (n_inst > 64) k_march_chunks_half<true><<<2 * mgrid, kMarchThreads / 2, 0, st>>>(ma);
      else k_march_chunks_half<false><<<2 * mgrid, kMarchThreads / 2, 0, st>>>(ma);
    } else if (n_inst > 64) {
      k_march_chunks<true><<<mgrid, kMarchThreads, 0, st>>>(ma);
    } else {
      k_march_chunks<false><<<mgrid, kMarchThreads, 0, st>>>(ma);
    }
    if (!le.pending) {          // read the live count back on the side stream: shading never waits for it
      CUDA_TRY(cudaStreamWaitEvent(ax.s, ax.ev_cull, 0));
      CUDA_TRY(cudaMemcpyAsync(le.host, w.counts + n_inst, sizeof(unsigned), cudaMemcpyDeviceToHost, ax.s));
      CUDA_TRY(cudaEventRecord(le.ev, ax.s));
      le.pending = true;
    }
  }
  CUDA_TRY(cudaGetLastError());
  if ((rc = prof_mark(1, st))) return rc;
  if (mode == kModeScene) {
    if ((rc = run_shade(dp->inst, dp->qoff, n_inst, w, mode, w.lrgba, w.ldepth, w.P, counters, st, use_tc,
                        phi_smem, tab_smem, pl.qoff[(size_t)n_inst])))
      return rc;
    if ((rc = prof_mark(2, st))) return rc;
    ComposeArgs ca{};
    ca.n_pix = n_rays;
    ca.nhit = w.nhit;
    ca.K = 0;
    ca.rgba = w.lrgba;
    ca.depth = w.ldepth;
    ca.layer_stride = w.P;
    ca.tiles = reinterpret_cast<const TileParams *>(tiles_dev);
    ca.tile_stride = tile_stride;
    ca.cams = dp->cams;
    ca.n_cams = n_cams;
    ca.frame_layout = sout->layout;
    ca.peer = sout->peer;
    ca.alpha_vis = (float)alpha_vis;
    ca.out_rgba = sout->rgba;
    ca.out_depth = sout->depth;
    ca.out_rgba8 = sout->rgba8;
    ca.out_depth16 = sout->depth16;
    ca.depth_far = (float)sout->depth_far;
    ca.chunk_live = chunked ? w.chunk_live : nullptr;
    ca.prefilled = (sout->prefilled && !sout->rgba && !sout->depth) ? 1 : 0;
    ca.four = (tile_stride % 4 == 0 && n_rays % 4 == 0 && ((uintptr_t)w.nhit & 3) == 0 &&
               ((uintptr_t)sout->rgba8 & 15) == 0 && ((uintptr_t)sout->depth16 & 7) == 0) ? 1 : 0;
    if (ca.four && tile_stride % 8 == 0 && ((uintptr_t)w.nhit & 7) == 0 && ((uintptr_t)sout->rgba8 & 31) == 0 &&
        ((uintptr_t)sout->depth16 & 15) == 0)
      ca.four = 2;
    const long long n_thr = ca.four == 2 ? n_rays / 8 : ca.four ? n_rays / 4 : n_rays;
    ca.errors = errs->dev;
    const bool pack = sout->pack || sout->pack_ids || sout->pack_count;
    if (pack) {
      if (!sout->pack || !sout->pack_ids || !sout->pack_count)
        return fail(NOLF_EINVAL, "sparse frame: pack, pack_ids and pack_count are all required");
      if (!(chunked && ca.prefilled && ca.four == 2))
        return fail(NOLF_EINVAL, "sparse frame needs prefilled u8 outputs and 8-slot-aligned, 128-slot tiles");
      ca.pack = sout->pack;
      ca.pack_ids = sout->pack_ids;
      ca.pack_count = sout->pack_count;
      CUDA_TRY(cudaMemsetAsync(sout->pack_count + 1, 0, sizeof(uint32_t), st));   // run allocator
    }
    if (sout->chunk_state) {
      if (!(chunked && ca.prefilled && ca.four == 2 && sout->layout == 1 && sout->rgba8 && sout->depth16 && !pack))
        return fail(NOLF_EINVAL, "chunk_state needs prefilled u8 frame-layout outputs and 128-slot tiles");
      ca.chunk_state = sout->chunk_state;     // run-level dirty bits (compose_eight_state)
    }
    if (chunked && ca.prefilled && ca.four == 2) {
      // misses are already in place: only the live chunks (grid from the
      // earlier frame's live count, grid-stride for any size)
      const long long n_chunks = n_rays / kMarchThreads;
      const long long live = std::min<long long>(n_chunks, g_live.last + g_live.last / 8 + 2ll * num_sms());
      // 8 slots per thread, or 4 when that leaves under ~1024 threads per SM
      const int g_opt = options().compose_slots;
      const int G = (pack || sout->chunk_state) ? 8 : g_opt == 4 || g_opt == 8 ? g_opt : (live * 16 >= 1024ll * num_sms() ? 8 : 4);
      g_last_launch[2] = G;
      const long long threads = live * (128 / G);
      const unsigned cgrid = (unsigned)std::max<long long>(1, (threads + 255) / 256);
      if (G == 8) k_compose_live<8><<<cgrid, 256, 0, st>>>(ca, w.chunk_list, w.counts + n_inst, n_chunks);
      else k_compose_live<4><<<cgrid, 256, 0, st>>>(ca, w.chunk_list, w.counts + n_inst, n_chunks);
    } else {
      k_compose<<<(unsigned)((n_thr + 255) / 256), 256, 0, st>>>(ca);
    }
    CUDA_TRY(cudaGetLastError());
    if (sout->chunk_state) {   // after compose: reset chunks written last time that are dead now, state = live
      const long long n_chunks = n_rays / kMarchThreads;
      k_clear_stale<<<(unsigned)((n_chunks * 16 + 255) / 256), 256, 0, st>>>(ca, n_chunks);
      CUDA_TRY(cudaGetLastError());
    }
    if ((rc = prof_mark(3, st))) return rc;
    if ((rc = ring_release(slot, st))) return rc;   // the block is reusable once this frame is done
  } else {
    if ((rc = run_shade(dp->inst, dp->qoff, n_inst, w, mode, rgba, depth, 0, counters, st, use_tc, phi_smem, tab_smem,
                        pl.qoff[(size_t)n_inst])))
      return rc;
    if ((rc = prof_mark(2, st))) return rc;
    if ((rc = prof_mark(3, st))) return rc;
    if ((rc = ring_release(slot, st))) return rc;
  }
  return post_errors(st, ax.s);
}

}  // namespace

extern "C" {

int nolf_render_rays(const NolfInstance *inst, const double *origins, int32_t origin_stride, const double *dirs,
                     int64_t n, float *rgba, float *depth, unsigned long long *counters, void *workspace,
                     size_t ws_bytes, void *stream) {
  if (n < 0) return fail(NOLF_EINVAL, "negative ray count");
  if (n > 0 && (!origins || !dirs || !rgba || !depth)) return fail(NOLF_EINVAL, "null buffer");
  if (n >= (1ll << 32)) return fail(NOLF_EINVAL, "too many rays for one launch");
  TileParams rect{0, 0, 0, 0, 0};
  return launch_march_shade(kModeRays, inst, 1, nullptr, 0, nullptr, 0, rect, n, 0, origins,
                            origin_stride ? 1 : 0, dirs, rgba, depth, nullptr, 0.5, counters, workspace,
                            ws_bytes, static_cast<cudaStream_t>(stream));
}

int nolf_render_rect(const NolfInstance *inst, const NolfCamera *cam, int32_t x0, int32_t y0, int32_t x1,
                     int32_t y1, float *rgba, float *depth, unsigned long long *counters, void *workspace,
                     size_t ws_bytes, void *stream) {
  if (!cam) return fail(NOLF_EINVAL, "null camera");
  if (!(0 <= x0 && x0 < x1 && x1 <= cam->width)) return fail(NOLF_EINVAL, "ray range x bounds outside frame");
  if (!(0 <= y0 && y0 < y1 && y1 <= cam->height)) return fail(NOLF_EINVAL, "ray range y bounds outside frame");
  TileParams rect{0, x0, y0, x1, y1};
  const long long n = (long long)(x1 - x0) * (y1 - y0);
  return launch_march_shade(kModeRect, inst, 1, cam, 1, nullptr, 0, rect, n, 0, nullptr, 0, nullptr, rgba,
                            depth, nullptr, 0.5, counters, workspace, ws_bytes, static_cast<cudaStream_t>(stream));
}

int nolf_render_scene(const NolfInstance *inst, int32_t n_inst, const NolfCamera *cams, int32_t n_cams,
                      const NolfTile *tiles, int32_t n_tiles, const NolfSceneOut *out, double alpha_vis,
                      unsigned long long *counters, void *workspace, size_t ws_bytes, void *stream) {
  if (!out || !cams || n_cams < 1) return fail(NOLF_EINVAL, "null scene argument");
  if (n_tiles < 0 || (n_tiles > 0 && !tiles)) return fail(NOLF_EINVAL, "bad tile list");
  if (out->tile_stride < 1) return fail(NOLF_EINVAL, "tile_stride must be positive");
  const long long n = (long long)n_tiles * out->tile_stride;
  if (n >= (1ll << 32)) return fail(NOLF_EINVAL, "too many pixels for one launch");
  TileParams rect{0, 0, 0, 0, 0};
  return launch_march_shade(kModeScene, inst, n_inst, cams, n_cams, tiles, n_tiles, rect, n, out->tile_stride,
                            nullptr, 0, nullptr, nullptr, nullptr, out, alpha_vis, counters, workspace, ws_bytes,
                            static_cast<cudaStream_t>(stream));
}

int nolf_march_rays(nolf_asset_t asset, const double *origins, int32_t origin_stride, const double *dirs, int64_t n,
                    uint8_t *hit, double *t_hit, double *alpha_c, int64_t *samples, double *p_h, void *workspace,
                    size_t ws_bytes, void *stream) {
  if (!asset) return fail(NOLF_EINVAL, "null asset");
  if (n < 0 || n >= (1ll << 32)) return fail(NOLF_EINVAL, "bad ray count");
  if (n == 0) return 0;
  if (!origins || !dirs || !hit || !t_hit || !alpha_c || !samples || !p_h) return fail(NOLF_EINVAL, "null buffer");
  (void)workspace;
  (void)ws_bytes;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const ParamLayout PL = param_layout(1, 0);
  char *hraw, *draw;
  int slot, rc;
  if ((rc = ring_acquire(PL.total, &hraw, &draw, &slot))) return rc;
  ParamBlock hb = param_view(hraw, PL), db = param_view(draw, PL);
  ParamBlock *hp = &hb, *dp = &db;
  memset(&hp->inst[0], 0, sizeof(DevInst));
  hp->inst[0].a = asset->dev;
  hp->inst[0].scale = 1.0;
  hp->qoff[0] = 0;
  hp->qoff[1] = 0;
  CUDA_TRY(cudaMemcpyAsync(draw, hraw, PL.total, cudaMemcpyHostToDevice, st));
  if ((rc = ring_release(slot, st))) return rc;
  MarchArgs ma{};
  ma.inst = dp->inst;
  ma.n_inst = 1;
  ma.origins = origins;
  ma.origin_stride = origin_stride ? 1 : 0;
  ma.dirs = dirs;
  ma.n_rays = n;
  ma.raw_rays = 1;
  ma.out_hit = hit;
  ma.out_t_hit = t_hit;
  ma.out_alpha_c = alpha_c;
  ma.out_samples = reinterpret_cast<long long *>(samples);
  ma.out_p_h = p_h;
  unsigned long long *dummy = nullptr;
  ma.counters = dummy;
  ErrState *errs;
  if ((rc = poll_errors())) return rc;
  if ((rc = err_state(&errs))) return rc;
  ma.errors = errs->dev;
  k_march<kModeRays><<<(unsigned)((n + 127) / 128), 128, 0, st>>>(ma);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int nolf_eval_diffuse(nolf_asset_t asset, const double *points, int64_t n, float *out, void *stream) {
  if (!asset) return fail(NOLF_EINVAL, "null asset");
  if (!asset->host.fd.params || asset->host.hg_levels < 1) return fail(NOLF_ESTATE, "asset has no diffuse network");
  if (asset->host.fd.in != asset->host.hg_levels * asset->host.hg_F)
    return fail(NOLF_EINVAL, "diffuse MLP input width mismatch");
  if (n < 0) return fail(NOLF_EINVAL, "negative point count");
  if (n == 0) return 0;
  if (!points || !out) return fail(NOLF_EINVAL, "null buffer");
  int rc;
  if ((rc = ensure_attrs())) return rc;
  const long long blocks = std::min<long long>((n + kShadeThreads - 1) / kShadeThreads, (long long)num_sms() * 8);
  k_eval_diffuse<<<(unsigned)blocks, kShadeThreads, kShadeSmem, static_cast<cudaStream_t>(stream)>>>(asset->dev, points,
                                                                                                    n, out);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int nolf_mlp_eval(nolf_asset_t asset, int mode, const float *x, int64_t n, float *out, void *stream) {
  if (!asset) return fail(NOLF_EINVAL, "null asset");
  if (n < 0) return fail(NOLF_EINVAL, "negative row count");
  if (n == 0) return 0;
  if (!x || !out) return fail(NOLF_EINVAL, "null buffer");
  int rc;
  if ((rc = ensure_attrs())) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (mode == NOLF_MLP_BF16) {
    if (!asset->host.tc_w) return fail(NOLF_EINVAL, "asset has no tensor-core weights");
    const long long blocks = std::min<long long>((n + kTcThreads - 1) / kTcThreads, (long long)num_sms() * 2);
    k_mlp_tc<<<(unsigned)blocks, kTcThreads, kTcSmem, st>>>(asset->dev, x, n, out);
  } else if (mode == NOLF_MLP_FP32) {
    const long long blocks = std::min<long long>((n + kShadeThreads - 1) / kShadeThreads, (long long)num_sms() * 4);
    k_mlp_fp32<<<(unsigned)blocks, kShadeThreads, kShadeSmem, st>>>(asset->dev, x, n, out);
  } else {
    return fail(NOLF_EINVAL, "unknown MLP mode %d", mode);
  }
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int nolf_set_option(int32_t key, int64_t value) {
  Options &o = options();
  switch (key) {
    case NOLF_OPT_MARCH_ORDER:
      if (value < 0 || value > 2) return fail(NOLF_EINVAL, "march order %lld outside 0..2", (long long)value);
      o.march_order = (int)value;
      return 0;
    case NOLF_OPT_COMPOSE_SLOTS:
      if (value != 0 && value != 4 && value != 8) return fail(NOLF_EINVAL, "compose slots must be 0, 4 or 8");
      o.compose_slots = (int)value;
      return 0;
    case NOLF_OPT_MARCH_SPLIT:
      if (value != 1 && value != 2) return fail(NOLF_EINVAL, "march split must be 1 or 2");
      o.march_split = (int)value;
      return 0;
    case NOLF_OPT_HEAVY_WAVES:
      if (value < 0) return fail(NOLF_EINVAL, "heavy waves must be >= 0");
      o.heavy_waves = value;
      return 0;
    case NOLF_OPT_CHUNK_COST:
      if (value != 0 && value != 1) return fail(NOLF_EINVAL, "chunk cost must be 0 or 1");
      o.chunk_cost = (int)value;
      return 0;
    default:
      return fail(NOLF_EINVAL, "unknown option %d", key);
  }
}

int nolf_check_errors(void *stream) {
  ErrState *E;
  int rc;
  if ((rc = err_state(&E))) return rc;
  CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  if (E->pending) CUDA_TRY(cudaEventSynchronize(E->ev_done));
  E->pending = false;
  CUDA_TRY(cudaMemcpy(E->host, E->dev, sizeof(unsigned) * kNumErr, cudaMemcpyDeviceToHost));
  return report_errors(*E);
}

int nolf_last_launch(int32_t *info) {
  if (!info) return fail(NOLF_EINVAL, "null argument");
  for (int i = 0; i < 4; ++i) info[i] = g_last_launch[i];
  return 0;
}

int nolf_debug_psh_slots(uint32_t *slots, int64_t capacity_rows) {
  if (slots && capacity_rows < 0) return fail(NOLF_EINVAL, "negative capacity");
  g_dbg_slots = slots;
  g_dbg_rows = slots ? capacity_rows : 0;
  return 0;
}

int nolf_profile(int enable) {
  if (enable && !g_prof) {
    g_prof = new Prof();
    for (int c = 0; c < kProfRing; ++c)
      for (int i = 0; i < 4; ++i) CUDA_TRY(cudaEventCreate(&g_prof->ev[c][i]));
    g_prof->created = true;
  }
  if (g_prof) {
    g_prof->on = enable != 0;
    if (enable) g_prof->calls = 0;
  }
  return 0;
}

// Sum of per-kernel durations over every render call recorded since
// nolf_profile(1): ms[0..2] = k_march, k_shade, k_compose; returns calls.
int nolf_profile_read(float *ms) {
  if (!g_prof) return fail(NOLF_ESTATE, "profiling was never enabled");
  ms[0] = ms[1] = ms[2] = 0.f;
  const int n = g_prof->calls;
  if (n == 0) return 0;
  CUDA_TRY(cudaEventSynchronize(g_prof->ev[n - 1][3]));
  for (int c = 0; c < n; ++c)
    for (int i = 0; i < 3; ++i) {
      float t = 0.f;
      CUDA_TRY(cudaEventElapsedTime(&t, g_prof->ev[c][i], g_prof->ev[c][i + 1]));
      ms[i] += t;
    }
  return n;
}

size_t nolf_launch_param_bytes(int32_t n_inst, int32_t n_cams) { return param_bytes(n_inst, n_cams); }

int nolf_unpack_gathered(const uint8_t *gathered, int32_t world, int32_t n_per_rank, int64_t tile_stride,
                         const NolfTile *slot_tiles, int32_t width, int32_t height, uint8_t *rgba8, uint16_t *depth16,
                         void *stream) {
  if (world < 1 || n_per_rank < 0 || tile_stride < 1 || width < 1 || height < 1)
    return fail(NOLF_EINVAL, "bad unpack geometry");
  const long long n_slots = (long long)world * n_per_rank;
  const long long n = n_slots * tile_stride;
  if (n == 0) return 0;
  if (!gathered || !slot_tiles || !rgba8 || !depth16) return fail(NOLF_EINVAL, "null buffer");
  const long long rank_bytes = (long long)n_per_rank * tile_stride * 6;
  k_unpack<<<(unsigned)((n + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      gathered, rank_bytes, n_per_rank, tile_stride, reinterpret_cast<const TileParams *>(slot_tiles), n_slots,
      width, height, reinterpret_cast<uchar4 *>(rgba8), depth16);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int nolf_device_alloc(size_t bytes, void **ptr) {
  if (!ptr) return fail(NOLF_EINVAL, "null out pointer");
  *ptr = nullptr;
  cudaError_t e = cudaMalloc(ptr, bytes ? bytes : 1);
  if (e != cudaSuccess) return fail(NOLF_ENOMEM, "cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
  return 0;
}

int nolf_device_free(void *ptr) {
  if (ptr) CUDA_TRY(cudaFree(ptr));
  return 0;
}

int nolf_ipc_get_handle(void *ptr, void *handle64) {
  if (!ptr || !handle64) return fail(NOLF_EINVAL, "null argument");
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, ptr));
  memcpy(handle64, &h, sizeof(h));
  return 0;
}

int nolf_ipc_open_handle(const void *handle64, void **ptr) {
  if (!ptr || !handle64) return fail(NOLF_EINVAL, "null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  CUDA_TRY(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return 0;
}

int nolf_flag_set(uint32_t *flag, uint32_t value, void *stream) {
  if (!flag) return fail(NOLF_EINVAL, "null flag");
  k_flag_set<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(flag, value);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int nolf_flag_wait(const uint32_t *flags, int32_t n, uint32_t value, uint32_t *timed_out, void *stream) {
  if (n < 0 || n > 32 || (n > 0 && !flags)) return fail(NOLF_EINVAL, "flag count %d outside 0..32", n);
  if (n == 0) return 0;
  k_flag_wait<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(flags, n, value, timed_out);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int nolf_ipc_close_handle(void *ptr) {
  if (ptr) CUDA_TRY(cudaIpcCloseMemHandle(ptr));
  return 0;
}

int nolf_store_u32(uint32_t *dst, const uint32_t *src, int32_t n, void *stream) {
  if (n < 0 || n > 1024 || (n && (!dst || !src))) return fail(NOLF_EINVAL, "bad store arguments");
  if (n == 0) return 0;
  k_store_u32<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(dst, src, n);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int nolf_memset_async(void *dst, int32_t byte_value, size_t bytes, void *stream) {
  if (bytes == 0) return 0;
  if (!dst) return fail(NOLF_EINVAL, "null buffer");
  CUDA_TRY(cudaMemsetAsync(dst, byte_value, bytes, static_cast<cudaStream_t>(stream)));
  return 0;
}

int nolf_memcpy_async(void *dst, const void *src, size_t bytes, void *stream) {
  if (bytes == 0) return 0;
  if (!dst || !src) return fail(NOLF_EINVAL, "null buffer");
  CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, static_cast<cudaStream_t>(stream)));
  return 0;
}

int nolf_memcpy2d_async(void *dst, size_t dpitch, const void *src, size_t spitch, size_t width_bytes, size_t height,
                        void *stream) {
  if (width_bytes == 0 || height == 0) return 0;
  if (!dst || !src) return fail(NOLF_EINVAL, "null buffer");
  CUDA_TRY(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width_bytes, height, cudaMemcpyDefault,
                             static_cast<cudaStream_t>(stream)));
  return 0;
}

int nolf_host_register(void *host_ptr, size_t bytes, void **dev_ptr) {
  if (!host_ptr || !dev_ptr || bytes == 0) return fail(NOLF_EINVAL, "bad host buffer");
  CUDA_TRY(cudaHostRegister(host_ptr, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
  CUDA_TRY(cudaHostGetDevicePointer(dev_ptr, host_ptr, 0));
  return 0;
}

int nolf_host_unregister(void *host_ptr) {
  if (host_ptr) CUDA_TRY(cudaHostUnregister(host_ptr));
  return 0;
}

int nolf_encode_frame(const float *rgba, const float *depth, int64_t n, double depth_far, uint8_t *rgba8,
                      uint16_t *depth16, void *stream) {
  if (n < 0 || !(depth_far > 0.0)) return fail(NOLF_EINVAL, "bad frame encode arguments");
  if (n == 0) return 0;
  if (!rgba || !depth || !rgba8 || !depth16) return fail(NOLF_EINVAL, "null buffer");
  if ((uintptr_t)rgba & 15) return fail(NOLF_EINVAL, "rgba must be 16-byte aligned");
  const long long blocks = std::min<long long>((n + 255) / 256, (long long)num_sms() * 16);
  k_encode_frame<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const float4 *>(rgba), depth, n, (float)depth_far, reinterpret_cast<uchar4 *>(rgba8), depth16);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int nolf_deflate(const void *src, size_t n, int32_t level, void *dst, size_t *dst_len) {
  if ((n && !src) || !dst_len || level < -1 || level > 9) return fail(NOLF_EINVAL, "bad deflate arguments");
  const size_t bound = compressBound((uLong)n);
  if (!dst) {
    *dst_len = bound;
    return 0;
  }
  uLongf out = (uLongf)*dst_len;
  const int z = compress2(static_cast<Bytef *>(dst), &out, static_cast<const Bytef *>(src), (uLong)n, level);
  if (z != Z_OK) return fail(z == Z_BUF_ERROR ? NOLF_EINVAL : NOLF_ENOMEM, "zlib compress2 failed (%d)", z);
  *dst_len = (size_t)out;
  return 0;
}

const char *nolf_zlib_version(void) { return zlibVersion(); }

int nolf_compose(int32_t K, int64_t P, const float *rgba, const float *depth, double alpha_vis, float *out_rgba,
                 float *out_depth, void *stream) {
  if (K < 1) return fail(NOLF_EINVAL, "compose needs at least one frame");
  if (P == 0) return 0;
  if (!rgba || !depth || !out_rgba || !out_depth) return fail(NOLF_EINVAL, "null buffer");
  ComposeArgs ca{};
  ca.n_pix = P;
  ca.nhit = nullptr;
  ca.K = K;
  ca.rgba = rgba;
  ca.depth = depth;
  ca.layer_stride = P;
  ca.tiles = nullptr;
  ca.alpha_vis = (float)alpha_vis;
  ca.out_rgba = out_rgba;
  ca.out_depth = out_depth;
  k_compose<<<(unsigned)((P + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(ca);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

}  // extern "C"

#ifdef NOLF_STATS
extern "C" int nolf_stats_cta(unsigned long long *start, unsigned long long *end, int n) {
  cudaMemcpyFromSymbol(start, nolf::g_cta_start, sizeof(unsigned long long) * n);
  cudaMemcpyFromSymbol(end, nolf::g_cta_end, sizeof(unsigned long long) * n);
  static unsigned long long z[1 << 20];
  cudaMemcpyToSymbol(nolf::g_cta_end, z, sizeof(z));
  return (int)cudaGetLastError();
}
extern "C" int nolf_stats_work(unsigned *out, int n) {   // g_cta_work[0..n) (then zeroed)
  cudaMemcpyFromSymbol(out, nolf::g_cta_work, sizeof(unsigned) * 4 * n);
  static unsigned z[4 << 20];
  cudaMemcpyToSymbol(nolf::g_cta_work, z, sizeof(z));
  return (int)cudaGetLastError();
}
extern "C" int nolf_stats_read(unsigned long long *out, int reset) {
  cudaMemcpyFromSymbol(out, nolf::g_stats, sizeof(unsigned long long) * 16);
  if (reset) {
    static const unsigned long long z[16] = {};
    cudaMemcpyToSymbol(nolf::g_stats, z, sizeof(z));
  }
  return (int)cudaGetLastError();
}
#endif

// ---------------------------------------------------------------- native .nolf loading
// assetio.read_asset (assetio.py:174-255) without Python: container, CRC32,
// gzip, meta JSON -> NolfAssetDesc -> nolf_asset_create.
// Bounded products of untrusted meta fields: false if any factor is
// negative or the product exceeds `limit` (no int64 overflow on the way).
static bool checked_product(std::initializer_list<int64_t> f, int64_t limit, int64_t &out) {
  int64_t p = 1;
  for (int64_t v : f) {
    if (v < 0 || (v > 0 && p > limit / v)) return false;
    p *= v;
  }
  out = p;
  return p <= limit;
}

static int asset_load_mem(const void *data, size_t n, int device, nolf_asset_t *out, double object_to_world[16]);

extern "C" int nolf_asset_load_mem(const void *data, size_t n, int device, nolf_asset_t *out,
                                   double object_to_world[16]) {
  try {                        // nothing may escape the C ABI (bad_alloc on a hostile size, ...)
    return asset_load_mem(data, n, device, out, object_to_world);
  } catch (const std::exception &e) {
    return fail(NOLF_EDATA, "asset load failed: %s", e.what());
  } catch (...) {
    return fail(NOLF_EDATA, "asset load failed");
  }
}

static int asset_load_mem(const void *data, size_t n, int device, nolf_asset_t *out, double object_to_world[16]) {
  using namespace nolf_load;
  if (!data || !out) return fail(NOLF_EINVAL, "null argument");
  *out = nullptr;
  Container c;
  std::string err;
  if (!parse_container(std::vector<uint8_t>(static_cast<const uint8_t *>(data), static_cast<const uint8_t *>(data) + n),
                       c, err))
    return fail(NOLF_EDATA, "%s", err.c_str());
  const Json &m = c.meta;
  auto bad = [&](const char *what) { return fail(NOLF_EDATA, "bad asset meta: %s", what); };
  NolfAssetDesc d{};
  // keep-alive storage for the aligned copies handed to nolf_asset_create
  std::vector<int32_t> den_index, dif_index, tris;
  std::vector<float> den_cubes, dif_cubes, feats;
  std::vector<int64_t> offsets;
  std::vector<double> verts;
  std::vector<std::vector<float>> hg, mw;

  auto atlas = [&](const char *key, const char *tag, int ch, NolfAtlasDesc &a, std::vector<int32_t> &idx,
                   std::vector<float> &cubes) -> int {
    const Json *j = m.get(key);
    int64_t b, r, nc, ncell, ncube;
    if (!inum(j ? j->get("b") : nullptr, b) || !inum(j->get("r"), r) || !inum(j->get("cubes"), nc) || b < 1 ||
        b > 1024 || r < 1 || r > 64 || nc < 0)
      return bad(key);
    const int64_t s1 = r + 1;
    if (!checked_product({b, b, b}, 1ll << 30, ncell) || nc > ncell ||
        !checked_product({nc, s1, s1, s1, (int64_t)ch}, 1ll << 34, ncube))
      return bad(key);
    if (!aligned(c, std::string(tag) + "_index", (size_t)ncell, idx, err) ||
        !aligned(c, std::string(tag) + "_cubes", (size_t)ncube, cubes, err))
      return fail(NOLF_EDATA, "%s", err.c_str());
    a.b = (int32_t)b;
    a.r = (int32_t)r;
    a.channels = ch;
    a.n_cubes = nc;
    a.index = idx.data();
    a.cubes = cubes.empty() ? nullptr : cubes.data();
    return 0;
  };
  int rc;
  if ((rc = atlas("density_atlas", "den", 1, d.density, den_index, den_cubes))) return rc;
  if (flag(m.get("has_diffuse_atlas"), false)) {
    d.has_diffuse_atlas = 1;
    if ((rc = atlas("diffuse_atlas", "dif", 4, d.diffuse, dif_index, dif_cubes))) return rc;
  }
  // PSH (assetio.py: psh meta + psh_offsets int64 + psh_features f32)
  const Json *pm = m.get("psh");
  int64_t res, tsz, osz, F;
  if (!pm || !inum(pm->get("resolution"), res) || !inum(pm->get("table_size"), tsz) ||
      !inum(pm->get("offset_size"), osz) || !inum(pm->get("features"), F) || F < 1 || F > 4 || res < 1 ||
      res > (1 << 20) || tsz < 1 || tsz >= (1ll << 30) || osz < 1 || osz >= (1ll << 30))
    return bad("psh");
  const Json *p0 = pm->get("primes_h0"), *p1 = pm->get("primes_h1");
  if (!p0 || !p1 || p0->kind != Json::Arr || p1->kind != Json::Arr || p0->arr.size() != 3 || p1->arr.size() != 3)
    return bad("psh primes");
  for (int k = 0; k < 3; ++k) {
    int64_t a, b;
    if (!inum(&p0->arr[k], a) || !inum(&p1->arr[k], b) || a < 0 || b < 0) return bad("psh primes");
    d.primes_h0[k] = (uint64_t)a;
    d.primes_h1[k] = (uint64_t)b;
  }
  if (!aligned(c, "psh_offsets", (size_t)osz, offsets, err) || !aligned(c, "psh_features", (size_t)(tsz * F), feats, err))
    return fail(NOLF_EDATA, "%s", err.c_str());
  d.psh_resolution = (int32_t)res;
  d.psh_table_size = tsz;
  d.psh_offset_size = osz;
  d.psh_offsets = offsets.data();
  d.psh_features = feats.data();
  d.psh_features_dim = (int32_t)F;
  // hash-grid diffuse encoder (encoding.py:415-424 resolutions / dense rows)
  const Json *em = m.get("diffuse_encoder");
  int64_t lv, base, hts, fpl;
  double growth;
  if (!em || !inum(em->get("levels"), lv) || !inum(em->get("base_resolution"), base) || !num(em->get("growth"), growth) ||
      !inum(em->get("table_size"), hts) || !inum(em->get("features_per_level"), fpl) || lv < 0 || lv > 16 ||
      base < 1 || base > 4096 || !(growth >= 1.0 && growth <= 16.0) || hts < 1 || hts >= (1ll << 30) || fpl < 1 ||
      fpl > 8)
    return bad("diffuse_encoder");
  d.hg_levels = (int32_t)lv;
  d.hg_features = (int32_t)fpl;
  d.hg_table_size = hts;
  hg.resize((size_t)lv);
  for (int l = 0; l < lv; ++l) {
    const double fres = std::floor((double)base * std::pow(growth, (double)l));
    if (!(fres < 1e6)) return bad("diffuse_encoder resolution");
    const int64_t nres = std::max<int64_t>(2, (int64_t)fres);
    const bool dense = (nres + 1) * (nres + 1) * (nres + 1) <= hts;
    const int64_t rows = dense ? (nres + 1) * (nres + 1) * (nres + 1) : hts;
    if (!aligned(c, "ed_feat_" + std::to_string(l), (size_t)(rows * fpl), hg[(size_t)l], err))
      return fail(NOLF_EDATA, "%s", err.c_str());
    d.hg_resolution[l] = (int32_t)nres;
    d.hg_dense[l] = dense ? 1 : 0;
    d.hg_rows[l] = rows;
    d.hg_feat[l] = hg[(size_t)l].data();
  }
  // MLPs (assetio.py mlp meta: widths + heads; sections {tag}_w{i} (out,in), {tag}_b{i})
  mw.reserve(16);
  auto mlp = [&](const char *key, const char *tag, NolfMlpDesc &md) -> int {
    const Json *j = m.get(key);
    const Json *w = j ? j->get("widths") : nullptr, *h = j ? j->get("heads") : nullptr;
    if (!w || w->kind != Json::Arr || w->arr.size() < 2 || w->arr.size() > 5 || !h || h->kind != Json::Arr ||
        h->arr.size() > 8)
      return bad(key);
    int64_t wd[5];
    for (size_t i = 0; i < w->arr.size(); ++i)
      if (!inum(&w->arr[i], wd[i]) || wd[i] < 1 || wd[i] > 4096) return bad(key);
    md.n_layers = (int32_t)w->arr.size() - 1;
    md.widths[0] = (int32_t)wd[0];
    for (int i = 0; i < md.n_layers; ++i) {
      mw.emplace_back();
      std::vector<float> &W = mw.back();
      if (!aligned(c, std::string(tag) + "_w" + std::to_string(i), (size_t)(wd[i + 1] * wd[i]), W, err))
        return fail(NOLF_EDATA, "%s", err.c_str());
      mw.emplace_back();
      std::vector<float> &B = mw.back();
      if (!aligned(c, std::string(tag) + "_b" + std::to_string(i), (size_t)wd[i + 1], B, err))
        return fail(NOLF_EDATA, "%s", err.c_str());
      md.widths[i + 1] = (int32_t)wd[i + 1];
      md.w[i] = mw[mw.size() - 2].data();
      md.b[i] = B.data();
    }
    md.n_heads = (int32_t)h->arr.size();
    for (size_t i = 0; i < h->arr.size(); ++i) {
      const Json &e = h->arr[i];
      int64_t hw;
      if (e.kind != Json::Arr || e.arr.size() != 2 || e.arr[0].kind != Json::Str || !inum(&e.arr[1], hw))
        return bad(key);
      const std::string &act = e.arr[0].str;
      md.head_act[i] = act == "identity" ? NOLF_HEAD_IDENTITY : act == "sigmoid" ? NOLF_HEAD_SIGMOID
                     : act == "exponential" ? NOLF_HEAD_EXP : -1;
      if (md.head_act[i] < 0) return bad("head activation");
      md.head_w[i] = (int32_t)hw;
    }
    return 0;
  };
  if ((rc = mlp("specular_mlp", "fs", d.specular)) || (rc = mlp("diffuse_mlp", "fd", d.diffuse_mlp))) return rc;
  // march params, proxy, wiring, transform
  const Json *mm = m.get("march");
  if (!mm || !num(mm->get("step"), d.step) || !num(mm->get("t_stop"), d.t_stop) ||
      !num(mm->get("alpha_floor"), d.alpha_floor))
    return bad("march");
  const Json *px = m.get("proxy");
  const Json *pmin = px ? px->get("min") : nullptr, *pmax = px ? px->get("max") : nullptr;
  if (!pmin || !pmax || pmin->kind != Json::Arr || pmax->kind != Json::Arr || pmin->arr.size() != 3 ||
      pmax->arr.size() != 3)
    return bad("proxy");
  for (int k = 0; k < 3; ++k)
    if (!num(&pmin->arr[k], d.proxy_min[k]) || !num(&pmax->arr[k], d.proxy_max[k])) return bad("proxy");
  const Json *wi = m.get("wiring");
  d.use_hit_point = flag(wi ? wi->get("use_hit_point") : nullptr, true);
  d.use_opacity = flag(wi ? wi->get("use_opacity") : nullptr, true);
  d.refine_opacity = flag(wi ? wi->get("refine_opacity") : nullptr, true);
  d.use_tint = flag(wi ? wi->get("use_tint") : nullptr, true);
  d.use_diffuse_color = flag(wi ? wi->get("use_diffuse_color") : nullptr, true);
  const Json *tf = m.get("transform");
  if (!tf || tf->kind != Json::Arr || tf->arr.size() != 16) return bad("transform");
  double o2w[16];
  for (int k = 0; k < 16; ++k)
    if (!num(&tf->arr[k], o2w[k])) return bad("transform");
  if (const Json *pm2 = m.get("proxy_mesh")) {   // extension sections (nolf_io.py), absent in reference files
    int64_t nv, nt;
    if (!inum(pm2->get("vertices"), nv) || !inum(pm2->get("triangles"), nt) || nv < 0 || nt < 0 || nv >= (1ll << 30) ||
        nt >= (1ll << 30))
      return bad("proxy_mesh");
    if (!aligned(c, "mesh_vertices", (size_t)nv * 3, verts, err) || !aligned(c, "mesh_triangles", (size_t)nt * 3, tris, err))
      return fail(NOLF_EDATA, "%s", err.c_str());
    d.mesh_vertices = verts.data();
    d.mesh_n_vertices = nv;
    d.mesh_triangles = tris.data();
    d.mesh_n_triangles = nt;
  }
  if ((rc = nolf_asset_create(&d, device, out))) return rc;
  if (object_to_world) memcpy(object_to_world, o2w, sizeof o2w);
  return 0;
}

extern "C" int nolf_asset_load(const char *path, int device, nolf_asset_t *out, double object_to_world[16]) {
  if (!path || !out) return fail(NOLF_EINVAL, "null argument");
  FILE *f = fopen(path, "rb");
  if (!f) return fail(NOLF_EDATA, "cannot open %s", path);
  std::vector<uint8_t> buf;
  uint8_t tmp[1 << 16];
  size_t got;
  while ((got = fread(tmp, 1, sizeof tmp, f)) > 0) buf.insert(buf.end(), tmp, tmp + got);
  const bool err = ferror(f) != 0;
  fclose(f);
  if (err) return fail(NOLF_EDATA, "read error on %s", path);
  return nolf_asset_load_mem(buf.data(), buf.size(), device, out, object_to_world);
}

// ---------------------------------------------------------------- sparse frame, host side
extern "C" int nolf_host_scatter(const uint8_t *runs, const uint32_t *heads, uint32_t n, const NolfTile *tiles,
                                 int32_t n_tiles, int64_t tile_stride, int32_t width, int32_t height, uint8_t *rgba8,
                                 uint16_t *depth16, uint16_t *dirty, int32_t n_threads) {
  if ((n && !heads) || !tiles || n_tiles < 0 || tile_stride < 128 || tile_stride % 128 || width < 1 || height < 1 ||
      !rgba8 || !depth16 || !dirty)
    return fail(NOLF_EINVAL, "bad sparse frame arguments");
  const uint64_t n_chunks = (uint64_t)n_tiles * (uint64_t)(tile_stride / 128);
  uint64_t total_runs = 0;
  for (uint32_t i = 0; i < n; ++i) {
    if (heads[3 * i] >= n_chunks || heads[3 * i + 1] > 0xffffu)
      return fail(NOLF_EDATA, "packed chunk %u: bad header", i);
    total_runs = std::max<uint64_t>(total_runs, (uint64_t)heads[3 * i + 2] + __builtin_popcount(heads[3 * i + 1]));
  }
  if (total_runs && !runs) return fail(NOLF_EINVAL, "null run payload");
  nolf_host::ScatterJob job{runs, heads, n, tiles, n_tiles, tile_stride, width, height, rgba8, depth16, dirty};
  if (nolf_host::scatter(job, n_threads))
    return fail(NOLF_EDATA, "sparse frame: tile of a packed chunk is not in the 8x4-block layout");
  return 0;
}

// ---------------------------------------------------------------- stage-2 training step
extern "C" int nolf_train_shade(nolf_asset_t asset, const float *params, const int64_t *offsets, double *grads,
                                int64_t n, const double *p_h, const double *alpha_c, const double *dirs,
                                const float *rgb, const float *alpha_t, double batch, float *pred, double *loss,
                                uint32_t *nonfinite, void *stream) {
  if (!asset || !params || !offsets || !grads || !nonfinite) return fail(NOLF_EINVAL, "null argument");
  if (n < 0 || !(batch > 0.0)) return fail(NOLF_EINVAL, "bad batch");
  if (n == 0) return 0;
  if (!p_h || !alpha_c || !dirs || !rgb || !alpha_t || !pred || !loss) return fail(NOLF_EINVAL, "null buffer");
  const DevAsset &H = asset->host;
  if (H.fs.n_layers != 3 || (H.use_diffuse_color && (!H.fd.params || H.fd.n_layers != 2)))
    return fail(NOLF_EINVAL, "training needs a 3-layer specular and a 2-layer diffuse network");
  TrainArgs a{};
  a.asset = asset->dev;
  a.params = params;
  a.grads = grads;
  for (int i = 0; i < kTpCount; ++i) a.L.off[i] = offsets[i];
  a.fs_in = H.fs.in;
  a.fd_in = H.fd.params ? H.fd.in : 0;
  a.p_h = p_h;
  a.alpha_c = alpha_c;
  a.dirs = dirs;
  a.rgb = rgb;
  a.alpha_t = alpha_t;
  a.n = n;
  a.batch = batch;
  a.pred = pred;
  a.loss = loss;
  a.nonfinite = reinterpret_cast<unsigned *>(nonfinite);
  const size_t smem = sizeof(float) * 2 * 128 * kHid;     // the staged per-layer vectors
  CUDA_TRY(cudaFuncSetAttribute(k_train_shade, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_train_shade<<<(unsigned)((n + 127) / 128), 128, smem, static_cast<cudaStream_t>(stream)>>>(a);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

extern "C" int nolf_adam(float *param, const double *grad, float *m, float *v, int64_t n, double lr, double beta1,
                         double beta2, double eps, int64_t step, uint32_t *nonfinite, void *stream) {
  if (!param || !grad || !m || !v || !nonfinite || n < 0 || step < 1) return fail(NOLF_EINVAL, "bad adam arguments");
  if (n == 0) return 0;
  // neural.py:167-177: c1 = 1 - beta1**t, c2 = 1 - beta2**t in f64; every
  // scalar enters the f32 arithmetic rounded to f32 (numpy weak scalars)
  const double c1 = 1.0 - pow(beta1, (double)step), c2 = 1.0 - pow(beta2, (double)step);
  const long long blocks = std::min<long long>((n + 255) / 256, (long long)num_sms() * 16);
  k_adam<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      param, grad, m, v, n, (float)lr, (float)beta1, (float)beta2, (float)(1.0 - beta1), (float)(1.0 - beta2),
      (float)c1, (float)c2, (float)eps, reinterpret_cast<unsigned *>(nonfinite));
  CUDA_TRY(cudaGetLastError());
  return 0;
}
