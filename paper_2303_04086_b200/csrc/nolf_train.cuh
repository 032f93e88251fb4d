// nolf_train.cuh -- stage-2 training step of an i-NOLF asset on the GPU
// (SURVEY.md 8(f) rank 4): the per-step work of train_light_field
// (lightfield.py:654-749) after the frozen march --
//
//   shade_batch(..., want_cache, force_live_diffuse)   lightfield.py:267-336
//   loss, d_c = 2 err_c / b, d_alpha = 2 err_a / b      lightfield.py:714-733
//   shade_backward                                      lightfield.py:358-397
//     mlp_backward (heads, ReLU masks, W / b grads)     neural.py:111-148
//     psh_backward / hashgrid_backward (scatter-add)    encoding.py:397-402, 481-489
//   adam_step                                            neural.py:162-177
//
// k_train_shade: one thread per hit ray, forward + backward fused; the MLP
// weight / bias gradients are reduced per CTA in shared memory (f64) and
// added to the global f64 gradient buffer once per CTA; feature gradients
// are scattered with f64 atomics (the reference sums the f64 contributions
// with bincount and adds the f32 cast).  k_adam: the reference's f32 update
// arithmetic, operation for operation.
//
// Trainable parameters live in one flat f32 buffer (reference layouts:
// W (out, in) row-major), gradients in a parallel f64 buffer:
//   TrainLayout.off[kTp*] = offsets (floats) of each tensor.
#pragma once
#include "nolf_kernels.cuh"

namespace nolf {

enum {
  kTpPsh = 0,          // psh features (m, F)
  kTpFsW0, kTpFsB0, kTpFsW1, kTpFsB1, kTpFsW2, kTpFsB2,   // specular MLP [in -> 64 -> 64 -> 4]
  kTpFdW0, kTpFdB0, kTpFdW1, kTpFdB1,                     // diffuse MLP [L*F -> 64 -> 4]
  kTpHg,               // hash-grid level l features at off[kTpHg + l] (rows_l, F)
  kTpCount = kTpHg + kMaxLevels
};

struct TrainLayout {
  long long off[kTpCount];
};

struct TrainArgs {
  const DevAsset *asset;       // fixed tables (PSH addressing, hash-grid config, wiring)
  const float *params;
  double *grads;
  TrainLayout L;
  int fs_in, fd_in;            // MLP input widths
  const double *p_h, *alpha_c, *dirs;
  const float *rgb, *alpha_t;
  long long n;
  double batch;                // b: d_c = 2 err_c / b (lightfield.py:729-730)
  float *pred;                 // (n, 4): c, alpha
  double *loss;                // (n): |c - rgb|^2 + (alpha - alpha_t)^2
  unsigned *nonfinite;         // set when a forward value is not finite
};

// per-CTA shared gradient block (doubles): fs then fd weights / biases
struct TrainSmem {
  int fs_w0, fs_b0, fs_w1, fs_b1, fs_w2, fs_b2, fd_w0, fd_b0, fd_w1, fd_b1, total;
};
__host__ __device__ inline TrainSmem train_smem(int fs_in, int fd_in) {
  TrainSmem S;
  int o = 0;
  S.fs_w0 = o; o += kHid * fs_in;
  S.fs_b0 = o; o += kHid;
  S.fs_w1 = o; o += kHid * kHid;
  S.fs_b1 = o; o += kHid;
  S.fs_w2 = o; o += 4 * kHid;
  S.fs_b2 = o; o += 4;
  S.fd_w0 = o; o += kHid * fd_in;
  S.fd_b0 = o; o += kHid;
  S.fd_w1 = o; o += 4 * kHid;
  S.fd_b1 = o; o += 4;
  S.total = o;
  return S;
}
// the global gradient offset of each shared block entry
__device__ __forceinline__ long long train_goff(const TrainArgs &a, const TrainSmem &S, int i) {
  if (i < S.fs_b0) return a.L.off[kTpFsW0] + i;
  if (i < S.fs_w1) return a.L.off[kTpFsB0] + (i - S.fs_b0);
  if (i < S.fs_b1) return a.L.off[kTpFsW1] + (i - S.fs_w1);
  if (i < S.fs_w2) return a.L.off[kTpFsB1] + (i - S.fs_b1);
  if (i < S.fs_b2) return a.L.off[kTpFsW2] + (i - S.fs_w2);
  if (i < S.fd_w0) return a.L.off[kTpFsB2] + (i - S.fs_b2);
  if (i < S.fd_b0) return a.L.off[kTpFdW0] + (i - S.fd_w0);
  if (i < S.fd_w1) return a.L.off[kTpFdB0] + (i - S.fd_b0);
  if (i < S.fd_b1) return a.L.off[kTpFdW1] + (i - S.fd_w1);
  return a.L.off[kTpFdB1] + (i - S.fd_b1);
}

// z = W x + b (W (out, in) row-major), sequential in the input index
__device__ __forceinline__ float dense_row(const float *W, const float *b, int o, int in, const float *x) {
  float acc = 0.f;
  for (int i = 0; i < in; ++i) acc = fmaf(x[i], W[o * in + i], acc);
  return acc + b[o];
}

__device__ __forceinline__ double sigmoid_d(double z) { return sigmoid_np(z); }

__global__ void __launch_bounds__(128) k_train_shade(TrainArgs a) {
  // Weight gradients are per-CTA matrix products over its 128 rays: each
  // layer stages every ray's upstream vector and input activations in shared
  // memory, then thread t sums (double) g[r][o] * (double) in[r][i] over the
  // rays for its weights (f64, as the reference's f64 accumulation) and adds
  // one value per weight to the global gradient -- no per-ray atomics.
  extern __shared__ float stage[];               // [128][kHid] upstream | [128][kHid] inputs
  const int fs_in = a.fs_in, fd_in = a.fd_in;
  const TrainSmem S = train_smem(fs_in, fd_in);
  const DevAsset &A = *a.asset;
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = r < a.n;
  const bool dif = A.use_diffuse_color;          // uniform
  // per-ray vectors kept for the staged reductions (zero for padding rays)
  float x[kInp], h1[kHid], h2[kHid], g2[4] = {0.f, 0.f, 0.f, 0.f}, g1[kHid], g0[kHid];
  float ed[kInp], hd[kHid], gd[4] = {0.f, 0.f, 0.f, 0.f}, gd0[kHid];
  for (int i = 0; i < kInp; ++i) { x[i] = 0.f; ed[i] = 0.f; }
  for (int o = 0; o < kHid; ++o) { h1[o] = h2[o] = g1[o] = g0[o] = hd[o] = gd0[o] = 0.f; }
  if (valid) {
    const float *P = a.params;
    const double p[3] = {a.p_h[3 * r], a.p_h[3 * r + 1], a.p_h[3 * r + 2]};
    const double dv[3] = {a.dirs[3 * r], a.dirs[3 * r + 1], a.dirs[3 * r + 2]};
    // ---- forward: PSH features (encoding.py:390-394), f64 accumulation
    int base[3];
    double w8[8];
    uint32_t slots[8];
    base_weights(p, A.N, base, w8);
    const int F = A.F;
    double es[4] = {0.0, 0.0, 0.0, 0.0};
    const float *feat = P + a.L.off[kTpPsh];
    for (int c = 0; c < 8; ++c) {
      slots[c] = psh_slot(A.tab, A.phi, A.N, A.m, A.mphi, base[0] + (c & 1), base[1] + ((c >> 1) & 1),
                          base[2] + ((c >> 2) & 1));
      for (int f = 0; f < F; ++f) es[f] = __dadd_rn(es[f], __dmul_rn((double)feat[(size_t)slots[c] * F + f], w8[c]));
    }
    int nin = 0;
    for (int f = 0; f < F; ++f) x[nin++] = (float)es[f];
    double sh[16];
    sh_encode(dv, sh);
    for (int q = 0; q < 16; ++q) x[nin++] = (float)sh[q];
    const double ac = clampd(a.alpha_c[r], 1e-4, 1.0 - 1e-4);
    if (A.refine_opacity) x[nin++] = (float)ac;
    // ---- specular MLP [in -> 64 -> 64 -> 4] (neural.py:89-108), f32
    const float *W0 = P + a.L.off[kTpFsW0], *B0 = P + a.L.off[kTpFsB0], *W1 = P + a.L.off[kTpFsW1],
                *B1 = P + a.L.off[kTpFsB1], *W2 = P + a.L.off[kTpFsW2], *B2 = P + a.L.off[kTpFsB2];
    float zs[4], fs[4];
    for (int o = 0; o < kHid; ++o) h1[o] = fmaxf(dense_row(W0, B0, o, fs_in, x), 0.f);
    for (int o = 0; o < kHid; ++o) h2[o] = fmaxf(dense_row(W1, B1, o, kHid, h1), 0.f);
    for (int j = 0; j < 4; ++j) {
      zs[j] = dense_row(W2, B2, j, kHid, h2);
      fs[j] = A.fs.act[j] == 0 ? zs[j] : (A.fs.act[j] == 1 ? sigmoidf_np(zs[j]) : expf(zs[j]));
    }
    const double cs[3] = {(double)fs[0], (double)fs[1], (double)fs[2]};
    const double z = (double)fs[3];
    double alpha;
    if (!A.use_opacity) alpha = clampd(a.alpha_c[r], 0.0, 1.0);
    else if (A.refine_opacity) alpha = sigmoid_d(z + log(ac / (1.0 - ac)));
    else alpha = sigmoid_d(z);
    // ---- live diffuse: hash grid (encoding.py:467-478) + diffuse MLP
    float fd[4] = {0.f, 0.f, 0.f, 1.f};
    int led = 0;
    int hb[kMaxLevels][3];
    double hw[kMaxLevels][8];
    long long hidx[kMaxLevels][8];
    if (dif) {
      for (int l = 0; l < A.hg_levels; ++l) {
        base_weights(p, A.hg_res[l], hb[l], hw[l]);
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        const float *hf = P + a.L.off[kTpHg + l];
        for (int c = 0; c < 8; ++c) {
          const int cx = c & 1, cy = (c >> 1) & 1, cz = (c >> 2) & 1;
          long long idx;
          if (A.hg_dense[l]) {
            const long long side = A.hg_res[l] + 1;
            idx = ((hb[l][0] * side + hb[l][1]) * side + hb[l][2]) + ((cx * side + cy) * side + cz);
          } else {
            const unsigned long long h = ((unsigned long long)(hb[l][0] + cx) * 1ull) ^
                                         ((unsigned long long)(hb[l][1] + cy) * 2654435761ull) ^
                                         ((unsigned long long)(hb[l][2] + cz) * 805459861ull);
            idx = (long long)(h % A.hg_table);
          }
          hidx[l][c] = idx;
          for (int f = 0; f < A.hg_F; ++f)
            acc[f] = __dadd_rn(acc[f], __dmul_rn((double)hf[idx * A.hg_F + f], hw[l][c]));
        }
        for (int f = 0; f < A.hg_F; ++f) ed[led++] = (float)acc[f];
      }
      const float *V0 = P + a.L.off[kTpFdW0], *C0 = P + a.L.off[kTpFdB0], *V1 = P + a.L.off[kTpFdW1],
                  *C1 = P + a.L.off[kTpFdB1];
      for (int o = 0; o < kHid; ++o) hd[o] = fmaxf(dense_row(V0, C0, o, fd_in, ed), 0.f);
      for (int j = 0; j < 4; ++j) {
        const float zz = dense_row(V1, C1, j, kHid, hd);
        fd[j] = A.fd.act[j] == 0 ? zz : (A.fd.act[j] == 1 ? sigmoidf_np(zz) : expf(zz));
      }
    }
    double cd[3] = {0.0, 0.0, 0.0}, t = 1.0;
    if (dif) { cd[0] = fd[0]; cd[1] = fd[1]; cd[2] = fd[2]; t = fd[3]; }
    if (!A.use_tint) t = 0.5;
    double cpre[3], c[3];
    for (int k = 0; k < 3; ++k) {
      cpre[k] = __dadd_rn(cd[k], __dmul_rn(t, cs[k]));
      c[k] = clampd(cpre[k], 0.0, 1.0);
    }
    // ---- loss and its gradient (lightfield.py:714-730)
    double errc[3], loss = 0.0;
    for (int k = 0; k < 3; ++k) {
      errc[k] = __dsub_rn(c[k], (double)a.rgb[3 * r + k]);
      loss = __dadd_rn(loss, __dmul_rn(errc[k], errc[k]));
    }
    const double erra = __dsub_rn(alpha, (double)a.alpha_t[r]);
    loss = __dadd_rn(loss, __dmul_rn(erra, erra));
    a.loss[r] = loss;
    a.pred[4 * r + 0] = (float)c[0];
    a.pred[4 * r + 1] = (float)c[1];
    a.pred[4 * r + 2] = (float)c[2];
    a.pred[4 * r + 3] = (float)alpha;
    if (!(loss == loss) || loss > 1e300) atomicOr(a.nonfinite, 1u);
    // ---- shade_backward (lightfield.py:358-397)
    double dcpre[3];
    for (int k = 0; k < 3; ++k) {
      const double dc = __ddiv_rn(__dmul_rn(2.0, errc[k]), a.batch);
      dcpre[k] = (cpre[k] > 0.0 && cpre[k] < 1.0) ? dc : 0.0;
    }
    const double da = __ddiv_rn(__dmul_rn(2.0, erra), a.batch);
    const double dz = A.use_opacity ? __dmul_rn(__dmul_rn(da, alpha), __dsub_rn(1.0, alpha)) : 0.0;
    // specular: upstream (f32, neural.py:119) through the heads
    float up[4] = {(float)__dmul_rn(dcpre[0], t), (float)__dmul_rn(dcpre[1], t), (float)__dmul_rn(dcpre[2], t),
                   (float)dz};
    for (int j = 0; j < 4; ++j)
      g2[j] = A.fs.act[j] == 0 ? up[j] : (A.fs.act[j] == 1 ? up[j] * fs[j] * (1.0f - fs[j]) : up[j] * fs[j]);
    // layer 2 -> dh2
    float dh2[kHid];
    for (int o = 0; o < kHid; ++o) dh2[o] = 0.f;
    for (int j = 0; j < 4; ++j)
      for (int o = 0; o < kHid; ++o) dh2[o] = fmaf(g2[j], W2[j * kHid + o], dh2[o]);
    // layer 1 -> dh1
    float dh1[kHid];
    for (int i = 0; i < kHid; ++i) dh1[i] = 0.f;
    for (int o = 0; o < kHid; ++o) {
      const float g = h2[o] > 0.f ? dh2[o] : 0.f;
      g1[o] = g;
      if (g == 0.f) continue;
      for (int i = 0; i < kHid; ++i) dh1[i] = fmaf(g, W1[o * kHid + i], dh1[i]);
    }
    // layer 0 -> input gradient
    float dx[kInp];
    for (int i = 0; i < fs_in; ++i) dx[i] = 0.f;
    for (int o = 0; o < kHid; ++o) {
      const float g = h1[o] > 0.f ? dh1[o] : 0.f;
      g0[o] = g;
      if (g == 0.f) continue;
      for (int i = 0; i < fs_in; ++i) dx[i] = fmaf(g, W0[o * fs_in + i], dx[i]);
    }
    // psh_backward: trilinear weight x upstream, scattered (f64)
    double *gfeat = a.grads + a.L.off[kTpPsh];
    for (int c = 0; c < 8; ++c)
      for (int f = 0; f < F; ++f)
        if (dx[f] != 0.f) atomicAdd(&gfeat[(size_t)slots[c] * F + f], __dmul_rn(w8[c], (double)dx[f]));
    // diffuse network (live path): upstream [d_cd, d_t]
    if (dif) {
      double dt = 0.0;
      if (A.use_tint)
        for (int k = 0; k < 3; ++k) dt = __dadd_rn(dt, __dmul_rn(dcpre[k], cs[k]));
      const float upd[4] = {(float)dcpre[0], (float)dcpre[1], (float)dcpre[2], (float)dt};
      for (int j = 0; j < 4; ++j)
        gd[j] = A.fd.act[j] == 0 ? upd[j] : (A.fd.act[j] == 1 ? upd[j] * fd[j] * (1.0f - fd[j]) : upd[j] * fd[j]);
      const float *V0 = P + a.L.off[kTpFdW0], *V1 = P + a.L.off[kTpFdW1];
      float dhd[kHid];
      for (int o = 0; o < kHid; ++o) dhd[o] = 0.f;
      for (int j = 0; j < 4; ++j)
        for (int o = 0; o < kHid; ++o) dhd[o] = fmaf(gd[j], V1[j * kHid + o], dhd[o]);
      float ded[kInp];
      for (int i = 0; i < fd_in; ++i) ded[i] = 0.f;
      for (int o = 0; o < kHid; ++o) {
        const float g = hd[o] > 0.f ? dhd[o] : 0.f;
        gd0[o] = g;
        if (g == 0.f) continue;
        for (int i = 0; i < fd_in; ++i) ded[i] = fmaf(g, V0[o * fd_in + i], ded[i]);
      }
      // hashgrid_backward (encoding.py:481-489)
      for (int l = 0; l < A.hg_levels; ++l) {
        double *gh = a.grads + a.L.off[kTpHg + l];
        for (int c = 0; c < 8; ++c)
          for (int f = 0; f < A.hg_F; ++f) {
            const float u = ded[l * A.hg_F + f];
            if (u != 0.f) atomicAdd(&gh[hidx[l][c] * A.hg_F + f], __dmul_rn(hw[l][c], (double)u));
          }
      }
    }
  }
  // ---- weight gradients, one layer at a time (all threads: uniform)
  float *G = stage, *IN = stage + 128 * kHid;
  const int t = threadIdx.x;
  // dW[o][i] = sum_r G[r][o] * IN[r][i] and db[o] = sum_r G[r][o] over the
  // CTA's rays; w_off / b_off: the blocks' offsets in the TrainSmem layout
  auto layer = [&](const float *g, int O, const float *in, int I, int w_off, int b_off) {
    __syncthreads();
    for (int o = 0; o < O; ++o) G[t * kHid + o] = g[o];
    for (int i = 0; i < I; ++i) IN[t * kHid + i] = in[i];
    __syncthreads();
    for (int w = t; w < O * I + O; w += 128) {
      double acc = 0.0;
      if (w < O * I) {
        const int o = w / I, i = w % I;
        for (int q = 0; q < 128; ++q) acc = __dadd_rn(acc, __dmul_rn((double)G[q * kHid + o], (double)IN[q * kHid + i]));
        if (acc != 0.0) atomicAdd(a.grads + train_goff(a, S, w_off + w), acc);
      } else {
        const int o = w - O * I;
        for (int q = 0; q < 128; ++q) acc = __dadd_rn(acc, (double)G[q * kHid + o]);
        if (acc != 0.0) atomicAdd(a.grads + train_goff(a, S, b_off + o), acc);
      }
    }
  };
  layer(g2, 4, h2, kHid, S.fs_w2, S.fs_b2);
  layer(g1, kHid, h1, kHid, S.fs_w1, S.fs_b1);
  layer(g0, kHid, x, fs_in, S.fs_w0, S.fs_b0);
  if (dif) {
    layer(gd, 4, hd, kHid, S.fd_w1, S.fd_b1);
    layer(gd0, kHid, ed, fd_in, S.fd_w0, S.fd_b0);
  }
}

// adam_step (neural.py:162-177) on one parameter group, in the reference's
// f32 arithmetic: m = m*b1 + (1-b1)*g ; v = v*b2 + (1-b2)*g^2 ;
// p -= lr * (m / c1) / (sqrt(v / c2) + eps).  g = f32(sum of f64 grads).
__global__ void __launch_bounds__(256) k_adam(float *p, const double *grad, float *m, float *v, long long n, float lr,
                                              float b1, float b2, float one_m_b1, float one_m_b2, float c1, float c2,
                                              float eps, unsigned *nonfinite) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float g = (float)grad[i];
    if (!isfinite(g)) atomicOr(nonfinite, 2u);
    float mi = __fmul_rn(m[i], b1);
    mi = __fadd_rn(mi, __fmul_rn(one_m_b1, g));
    float vi = __fmul_rn(v[i], b2);
    vi = __fadd_rn(vi, __fmul_rn(one_m_b2, __fmul_rn(g, g)));
    m[i] = mi;
    v[i] = vi;
    const float upd = __fdiv_rn(__fmul_rn(lr, __fdiv_rn(mi, c1)), __fadd_rn(__fsqrt_rn(__fdiv_rn(vi, c2)), eps));
    p[i] = __fsub_rn(p[i], upd);
  }
}

}  // namespace nolf
