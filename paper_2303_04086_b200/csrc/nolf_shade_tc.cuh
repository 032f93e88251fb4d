// nolf_shade_tc.cuh -- fused shading kernel on the 5th-generation tensor cores.
//
// Per CTA: tiles of 128 hit records of ONE placed asset (thread t owns row t).
//   * Phi (the PSH offset table, narrowed to u16 when m <= 65536) and the bf16
//     specular weights are staged into shared memory with TMA bulk copies
//     (cp.async.bulk -> mbarrier complete_tx) whenever the asset changes.
//   * Each thread gathers its PSH corners (Phi from smem), SH(d_obj), the
//     clamped coarse opacity and the diffuse atlas, and writes its 19-wide
//     input row as bf16 into a K-major UMMA operand tile.
//   * Layer 0 [19->64] and layer 1 [64->64] run as tcgen05.mma kind::f16
//     (M=128, N=64, K=16 steps) into a 64-column TMEM accumulator issued by
//     one thread; tcgen05.commit arrives on an mbarrier; the 4 warps read
//     their 32 TMEM lanes back with tcgen05.ld (bias + ReLU in fp32, H1
//     re-quantised to bf16 as the next A operand).
//   * Layer 2 [64->4] is a third tcgen05.mma with W2 zero-padded to N = 16
//     (TMEM columns 64..79); heads + the c = c_d + t*c_s combine run in fp32
//     in the epilogue (-DNOLF_SHADE_L2_FP32: layer 2 on the CUDA cores).
// Numerics: bf16 inputs/weights, fp32 accumulation -> north-star tolerance
// 2/255 (lightfield.py:632-637 network, lightfield.py:291-336 combine).
#pragma once
#include "nolf_kernels.cuh"
#include "nolf_tc.cuh"

namespace nolf {

constexpr int kTcThreads = 128;
constexpr int kTcK0 = 32;                    // layer-0 K padded (inputs <= kTcIn)
constexpr int kTcIn = kTcK0 - 2;             // K columns 30, 31: constant 1 (layer-0 bias hi / lo)
constexpr uint32_t kTcA = 16384;             // A tile: 128 x 64 bf16
constexpr uint32_t kTcW0 = 64 * kTcK0 * 2;   // 4 KB (bias hi / lo in K columns 30, 31)
constexpr uint32_t kTcW1 = 64 * 64 * 2;      // 8 KB
constexpr uint32_t kTcW2 = 16 * 64 * 2;      // 2 KB: W2 (4 x 64) zero-padded to N = 16 rows
// Biases of layers 1 and 2 as one more K=16 MMA step each: A = a broadcast
// "ones" operand (every row {1, 1, 0 x 6}: one 128 B core matrix re-read for
// all row groups, SBO = 0; its second K chunk is a zero core matrix -- the
// zero-padded rows 8..15 of W2, LBO = 256), B = one K chunk holding (bias hi,
// bias lo) per output row (its second K chunk aliases the first, LBO = 0, and
// meets the zeros of A).  hi + lo = the fp32 bias to 2^-17 relative.
// Image layout (byte offsets; one TMA bulk copy):
constexpr uint32_t kTcW1b = 64 * 8 * 2;      // 1 KB
constexpr uint32_t kTcW2b = 16 * 8 * 2;      // 256 B
constexpr uint32_t kOffW1 = kTcW0;
constexpr uint32_t kOffOne = kOffW1 + kTcW1;
constexpr uint32_t kOffW2 = kOffOne + 128;
constexpr uint32_t kOffW1b = kOffW2 + kTcW2;
constexpr uint32_t kOffW2b = kOffW1b + kTcW1b;
constexpr uint32_t kTcWBytes = kOffW2b + kTcW2b;
constexpr uint32_t kOneLbo = kOffW2 + 128 - kOffOne;   // -> W2 row group 1 of K chunk 0: zeros
#ifndef NOLF_SHADE_L2_FP32
constexpr int kTcCols = 128;                 // TMEM columns per tile group: hidden (64) + layer 2 (16)
constexpr int kTcF32 = 0;                    // no fp32 block staged
#else
constexpr int kTcCols = 64;
constexpr int kTcF32 = 64 + 64 + 4 * 64 + 4; // (b0, b1 unused: folded), W2 hidden-major, b2
#endif
#ifndef NOLF_TC_PHIMAX
#define NOLF_TC_PHIMAX (64 * 1024)
#endif
constexpr uint32_t kTcPhiMax = NOLF_TC_PHIMAX;   // Phi bytes staged in smem
constexpr uint32_t kTcTabMax = 776;          // residue tables 6*(N+1) for N <= 128 (16-B multiple)
constexpr uint32_t kTcAlign = 16;            // SWIZZLE_NONE operands, TMA bulk copies and mbarriers need <= 16 B

// Residue-table bytes of an asset's shared-memory image (0: read from global).
__host__ __device__ constexpr uint32_t tc_tab_bytes(int N) {
  return 6 * (N + 1) <= (int)kTcTabMax ? (uint32_t)(6 * (N + 1) * 4 + 15) / 16 * 16 : 0u;
}

// ReLU of this thread's 64 TMEM accumulator columns, re-quantised to bf16
// into its row of the K-major A tile (16 columns per TMEM load, one cvt per
// pair).
__device__ __forceinline__ void tc_relu_store(uint32_t trow, uint32_t rowa) {
#pragma unroll
  for (int c4 = 0; c4 < 4; ++c4) {
    uint32_t r[16];
    tc::tmem_ld16(trow + 16 * c4, r);
#pragma unroll
    for (int hcol = 0; hcol < 2; ++hcol) {
      const uint32_t *v = r + 8 * hcol;
      uint4 q;
      q.x = tc::pack_bf16_relu(v[0], v[1]);
      q.y = tc::pack_bf16_relu(v[2], v[3]);
      q.z = tc::pack_bf16_relu(v[4], v[5]);
      q.w = tc::pack_bf16_relu(v[6], v[7]);
      tc::sts128(rowa + (2 * c4 + hcol) * 2048, q);
    }
  }
}

// Two layers on tcgen05 for the 128 rows already written to A (layer-0 input,
// bf16, K-major) by one 128-thread tile group (named barrier `bar_id`,
// group thread gt, TMEM columns [tmem, tmem+64)); returns this thread's 4
// pre-head outputs (fp32).  TMEM is read back 16 columns at a time so the
// hidden layer never occupies more than 16 registers.
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};

template <class Hook = NoHook>
__device__ __forceinline__ void tc_mlp_rows(uint8_t *A, const uint8_t *W, const float *fp, uint32_t tmem,
                                            uint64_t *bar, uint32_t &phase, int gt, int bar_id, float out4[4],
                                            const Hook &while_mma = Hook()) {
  const uint32_t aA = tc::smem_u32(A), aW0 = tc::smem_u32(W), aW1 = aW0 + kOffW1;
  const uint32_t aW1b = aW0 + kOffW1b, aW2b = aW0 + kOffW2b, aOne = aW0 + kOffOne;
  constexpr uint32_t idesc = tc::idesc_bf16_f32(128, 64);
  const uint32_t trow = tmem + ((uint32_t)((gt >> 5) * 32) << 16);   // this warp's TMEM lane quadrant
  // ---- layer 0: D = X[128x32] * W0[64x32]^T
  tc::fence_async_smem();
  tc::bar_sync(bar_id, 128);
  if (gt == 0) {
    tc::tc_fence_after();
#pragma unroll
    for (int s = 0; s < kTcK0 / 16; ++s)
      tc::umma_bf16(tmem, tc::smem_desc(aA + s * 2 * 2048, 2048, 128), tc::smem_desc(aW0 + s * 2 * 1024, 1024, 128),
                    idesc, s > 0);
    tc::umma_commit(bar);
  }
  while_mma();                 // independent work while layer 0 runs
  tc::mbar_wait(bar, phase);
  phase ^= 1;
  tc::tc_fence_after();
  // ReLU (bias already in the accumulator), re-quantised as the layer-1 A
  // operand (K=64), 16 columns at a time
  const uint32_t rowa = aA + (gt >> 3) * 128 + (gt & 7) * 16;
  tc_relu_store(trow, rowa);
  tc::tc_fence_before();
  tc::fence_async_smem();
  tc::bar_sync(bar_id, 128);
  // ---- layer 1: D = H1[128x64] * W1[64x64]^T + 1 * b1 (reuses the TMEM columns)
  if (gt == 0) {
    tc::tc_fence_after();
#pragma unroll
    for (int s = 0; s < 4; ++s)
      tc::umma_bf16(tmem, tc::smem_desc(aA + s * 2 * 2048, 2048, 128), tc::smem_desc(aW1 + s * 2 * 1024, 1024, 128),
                    idesc, s > 0);
    tc::umma_bf16(tmem, tc::smem_desc(aOne, kOneLbo, 0), tc::smem_desc(aW1b, 0, 128), idesc, 1);
    tc::umma_commit(bar);
  }
  tc::mbar_wait(bar, phase);
  phase ^= 1;
  tc::tc_fence_after();
#ifndef NOLF_SHADE_L2_FP32
  // ---- layer 2 on the tensor cores too: H2 = relu(D) re-quantised as the A
  // operand, D2[128 x 16] = H2 * W2p^T + 1 * b2 (W2 zero-padded to 16 rows)
  tc_relu_store(trow, rowa);
  tc::tc_fence_before();
  tc::fence_async_smem();
  tc::bar_sync(bar_id, 128);
  if (gt == 0) {
    tc::tc_fence_after();
    constexpr uint32_t idesc2 = tc::idesc_bf16_f32(128, 16);
    const uint32_t aW2 = aW0 + kOffW2;
#pragma unroll
    for (int s = 0; s < 4; ++s)
      tc::umma_bf16(tmem + 64, tc::smem_desc(aA + s * 2 * 2048, 2048, 128), tc::smem_desc(aW2 + s * 2 * 256, 256, 128),
                    idesc2, s > 0);
    tc::umma_bf16(tmem + 64, tc::smem_desc(aOne, kOneLbo, 0), tc::smem_desc(aW2b, 0, 128), idesc2, 1);
    tc::umma_commit(bar);
  }
  tc::mbar_wait(bar, phase);
  phase ^= 1;
  tc::tc_fence_after();
  uint32_t r4[4];
  tc::tmem_ld4(trow + 64, r4);
  tc::tc_fence_before();
#pragma unroll
  for (int j = 0; j < 4; ++j) out4[j] = __uint_as_float(r4[j]);
}
#else
  // ---- layer 2 (fp32, CUDA cores): 64 -> 4, sequential in the hidden index;
  // W2 is staged hidden-major ([o][4]) so one 16 B load feeds the 4 outputs
  // W2 at fp + 128, b2 at fp + 384 (floats; b1 is folded into the MMA)
  const uint32_t fpa = tc::smem_u32(fp);
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int c4 = 0; c4 < 4; ++c4) {
    uint32_t r[16];
    tc::tmem_ld16(trow + 16 * c4, r);
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
      const int o4 = 4 * c4 + q4;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int o = 4 * o4 + e;
        float z = __uint_as_float(r[4 * q4 + e]);
        z = z > 0.f ? z : 0.f;
        const float4 wv = tc::lds128(fpa + 512 + 16 * o);
        acc[0] = fmaf(z, wv.x, acc[0]);
        acc[1] = fmaf(z, wv.y, acc[1]);
        acc[2] = fmaf(z, wv.z, acc[2]);
        acc[3] = fmaf(z, wv.w, acc[3]);
      }
    }
  }
  tc::tc_fence_before();
  const float4 b2 = tc::lds128(fpa + 1536);
  out4[0] = acc[0] + b2.x;
  out4[1] = acc[1] + b2.y;
  out4[2] = acc[2] + b2.z;
  out4[3] = acc[3] + b2.w;
}
#endif

// Write one bf16 input row (n <= kTcIn values of x, zero padded; columns
// kTcIn.. = 1, the layer-0 bias inputs) to A.
__device__ __forceinline__ void tc_write_x(uint8_t *A, int gt, const float *x, int n) {
  const uint32_t rowa = tc::smem_u32(A) + (gt >> 3) * 128 + (gt & 7) * 16;
#pragma unroll
  for (int c = 0; c < kTcK0 / 8; ++c) {
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = 8 * c + e >= kTcIn ? 1.f : ((8 * c + e < n) ? x[8 * c + e] : 0.f);
    uint4 q;
    q.x = tc::pack_bf16(v[0], v[1]);
    q.y = tc::pack_bf16(v[2], v[3]);
    q.z = tc::pack_bf16(v[4], v[5]);
    q.w = tc::pack_bf16(v[6], v[7]);
    tc::sts128(rowa + c * 2048, q);
  }
}

struct TcSmemPtrs {
  uint8_t *A, *W;              // A: the tile groups' operand tiles, kTcA bytes each
  float *fp;
  uint32_t *tab;
  uint64_t *bar_mma, *bar_tma; // bar_mma: one per tile group
  uint32_t *tmem_slot;
  uint8_t *phi;
};

// Shared-memory carve-up for `groups` 128-thread tile groups: the operand
// tiles, then the asset image (bf16 weights, bias chunks, ones operand,
// [fp32 block], residue tables of up to tab_bytes) exactly as the host laid
// it out for one bulk copy, the barriers and Phi.
__host__ __device__ constexpr uint32_t tc_smem_bytes(int groups, uint32_t phi_bytes, uint32_t tab_bytes) {
  return kTcAlign + groups * kTcA + kTcWBytes + kTcF32 * 4 + tab_bytes + 64 + phi_bytes;
}
constexpr uint32_t kTcSmem = tc_smem_bytes(1, kTcPhiMax, kTcTabMax * 4);

__device__ __forceinline__ TcSmemPtrs tc_carve(uint8_t *raw, int groups, uint32_t tab_bytes) {
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + kTcAlign - 1) &
                                              ~uintptr_t(kTcAlign - 1));
  TcSmemPtrs p;
  p.A = base;
  p.W = p.A + groups * kTcA;
  p.fp = reinterpret_cast<float *>(p.W + kTcWBytes);
  p.tab = reinterpret_cast<uint32_t *>(p.fp + kTcF32);
  p.bar_mma = reinterpret_cast<uint64_t *>(reinterpret_cast<uint8_t *>(p.tab) + tab_bytes);
  p.bar_tma = p.bar_mma + groups;
  p.tmem_slot = reinterpret_cast<uint32_t *>(p.bar_tma + 1);
  p.phi = reinterpret_cast<uint8_t *>(p.bar_mma) + 64;
  return p;
}

// Stage an asset's specular tables: TMA for the bf16 weights and Phi,
// ordinary loads for the small fp32 block and the PSH residue tables.
__device__ __forceinline__ void tc_stage_asset(const DevAsset &A, const TcSmemPtrs &S, uint32_t &tma_phase,
                                               int tid, bool &phi_smem) {
  phi_smem = A.phi16 != nullptr && A.phi16_bytes <= kTcPhiMax;
  // one bulk copy: bf16 weights, fp32 block and residue tables (the host
  // laid them out as the shared-memory image, tc_w_bytes), plus Phi
  if (tid == 0) {
    const uint32_t bytes = A.tc_w_bytes + (phi_smem ? A.phi16_bytes : 0u);
    tc::mbar_arrive_expect_tx(S.bar_tma, bytes);
    tc::bulk_g2s(S.W, A.tc_w, A.tc_w_bytes, S.bar_tma);
    if (phi_smem) tc::bulk_g2s(S.phi, A.phi16, A.phi16_bytes, S.bar_tma);
  }
  tc::mbar_wait(S.bar_tma, tma_phase);
  tma_phase ^= 1;
}

// Layer-0 input row of one hit (lightfield.py:300-331): PSH features
// (trilinear over 8 corner slots, f64 accumulation), SH degree-3 of the view
// direction, and the clamped opacity when refining.  FIXED_F = 2 makes every
// index static (the row stays in registers); 0 = any F (local array).
template <int FIXED_F>
__device__ __forceinline__ void tc_gather_inputs(const DevAsset &A, const TcSmemPtrs &S, bool tab_smem,
                                                 bool phi_smem, const HitRec &rec, float x[kTcK0],
                                                 uint32_t *dbg_slots) {
  const int F = FIXED_F ? FIXED_F : A.F;
  int base[3];
  double w8[8];
  float w8f[8];
  if (FIXED_F == 2) {
    // bf16 path: the corner (integer) addresses exactly as encoding.py, the
    // weights and sums in fp32 -- they feed bf16 MLP inputs (2/255 budget)
    float f[3], g[3];
    const double rd = (double)A.N;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double scaled = __dmul_rn(rec.p[k], rd);
      const double fl = floor(scaled);
      int bb = fl > (double)(A.N - 1) ? A.N - 1 : (int)fl;
      if (bb < 0) bb = 0;
      base[k] = bb;
      f[k] = (float)(scaled - (double)bb);
      g[k] = 1.0f - f[k];
    }
    const float gygz = g[1] * g[2], fygz = f[1] * g[2], gyfz = g[1] * f[2], fyfz = f[1] * f[2];
    w8f[0] = g[0] * gygz; w8f[1] = f[0] * gygz; w8f[2] = g[0] * fygz; w8f[3] = f[0] * fygz;
    w8f[4] = g[0] * gyfz; w8f[5] = f[0] * gyfz; w8f[6] = g[0] * fyfz; w8f[7] = f[0] * fyfz;
  } else {
    base_weights(rec.p, A.N, base, w8);
  }
  double es[FIXED_F ? FIXED_F : kTcK0] = {};
  uint32_t slots[8];
  const int s1 = A.N + 1;
  const uint32_t taba = tc::smem_u32(S.tab), phia = tc::smem_u32(S.phi);
  auto tab = [&](int i) -> uint32_t { return tab_smem ? tc::lds32(taba + 4u * (uint32_t)i) : __ldg(A.tab + i); };
  // the 8 corners touch only 2 residues per (table, axis): load those 12
  // once (the volatile shared loads are never merged by the compiler)
  uint32_t rt[6][2];
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    const int ax = j % 3;
    rt[j][0] = tab(j * s1 + base[ax]);
    rt[j][1] = tab(j * s1 + base[ax] + 1);
  }
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int cx = c & 1, cy = (c >> 1) & 1, cz = (c >> 2) & 1;
    uint32_t h0 = rt[0][cx] + rt[1][cy];
    h0 = h0 >= A.m ? h0 - A.m : h0;
    h0 += rt[2][cz];
    h0 = h0 >= A.m ? h0 - A.m : h0;
    uint32_t h1 = rt[3][cx] + rt[4][cy];
    h1 = h1 >= A.mphi ? h1 - A.mphi : h1;
    h1 += rt[5][cz];
    h1 = h1 >= A.mphi ? h1 - A.mphi : h1;
    const uint32_t off = phi_smem ? tc::lds16(phia + 2u * h1) : __ldg(A.phi + h1);
    uint32_t slot = h0 + off;
    slots[c] = slot >= A.m ? slot - A.m : slot;
  }
  if (dbg_slots) {             // debug read-back of the addresses the gathers below use
#pragma unroll
    for (int c = 0; c < 8; ++c) dbg_slots[c] = slots[c];
  }
  if (FIXED_F == 2) {
    float2 f[8];               // all 8 gathers in flight before the sum
#pragma unroll
    for (int c = 0; c < 8; ++c) f[c] = __ldg(reinterpret_cast<const float2 *>(A.feat) + slots[c]);
    float e0 = 0.f, e1 = 0.f;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      e0 = fmaf(f[c].x, w8f[c], e0);
      e1 = fmaf(f[c].y, w8f[c], e1);
    }
    x[0] = e0;
    x[1] = e1;
    // SH degree 3 of d_obj (core.py:239-261) in fp32
    float sh[16];
    sh_encode_f(rec.d, sh);
#pragma unroll
    for (int q = 0; q < 16; ++q) x[2 + q] = sh[q];
    if (A.refine_opacity) x[18] = (float)clampd(rec.alpha_c, 1e-4, 1.0 - 1e-4);
    return;
  } else {
    for (int c = 0; c < 8; ++c)
      for (int q = 0; q < F; ++q)
        es[q] = __dadd_rn(es[q], __dmul_rn((double)__ldg(A.feat + (size_t)slots[c] * F + q), w8[c]));
  }
  for (int q = 0; q < F; ++q) x[q] = (float)es[q];
  double sh[16];
  sh_encode(rec.d, sh);
#pragma unroll
  for (int q = 0; q < 16; ++q) x[F + q] = (float)sh[q];
  if (A.refine_opacity) x[F + 16] = (float)clampd(rec.alpha_c, 1e-4, 1.0 - 1e-4);
}

// Heads of the bf16 path (its inputs already carry bf16 rounding; the
// 2/255 budget dwarfs the ~2 ulp of the fast exp / reciprocal / log).
#ifdef NOLF_SHADE_EXACT_ACT
__device__ __forceinline__ float tc_sigmoid(float z) { return sigmoidf_np(z); }
__device__ __forceinline__ float tc_exp(float z) { return expf(z); }
__device__ __forceinline__ float tc_log(float z) { return logf(z); }
#else
__device__ __forceinline__ float tc_sigmoid(float z) {   // 1 / (1 + e^-z): MUFU ex2 + rcp (rcp(inf) = 0)
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + __expf(-z)));
  return r;
}
__device__ __forceinline__ float tc_exp(float z) { return __expf(z); }
__device__ __forceinline__ float tc_log(float z) { return __logf(z); }
#endif

// Shading of one 128-hit tile by one tile group (group thread gt owns row
// gt): gather -> bf16 operand tile -> two tcgen05 layers -> fp32 layer 2,
// heads and the combine (lightfield.py:267-336, 446-455).  Only the values
// the epilogue needs stay in registers across the MMA chain.
template <int TG>
__device__ __forceinline__ void tc_shade_tile(const ShadeArgs &args, const DevAsset &A, const TcSmemPtrs &S,
                                              uint8_t *Ag, uint32_t tmem_g, uint64_t *bar_g, uint32_t &mma_phase,
                                              int gt, int bar_id, bool tab_smem, bool phi_smem, double scale,
                                              const HitRec &rec, bool valid, const HitRec *next, HitRec &nxt,
                                              bool std_heads, unsigned long long &n_fs) {
  float cd0 = 0.f, cd1 = 0.f, cd2 = 0.f, tint = 1.f, aterm = 0.f, dep = 0.f;
  long long orow = 0;
  {
    float x[kTcK0];
#pragma unroll
    for (int q = 0; q < kTcK0; ++q) x[q] = 0.f;
    if (valid) {
      orow = args.mode == kModeScene ? (long long)rec.ordinal * args.layer_stride + rec.out_idx
                                     : (long long)rec.out_idx;
      uint32_t *dbg = (args.dbg_slots && orow < args.dbg_rows) ? args.dbg_slots + 8 * orow : nullptr;
      const bool want_dif = A.use_diffuse_color && A.has_dif;
      const int dif_cid = want_dif ? atlas_cell_id(A.dif, rec.p) : -1;   // overlaps the PSH gather
      if (A.F == 2) {            // the common layout: every input index is static -> registers
        tc_gather_inputs<2>(A, S, tab_smem, phi_smem, rec, x, dbg);
      } else {
        float xl[kTcK0] = {};
        tc_gather_inputs<0>(A, S, tab_smem, phi_smem, rec, xl, dbg);
#pragma unroll
        for (int q = 0; q < kTcK0; ++q) x[q] = xl[q];
      }
      if (want_dif) {
        float dv[4];
        atlas_query4_f(A.dif, dif_cid, rec.p, dv);
        cd0 = dv[0]; cd1 = dv[1]; cd2 = dv[2];
        tint = dv[3];
      }
      if (!A.use_tint) tint = 0.5f;
      // opacity input of the combine (lightfield.py:305-310), fp32 (bf16 path budget)
      if (!A.use_opacity) {
        aterm = (float)clampd(rec.alpha_c, 0.0, 1.0);
      } else if (A.refine_opacity) {
        const float ac = (float)clampd(rec.alpha_c, 1e-4, 1.0 - 1e-4);
        aterm = tc_log(__fdividef(ac, 1.0f - ac));
      }
      dep = (float)__ddiv_rn(rec.t_obj, scale);
      ++n_fs;
    }
    tc_write_x(Ag, gt, x, kTcIn);   // unused inputs are 0 (W0 is zero-padded too)
  }
  // the next tile's record, in flight across this tile's MMA chain
  if (next) nxt = *next;
  float z4[4];
#ifdef NOLF_SHADE_PREFETCH_DIF
  // and its diffuse-atlas corners pulled into L2 while layer 0 runs
  auto prefetch = [&]() {
    if (next && A.use_diffuse_color && A.has_dif) atlas_prefetch4(A.dif, nxt.p);
  };
  tc_mlp_rows(Ag, S.W, S.fp, tmem_g, bar_g, mma_phase, gt, bar_id, z4, prefetch);
#else
  tc_mlp_rows(Ag, S.W, S.fp, tmem_g, bar_g, mma_phase, gt, bar_id, z4);
#endif
  if (valid) {
    float fs_out[4];
    if (std_heads) {             // the reference's (sigmoid x 3, identity) head (lightfield.py:635)
#pragma unroll
      for (int j = 0; j < 3; ++j) fs_out[j] = tc_sigmoid(z4[j]);
      fs_out[3] = z4[3];
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        fs_out[j] = A.fs.act[j] == 0 ? z4[j] : (A.fs.act[j] == 1 ? tc_sigmoid(z4[j]) : tc_exp(z4[j]));
    }
    float alpha;
    if (!A.use_opacity) alpha = aterm;
    else if (A.refine_opacity) alpha = tc_sigmoid(fs_out[3] + aterm);
    else alpha = tc_sigmoid(fs_out[3]);
    float4 o;
    o.x = fminf(fmaxf(fmaf(tint, fs_out[0], cd0), 0.f), 1.f);
    o.y = fminf(fmaxf(fmaf(tint, fs_out[1], cd1), 0.f), 1.f);
    o.z = fminf(fmaxf(fmaf(tint, fs_out[2], cd2), 0.f), 1.f);
    o.w = alpha;
    if (o.w <= 0.f) {            // lightfield.py:453-455
      o = make_float4(0.f, 0.f, 0.f, 0.f);
      dep = __int_as_float(0x7f800000);
    }
    reinterpret_cast<float4 *>(args.rgba)[orow] = o;
    args.depth[orow] = dep;
  }
}

// bf16 tcgen05 shading: TG tile groups of 128 threads per CTA, each with its
// own operand tile, TMEM columns and MMA barrier, sharing one staged copy of
// the asset's tables (TMA) -- while one group waits on its gathers the
// other's MMA chain and epilogue run, and the staged tables cost shared
// memory once per CTA.  Tiles (128 hit records of one instance) are dealt
// to the CTAs in blocked ranges; inside an instance the groups take
// alternate tiles.
#ifndef NOLF_SHADE_TG
#define NOLF_SHADE_TG 1
#endif
constexpr int kShadeTG = NOLF_SHADE_TG;

template <int TG>
__global__ void __launch_bounds__(128 * TG, TG == 1 ? 4 : (TG == 2 ? 3 : 2)) k_shade_tc(ShadeArgs args) {
  extern __shared__ uint8_t smem_raw[];
  const TcSmemPtrs S = tc_carve(smem_raw, TG, args.tab_bytes);
  const int tid = threadIdx.x, warp = tid >> 5, g = tid >> 7, gt = tid & 127;
  if (warp == 0) tc::tmem_alloc<kTcCols * TG>(S.tmem_slot);
  __shared__ DevAsset s_asset;
  __shared__ double s_scale;
  if (tid == 0) {
#pragma unroll
    for (int q = 0; q < TG; ++q) tc::mbar_init(S.bar_mma + q, 1);
    tc::mbar_init(S.bar_tma, 1);
    tc::mbar_fence_init();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_g = *S.tmem_slot + (uint32_t)kTcCols * (uint32_t)g;
  uint8_t *Ag = S.A + g * kTcA;
  uint32_t mma_phase = 0, tma_phase = 0;
  bool phi_smem = false, tab_smem = false;
  unsigned long long n_fs = 0;
  const unsigned lane = tid & 31;
  // hits of instance q (its queue may have overflowed: capped), read by the
  // lanes of every warp in chunks of 32 instances and shared by shuffles
  auto inst_hits = [&](int q) -> unsigned {
    return q < args.n_inst ? (unsigned)min((long long)args.counts[q], args.qoff[q + 1] - args.qoff[q]) : 0u;
  };
  long long total_tiles = 0;
  for (int b0 = 0; b0 < args.n_inst; b0 += 32)
    total_tiles += __reduce_add_sync(0xffffffffu, (inst_hits(b0 + (int)lane) + 127u) / 128u);
  const long long tile_lo = total_tiles * blockIdx.x / gridDim.x;
  const long long tile_hi = total_tiles * (blockIdx.x + 1) / gridDim.x;
  // walk the instances overlapping [tile_lo, tile_hi)
  long long t_skip = tile_lo, left = tile_hi - tile_lo;
  unsigned lane_hits = 0;
  for (int k = 0; k < args.n_inst && left > 0; ++k) {
    if ((k & 31) == 0) lane_hits = inst_hits(k + (int)lane);
    const unsigned cnt = __shfl_sync(0xffffffffu, lane_hits, k & 31);
    const long long nt = (cnt + 127) / 128;
    if (t_skip >= nt) { t_skip -= nt; continue; }
    const long long first = t_skip, n_here = min(nt - first, left);
    t_skip = 0;
    left -= n_here;
    // this group's first record, in flight while the tables are staged
    const HitRec *recs = args.queue + args.qoff[k];
    long long r = (first + g) * 128 + gt;
    HitRec cur, nxt;
    if (g < n_here && r < cnt) cur = recs[r];
    // the instance's asset record and tables, once per CTA (record as shared
    // memory: the tile loop's field reads never miss a gather-thrashed L1)
    __syncthreads();
    {
      const uint32_t *src = reinterpret_cast<const uint32_t *>(args.inst[k].a);
      uint32_t *dst = reinterpret_cast<uint32_t *>(&s_asset);
      for (int q = tid; q < (int)(sizeof(DevAsset) / 4); q += 128 * TG) dst[q] = __ldg(src + q);
      if (tid == 0) s_scale = args.inst[k].scale;
    }
    __syncthreads();
    const DevAsset &A = s_asset;
    tc_stage_asset(A, S, tma_phase, tid, phi_smem);
    tab_smem = tc_tab_bytes(A.N) != 0;   // the launch sized the carve for it
    __syncthreads();
    const double scale = s_scale;
    const bool std_heads = A.fs.act[0] == NOLF_HEAD_SIGMOID && A.fs.act[1] == NOLF_HEAD_SIGMOID &&
                           A.fs.act[2] == NOLF_HEAD_SIGMOID && A.fs.act[3] == NOLF_HEAD_IDENTITY;
    for (long long q = g; q < n_here; q += TG, r += 128 * TG) {
      const bool has_next = q + TG < n_here && r + 128 * TG < cnt;
      tc_shade_tile<TG>(args, A, S, Ag, tmem_g, S.bar_mma + g, mma_phase, gt, 1 + g, tab_smem, phi_smem, scale,
                        cur, r < cnt, has_next ? recs + r + 128 * TG : nullptr, nxt, std_heads, n_fs);
      cur = nxt;
    }
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) n_fs += __shfl_xor_sync(0xffffffffu, n_fs, off);
  if (lane == 0 && n_fs) {
    atomicAdd(args.counters + 0, n_fs);
    atomicAdd(args.counters + 2, n_fs);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<kTcCols * TG>(*S.tmem_slot);
}

// The specular MLP alone on n input rows (numerics tests): X (n, in) f32 ->
// out (n, 4) post-head, via the same tcgen05 routine (mode BF16) or the fp32
// CUDA-core routine (mode FP32).
__global__ void __launch_bounds__(kTcThreads) k_mlp_tc(const DevAsset *Ap, const float *X, long long n, float *out) {
  extern __shared__ uint8_t smem_raw[];
  const TcSmemPtrs S = tc_carve(smem_raw, 1, kTcTabMax * 4);
  const int tid = threadIdx.x, warp = tid >> 5;
  const DevAsset &A = *Ap;
  if (warp == 0) tc::tmem_alloc<kTcCols>(S.tmem_slot);
  if (tid == 0) {
    tc::mbar_init(S.bar_mma, 1);
    tc::mbar_init(S.bar_tma, 1);
    tc::mbar_fence_init();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *S.tmem_slot;
  uint32_t mma_phase = 0, tma_phase = 0;
  bool phi_smem;
  tc_stage_asset(A, S, tma_phase, tid, phi_smem);
  __syncthreads();
  const int in = A.fs.in;
  for (long long row0 = (long long)blockIdx.x * kTcThreads; row0 < n; row0 += (long long)gridDim.x * kTcThreads) {
    const long long r = row0 + tid;
    float x[kTcK0];
    for (int i = 0; i < in; ++i) x[i] = r < n ? X[r * in + i] : 0.f;
    tc_write_x(S.A, tid, x, r < n ? in : 0);
    float z4[4];
    tc_mlp_rows(S.A, S.W, S.fp, tmem, S.bar_mma, mma_phase, tid, 1, z4);
    if (r < n)
      for (int j = 0; j < 4; ++j)
        out[r * 4 + j] = A.fs.act[j] == 0 ? z4[j] : (A.fs.act[j] == 1 ? sigmoidf_np(z4[j]) : expf(z4[j]));
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<kTcCols>(tmem);
}

__global__ void __launch_bounds__(kShadeThreads) k_mlp_fp32(const DevAsset *Ap, const float *X, long long n,
                                                            float *out) {
  extern __shared__ __align__(16) float smem[];
  float *s_fs = smem;
  float *s_x = smem + MlpOff::total;
  const DevAsset &A = *Ap;
  for (int q = threadIdx.x; q < MlpOff::total; q += kShadeThreads) s_fs[q] = A.fs.params[q];
  __syncthreads();
  for (long long r = (long long)blockIdx.x * kShadeThreads + threadIdx.x; r < n;
       r += (long long)gridDim.x * kShadeThreads) {
    float *xcol = s_x + threadIdx.x;
    for (int i = 0; i < A.fs.in; ++i) xcol[i * kShadeThreads] = X[r * A.fs.in + i];
    float o[4];
    mlp_row(s_fs, A.fs.n_layers, A.fs.in, A.fs.act, xcol, o);
    for (int j = 0; j < 4; ++j) out[r * 4 + j] = o[j];
  }
}

}  // namespace nolf
