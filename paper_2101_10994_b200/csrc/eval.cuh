// Warp-cooperative SDF evaluation: the per-LOD trilinear feature gather and
// the per-LOD decoder (field.py:104-218, render.py:155-171).
//
// A warp evaluates 32 points at once, one per lane.
//  1. Lane = point: fp64 binning of x at the finest gathered level, then per
//     level a bitmap rank lookup (locate, octree.py:259-282), the voxel's 8
//     corner ids and the 8 trilinear weights (field.py:104-135), staged in
//     shared memory.
//  2. Lane = feature channel: for every point with the level present, the 8
//     corner rows Z[id, 0:32] are read as coalesced 128-byte loads (one
//     feature per lane), weighted and added into the shared z tile, so the
//     running level sum (sum_features, field.py:154-169) never leaves SMEM.
//  3. Lane = point again: at each requested decoder level L the lane reads
//     its z_L row and runs the 35 -> h -> 1 MLP (decode, field.py:172-182)
//     in fp32 with the decoder weights broadcast from shared memory.
#pragma once

#include "common.cuh"

#ifndef NG_GATHER_BATCH
#define NG_GATHER_BATCH 8  // points whose 8 corner rows are in flight together per warp (2 quad loads)
#endif
#ifndef NG_PROF_SLOTS
#define NG_PROF_SLOTS 32   // NG_PROFILE builds: uint64 counters per march group (tools/march_profile.py)
#endif
#ifndef NG_STAGE_GATHER
// presummed direct-z gather: 4 more points per round staged in shared
// memory with cp.async (experiment knob; measured slower on the 720p frame:
// 0.650 vs 0.630 ms with .ca, 0.646 with .cg)
#define NG_STAGE_GATHER 0
#endif
#ifndef NG_QUAD_GATHER
#define NG_QUAD_GATHER 1   // warp_eval: 16-byte row loads, 4 points per load instruction
#endif

namespace ng {

// zt row stride in floats: 36 keeps rows 16-byte aligned, so the quad
// gather's per-point update and the decoder's row read are 128-bit accesses
// (conflict-free per quarter warp); 33 (A/B builds) is the scalar layout
#ifndef NG_ZT_STRIDE
#define NG_ZT_STRIDE 36
#endif
struct WarpScratch {
  int4 ids[32][2];      // corner ids of each lane's point at the current level
  float4 w[32][2];      // trilinear weights
  float zt[32][NG_ZT_STRIDE];  // running feature sum, row = point, col = channel (+ pad);
                        // the presummed direct-z gather stages 4 points' rows here instead
};

// A point's 32 channels from its zt row.
__device__ __forceinline__ void load_zrow(const float* zrow, float z[32]) {
  if constexpr (NG_ZT_STRIDE % 4 == 0) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float4 q = reinterpret_cast<const float4*>(zrow)[k];
      z[4 * k] = q.x;
      z[4 * k + 1] = q.y;
      z[4 * k + 2] = q.z;
      z[4 * k + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < 32; ++k) z[k] = zrow[k];
  }
}

// zt[p][4 sub .. 4 sub + 3] (+)= acc
template <bool kAdd>
__device__ __forceinline__ void zt_quad(float* zr, const float acc[4]) {
  if constexpr (NG_ZT_STRIDE % 4 == 0) {
    float4* z4 = reinterpret_cast<float4*>(zr);
    if constexpr (kAdd) {
      float4 q = *z4;
      q.x += acc[0];
      q.y += acc[1];
      q.z += acc[2];
      q.w += acc[3];
      *z4 = q;
    } else {
      *z4 = make_float4(acc[0], acc[1], acc[2], acc[3]);
    }
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) zr[e] = kAdd ? zr[e] + acc[e] : acc[e];
  }
}

// Asynchronous 16-byte global -> shared copies (LDGSTS): rows land in
// shared memory without occupying registers while in flight.
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// sum_j w_j * v_j over a point's 8 corner rows, 4 channels, as packed
// FFMA2s (two channels per instruction, half the FMA issue slots). Each
// channel is the scalar chain w_0 v_0, fma(w_1, v_1, .), ... bit for bit:
// the chain starts from fma(w_0, v_0, -0) = w_0 * v_0 (sign of zero included).
// Used by the level-by-level gather (the batched query: 11.16 -> 11.06 ms);
// the march's presummed gather keeps the scalar chain (FFMA2 there measured
// 0.462 -> 0.477 ms per 720p frame at 16 frames per launch). NG_FFMA2=0 off.
#ifndef NG_FFMA2
#define NG_FFMA2 1
#endif
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<const unsigned long long*>(&a)), "l"(*reinterpret_cast<const unsigned long long*>(&b)),
        "l"(*reinterpret_cast<const unsigned long long*>(&c)));
  return *reinterpret_cast<const float2*>(&d);
}
template <bool kPacked>
__device__ __forceinline__ void corner_sum4(const float wj[8], const float4 v[8], float acc[4]) {
  if constexpr (kPacked) {
  float2 a01 = make_float2(-0.f, -0.f), a23 = a01;
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) {
    const float2 w2 = make_float2(wj[jj], wj[jj]);
    a01 = ffma2(w2, make_float2(v[jj].x, v[jj].y), a01);
    a23 = ffma2(w2, make_float2(v[jj].z, v[jj].w), a23);
  }
  acc[0] = a01.x;
  acc[1] = a01.y;
  acc[2] = a23.x;
  acc[3] = a23.y;
  } else {
  acc[0] = wj[0] * v[0].x;
  acc[1] = wj[0] * v[0].y;
  acc[2] = wj[0] * v[0].z;
  acc[3] = wj[0] * v[0].w;
#pragma unroll
  for (int jj = 1; jj < 8; ++jj) {
    acc[0] = fmaf(wj[jj], v[jj].x, acc[0]);
    acc[1] = fmaf(wj[jj], v[jj].y, acc[1]);
    acc[2] = fmaf(wj[jj], v[jj].z, acc[2]);
    acc[3] = fmaf(wj[jj], v[jj].w, acc[3]);
  }
  }
}

struct EvalCtx {
  const float* __restrict__ Z;       // (C, 32)
  const float* dec;                  // shared-memory decoders, level dec_first first
  int dec_first;                     // decoder level of the first staged block
  int dec_stride;                    // floats per decoder block
  int h;
  int gather_level;                  // G: highest level interpolated
  int inside_level;                  // -1 or query_field level
  int out_mask;                      // decoder levels evaluated (bit L-1)
  unsigned long long* dbg = nullptr; // debug (lane 0): ns in prologue, staging, gather, decoder
  // presummed tables (presum.cu): S_L on the gather level's corner ids, one
  // (corners, 32) block per output level; only valid with inside_level == G
  const float* __restrict__ presum = nullptr;
  int64_t presum_offset = 0;
  int64_t presum_corners = 0;
};

__device__ __forceinline__ unsigned long long dbg_now() {  // NG_PROFILE laps: SM clock cycles
  return (unsigned long long)clock64();
}

// empty_space_value (field.py:185-191) in float64, numpy operation order.
__device__ __forceinline__ double empty_value(const ng_octree& t, const double x[3]) {
  double g[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double lo = np_max(dsub(t.region_lo[a], x[a]), 0.0);
    double hi = np_max(dsub(x[a], t.region_hi[a]), 0.0);
    g[a] = dadd(lo, hi);
  }
  double s = dadd(dadd(dmul(g[0], g[0]), dmul(g[1], g[1])), dmul(g[2], g[2]));
  return dadd(__dsqrt_rn(s), t.half_diag_finest);
}

__device__ __forceinline__ int64_t locate_point(const ng_octree& t, const double x[3], int level) {
  const int res = t.r0 << level;
  const int tl = level + t.n_virtual;
  uint64_t code = morton(bin_axis(x[0], res), bin_axis(x[1], res), bin_axis(x[2], res));
  return rank_lookup(t.bitmap[tl], t.rank[tl], code);
}

// 35 -> h -> 1 decoder in fp32; weights broadcast from shared memory.
__device__ __forceinline__ float mlp_eval(const float* __restrict__ dec, int h, const float xin[3],
                                          const float* zrow, bool& nonfinite) {
  float in[35];
  in[0] = xin[0];
  in[1] = xin[1];
  in[2] = xin[2];
  load_zrow(zrow, in + 3);
  float chk = 0.f;
#pragma unroll
  for (int k = 0; k < 35; ++k) chk += in[k] - in[k];
  nonfinite = !(chk == 0.f);
  const float* W2 = dec + h * NG_W1_STRIDE;
  float out = W2[h];  // b2
#pragma unroll 2
  for (int j = 0; j < h; ++j) {
    const float4* row = reinterpret_cast<const float4*>(dec + j * NG_W1_STRIDE);
    float4 r0 = row[0], r1 = row[1], r2 = row[2], r3 = row[3], r4 = row[4];
    float4 r5 = row[5], r6 = row[6], r7 = row[7], r8 = row[8];
    float a0 = r8.w;  // b1
    float a1 = 0.f, a2 = 0.f, a3 = 0.f;
    a0 = fmaf(r0.x, in[0], a0); a1 = fmaf(r0.y, in[1], a1); a2 = fmaf(r0.z, in[2], a2); a3 = fmaf(r0.w, in[3], a3);
    a0 = fmaf(r1.x, in[4], a0); a1 = fmaf(r1.y, in[5], a1); a2 = fmaf(r1.z, in[6], a2); a3 = fmaf(r1.w, in[7], a3);
    a0 = fmaf(r2.x, in[8], a0); a1 = fmaf(r2.y, in[9], a1); a2 = fmaf(r2.z, in[10], a2); a3 = fmaf(r2.w, in[11], a3);
    a0 = fmaf(r3.x, in[12], a0); a1 = fmaf(r3.y, in[13], a1); a2 = fmaf(r3.z, in[14], a2); a3 = fmaf(r3.w, in[15], a3);
    a0 = fmaf(r4.x, in[16], a0); a1 = fmaf(r4.y, in[17], a1); a2 = fmaf(r4.z, in[18], a2); a3 = fmaf(r4.w, in[19], a3);
    a0 = fmaf(r5.x, in[20], a0); a1 = fmaf(r5.y, in[21], a1); a2 = fmaf(r5.z, in[22], a2); a3 = fmaf(r5.w, in[23], a3);
    a0 = fmaf(r6.x, in[24], a0); a1 = fmaf(r6.y, in[25], a1); a2 = fmaf(r6.z, in[26], a2); a3 = fmaf(r6.w, in[27], a3);
    a0 = fmaf(r7.x, in[28], a0); a1 = fmaf(r7.y, in[29], a1); a2 = fmaf(r7.z, in[30], a2); a3 = fmaf(r7.w, in[31], a3);
    a0 = fmaf(r8.x, in[32], a0); a1 = fmaf(r8.y, in[33], a1); a2 = fmaf(r8.z, in[34], a2);
    float pre = (a0 + a1) + (a2 + a3);
    out = fmaf(W2[j], fmaxf(pre, 0.f), out);
  }
  return out;
}

// Per-lane outcome of one evaluation.
struct EvalLane {
  unsigned present;   // bit l-1: voxel exists at level l
  bool inside;        // inside the query_field level (true when not tested)
};

// SIMT decoder policy: each lane runs its point's MLP (skipped when no lane
// of the warp needs a decode).
struct SimtMlp {
  const EvalCtx& c;
  static constexpr bool kDirectZ = false;  // reads z rows from the warp's z tile
  __device__ __forceinline__ void prepare(int) const {}
  __device__ __forceinline__ void put_z4(int, int, const float*) const {}
  __device__ __forceinline__ float decode_direct(int, const float*, bool&) const { return 0.f; }
  __device__ __forceinline__ float operator()(int l, const float xf[3], const float* zrow, bool any,
                                              bool& bad) const {
    bad = false;
    if (!any) return 0.f;
    return mlp_eval(c.dec + (l - c.dec_first) * c.dec_stride, c.h, xf, zrow, bad);
  }
};

// Evaluate the warp's 32 points. At every decoder level L in ctx.out_mask
// (ascending) the decoder policy `mlp` turns the lane's z_L into a value and
// `emit(L, value_f32, nonfinite, lane)` is called warp-uniformly; lanes
// decide what to do with it.
template <int GB = NG_GATHER_BATCH, class Mlp, class Emit>
__device__ __forceinline__ EvalLane warp_eval(const ng_octree& tree, const EvalCtx& c, WarpScratch& ws,
                                              bool act, const double x[3], const Mlp& mlp, Emit&& emit) {
  const int lane = (int)lane_id();
#ifdef NG_PROFILE
  const bool dbg = c.dbg && lane == 0;
  unsigned long long t_mark = dbg ? dbg_now() : 0;
  auto lap = [&](int slot) {
    if (dbg) {
      const unsigned long long t = dbg_now();
      c.dbg[slot] += t - t_mark;
      t_mark = t;
    }
  };
#else
  auto lap = [](int) {};
#endif
  EvalLane res;
  res.present = 0;
  res.inside = true;
  bool dec = act;
  if (act && c.inside_level >= 0) {
    res.inside = locate_point(tree, x, c.inside_level) >= 0;
    dec = res.inside;
  }
  const int G = c.gather_level;
  const int resG = tree.r0 << G;
  int cell[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) cell[a] = bin_axis(x[a], resG);
  const float xf[3] = {(float)x[0], (float)x[1], (float)x[2]};
#pragma unroll
  for (int p = 0; p < 32; ++p) ws.zt[p][lane] = 0.f;

  // Per-lane lookups are software-pipelined across levels so their latency
  // hides behind the gather: while level l is gathered, level l+1's corner
  // ids and level l+2's bitmap / rank words are already in flight.
  auto level_code = [&](int l) -> uint64_t {
    const int sh = G - l;
    return morton(cell[0] >> sh, cell[1] >> sh, cell[2] >> sh);
  };
  auto words = [&](int l, uint64_t& w, uint32_t& r) {
    const int tl = l + tree.n_virtual;
    const uint64_t code = level_code(l);
    w = __ldg(tree.bitmap[tl] + (code >> 6));
    r = __ldg(tree.rank[tl] + (code >> 6));
  };
  auto index_of = [&](int l, uint64_t w, uint32_t r) -> int64_t {
    const uint32_t b = (uint32_t)(level_code(l) & 63);
    return ((w >> b) & 1ull) ? (int64_t)r + __popcll(w & ((1ull << b) - 1ull)) : -1;
  };
  auto corners = [&](int l, int64_t idx, int4& a, int4& b) {
    if (idx >= 0) {
      const int4* cr = reinterpret_cast<const int4*>(tree.corners[l + tree.n_virtual] + 8 * idx);
      a = __ldg(cr);
      b = __ldg(cr + 1);
    }
  };
  int64_t idx_cur = -1, idx_nxt = -1;
  int4 ca = make_int4(0, 0, 0, 0), cb = ca, na = ca, nb = ca;
  uint64_t w_nxt = 0;
  uint32_t r_nxt = 0;
  if (dec) {
    uint64_t w1;
    uint32_t r1;
    words(1, w1, r1);
    if (G >= 2) words(2, w_nxt, r_nxt);
    idx_cur = index_of(1, w1, r1);
    corners(1, idx_cur, ca, cb);
  }

  lap(0);
  for (int l = 1; l <= G; ++l) {
    const int sh = G - l;
    const int resl = resG >> sh;
    const int ci = cell[0] >> sh, cj = cell[1] >> sh, ck = cell[2] >> sh;
    const int64_t idx = idx_cur;
    const bool pres = idx >= 0;
    int4 ia = make_int4(0, 0, 0, 0), ib = ia;
    float4 wa = make_float4(0.f, 0.f, 0.f, 0.f), wb = wa;
    if (pres) {
      res.present |= 1u << (l - 1);
      ia = ca;
      ib = cb;
      // u = clip(f - cell, 0, 1) with f = (x + 1) * (res / 2)  (field.py:115-116)
      const double half = 0.5 * (double)resl;
      float u[3];
      const int cc[3] = {ci, cj, ck};
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        double f = dsub(dmul(dadd(x[a], 1.0), half), (double)cc[a]);
        f = f < 0.0 ? 0.0 : (f > 1.0 ? 1.0 : f);
        u[a] = (float)f;
      }
      const float wx0 = 1.f - u[0], wy0 = 1.f - u[1], wz0 = 1.f - u[2];
      // corner j weight = wx[j&1] * wy[j>>1&1] * wz[j>>2&1]  (field.py:122-135)
      wa = make_float4(wx0 * wy0 * wz0, u[0] * wy0 * wz0, wx0 * u[1] * wz0, u[0] * u[1] * wz0);
      wb = make_float4(wx0 * wy0 * u[2], u[0] * wy0 * u[2], wx0 * u[1] * u[2], u[0] * u[1] * u[2]);
    }
    // prefetch: corners of level l+1, words of level l+2
    if (dec && l < G) {
      idx_nxt = index_of(l + 1, w_nxt, r_nxt);
      corners(l + 1, idx_nxt, na, nb);
      if (l + 2 <= G) words(l + 2, w_nxt, r_nxt);
    }
    ws.ids[lane][0] = ia;
    ws.ids[lane][1] = ib;
    ws.w[lane][0] = wa;
    ws.w[lane][1] = wb;
    unsigned pm = __ballot_sync(FULL, pres);
    __syncwarp();
    lap(1);
#if NG_QUAD_GATHER
    // lane = (point slot lane / 8, channel quad lane % 8): a 128-byte corner
    // row is 8 lanes' 16-byte loads, so one load instruction covers 4
    // points' rows; GB points (2 GB rows per lane) are in flight per
    // iteration; absent slots re-read a present point and are dropped
    if constexpr (GB % 4 == 0) {
      const int grp = lane >> 3, sub = lane & 7;
      const float4* __restrict__ Z4 = reinterpret_cast<const float4*>(c.Z) + sub;
      while (pm) {
        int pp[GB];
#pragma unroll
        for (int q = 0; q < GB; ++q) {
          pp[q] = pm ? __ffs(pm) - 1 : -1;
          pm &= pm ? pm - 1 : 0u;
        }
        int mine[GB / 4];
        float4 v[GB / 4][8];
#pragma unroll
        for (int k = 0; k < GB / 4; ++k) {
          const int a0 = pp[4 * k], a1 = pp[4 * k + 1], a2 = pp[4 * k + 2], a3 = pp[4 * k + 3];
          mine[k] = grp == 0 ? a0 : (grp == 1 ? a1 : (grp == 2 ? a2 : a3));
          const int p = mine[k] >= 0 ? mine[k] : pp[0];
          const int4 a = ws.ids[p][0], b = ws.ids[p][1];
          v[k][0] = __ldg(Z4 + 8 * (int64_t)a.x);
          v[k][1] = __ldg(Z4 + 8 * (int64_t)a.y);
          v[k][2] = __ldg(Z4 + 8 * (int64_t)a.z);
          v[k][3] = __ldg(Z4 + 8 * (int64_t)a.w);
          v[k][4] = __ldg(Z4 + 8 * (int64_t)b.x);
          v[k][5] = __ldg(Z4 + 8 * (int64_t)b.y);
          v[k][6] = __ldg(Z4 + 8 * (int64_t)b.z);
          v[k][7] = __ldg(Z4 + 8 * (int64_t)b.w);
        }
#pragma unroll
        for (int k = 0; k < GB / 4; ++k) {
          if (mine[k] < 0) continue;
          const float4 u0 = ws.w[mine[k]][0], u1 = ws.w[mine[k]][1];
          const float wj[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
          float acc[4];
          corner_sum4<NG_FFMA2 != 0>(wj, v[k], acc);
          zt_quad<true>(&ws.zt[mine[k]][4 * sub], acc);
        }
      }
    } else
#endif
    {
    // lane = channel: coalesced 128-byte corner rows, 4 points (32 loads) in
    // flight per iteration; absent slots re-read a present point and are
    // masked out of the accumulation
    const float* __restrict__ Zc = c.Z + lane;
    while (pm) {
      int pp[GB];
#pragma unroll
      for (int q = 0; q < GB; ++q) {
        pp[q] = pm ? __ffs(pm) - 1 : -1;
        pm &= pm ? pm - 1 : 0u;
      }
      float v[GB][8];
#pragma unroll
      for (int q = 0; q < GB; ++q) {
        const int p = pp[q] >= 0 ? pp[q] : pp[0];
        const int4 a = ws.ids[p][0], b = ws.ids[p][1];
        v[q][0] = __ldg(Zc + 32 * (int64_t)a.x);
        v[q][1] = __ldg(Zc + 32 * (int64_t)a.y);
        v[q][2] = __ldg(Zc + 32 * (int64_t)a.z);
        v[q][3] = __ldg(Zc + 32 * (int64_t)a.w);
        v[q][4] = __ldg(Zc + 32 * (int64_t)b.x);
        v[q][5] = __ldg(Zc + 32 * (int64_t)b.y);
        v[q][6] = __ldg(Zc + 32 * (int64_t)b.z);
        v[q][7] = __ldg(Zc + 32 * (int64_t)b.w);
      }
#pragma unroll
      for (int q = 0; q < GB; ++q) {
        if (pp[q] < 0) continue;
        const float4 u0 = ws.w[pp[q]][0], u1 = ws.w[pp[q]][1];
        float acc = u0.x * v[q][0];
        acc = fmaf(u0.y, v[q][1], acc);
        acc = fmaf(u0.z, v[q][2], acc);
        acc = fmaf(u0.w, v[q][3], acc);
        acc = fmaf(u1.x, v[q][4], acc);
        acc = fmaf(u1.y, v[q][5], acc);
        acc = fmaf(u1.z, v[q][6], acc);
        acc = fmaf(u1.w, v[q][7], acc);
        ws.zt[pp[q]][lane] += acc;
      }
    }
    }
    __syncwarp();
    if ((c.out_mask >> (l - 1)) & 1) {
      lap(2);
      mlp.prepare(l);  // decoder policies that stage one level at a time (k_query_tc)
      const bool any = __any_sync(FULL, dec && (res.present != 0));
      bool bad = false;
      const float d = mlp(l, xf, &ws.zt[lane][0], any, bad);
      emit(l, d, bad && dec && res.present != 0, res);
      lap(3);
    }
    idx_cur = idx_nxt;
    ca = na;
    cb = nb;
  }
  __syncwarp();
  return res;
}

// warp_eval for points that are decoded only inside a level-G voxel
// (query_field with inside_level == G: the march and the normal probes).
// Every ancestor of the voxel exists, so all levels 1..G are present and
// z_L = sum_j w_j^G S_L[c_j] (presum.cu): one voxel lookup and 8 corner rows
// per output level instead of a lookup and 8 rows per level 1..L.
template <int GB = NG_GATHER_BATCH, class Mlp, class Emit>
__device__ __forceinline__ EvalLane warp_eval_presum(const ng_octree& tree, const EvalCtx& c, WarpScratch& ws,
                                                     bool act, const double x[3], const Mlp& mlp, Emit&& emit,
                                                     int64_t known = -1) {
  const int lane = (int)lane_id();
#ifdef NG_PROFILE
  const bool dbg = c.dbg && lane == 0;
  unsigned long long t_mark = dbg ? dbg_now() : 0;
  auto lap = [&](int slot) {
    if (dbg) {
      const unsigned long long t = dbg_now();
      c.dbg[slot] += t - t_mark;
      t_mark = t;
    }
  };
#else
  auto lap = [](int) {};
#endif
  EvalLane res;
  res.present = 0;
  res.inside = true;
  const int G = c.gather_level;
  const int resG = tree.r0 << G;
  const int tl = G + tree.n_virtual;
  int cell[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) cell[a] = bin_axis(x[a], resG);
  int64_t idx = -1;
  int4 ia = make_int4(0, 0, 0, 0), ib = ia;
  if (act) {
    // `known`: the caller already holds the level-G voxel containing x
    idx = known >= 0 ? known : rank_lookup(tree.bitmap[tl], tree.rank[tl], morton(cell[0], cell[1], cell[2]));
    res.inside = idx >= 0;  // query_field's inside test at the trace level (render.py:159-166)
    if (idx >= 0) {
      const int4* cr = reinterpret_cast<const int4*>(tree.corners[tl] + 8 * idx);
      ia = __ldg(cr);
      ib = __ldg(cr + 1);
    }
  }
  const bool pres = act && idx >= 0;
  lap(0);
  float4 wa = make_float4(0.f, 0.f, 0.f, 0.f), wb = wa;
  if (pres) {
    res.present = (G >= 32) ? 0xffffffffu : ((1u << G) - 1u);
    const double half = 0.5 * (double)resG;
    float u[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double f = dsub(dmul(dadd(x[a], 1.0), half), (double)cell[a]);
      f = f < 0.0 ? 0.0 : (f > 1.0 ? 1.0 : f);
      u[a] = (float)f;
    }
    const float wx0 = 1.f - u[0], wy0 = 1.f - u[1], wz0 = 1.f - u[2];
    wa = make_float4(wx0 * wy0 * wz0, u[0] * wy0 * wz0, wx0 * u[1] * wz0, u[0] * u[1] * wz0);
    wb = make_float4(wx0 * wy0 * u[2], u[0] * wy0 * u[2], wx0 * u[1] * u[2], u[0] * u[1] * u[2]);
    const int off = (int)c.presum_offset;
    ia = make_int4(ia.x - off, ia.y - off, ia.z - off, ia.w - off);
    ib = make_int4(ib.x - off, ib.y - off, ib.z - off, ib.w - off);
  }
  ws.ids[lane][0] = ia;
  ws.ids[lane][1] = ib;
  ws.w[lane][0] = wa;
  ws.w[lane][1] = wb;
  const unsigned pm0 = __ballot_sync(FULL, pres);
  const float xf[3] = {(float)x[0], (float)x[1], (float)x[2]};
  __syncwarp();
  lap(1);
  int slot = 0;
  for (int L = 1; L <= G; ++L) {
    if (!((c.out_mask >> (L - 1)) & 1)) continue;
    const float* __restrict__ Sc = c.presum + (int64_t)slot * c.presum_corners * 32 + lane;
    ++slot;
    unsigned pm = pm0;
    unsigned zbad = 0;  // (direct z) points whose z has a non-finite channel on this lane
#if NG_QUAD_GATHER
    if constexpr (GB % 4 == 0) {
      // 16-byte row loads: lane = (point slot lane / 8, channel quad lane % 8)
      const int grp = lane >> 3, sub = lane & 7;
      const float4* __restrict__ S4 = reinterpret_cast<const float4*>(Sc - lane) + sub;
      // With the direct-z decoder the zt scratch is free: 4 more points per
      // round stage their rows there with cp.async (no registers in flight)
      // while the register path loads and sums its GB points; they are summed
      // after, from shared memory, with the same FMA order.
      constexpr bool kStage = Mlp::kDirectZ && NG_STAGE_GATHER;
      float4* const stage = reinterpret_cast<float4*>(&ws.zt[0][0]);  // [grp][row][sub]
      while (pm) {
        int pp[GB];
#pragma unroll
        for (int q = 0; q < GB; ++q) {
          pp[q] = pm ? __ffs(pm) - 1 : -1;
          pm &= pm ? pm - 1 : 0u;
        }
        int smine = -1;
        if constexpr (kStage) {
          int ps[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            ps[q] = pm ? __ffs(pm) - 1 : -1;
            pm &= pm ? pm - 1 : 0u;
          }
          smine = grp == 0 ? ps[0] : (grp == 1 ? ps[1] : (grp == 2 ? ps[2] : ps[3]));
          if (smine >= 0) {
            const int4 a = ws.ids[smine][0], b = ws.ids[smine][1];
            const int id[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
            for (int j = 0; j < 8; ++j) cp_async16(stage + (grp * 8 + j) * 8 + sub, S4 + 8 * (int64_t)id[j]);
          }
          cp_async_commit();
        }
        int mine[GB / 4];
        float4 v[GB / 4][8];
#pragma unroll
        for (int k = 0; k < GB / 4; ++k) {
          const int a0 = pp[4 * k], a1 = pp[4 * k + 1], a2 = pp[4 * k + 2], a3 = pp[4 * k + 3];
          mine[k] = grp == 0 ? a0 : (grp == 1 ? a1 : (grp == 2 ? a2 : a3));
          const int p = mine[k] >= 0 ? mine[k] : pp[0];
          const int4 a = ws.ids[p][0], b = ws.ids[p][1];
          v[k][0] = __ldg(S4 + 8 * (int64_t)a.x);
          v[k][1] = __ldg(S4 + 8 * (int64_t)a.y);
          v[k][2] = __ldg(S4 + 8 * (int64_t)a.z);
          v[k][3] = __ldg(S4 + 8 * (int64_t)a.w);
          v[k][4] = __ldg(S4 + 8 * (int64_t)b.x);
          v[k][5] = __ldg(S4 + 8 * (int64_t)b.y);
          v[k][6] = __ldg(S4 + 8 * (int64_t)b.z);
          v[k][7] = __ldg(S4 + 8 * (int64_t)b.w);
        }
#pragma unroll
        for (int k = 0; k < GB / 4; ++k) {
          if (mine[k] < 0) continue;
          const float4 u0 = ws.w[mine[k]][0], u1 = ws.w[mine[k]][1];
          const float wj[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
          float acc[4];
          corner_sum4<false>(wj, v[k], acc);
          if constexpr (Mlp::kDirectZ) {  // z straight into the decoder's operand row
            mlp.put_z4(mine[k], sub, acc);
            zbad |= (isfinite(acc[0]) && isfinite(acc[1]) && isfinite(acc[2]) && isfinite(acc[3]) ? 0u : 1u)
                    << mine[k];
          } else {
            zt_quad<false>(&ws.zt[mine[k]][4 * sub], acc);
          }
        }
        if constexpr (kStage) {  // the staged point: each lane reads back the rows it copied
          cp_async_wait_all();
          if (smine >= 0) {
            const float4 u0 = ws.w[smine][0], u1 = ws.w[smine][1];
            const float wj[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
            float4 r[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = stage[(grp * 8 + j) * 8 + sub];
            float acc[4];
            acc[0] = wj[0] * r[0].x;
            acc[1] = wj[0] * r[0].y;
            acc[2] = wj[0] * r[0].z;
            acc[3] = wj[0] * r[0].w;
#pragma unroll
            for (int jj = 1; jj < 8; ++jj) {
              acc[0] = fmaf(wj[jj], r[jj].x, acc[0]);
              acc[1] = fmaf(wj[jj], r[jj].y, acc[1]);
              acc[2] = fmaf(wj[jj], r[jj].z, acc[2]);
              acc[3] = fmaf(wj[jj], r[jj].w, acc[3]);
            }
            mlp.put_z4(smine, sub, acc);
            zbad |= (isfinite(acc[0]) && isfinite(acc[1]) && isfinite(acc[2]) && isfinite(acc[3]) ? 0u : 1u)
                    << smine;
          }
          __syncwarp();  // the stage is rewritten next round
        }
      }
    } else
#endif
    {
    while (pm) {
      int pp[GB];
#pragma unroll
      for (int q = 0; q < GB; ++q) {
        pp[q] = pm ? __ffs(pm) - 1 : -1;
        pm &= pm ? pm - 1 : 0u;
      }
      float v[GB][8];
#pragma unroll
      for (int q = 0; q < GB; ++q) {
        const int p = pp[q] >= 0 ? pp[q] : pp[0];
        const int4 a = ws.ids[p][0], b = ws.ids[p][1];
        v[q][0] = __ldg(Sc + 32 * (int64_t)a.x);
        v[q][1] = __ldg(Sc + 32 * (int64_t)a.y);
        v[q][2] = __ldg(Sc + 32 * (int64_t)a.z);
        v[q][3] = __ldg(Sc + 32 * (int64_t)a.w);
        v[q][4] = __ldg(Sc + 32 * (int64_t)b.x);
        v[q][5] = __ldg(Sc + 32 * (int64_t)b.y);
        v[q][6] = __ldg(Sc + 32 * (int64_t)b.z);
        v[q][7] = __ldg(Sc + 32 * (int64_t)b.w);
      }
#pragma unroll
      for (int q = 0; q < GB; ++q) {
        if (pp[q] < 0) continue;
        const float4 u0 = ws.w[pp[q]][0], u1 = ws.w[pp[q]][1];
        float acc = u0.x * v[q][0];
        acc = fmaf(u0.y, v[q][1], acc);
        acc = fmaf(u0.z, v[q][2], acc);
        acc = fmaf(u0.w, v[q][3], acc);
        acc = fmaf(u1.x, v[q][4], acc);
        acc = fmaf(u1.y, v[q][5], acc);
        acc = fmaf(u1.z, v[q][6], acc);
        acc = fmaf(u1.w, v[q][7], acc);
        ws.zt[pp[q]][lane] = acc;
      }
    }
    }
    __syncwarp();
    lap(2);
    bool bad = false;
    float d;
    if constexpr (Mlp::kDirectZ && GB % 4 == 0 && NG_QUAD_GATHER) {
      // this lane's point: non-finite z on any channel lane, or non-finite x
      const unsigned zb = __reduce_or_sync(FULL, zbad);
      d = mlp.decode_direct(L, xf, bad);
      bad = bad || ((zb >> lane) & 1u);
    } else {
      const bool any = __any_sync(FULL, pres);
      d = mlp(L, xf, &ws.zt[lane][0], any, bad);
    }
    emit(L, d, bad && pres, res);
    lap(3);
  }
  __syncwarp();
  return res;
}

// Stage decoder blocks [first, last] into shared memory (whole CTA).
__device__ __forceinline__ void stage_decoders(float* dst, const float* __restrict__ src, int first,
                                               int last, int stride) {
  const int n = (last - first + 1) * stride;
  const float4* s4 = reinterpret_cast<const float4*>(src + (first - 1) * stride);
  float4* d4 = reinterpret_cast<float4*>(dst);
  for (int i = threadIdx.x; i < n / 4; i += blockDim.x) d4[i] = __ldg(s4 + i);
  __syncthreads();
}

// Counters accumulated per lane and flushed once per warp.
struct LaneCounters {
  long long evals = 0, missing = 0, empty = 0, nonfinite = 0;
  __device__ __forceinline__ void flush(ng_counters* d) {
    long long v[4] = {evals, missing, empty, nonfinite};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
#pragma unroll
      for (int o = 16; o; o >>= 1) v[k] += __shfl_xor_sync(FULL, v[k], o);
    }
    if (lane_id() == 0 && d != nullptr) {
      if (v[0]) atomicAdd((unsigned long long*)&d->decoder_evals, (unsigned long long)v[0]);
      if (v[1]) atomicAdd((unsigned long long*)&d->evals_missing_level, (unsigned long long)v[1]);
      if (v[2]) atomicAdd((unsigned long long*)&d->empty_fallbacks, (unsigned long long)v[2]);
      if (v[3]) atomicAdd((unsigned long long*)&d->nonfinite_inputs, (unsigned long long)v[3]);
    }
  }
};

// Full query_field / blend / predict semantics for one lane: combines the
// emitted decoder outputs into the value the reference returns.
struct BlendAcc {
  int base;        // decoder level for predict / lower blend level
  double alpha;    // 0 -> plain predict(base)
  double lo = 0.0, hi = 0.0;
};

}  // namespace ng
