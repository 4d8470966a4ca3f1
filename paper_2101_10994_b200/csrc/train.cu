// Training step of the neural field on sm_100a: loss, reverse-mode gradients
// and Adam.
//
// Reference: octfield/field.py:286-409 (forward cache, backward,
// scatter_add_rows) and octfield/trainer.py:87-144, 165-296 (adam_step,
// loss_batch, train, _batch_pass). The reference keeps float64 master
// weights and computes in float64; so does this path (B200 has full-rate
// fp64 relative to the work here, which is tiny per batch and bound by the
// dense Adam sweep over Z).
//
// One batch step, all on one stream, deterministic (no fp atomics):
//   memset      corner counts / fill cursors / decoder-touched flags
//   k_train_points   warp per point: locate + corner ids + trilinear weights at
//                    levels 1..Lmax (fp64), running feature sums, then per active
//                    level L the 35->h->1 decoder forward, residual, dout,
//                    dpre (relu mask) and dz = dpre W1[:,3:]; the per-level
//                    feature gradient G_l = sum_{L>=l} dz_L; integer counts of
//                    (corner, record) contributions
//   exclusive scan   counts -> segment offsets (scan.cu)
//   k_train_fill     records -> corner segments (slot order is arbitrary)
//   k_train_dec_grads  dW1|db1 = dpre^T [x z 1], dW2 = dout^T relu(pre), db2,
//                      per-level residual sums; fixed-order reductions
//   k_train_rows     warp per corner row: sort the segment's record keys,
//                    sum w * G in key order (= dZ row, field.py:388-394),
//                    Adam update of the row (dense: every row decays m, v)
//   k_train_dec_adam Adam on the decoders that received a gradient
#include "common.cuh"

namespace ng {

constexpr int TR_WARPS = 4;    // points per CTA in k_train_points
constexpr int TR_LM = 12;      // max feature levels handled by the trainer
constexpr int TR_HMAX = 128;   // max decoder width
constexpr int W1S = 37;        // smem row stride (doubles) of the staged W1b block
constexpr double BETA1 = 0.9, BETA2 = 0.999, ADAM_EPS = 1e-8;  // trainer.py:29-31

static inline int tr_grid(int64_t n, int nt) { return (int)((n + nt - 1) / nt); }

struct TrainLayout {
  size_t rec_w, rec_id, G, inp, pre, dpre, dout, sq, cnt, off, fill, list, sorted, scan, gdec, touched, total;
};

// Workspace carve-up for a batch capacity B, max level LM, A active-level
// slots (= n_decoders), decoder width h, C corners and dec_stride doubles.
static TrainLayout train_layout(int64_t B, int LM, int A, int h, int64_t C, int dec_stride) {
  TrainLayout L;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o += (bytes + 255) & ~(size_t)255;
    return at;
  };
  L.rec_w = take(sizeof(double) * B * LM * 8);
  L.rec_id = take(sizeof(int32_t) * B * LM * 8);
  L.G = take(sizeof(double) * B * LM * 32);
  L.inp = take(sizeof(double) * A * B * 36);
  L.pre = take(sizeof(double) * A * B * h);
  L.dpre = take(sizeof(double) * A * B * h);
  L.dout = take(sizeof(double) * A * B);
  L.sq = take(sizeof(double) * A * B);
  L.cnt = take(sizeof(int64_t) * C);
  L.fill = take(sizeof(int32_t) * C);
  L.touched = take(sizeof(int32_t) * 32);
  L.off = take(sizeof(int64_t) * C);
  L.list = take(sizeof(int32_t) * B * LM * 8);
  L.sorted = take(sizeof(int32_t) * B * LM * 8);
  L.scan = take(ng_scan_scratch_bytes(C > 0 ? C : 1));
  L.gdec = take(sizeof(double) * A * dec_stride);
  L.total = o;
  return L;
}

struct TrainArgs {
  // parameters (fp64 masters)
  double* Z;
  double* Zm;
  double* Zv;
  double* dec;
  double* decm;
  double* decv;
  int m, h, n_dec, dec_stride;
  int64_t C;
  // batch
  const double* pts;
  const double* dist;
  const double* upstream;  // backward(cache, upstream) mode: dout = upstream[p]
  int64_t n;
  int LM;                  // levels interpolated: highest active level
  int active_mask;
  int update_decoders;
  int mode;                // 0 Adam, 1 gradients only
  double two_over_n;       // 2.0 / denom (trainer.py:143)
  double lr, c1, c2;
  int64_t batch_index;
  // workspace
  double* rec_w;
  int32_t* rec_id;
  double* G;
  double* inp;
  double* pre;
  double* dpre;
  double* dout;
  double* sq;
  int64_t* cnt;
  int64_t* off;
  int32_t* fill;
  int32_t* list;
  int32_t* sorted;
  double* gdec;
  int32_t* touched;
  // outputs
  double* level_sums;      // (n_dec): += residual sums (mode 0: epoch accumulators)
  double* grad_Z;          // mode 1: (C, 32) +=
  double* grad_dec;        // mode 1: n_dec * dec_stride +=
  int32_t* dec_touched;    // mode 1: 1 where a decoder received a gradient
  double* psi_out;         // optional (n, LM, 32): per-level interpolated features
  int64_t* status;         // [0] = 1 + batch index of the first divergence
};

__device__ __forceinline__ int level_slot(int mask, int L) { return __popc(mask & ((1 << (L - 1)) - 1)); }

__device__ __forceinline__ void flag_divergence(int64_t* status, int64_t batch) {
  atomicCAS((unsigned long long*)status, 0ull, (unsigned long long)(batch + 1));
}

struct TrainWarp {
  int ids[TR_LM][8];
  double w[TR_LM][8];
  double z[TR_LM][32];   // running feature sum through level l
  double dz[TR_LM][32];  // dz of active slot a
  double dpre[TR_HMAX];
  double inp[36];
};

// Per point (one warp): interpolation, decoder forward/backward at every
// active level, feature-gradient records (field.py:337-394, trainer.py:132-143).
__global__ void __launch_bounds__(TR_WARPS * 32) k_train_points(const __grid_constant__ ng_octree tree,
                                                                const __grid_constant__ TrainArgs A) {
  extern __shared__ __align__(16) double tr_smem[];
  double* sW1 = tr_smem;              // h x W1S: x weights, feature weights, (col 35) b1
  double* sW2 = sW1 + TR_HMAX * W1S;  // h weights, then b2
  TrainWarp* tws = reinterpret_cast<TrainWarp*>(sW2 + TR_HMAX + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  TrainWarp& tw = tws[warp];
  const int64_t p = (int64_t)blockIdx.x * TR_WARPS + warp;
  const bool valid = p < A.n;
  const int LM = A.LM, h = A.h, m = A.m;

  double x[3] = {0.0, 0.0, 0.0};
  if (valid) {
    x[0] = __ldg(A.pts + 3 * p);
    x[1] = __ldg(A.pts + 3 * p + 1);
    x[2] = __ldg(A.pts + 3 * p + 2);
  }
  // ---- locate + corner ids + weights, lane l-1 handles level l (field.py:104-119)
  bool pres = false;
  if (valid && lane < LM) {
    const int l = lane + 1;
    const int res = tree.r0 << l;
    const int tl = l + tree.n_virtual;
    const int c0 = bin_axis(x[0], res), c1 = bin_axis(x[1], res), c2 = bin_axis(x[2], res);
    const int64_t idx = rank_lookup(tree.bitmap[tl], tree.rank[tl], morton(c0, c1, c2));
    pres = idx >= 0;
    if (pres) {
      const int4* cr = reinterpret_cast<const int4*>(tree.corners[tl] + 8 * idx);
      const int4 a = __ldg(cr), b = __ldg(cr + 1);
      tw.ids[lane][0] = a.x; tw.ids[lane][1] = a.y; tw.ids[lane][2] = a.z; tw.ids[lane][3] = a.w;
      tw.ids[lane][4] = b.x; tw.ids[lane][5] = b.y; tw.ids[lane][6] = b.z; tw.ids[lane][7] = b.w;
      // u = clip((x - DOMAIN_MIN) * (res / span) - cell, 0, 1); w_j = cx * cy * cz (field.py:115-135)
      const double half = 0.5 * (double)res;
      const int cc[3] = {c0, c1, c2};
      double u[3];
#pragma unroll
      for (int a3 = 0; a3 < 3; ++a3) {
        double f = dsub(dmul(dadd(x[a3], 1.0), half), (double)cc[a3]);
        u[a3] = f < 0.0 ? 0.0 : (f > 1.0 ? 1.0 : f);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double wx = (j & 1) ? u[0] : dsub(1.0, u[0]);
        const double wy = ((j >> 1) & 1) ? u[1] : dsub(1.0, u[1]);
        const double wz = ((j >> 2) & 1) ? u[2] : dsub(1.0, u[2]);
        tw.w[lane][j] = dmul(dmul(wx, wy), wz);
      }
    }
  }
  const unsigned present = __ballot_sync(FULL, pres);
  __syncwarp();

  // ---- running feature sums, lane = channel (field.py:119, 154-169)
  {
    double zrun = 0.0;
    for (int l = 1; l <= LM; ++l) {
      double psi = 0.0;
      if ((present >> (l - 1)) & 1) {
        const double* Zc = A.Z + lane;
#pragma unroll
        for (int j = 0; j < 8; ++j) psi = dadd(psi, dmul(tw.w[l - 1][j], __ldg(Zc + 32 * (int64_t)tw.ids[l - 1][j])));
      }
      zrun = dadd(zrun, psi);
      tw.z[l - 1][lane] = zrun;
      if (A.psi_out && valid) A.psi_out[(p * LM + (l - 1)) * 32 + lane] = psi;
    }
  }
  double dval = 0.0, upv = 0.0;
  if (valid) {
    if (A.upstream) upv = __ldg(A.upstream + p);
    else if (A.dist) dval = __ldg(A.dist + p);
  }

  // ---- active levels, ascending (trainer.py:132-143)
  for (int L = 1; L <= LM; ++L) {
    if (!((A.active_mask >> (L - 1)) & 1)) continue;
    const int a = level_slot(A.active_mask, L);
    __syncthreads();
    {
      const double* blk = A.dec + (int64_t)(L - 1) * A.dec_stride;
      for (int i = threadIdx.x; i < h * 36; i += blockDim.x) sW1[(i / 36) * W1S + (i % 36)] = blk[i];
      for (int i = threadIdx.x; i <= h; i += blockDim.x) sW2[i] = blk[h * 36 + i];
    }
    __syncthreads();
    const bool dec = valid && (present & ((1u << L) - 1u)) != 0u;
    const int64_t row = (int64_t)a * A.n + p;
    if (dec) {
      if (lane < 3) tw.inp[lane] = x[lane];
      tw.inp[3 + lane] = (lane < m) ? tw.z[L - 1][lane] : 0.0;
      if (lane == 0) tw.inp[35] = 1.0;
      __syncwarp();
      double prev[TR_HMAX / 32];
      double part = 0.0;
#pragma unroll
      for (int q = 0; q < TR_HMAX / 32; ++q) {
        const int j = lane + 32 * q;
        prev[q] = 0.0;
        if (j < h) {
          const double* wr = sW1 + j * W1S;
          double s = 0.0;
          for (int k = 0; k < 3 + m; ++k) s = fma(tw.inp[k], wr[k], s);
          const double pr = dadd(s, wr[35]);  // inp @ W1.T + b1 (field.py:350)
          prev[q] = pr;
          part = fma(pr > 0.0 ? pr : 0.0, sW2[j], part);
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(FULL, part, o);
      const double out = dadd(part, sW2[h]);
      // resid = where(mask_L, out - d, 0); upstream = (2/n) resid (trainer.py:139-143)
      const bool inL = (present >> (L - 1)) & 1;
      const double resid = inL ? dsub(out, dval) : 0.0;
      const double dout = A.upstream ? upv : dmul(A.two_over_n, resid);
      // dhidden = dout * W2; dpre = where(pre > 0, dhidden, 0) (field.py:381-383)
#pragma unroll
      for (int q = 0; q < TR_HMAX / 32; ++q) {
        const int j = lane + 32 * q;
        if (j < h) {
          const double dp = prev[q] > 0.0 ? dmul(dout, sW2[j]) : 0.0;
          tw.dpre[j] = dp;
          A.dpre[row * h + j] = dp;
          A.pre[row * h + j] = prev[q];
        }
      }
      A.inp[row * 36 + lane] = tw.inp[lane];
      if (lane < 4) A.inp[row * 36 + 32 + lane] = tw.inp[32 + lane];
      if (lane == 0) {
        A.dout[row] = dout;
        A.sq[row] = dmul(resid, resid);
        A.touched[L - 1] = 1;
      }
      __syncwarp();
      // dz = (dpre @ W1)[:, 3:] (field.py:386-387), lane = channel
      double s = 0.0;
      if (lane < m)
        for (int j = 0; j < h; ++j) s = fma(tw.dpre[j], sW1[j * W1S + 3 + lane], s);
      tw.dz[a][lane] = s;
    } else if (valid) {
      for (int j = lane; j < h; j += 32) {
        A.dpre[row * h + j] = 0.0;
        A.pre[row * h + j] = 0.0;
      }
      A.inp[row * 36 + lane] = 0.0;
      if (lane < 4) A.inp[row * 36 + 32 + lane] = 0.0;
      if (lane == 0) {
        A.dout[row] = 0.0;
        A.sq[row] = 0.0;
      }
      tw.dz[a][lane] = 0.0;
    }
  }
  if (!valid) return;
  __syncwarp();
  // ---- per-level feature gradient G_l = sum over active L >= l of dz_L (field.py:388-394)
  for (int l = 1; l <= LM; ++l) {
    if (!((present >> (l - 1)) & 1)) continue;
    double g = 0.0;
    for (int L = l; L <= LM; ++L)
      if ((A.active_mask >> (L - 1)) & 1) g = dadd(g, tw.dz[level_slot(A.active_mask, L)][lane]);
    A.G[(p * LM + (l - 1)) * 32 + lane] = g;
  }
  // ---- contribution records: key = (p * LM + l - 1) * 8 + j
  for (int s = lane; s < 8 * LM; s += 32) {
    const int l = s / 8 + 1, j = s % 8;
    const int64_t key = (p * LM + (l - 1)) * 8 + j;
    if ((present >> (l - 1)) & 1) {
      const int id = tw.ids[l - 1][j];
      A.rec_id[key] = id;
      A.rec_w[key] = tw.w[l - 1][j];
      atomicAdd((unsigned long long*)(A.cnt + id), 1ull);
    } else {
      A.rec_id[key] = -1;
    }
  }
}

// Records into their corner's segment.
__global__ void k_train_fill(const __grid_constant__ TrainArgs A, int64_t n_rec) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rec) return;
  const int id = A.rec_id[r];
  if (id < 0) return;
  const int64_t slot = A.off[id] + atomicAdd(A.fill + id, 1);
  A.list[slot] = (int32_t)r;
}

// Decoder gradients (field.py:377-385) and per-level residual sums
// (trainer.py:140): grid (active slot, 32-wide j block), 8 warps per CTA,
// warp w reduces points w, w+8, ... in order; warps are combined in order.
constexpr int DG_WARPS = 8;
__global__ void __launch_bounds__(DG_WARPS * 32) k_train_dec_grads(const __grid_constant__ TrainArgs A) {
  extern __shared__ __align__(16) double dg_smem[];  // [DG_WARPS][38][32]
  const int a = blockIdx.x, jb = blockIdx.y;
  int L = 0;
  for (int l = 1, k = 0; l <= 31; ++l)
    if ((A.active_mask >> (l - 1)) & 1) {
      if (k == a) { L = l; break; }
      ++k;
    }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = A.h;
  const int j = jb * 32 + lane;
  double acc[36];
#pragma unroll
  for (int k = 0; k < 36; ++k) acc[k] = 0.0;
  double aw2 = 0.0, ab2 = 0.0;
  if (j < h) {
    for (int64_t p = warp; p < A.n; p += DG_WARPS) {
      const int64_t row = (int64_t)a * A.n + p;
      const double d = A.dpre[row * h + j];
      const double dout = A.dout[row];
      const double pr = A.pre[row * h + j];
      aw2 = fma(dout, pr > 0.0 ? pr : 0.0, aw2);
      ab2 = dadd(ab2, dout);
      if (d != 0.0) {
        const double2* ir = reinterpret_cast<const double2*>(A.inp + row * 36);
#pragma unroll
        for (int k = 0; k < 18; ++k) {
          const double2 v = __ldg(ir + k);
          acc[2 * k] = fma(d, v.x, acc[2 * k]);
          acc[2 * k + 1] = fma(d, v.y, acc[2 * k + 1]);
        }
      }
    }
  }
  double* mine = dg_smem + (size_t)warp * 38 * 32;
#pragma unroll
  for (int k = 0; k < 36; ++k) mine[k * 32 + lane] = acc[k];
  mine[36 * 32 + lane] = aw2;
  mine[37 * 32 + lane] = ab2;
  __syncthreads();
  const bool adam = A.mode == 0;
  double* gblk = adam ? A.gdec + (int64_t)a * A.dec_stride : A.grad_dec + (int64_t)(L - 1) * A.dec_stride;
  bool bad = false;       // non-finite decoder gradient (adam_step raises, trainer.py:96-97)
  bool bad_loss = false;  // non-finite batch loss (trainer.py:233-236)
  for (int t = threadIdx.x; t < 38 * 32; t += blockDim.x) {
    const int k = t / 32, jj = jb * 32 + (t % 32);
    if (jj >= h) continue;
    if (k == 37 && (jb != 0 || jj != 0)) continue;  // b2 once
    double s = 0.0;
    for (int w = 0; w < DG_WARPS; ++w) s = dadd(s, dg_smem[(size_t)w * 38 * 32 + t]);
    int64_t dst;
    if (k < 36) {
      if (k >= 3 + A.m && k != 35) continue;  // padding columns stay zero
      dst = (int64_t)jj * 36 + k;
    } else if (k == 36) {
      dst = (int64_t)h * 36 + jj;
    } else {
      dst = (int64_t)h * 36 + h;
    }
    if (!isfinite(s)) bad = true;
    if (adam) gblk[dst] = s;
    else gblk[dst] += s;
  }
  // residual sum of this level: warp 0 of the first j block (fixed order)
  if (jb == 0 && warp == 0) {
    double s = 0.0;
    for (int64_t p = lane; p < A.n; p += 32) s = dadd(s, A.sq[(int64_t)a * A.n + p]);
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
    if (lane == 0) {
      if (!isfinite(s)) bad_loss = true;
      if (adam) A.level_sums[L - 1] = dadd(A.level_sums[L - 1], s);
      else A.level_sums[L - 1] = s;
      if (!adam && A.dec_touched && A.touched[L - 1]) A.dec_touched[L - 1] = 1;
    }
  }
  if (adam && (bad_loss || (bad && A.update_decoders && A.touched[L - 1])))
    flag_divergence(A.status, A.batch_index);
}

// Adam moment update and parameter step for one element (trainer.py:95-103),
// numpy's operation order, no contraction.
__device__ __forceinline__ void adam_elem(double& prm, double& mm, double& vv, double g, double lr, double c1,
                                          double c2) {
  mm = dadd(dmul(mm, BETA1), dmul(1.0 - BETA1, g));
  vv = dadd(dmul(vv, BETA2), dmul(1.0 - BETA2, dmul(g, g)));
  const double upd = __ddiv_rn(dmul(lr, __ddiv_rn(mm, c1)), dadd(__dsqrt_rn(__ddiv_rn(vv, c2)), ADAM_EPS));
  prm = dsub(prm, upd);
}

// One warp per corner row: dZ row = sum over the segment's records in key
// order, then Adam (mode 0) or accumulate into grad_Z (mode 1).
__global__ void __launch_bounds__(256) k_train_rows(const __grid_constant__ TrainArgs A) {
  const int lane = threadIdx.x & 31;
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= A.C) return;
  const int64_t S = A.cnt[c];
  const int64_t base = A.off[c];
  double g = 0.0;
  auto add_rec = [&](int key) {
    const int64_t gp = key >> 3;  // (p * LM + l - 1)
    g = dadd(g, dmul(A.rec_w[key], A.G[gp * 32 + lane]));
  };
  if (S > 0 && S <= 32) {
    const int key = lane < S ? A.list[base + lane] : 0x7fffffff;
    int rank = 0;
    for (int i = 0; i < (int)S; ++i) rank += __shfl_sync(FULL, key, i) < key;
    for (int r = 0; r < (int)S; ++r) {
      const unsigned who = __ballot_sync(FULL, lane < S && rank == r);
      add_rec(__shfl_sync(FULL, key, __ffs(who) - 1));
    }
  } else if (S > 32) {
    for (int64_t i0 = 0; i0 < S; i0 += 32) {
      const bool own = i0 + lane < S;
      const int key = own ? A.list[base + i0 + lane] : 0x7fffffff;
      int64_t rank = 0;
      for (int64_t i = 0; i < S; ++i) rank += A.list[base + i] < key;
      if (own) A.sorted[base + rank] = key;
    }
    __syncwarp();
    __threadfence_block();
    for (int64_t r = 0; r < S; ++r) add_rec(A.sorted[base + r]);
  }
  const int64_t e = c * 32 + lane;
  if (A.mode == 0) {
    if (*(volatile int64_t*)A.status) return;
    if (!isfinite(g)) {
      flag_divergence(A.status, A.batch_index);
      return;
    }
    double prm = A.Z[e], mm = A.Zm[e], vv = A.Zv[e];
    adam_elem(prm, mm, vv, g, A.lr, A.c1, A.c2);
    A.Z[e] = prm;
    A.Zm[e] = mm;
    A.Zv[e] = vv;
  } else if (S > 0) {
    A.grad_Z[e] = dadd(A.grad_Z[e], g);
  }
}

// Adam on every decoder that received a gradient this batch (trainer.py:100,
// 290-296: untouched decoders keep their moments).
__global__ void k_train_dec_adam(const __grid_constant__ TrainArgs A) {
  const int a = blockIdx.y;
  int L = 0;
  for (int l = 1, k = 0; l <= 31; ++l)
    if ((A.active_mask >> (l - 1)) & 1) {
      if (k == a) { L = l; break; }
      ++k;
    }
  if (!A.touched[L - 1] || *(volatile int64_t*)A.status) return;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t used = (int64_t)A.h * 36 + A.h + 1;
  if (i >= used) return;
  const int64_t e = (int64_t)(L - 1) * A.dec_stride + i;
  double prm = A.dec[e], mm = A.decm[e], vv = A.decv[e];
  adam_elem(prm, mm, vv, A.gdec[(int64_t)a * A.dec_stride + i], A.lr, A.c1, A.c2);
  A.dec[e] = prm;
  A.decm[e] = mm;
  A.decv[e] = vv;
}

// Generic Adam over one parameter array (adam_step, trainer.py:87-103):
// pass 1 flags non-finite gradients, pass 2 updates only if none.
__global__ void k_adam_check(const double* g, int64_t n, int64_t* d_bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool bad = i < n && !isfinite(g[i]);
  if (__any_sync(FULL, bad) && (threadIdx.x & 31) == 0) atomicExch((unsigned long long*)d_bad, 1ull);
}

__global__ void k_adam_apply(double* p, double* m, double* v, const double* g, int64_t n, double lr, double c1,
                             double c2, const int64_t* d_bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || *d_bad) return;
  double prm = p[i], mm = m[i], vv = v[i];
  adam_elem(prm, mm, vv, g[i], lr, c1, c2);
  p[i] = prm;
  m[i] = mm;
  v[i] = vv;
}

static size_t points_smem_bytes() {
  return sizeof(double) * (TR_HMAX * W1S + TR_HMAX + 4) + sizeof(TrainWarp) * TR_WARPS;
}

static int highest_level(int mask) { return 32 - __builtin_clz((unsigned)mask); }

}  // namespace ng

using namespace ng;

extern "C" {

size_t ng_train_workspace_bytes(const ng_octree* tree, int64_t batch_capacity, int32_t h, int32_t n_decoders,
                                int64_t corner_count, int32_t dec_stride) {
  return train_layout(batch_capacity, tree->max_level, n_decoders, h, corner_count, dec_stride).total;
}

int ng_train_batch(const ng_octree* tree, const ng_train_params* P, const ng_train_step* st, const double* pts,
                   const double* dist, const double* upstream, int64_t n, int64_t batch_capacity, void* ws,
                   size_t ws_bytes, double* level_sums, double* grad_Z, double* grad_dec, int32_t* dec_touched,
                   double* psi_out, int64_t* status, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (P->h < 1 || P->h > TR_HMAX || P->m < 1 || P->m > 32) {
    set_error("trainer supports 1 <= h <= %d and 1 <= m <= 32 (got h=%d, m=%d)", TR_HMAX, P->h, P->m);
    return NG_ERR_STRUCTURAL;
  }
  if (tree->max_level > TR_LM || P->n_decoders != tree->max_level) {
    set_error("trainer needs n_decoders == max_level <= %d", TR_LM);
    return NG_ERR_STRUCTURAL;
  }
  const int mask = st->active_mask;
  if (mask <= 0 || highest_level(mask) > tree->max_level) {
    set_error("active level mask 0x%x outside 1..%d", mask, tree->max_level);
    return NG_ERR_CONFIG;
  }
  if (n > batch_capacity) {
    set_error("batch of %lld points above the workspace capacity %lld", (long long)n, (long long)batch_capacity);
    return NG_ERR_CAPACITY;
  }
  if (n <= 0) return NG_OK;
  const TrainLayout Ly = train_layout(batch_capacity, tree->max_level, P->n_decoders, P->h, P->corner_count,
                                      P->dec_stride);
  if (ws_bytes < Ly.total) {
    set_error("train workspace %zu < %zu bytes", ws_bytes, Ly.total);
    return NG_ERR_CAPACITY;
  }
  char* b = (char*)ws;
  TrainArgs A;
  A.Z = P->Z; A.Zm = P->Zm; A.Zv = P->Zv;
  A.dec = P->dec; A.decm = P->decm; A.decv = P->decv;
  A.m = P->m; A.h = P->h; A.n_dec = P->n_decoders; A.dec_stride = P->dec_stride; A.C = P->corner_count;
  A.pts = pts; A.dist = dist; A.upstream = upstream; A.n = n;
  A.LM = highest_level(mask);
  A.active_mask = mask;
  A.update_decoders = st->update_decoders;
  A.mode = st->mode;
  A.two_over_n = 2.0 / st->denom;
  A.lr = st->lr; A.c1 = st->c1; A.c2 = st->c2;
  A.batch_index = st->batch_index;
  A.rec_w = (double*)(b + Ly.rec_w);
  A.rec_id = (int32_t*)(b + Ly.rec_id);
  A.G = (double*)(b + Ly.G);
  A.inp = (double*)(b + Ly.inp);
  A.pre = (double*)(b + Ly.pre);
  A.dpre = (double*)(b + Ly.dpre);
  A.dout = (double*)(b + Ly.dout);
  A.sq = (double*)(b + Ly.sq);
  A.cnt = (int64_t*)(b + Ly.cnt);
  A.off = (int64_t*)(b + Ly.off);
  A.fill = (int32_t*)(b + Ly.fill);
  A.list = (int32_t*)(b + Ly.list);
  A.sorted = (int32_t*)(b + Ly.sorted);
  A.gdec = (double*)(b + Ly.gdec);
  A.touched = (int32_t*)(b + Ly.touched);
  A.level_sums = level_sums;
  A.grad_Z = grad_Z;
  A.grad_dec = grad_dec;
  A.dec_touched = dec_touched;
  A.psi_out = psi_out;
  A.status = status;
  if (A.mode == 1 && (!grad_Z || !grad_dec)) {
    set_error("gradient mode needs grad_Z and grad_dec");
    return NG_ERR_STRUCTURAL;
  }
  // counts, fill cursors and touched flags are contiguous in the layout
  int r = cuda_status(cudaMemsetAsync(b + Ly.cnt, 0, Ly.off - Ly.cnt, s), "train memset");
  if (r) return r;
  const size_t smem = points_smem_bytes();
  static bool attr = false;
  if (!attr) {
    if ((r = cuda_status(cudaFuncSetAttribute(k_train_points, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)smem), "train smem attr")))
      return r;
    if ((r = cuda_status(cudaFuncSetAttribute(k_train_dec_grads, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)(sizeof(double) * DG_WARPS * 38 * 32)), "train smem attr")))
      return r;
    attr = true;
  }
  k_train_points<<<tr_grid(n, TR_WARPS), TR_WARPS * 32, smem, s>>>(*tree, A);
  NG_CHECK_LAUNCH("k_train_points");
  if (A.mode == 2) return NG_OK;  // forward cache only (ng_train_export)
  if ((r = ng_exclusive_sum_i64(A.cnt, A.C, A.off, b + Ly.scan, ng_scan_scratch_bytes(A.C), stream))) return r;
  const int64_t n_rec = n * A.LM * 8;
  k_train_fill<<<tr_grid(n_rec, 256), 256, 0, s>>>(A, n_rec);
  NG_CHECK_LAUNCH("k_train_fill");
  const int n_act = __builtin_popcount((unsigned)mask);
  k_train_dec_grads<<<dim3(n_act, (A.h + 31) / 32), DG_WARPS * 32, sizeof(double) * DG_WARPS * 38 * 32, s>>>(A);
  NG_CHECK_LAUNCH("k_train_dec_grads");
  k_train_rows<<<tr_grid(A.C * 32, 256), 256, 0, s>>>(A);
  NG_CHECK_LAUNCH("k_train_rows");
  if (A.mode == 0 && A.update_decoders) {
    const int64_t used = (int64_t)A.h * 36 + A.h + 1;
    k_train_dec_adam<<<dim3(tr_grid(used, 256), n_act), 256, 0, s>>>(A);
    NG_CHECK_LAUNCH("k_train_dec_adam");
  }
  return NG_OK;
}

int ng_train_epoch(const ng_octree* tree, const ng_train_params* P, const double* pts, const double* dist,
                   int64_t n, int64_t batch_size, int32_t active_mask, int32_t update_decoders, double lr,
                   int64_t step0, void* ws, size_t ws_bytes, double* level_sums, int64_t* status,
                   void* stream) {
  if (batch_size < 1) {
    set_error("batch_size must be positive");
    return NG_ERR_CONFIG;
  }
  int64_t step = step0;
  for (int64_t s0 = 0, bi = 0; s0 < n; s0 += batch_size, ++bi) {
    const int64_t cnt = (n - s0 < batch_size) ? n - s0 : batch_size;
    ++step;
    ng_train_step st;
    st.active_mask = active_mask;
    st.update_decoders = update_decoders;
    st.mode = 0;
    st.pad = 0;
    st.denom = (double)cnt;
    st.lr = lr;
    st.c1 = 1.0 - pow(BETA1, (double)step);  // trainer.py:92-93
    st.c2 = 1.0 - pow(BETA2, (double)step);
    st.batch_index = s0;
    int r = ng_train_batch(tree, P, &st, pts + 3 * s0, dist + s0, nullptr, cnt, batch_size, ws, ws_bytes,
                           level_sums, nullptr, nullptr, nullptr, nullptr, status, stream);
    if (r) return r;
  }
  return NG_OK;
}

int ng_train_export(const ng_octree* tree, const ng_train_params* P, int32_t level, const double* pts, int64_t n,
                    void* ws, size_t ws_bytes, int32_t* ids, double* weights, double* psi, double* pre, double* inp,
                    void* stream) {
  if (level < 1 || level > tree->max_level) {
    set_error("level %d outside 1..%d", level, tree->max_level);
    return NG_ERR_STRUCTURAL;
  }
  if (n <= 0) return NG_OK;
  ng_train_step st;
  st.active_mask = 1 << (level - 1);
  st.update_decoders = 0;
  st.mode = 2;
  st.pad = 0;
  st.denom = (double)n;
  st.lr = st.c1 = st.c2 = 0.0;
  st.batch_index = 0;
  int r = ng_train_batch(tree, P, &st, pts, nullptr, nullptr, n, n, ws, ws_bytes, nullptr, nullptr, nullptr,
                         nullptr, psi, nullptr, stream);
  if (r) return r;
  const TrainLayout Ly = train_layout(n, tree->max_level, P->n_decoders, P->h, P->corner_count, P->dec_stride);
  cudaStream_t s = (cudaStream_t)stream;
  const char* b = (const char*)ws;
  if ((r = cuda_status(cudaMemcpyAsync(ids, b + Ly.rec_id, sizeof(int32_t) * n * level * 8,
                                       cudaMemcpyDeviceToDevice, s), "export ids")))
    return r;
  if ((r = cuda_status(cudaMemcpyAsync(weights, b + Ly.rec_w, sizeof(double) * n * level * 8,
                                       cudaMemcpyDeviceToDevice, s), "export weights")))
    return r;
  if ((r = cuda_status(cudaMemcpyAsync(pre, b + Ly.pre, sizeof(double) * n * P->h, cudaMemcpyDeviceToDevice, s),
                       "export pre")))
    return r;
  return cuda_status(cudaMemcpyAsync(inp, b + Ly.inp, sizeof(double) * n * 36, cudaMemcpyDeviceToDevice, s),
                     "export inp");
}

int ng_adam_step(double* param, double* m, double* v, const double* grad, int64_t n, double lr, double c1,
                 double c2, int64_t* d_bad, void* stream) {
  if (n <= 0) return NG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  k_adam_check<<<tr_grid(n, 256), 256, 0, s>>>(grad, n, d_bad);
  NG_CHECK_LAUNCH("k_adam_check");
  k_adam_apply<<<tr_grid(n, 256), 256, 0, s>>>(param, m, v, grad, n, lr, c1, c2, d_bad);
  NG_CHECK_LAUNCH("k_adam_apply");
  return NG_OK;
}

}  // extern "C"
