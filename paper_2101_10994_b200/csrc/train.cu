// Training step of the neural field on sm_100a: loss, reverse-mode gradients
// and Adam.
//
// Reference: octfield/field.py:286-409 (forward cache, backward,
// scatter_add_rows) and octfield/trainer.py:87-144, 165-296 (adam_step,
// loss_batch, train, _batch_pass). The reference keeps float64 master
// weights and computes in float64; so does this path.
//
// One mini-batch, six launches on one stream, deterministic (no
// floating-point atomics; integer atomics only build index lists whose
// order never reaches the arithmetic):
//   k_train_locate   warp per point, lane = level: voxel lookup, 8 corner ids
//                    and trilinear weights per level (field.py:104-135);
//                    integer corner counts; first touch appends the corner
//                    row to the touched-row list
//   k_train_rowprep  warp per touched row: segment allocation; lazy Adam
//                    catch-up of the row to step s-1 (see below)
//   k_train_gather   warp per point, lane = channel: running feature sums z_l
//                    of levels 1..Lmax (field.py:119, 154-169)
//   k_train_dec      CTA per (active level L, 32-point group): decoder
//                    forward [x z_L 1] W1b^T, relu, W2 (field.py:346-
//                    357), residual + dout (trainer.py:139-143), dpre, dz =
//                    dpre W1[:,3:] (field.py:381-387) and the group's partial
//                    decoder gradients dW1b = dpre^T [x z 1], dW2, db2
//                    (field.py:377-385), all as small smem-tiled GEMMs;
//                    one extra row of blocks places the (corner, record) list
//   k_train_dec_reduce  fixed-order sum of the group partials, per-level
//                    residual sums (trainer.py:140), divergence flags; extra
//                    blocks form G_l = sum over active L >= l of dz_L per point
//   k_train_update   warp per touched row: record keys sorted, dZ row = sum
//                    of w * G_l in key order (field.py:388-394,
//                    scatter_add_rows 397-409), Adam step s; extra blocks run
//                    Adam on the decoders that received a gradient
//
// Lazy Adam. adam_step (trainer.py:87-103) decays the moments of EVERY
// parameter each step (the gradient dict always carries the dense dZ). A
// row with a zero gradient follows m = m*b1, v = v*b2, p -= lr*(m/c1)/
// (sqrt(v/c2)+eps): a fixed sequence of roundings that depends only on the
// row's own state and the step. Each row records the last step applied
// (Zlast) and replays the missed zero-gradient steps with the same
// operations before it is read or updated, so the result is bit-identical
// to a dense sweep while a batch touches only the rows it reads;
// ng_train_flush brings every row to the current step (every `flush_every`
// batches and at the end of an epoch). Rows whose moments are still zero
// are exact no-ops and are skipped.
#include "common.cuh"

namespace ng {

constexpr int TR_LM = 12;      // max feature levels handled by the trainer
constexpr int TR_HMAX = 128;   // max decoder width
constexpr int TR_GP = 16;      // points per decoder tile (one wave of tiles over the SMs at batch 512)
constexpr int TR_NT = 256;     // k_train_dec threads
constexpr int TR_PH = TR_GP / 2;            // points per thread half (forward / dpre)
constexpr int TR_PW = TR_GP / (TR_NT / 32); // points per warp (output / dz)
constexpr int W1S = 37;        // smem row stride (doubles) of the staged W1b block
constexpr double BETA1 = 0.9, BETA2 = 0.999, ADAM_EPS = 1e-8;  // trainer.py:29-31

static inline int tr_grid(int64_t n, int nt) { return (int)((n + nt - 1) / nt); }

struct TrainLayout {
  size_t rec_w, rec_id, pres, z, G, dz, sq, gpart, gdec, cnt, fill, seg, touched, list, sorted, ctr, total;
  int64_t max_rows;
};

// Workspace carve-up for a batch capacity B, LM levels, A level slots
// (= n_decoders), C corner rows. cnt must start zeroed (the caller
// zero-fills the workspace once); every batch leaves it zero.
static TrainLayout train_layout(int64_t B, int LM, int A, int64_t C, int dec_stride) {
  TrainLayout L;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o += (bytes + 255) & ~(size_t)255;
    return at;
  };
  const int64_t groups = (B + TR_GP - 1) / TR_GP;
  const int64_t n_rec = B * LM * 8;
  L.max_rows = n_rec < C ? n_rec : C;
  L.rec_w = take(sizeof(double) * n_rec);
  L.rec_id = take(sizeof(int32_t) * n_rec);
  L.pres = take(sizeof(uint32_t) * B);
  L.z = take(sizeof(double) * B * LM * 32);
  L.G = take(sizeof(double) * B * LM * 32);
  L.dz = take(sizeof(double) * B * A * 32);
  L.sq = take(sizeof(double) * A * B);
  L.gpart = take(sizeof(double) * A * groups * dec_stride);
  L.gdec = take(sizeof(double) * A * dec_stride);
  L.cnt = take(sizeof(int32_t) * C);
  L.fill = take(sizeof(int32_t) * C);
  L.seg = take(sizeof(int32_t) * C);
  L.touched = take(sizeof(int32_t) * L.max_rows);
  L.list = take(sizeof(int32_t) * n_rec);
  L.sorted = take(sizeof(int32_t) * n_rec);
  L.ctr = take(sizeof(int64_t) * 4 + sizeof(int32_t) * 32);  // n_touched, cursor, pad, pad | dtouch[32]
  L.total = o;
  return L;
}

struct TrainArgs {
  // parameters (fp64 masters)
  double* Z;
  double* Zm;
  double* Zv;
  int32_t* Zlast;
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
  int n_act;
  int update_decoders;
  int mode;                // 0 Adam, 1 gradients only, 2 forward cache export
  double two_over_n;       // 2.0 / denom (trainer.py:143)
  double lr;
  int64_t step;            // Adam step s of this batch (1-based)
  const double* adam_c;    // (c1, c2) of step t at [2(t-1)], [2(t-1)+1]
  int64_t batch_index;
  int64_t groups;
  int64_t max_rows;
  // workspace
  double* rec_w;
  int32_t* rec_id;
  uint32_t* pres;
  double* z;               // (n, LM, 32) running feature sums
  double* G;               // (n, LM, 32) feature-gradient per level
  double* dz;
  double* sq;
  double* gpart;
  double* gdec;
  int32_t* cnt;
  int32_t* fill;
  int32_t* seg;
  int32_t* touched;
  int32_t* list;
  int32_t* sorted;
  unsigned long long* ctr;  // [0] touched rows, [1] segment cursor
  int32_t* dtouch;          // per level: a decoded point this batch
  // outputs
  double* level_sums;      // mode 0: += per-level residual sums; mode 1: =
  double* grad_Z;          // mode 1: (C, 32) +=
  double* grad_dec;        // mode 1: n_dec * dec_stride +=
  int32_t* dec_touched;    // mode 1: 1 where a decoder received a gradient
  double* psi_out;         // mode 2: (n, LM, 32)
  double* pre_out;         // mode 2: (n, h)
  double* inp_out;         // mode 2: (n, 36)
  int64_t* status;         // [0] = 1 + batch index of the first divergence
};

__device__ __forceinline__ int level_slot(int mask, int L) { return __popc(mask & ((1 << (L - 1)) - 1)); }

__device__ __forceinline__ int slot_level(int mask, int a) {
  for (int l = 1, k = 0; l <= 31; ++l)
    if ((mask >> (l - 1)) & 1) {
      if (k == a) return l;
      ++k;
    }
  return 0;
}

__device__ __forceinline__ void flag_divergence(int64_t* status, int64_t batch) {
  atomicCAS((unsigned long long*)status, 0ull, (unsigned long long)(batch + 1));
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

// Zero-gradient Adam steps (last, upto] for one element: the dense sweep's
// exact operation sequence; zero moments stay zero and leave p unchanged.
__device__ __forceinline__ void adam_replay(double& prm, double& mm, double& vv, int64_t last, int64_t upto,
                                            double lr, const double* __restrict__ c) {
  if (mm == 0.0 && vv == 0.0) return;
  for (int64_t t = last + 1; t <= upto; ++t) adam_elem(prm, mm, vv, 0.0, lr, c[2 * (t - 1)], c[2 * (t - 1) + 1]);
}

// ---------------------------------------------------------------- locate
__global__ void __launch_bounds__(256) k_train_locate(const __grid_constant__ ng_octree tree,
                                                      const __grid_constant__ TrainArgs A) {
  const int lane = threadIdx.x & 31;
  const int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (p >= A.n) return;
  const int LM = A.LM;
  bool pres = false;
  int ids[8] = {-1, -1, -1, -1, -1, -1, -1, -1};
  if (lane < LM) {
    const double x0 = __ldg(A.pts + 3 * p), x1 = __ldg(A.pts + 3 * p + 1), x2 = __ldg(A.pts + 3 * p + 2);
    const int l = lane + 1;
    const int res = tree.r0 << l;
    const int tl = l + tree.n_virtual;
    const int c0 = bin_axis(x0, res), c1 = bin_axis(x1, res), c2 = bin_axis(x2, res);
    const int64_t idx = rank_lookup(tree.bitmap[tl], tree.rank[tl], morton(c0, c1, c2));
    const int64_t key0 = (p * LM + lane) * 8;
    pres = idx >= 0;
    if (pres) {
      const int4* cr = reinterpret_cast<const int4*>(tree.corners[tl] + 8 * idx);
      const int4 a = __ldg(cr), b = __ldg(cr + 1);
      ids[0] = a.x; ids[1] = a.y; ids[2] = a.z; ids[3] = a.w;
      ids[4] = b.x; ids[5] = b.y; ids[6] = b.z; ids[7] = b.w;
      // u = clip((x - DOMAIN_MIN) * (res / span) - cell, 0, 1); w_j = cx * cy * cz (field.py:115-135)
      const double half = 0.5 * (double)res;
      const double xs[3] = {x0, x1, x2};
      const int cc[3] = {c0, c1, c2};
      double u[3];
#pragma unroll
      for (int a3 = 0; a3 < 3; ++a3) {
        const double f = dsub(dmul(dadd(xs[a3], 1.0), half), (double)cc[a3]);
        u[a3] = f < 0.0 ? 0.0 : (f > 1.0 ? 1.0 : f);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double wx = (j & 1) ? u[0] : dsub(1.0, u[0]);
        const double wy = ((j >> 1) & 1) ? u[1] : dsub(1.0, u[1]);
        const double wz = ((j >> 2) & 1) ? u[2] : dsub(1.0, u[2]);
        A.rec_w[key0 + j] = dmul(dmul(wx, wy), wz);
        A.rec_id[key0 + j] = ids[j];
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) A.rec_id[key0 + j] = -1;
    }
  }
  // corner counts; first touches append the row, one cursor atomic per warp and corner slot
  if (A.mode != 2) {
    int old[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) old[j] = pres ? atomicAdd(A.cnt + ids[j], 1) : 1;
    int nfirst = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) nfirst += old[j] == 0;
    int incl = nfirst;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(FULL, incl, o);
      if ((int)lane >= o) incl += v;
    }
    const int total = __shfl_sync(FULL, incl, 31);
    if (total) {
      unsigned long long base = 0;
      if (lane == 31) base = atomicAdd(A.ctr, (unsigned long long)total);
      base = __shfl_sync(FULL, base, 31) + (unsigned long long)(incl - nfirst);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (old[j] == 0) A.touched[base++] = ids[j];
    }
  }
  const unsigned bits = __ballot_sync(FULL, pres);
  if (lane == 0) A.pres[p] = bits;
}

// ---------------------------------------------------------------- row prep
__global__ void __launch_bounds__(256) k_train_rowprep(const __grid_constant__ TrainArgs A) {
  __shared__ int s_cnt[8];
  __shared__ int s_base[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n_rows = (int64_t)A.ctr[0];
  // block-uniform loop: 8 rows per block iteration, one cursor atomic per block
  for (int64_t i0 = (int64_t)blockIdx.x * 8; i0 < n_rows; i0 += (int64_t)gridDim.x * 8) {
    const int64_t i = i0 + warp;
    const int id = i < n_rows ? A.touched[i] : -1;
    if (lane == 0) s_cnt[warp] = id >= 0 ? A.cnt[id] : 0;
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int q = 0; q < 8; ++q) tot += s_cnt[q];
      int base = (int)atomicAdd(A.ctr + 1, (unsigned long long)tot);
      for (int q = 0; q < 8; ++q) {
        s_base[q] = base;
        base += s_cnt[q];
      }
    }
    __syncthreads();
    if (id >= 0) {
      if (lane == 0) {
        A.seg[id] = s_base[warp];
        A.fill[id] = 0;
      }
      if (A.mode == 0) {
        const int64_t e = (int64_t)id * 32 + lane;
        const int64_t last = A.Zlast[id];
        if (last < A.step - 1) {
          double prm = A.Z[e], mm = A.Zm[e], vv = A.Zv[e];
          if (!(mm == 0.0 && vv == 0.0)) {
            adam_replay(prm, mm, vv, last, A.step - 1, A.lr, A.adam_c);
            A.Z[e] = prm;
            A.Zm[e] = mm;
            A.Zv[e] = vv;
          }
          __syncwarp();
          if (lane == 0) A.Zlast[id] = (int32_t)(A.step - 1);
        }
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- gather
// z_l = sum_{l' <= l} sum_j w_j Z[id_j] for l = 1..LM; a level's 8 corner
// rows are loaded together (lane = channel, 256 B per row).
__global__ void __launch_bounds__(256) k_train_gather(const __grid_constant__ TrainArgs A) {
  const int lane = threadIdx.x & 31;
  const int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (p >= A.n) return;
  const int LM = A.LM;
  const uint32_t pr = A.pres[p];
  const int64_t key0 = p * LM * 8;
  // lane i < 8 LM holds record i's (id, weight)
  int idv[3];
  double wv[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const int i = c * 32 + lane;
    const bool own = i < 8 * LM && ((pr >> (i >> 3)) & 1);
    idv[c] = own ? A.rec_id[key0 + i] : 0;
    wv[c] = own ? A.rec_w[key0 + i] : 0.0;
  }
  const double* Zc = A.Z + lane;
  double z = 0.0;
  for (int l = 1; l <= LM; ++l) {
    double psi = 0.0;
    if ((pr >> (l - 1)) & 1) {
      double v[8], w[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = (l - 1) * 8 + j;
        const int c = i >> 5;
        const int src = i & 31;
        const int id = __shfl_sync(FULL, c == 0 ? idv[0] : (c == 1 ? idv[1] : idv[2]), src);
        w[j] = __shfl_sync(FULL, c == 0 ? wv[0] : (c == 1 ? wv[1] : wv[2]), src);
        v[j] = Zc[32 * (int64_t)id];
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) psi = dadd(psi, dmul(w[j], v[j]));
    }
    z = dadd(z, psi);
    A.z[(p * LM + (l - 1)) * 32 + lane] = z;
    if (A.psi_out) A.psi_out[(p * LM + (l - 1)) * 32 + lane] = psi;
  }
}

// ---------------------------------------------------------------- decoder tiles
static size_t dec_smem_bytes() {
  return sizeof(double) * (TR_HMAX * W1S + TR_HMAX + 1 + TR_GP * 36 + 2 * TR_GP * TR_HMAX + TR_GP) +
         sizeof(int) * TR_GP + 64;
}

__global__ void __launch_bounds__(TR_NT) k_train_dec(const __grid_constant__ TrainArgs A) {
  extern __shared__ __align__(16) double dsm[];
  const int h = A.h, m = A.m;
  // one extra row of blocks (blockIdx.y == n_act): place records into their corner segments
  if ((int)blockIdx.y == A.n_act) {
    const int64_t n_rec = A.n * A.LM * 8;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rec; r += (int64_t)gridDim.x * blockDim.x) {
      const int id = A.rec_id[r];
      if (id < 0) continue;
      const int slot = A.seg[id] + atomicAdd(A.fill + id, 1);
      A.list[slot] = (int32_t)r;
    }
    return;
  }
  double* sW1 = dsm;                          // [h][W1S]
  double* sW2 = sW1 + TR_HMAX * W1S;          // [h + 1], b2 last
  double* sInp = sW2 + TR_HMAX + 1;           // [TR_GP][36]: x, z_L (padded to 32), 1
  double* sPre = sInp + TR_GP * 36;           // [TR_GP][TR_HMAX]
  double* sDpre = sPre + TR_GP * TR_HMAX;     // [TR_GP][TR_HMAX]
  double* sDout = sDpre + TR_GP * TR_HMAX;    // [TR_GP]
  int* sDec = reinterpret_cast<int*>(sDout + TR_GP);
  const int a = blockIdx.y;
  const int L = slot_level(A.active_mask, a);
  const int64_t g = blockIdx.x;
  const int64_t p0 = g * TR_GP;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;

  // ---- stage decoder L (W1b rows, W2, b2): 16-byte loads, all in flight
  {
    const double2* blk2 = reinterpret_cast<const double2*>(A.dec + (int64_t)(L - 1) * A.dec_stride);
    const int n2 = h * 18;
#pragma unroll 9
    for (int i = t; i < n2; i += TR_NT) {
      const double2 v = __ldg(blk2 + i);
      const int e = 2 * i;
      sW1[(e / 36) * W1S + (e % 36)] = v.x;
      sW1[((e + 1) / 36) * W1S + ((e + 1) % 36)] = v.y;
    }
    const double* blk = A.dec + (int64_t)(L - 1) * A.dec_stride;
    for (int i = t; i <= h; i += TR_NT) sW2[i] = __ldg(blk + h * 36 + i);
  }
  // ---- decoder inputs [x, z_L, 1] (field.py:347): warp w owns points w, w+8, ...; lane = channel
  for (int q = warp; q < TR_GP; q += TR_NT / 32) {
    const int64_t p = p0 + q;
    const bool valid = p < A.n;
    const uint32_t pr = valid ? A.pres[p] : 0u;
    const bool dec = valid && (pr & ((1u << L) - 1u)) != 0u;
    const double z = dec ? A.z[(p * A.LM + (L - 1)) * 32 + lane] : 0.0;
    double* ir = sInp + q * 36;
    if (lane < 3) ir[lane] = valid ? __ldg(A.pts + 3 * p + lane) : 0.0;
    ir[3 + lane] = (dec && lane < m) ? z : 0.0;
    if (lane == 0) {
      ir[35] = 1.0;
      sDec[q] = dec ? 1 : 0;
    }
  }
  __syncthreads();

  // ---- forward: pre[p][j] = [x z] . W1b[j][0:3+m] + b1[j]; thread = (j, TR_PH points)
  const int j = t & (TR_HMAX - 1);
  const int half = t >> 7;
  if (j < h) {
    double w[36];
#pragma unroll
    for (int k = 0; k < 36; ++k) w[k] = sW1[j * W1S + k];
    for (int q0 = half * TR_PH; q0 < half * TR_PH + TR_PH; q0 += 4) {
      double s[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int k = 0; k < 35; ++k)
        if (k < 3 + m) {
#pragma unroll
          for (int u = 0; u < 4; ++u) s[u] = fma(sInp[(q0 + u) * 36 + k], w[k], s[u]);
        }
#pragma unroll
      for (int u = 0; u < 4; ++u)  // inp @ W1.T + b1 (field.py:350)
        sPre[(q0 + u) * TR_HMAX + j] = sDec[q0 + u] ? dadd(s[u], w[35]) : 0.0;
    }
  }
  __syncthreads();

  // ---- output, residual, dout (warp: TR_PW points)
  for (int q = warp * TR_PW; q < warp * TR_PW + TR_PW; ++q) {
    double part = 0.0;
    for (int jj = lane; jj < h; jj += 32) {
      const double pr = sPre[q * TR_HMAX + jj];
      part = fma(pr > 0.0 ? pr : 0.0, sW2[jj], part);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(FULL, part, o);
    if (lane == 0) {
      const int64_t p = p0 + q;
      double dout = 0.0, sq = 0.0;
      if (sDec[q]) {
        const double out = dadd(part, sW2[h]);
        const bool inL = (A.pres[p] >> (L - 1)) & 1;
        if (A.upstream) {
          dout = __ldg(A.upstream + p);
        } else if (A.dist) {
          // resid = where(mask_L, out - d, 0); upstream = (2/n) resid (trainer.py:139-143)
          const double resid = inL ? dsub(out, __ldg(A.dist + p)) : 0.0;
          dout = dmul(A.two_over_n, resid);
          sq = dmul(resid, resid);
        }
      }
      sDout[q] = dout;
      if (p < A.n) A.sq[(int64_t)a * A.n + p] = sq;
    }
  }
  __syncthreads();

  // ---- dpre = where(pre > 0, dout * W2, 0) (field.py:381-383)
  if (j < h) {
    const double w2 = sW2[j];
    for (int q = half * TR_PH; q < half * TR_PH + TR_PH; ++q) {
      const double pr = sPre[q * TR_HMAX + j];
      sDpre[q * TR_HMAX + j] = (sDec[q] && pr > 0.0) ? dmul(sDout[q], w2) : 0.0;
    }
  }
  __syncthreads();

  if (A.mode == 2) {  // ForwardCache export
    for (int q = warp; q < TR_GP; q += TR_NT / 32) {
      const int64_t p = p0 + q;
      if (p >= A.n) break;
      for (int jj = lane; jj < h; jj += 32) A.pre_out[p * h + jj] = sPre[q * TR_HMAX + jj];
      A.inp_out[p * 36 + lane] = sInp[q * 36 + lane];
      if (lane < 4) A.inp_out[p * 36 + 32 + lane] = sInp[q * 36 + 32 + lane];
    }
    return;
  }

  // ---- dz = (dpre @ W1)[:, 3:] (field.py:386-387): thread = (channel, TR_PW points)
  {
    const int q0 = warp * TR_PW;
    double s[TR_PW];
#pragma unroll
    for (int u = 0; u < TR_PW; ++u) s[u] = 0.0;
    if (lane < m)
      for (int jj = 0; jj < h; ++jj) {
        const double wv = sW1[jj * W1S + 3 + lane];
#pragma unroll
        for (int u = 0; u < TR_PW; ++u) s[u] = fma(sDpre[(q0 + u) * TR_HMAX + jj], wv, s[u]);
      }
#pragma unroll
    for (int u = 0; u < TR_PW; ++u) {
      const int64_t p = p0 + q0 + u;
      if (p < A.n) A.dz[(p * A.n_dec + a) * 32 + lane] = sDec[q0 + u] ? s[u] : 0.0;
    }
  }
  // ---- this group's partial decoder gradients (field.py:377-385): thread = (j, 18 columns)
  if (j < h) {
    double acc[18];
#pragma unroll
    for (int k = 0; k < 18; ++k) acc[k] = 0.0;
    double aw2 = 0.0;
    const int k0 = half * 18;
    for (int q = 0; q < TR_GP; ++q) {
      const double d = sDpre[q * TR_HMAX + j];
      const double* ir = sInp + q * 36 + k0;
#pragma unroll
      for (int k = 0; k < 18; ++k) acc[k] = fma(d, ir[k], acc[k]);
      if (half == 0) {
        const double pr = sPre[q * TR_HMAX + j];
        aw2 = fma(sDout[q], pr > 0.0 ? pr : 0.0, aw2);
      }
    }
    double* gp = A.gpart + ((int64_t)a * A.groups + g) * A.dec_stride;
#pragma unroll
    for (int k = 0; k < 18; ++k) gp[j * 36 + k0 + k] = acc[k];
    if (half == 0) gp[h * 36 + j] = aw2;
    if (t == TR_HMAX) {  // db2 = sum dout
      double ab2 = 0.0;
      for (int q = 0; q < TR_GP; ++q) ab2 = dadd(ab2, sDout[q]);
      gp[h * 36 + h] = ab2;
    }
  }
  if (t == 0) {
    int any = 0;
    for (int q = 0; q < TR_GP; ++q) any |= sDec[q];
    if (any) A.dtouch[L - 1] = 1;
  }
}

// ---------------------------------------------------------------- decoder reduce
__global__ void __launch_bounds__(256) k_train_dec_reduce(const __grid_constant__ TrainArgs A) {
  if ((int)blockIdx.y == A.n_act) {  // G[p][l] = sum over active L >= l of dz_L (field.py:388-394)
    const int64_t total = A.n * A.LM * 32;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
      const int k = (int)(e & 31);
      const int64_t pl = e >> 5;
      const int64_t p = pl / A.LM;
      const int l = (int)(pl % A.LM) + 1;
      double v[TR_LM];
#pragma unroll
      for (int Lk = 1; Lk <= TR_LM; ++Lk)
        v[Lk - 1] = (Lk >= l && Lk <= A.LM && ((A.active_mask >> (Lk - 1)) & 1))
                        ? A.dz[(p * A.n_dec + level_slot(A.active_mask, Lk)) * 32 + k] : 0.0;
      double G = 0.0;
#pragma unroll
      for (int Lk = 1; Lk <= TR_LM; ++Lk)
        if (Lk >= l && Lk <= A.LM && ((A.active_mask >> (Lk - 1)) & 1)) G = dadd(G, v[Lk - 1]);
      A.G[e] = G;
    }
    return;
  }
  const int a = blockIdx.y;
  const int L = slot_level(A.active_mask, a);
  const int64_t used = (int64_t)A.h * 36 + A.h + 1;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool adam = A.mode == 0;
  bool bad = false;
  if (i < used) {
    double s = 0.0;
    for (int64_t g = 0; g < A.groups; ++g) s = dadd(s, A.gpart[((int64_t)a * A.groups + g) * A.dec_stride + i]);
    if (adam) A.gdec[(int64_t)a * A.dec_stride + i] = s;
    else if (A.dtouch[L - 1]) A.grad_dec[(int64_t)(L - 1) * A.dec_stride + i] += s;
    bad = !isfinite(s);
  }
  if (adam && A.update_decoders && A.dtouch[L - 1] && __any_sync(FULL, bad) && (threadIdx.x & 31) == 0)
    flag_divergence(A.status, A.batch_index);
  // residual sum of level L (trainer.py:140), fixed order
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double s = 0.0;
    for (int64_t p0 = lane; p0 < A.n; p0 += 128) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = p0 + 32 * u < A.n ? A.sq[(int64_t)a * A.n + p0 + 32 * u] : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (p0 + 32 * u < A.n) s = dadd(s, v[u]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
    if (lane == 0) {
      if (adam) {
        A.level_sums[L - 1] = dadd(A.level_sums[L - 1], s);
        if (!isfinite(s)) flag_divergence(A.status, A.batch_index);  // non-finite loss (trainer.py:233-236)
      } else {
        A.level_sums[L - 1] = s;
        if (A.dec_touched && A.dtouch[L - 1]) A.dec_touched[L - 1] = 1;
      }
    }
  }
}

// ---------------------------------------------------------------- update
// blocks [0, row_blocks): warp per touched row; the rest: decoder Adam.
__global__ void __launch_bounds__(256) k_train_update(const __grid_constant__ TrainArgs A, int row_blocks) {
  const int lane = threadIdx.x & 31;
  if ((int)blockIdx.x >= row_blocks) {
    if (A.mode != 0 || !A.update_decoders || *(volatile int64_t*)A.status) return;
    const int64_t per = (int64_t)A.h * 36 + A.h + 1;  // elements per decoder
    const double c1 = A.adam_c[2 * (A.step - 1)], c2 = A.adam_c[2 * (A.step - 1) + 1];
    for (int64_t e = (int64_t)(blockIdx.x - row_blocks) * blockDim.x + threadIdx.x; e < per * A.n_act;
         e += (int64_t)(gridDim.x - row_blocks) * blockDim.x) {
      const int a = (int)(e / per);
      const int64_t i = e % per;
      const int L = slot_level(A.active_mask, a);
      if (!A.dtouch[L - 1]) continue;  // untouched decoders keep their moments (trainer.py:100, 290-296)
      const int64_t o = (int64_t)(L - 1) * A.dec_stride + i;
      double prm = A.dec[o], mm = A.decm[o], vv = A.decv[o];
      adam_elem(prm, mm, vv, A.gdec[(int64_t)a * A.dec_stride + i], A.lr, c1, c2);
      A.dec[o] = prm;
      A.decm[o] = mm;
      A.decv[o] = vv;
    }
    return;
  }
  const int64_t n_rows = (int64_t)A.ctr[0];
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n_rows;
       i += ((int64_t)row_blocks * blockDim.x) >> 5) {
    const int id = A.touched[i];
    const int S = A.cnt[id];
    const int base = A.seg[id];
    double g = 0.0;
    // dZ row = sum of w * G over the records in key order: keys are ranked,
    // then contributions are loaded 8 records at a time
    auto accumulate = [&](const int* keys, int cnt) {
      for (int r0 = 0; r0 < cnt; r0 += 8) {
        double w[8], v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int key = keys[r0 + u < cnt ? r0 + u : r0];
          w[u] = A.rec_w[key];
          v[u] = A.G[(int64_t)(key >> 3) * 32 + lane];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (r0 + u < cnt) g = dadd(g, dmul(w[u], v[u]));
      }
    };
    if (S <= 32) {
      __shared__ int sk[8][32];
      const int wl = (threadIdx.x >> 5);
      const int key = lane < S ? A.list[base + lane] : 0x7fffffff;
      int rank = 0;
      for (int q = 0; q < S; ++q) rank += __shfl_sync(FULL, key, q) < key;
      if (lane < S) sk[wl][rank] = key;
      __syncwarp();
      accumulate(sk[wl], S);
      __syncwarp();
    } else {
      for (int i0 = 0; i0 < S; i0 += 32) {
        const bool own = i0 + lane < S;
        const int key = own ? A.list[base + i0 + lane] : 0x7fffffff;
        int rank = 0;
        for (int c0 = 0; c0 < S; c0 += 32) {
          const int other = c0 + lane < S ? A.list[base + c0 + lane] : 0x7fffffff;
          for (int q = 0; q < 32; ++q) rank += __shfl_sync(FULL, other, q) < key;
        }
        if (own) A.sorted[base + rank] = key;
      }
      __syncwarp();
      accumulate(A.sorted + base, S);
    }
    const int64_t e = (int64_t)id * 32 + lane;
    if (A.mode == 0) {
      if (!*(volatile int64_t*)A.status) {
        if (!isfinite(g)) {
          flag_divergence(A.status, A.batch_index);
        } else {
          double prm = A.Z[e], mm = A.Zm[e], vv = A.Zv[e];
          adam_elem(prm, mm, vv, g, A.lr, A.adam_c[2 * (A.step - 1)], A.adam_c[2 * (A.step - 1) + 1]);
          A.Z[e] = prm;
          A.Zm[e] = mm;
          A.Zv[e] = vv;
        }
      }
      __syncwarp();
      if (lane == 0) A.Zlast[id] = (int32_t)A.step;
    } else if (A.mode == 1) {
      A.grad_Z[e] = dadd(A.grad_Z[e], g);
    }
    __syncwarp();
    if (lane == 0) A.cnt[id] = 0;
  }
}

// ---------------------------------------------------------------- flush
__global__ void __launch_bounds__(256) k_train_flush(double* Z, double* Zm, double* Zv, int32_t* Zlast, int64_t C,
                                                     int64_t upto, double lr, const double* __restrict__ c) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= C) return;
  const int64_t last = Zlast[r];
  if (last >= upto) return;
  const int64_t e = r * 32 + lane;
  double prm = Z[e], mm = Zm[e], vv = Zv[e];
  if (!(mm == 0.0 && vv == 0.0)) {
    adam_replay(prm, mm, vv, last, upto, lr, c);
    Z[e] = prm;
    Zm[e] = mm;
    Zv[e] = vv;
  }
  __syncwarp();
  if (lane == 0) Zlast[r] = (int32_t)upto;
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

static int highest_level(int mask) { return 32 - __builtin_clz((unsigned)mask); }

// Debug (NG_TRAIN_EVENTS=1): per-kernel device time from CUDA events around
// each launch (one host sync per batch), read with ng_train_profile.
static double g_phase_ms[8];
static int64_t g_phase_batches = 0;

// parts: 1 = counters reset + point location, 2 = the rest of the step
static int launch_batch(const ng_octree* tree, TrainArgs& A, cudaStream_t s, int parts = 3) {
  // (a single-threaded debugging aid: the events belong to the device
  // current at the first batch)
  static cudaEvent_t ev[8];
  static const bool ev_env = [] {
    if (env_int("NG_TRAIN_EVENTS", 0) != 1) return false;
    for (int k = 0; k < 8; ++k) cudaEventCreate(&ev[k]);
    return true;
  }();
  int nev = 0;
  auto mark = [&]() {
    if (ev_env) cudaEventRecord(ev[nev++], s);
  };
  int r = 0;
  if ((r = set_smem_limit((const void*)k_train_dec, dec_smem_bytes()))) return r;  // per device
  const int cap_blocks = 4 * sm_count();
  const int row_blocks = tr_grid(A.max_rows * 32, 256) < cap_blocks ? tr_grid(A.max_rows * 32, 256) : cap_blocks;
  if (parts & 1) {
    mark();
    if ((r = cuda_status(cudaMemsetAsync(A.ctr, 0, 4 * sizeof(int64_t) + 32 * sizeof(int32_t), s), "train memset")))
      return r;
    k_train_locate<<<tr_grid(A.n * 32, 256), 256, 0, s>>>(*tree, A);
    NG_CHECK_LAUNCH("k_train_locate");
    mark();
  }
  if (!(parts & 2)) return NG_OK;
  if (A.mode != 2) {
    k_train_rowprep<<<row_blocks, 256, 0, s>>>(A);
    NG_CHECK_LAUNCH("k_train_rowprep");
    mark();
  }
  k_train_gather<<<tr_grid(A.n * 32, 256), 256, 0, s>>>(A);
  NG_CHECK_LAUNCH("k_train_gather");
  mark();
  // grid.y = n_act decoder slots, plus one row of record-placement blocks
  const int fill_rows = A.mode == 2 ? 0 : 1;
  k_train_dec<<<dim3((unsigned)A.groups, A.n_act + fill_rows), TR_NT, dec_smem_bytes(), s>>>(A);
  NG_CHECK_LAUNCH("k_train_dec");
  mark();
  if (A.mode == 2) return NG_OK;
  const int64_t used = (int64_t)A.h * 36 + A.h + 1;
  k_train_dec_reduce<<<dim3(tr_grid(used, 256), A.n_act + 1), 256, 0, s>>>(A);
  NG_CHECK_LAUNCH("k_train_dec_reduce");
  mark();
  const int dec_blocks = (A.mode == 0 && A.update_decoders) ? tr_grid(used * A.n_act, 256) : 0;
  k_train_update<<<row_blocks + dec_blocks, 256, 0, s>>>(A, row_blocks);
  NG_CHECK_LAUNCH("k_train_update");
  mark();
  if (ev_env && nev == 7) {
    cudaEventSynchronize(ev[6]);
    for (int k = 0; k < 6; ++k) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[k], ev[k + 1]);
      g_phase_ms[k] += ms;
    }
    ++g_phase_batches;
  }
  return NG_OK;
}

static int fill_args(const ng_octree* tree, const ng_train_params* P, const ng_train_step* st, const double* pts,
                     const double* dist, const double* upstream, int64_t n, int64_t batch_capacity, void* ws,
                     size_t ws_bytes, TrainArgs& A) {
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
  const TrainLayout Ly = train_layout(batch_capacity, tree->max_level, P->n_decoders, P->corner_count,
                                      P->dec_stride);
  if (ws_bytes < Ly.total) {
    set_error("train workspace %zu < %zu bytes", ws_bytes, Ly.total);
    return NG_ERR_CAPACITY;
  }
  if (st->mode == 0 && (!P->Zm || !P->Zv || !P->Zlast || !st->adam_c || st->step < 1)) {
    set_error("Adam mode needs moments, Zlast, the bias-correction table and step >= 1");
    return NG_ERR_STRUCTURAL;
  }
  char* b = (char*)ws;
  A.Z = P->Z; A.Zm = P->Zm; A.Zv = P->Zv; A.Zlast = P->Zlast;
  A.dec = P->dec; A.decm = P->decm; A.decv = P->decv;
  A.m = P->m; A.h = P->h; A.n_dec = P->n_decoders; A.dec_stride = P->dec_stride; A.C = P->corner_count;
  A.pts = pts; A.dist = dist; A.upstream = upstream; A.n = n;
  A.LM = highest_level(mask);
  A.active_mask = mask;
  A.n_act = __builtin_popcount((unsigned)mask);
  A.update_decoders = st->update_decoders;
  A.mode = st->mode;
  A.two_over_n = 2.0 / st->denom;
  A.lr = st->lr;
  A.step = st->step;
  A.adam_c = st->adam_c;
  A.batch_index = st->batch_index;
  A.groups = (n + TR_GP - 1) / TR_GP;
  A.max_rows = Ly.max_rows;
  A.rec_w = (double*)(b + Ly.rec_w);
  A.rec_id = (int32_t*)(b + Ly.rec_id);
  A.pres = (uint32_t*)(b + Ly.pres);
  A.z = (double*)(b + Ly.z);
  A.G = (double*)(b + Ly.G);
  A.dz = (double*)(b + Ly.dz);
  A.sq = (double*)(b + Ly.sq);
  A.gpart = (double*)(b + Ly.gpart);
  A.gdec = (double*)(b + Ly.gdec);
  A.cnt = (int32_t*)(b + Ly.cnt);
  A.fill = (int32_t*)(b + Ly.fill);
  A.seg = (int32_t*)(b + Ly.seg);
  A.touched = (int32_t*)(b + Ly.touched);
  A.list = (int32_t*)(b + Ly.list);
  A.sorted = (int32_t*)(b + Ly.sorted);
  A.ctr = (unsigned long long*)(b + Ly.ctr);
  A.dtouch = (int32_t*)(b + Ly.ctr + 4 * sizeof(int64_t));
  A.level_sums = A.grad_Z = A.grad_dec = nullptr;
  A.dec_touched = nullptr;
  A.psi_out = A.pre_out = A.inp_out = nullptr;
  A.status = nullptr;
  return NG_OK;
}

}  // namespace ng

using namespace ng;

extern "C" {

size_t ng_train_workspace_bytes(const ng_octree* tree, int64_t batch_capacity, int32_t h, int32_t n_decoders,
                                int64_t corner_count, int32_t dec_stride) {
  (void)h;
  // two batch buffers: ng_train_epoch locates batch b+1 in one while batch b
  // runs in the other (single-batch calls use the first)
  const size_t one = train_layout(batch_capacity, tree->max_level, n_decoders, corner_count, dec_stride).total;
  return 2 * ((one + 255) & ~(size_t)255);
}

int ng_train_batch(const ng_octree* tree, const ng_train_params* P, const ng_train_step* st, const double* pts,
                   const double* dist, const double* upstream, int64_t n, int64_t batch_capacity, void* ws,
                   size_t ws_bytes, double* level_sums, double* grad_Z, double* grad_dec, int32_t* dec_touched,
                   double* psi_out, int64_t* status, void* stream) {
  if (st->mode == 1 && (!grad_Z || !grad_dec)) {
    set_error("gradient mode needs grad_Z and grad_dec");
    return NG_ERR_STRUCTURAL;
  }
  if (st->mode != 2 && (!level_sums || !status)) {
    set_error("level_sums and status are required");
    return NG_ERR_STRUCTURAL;
  }
  TrainArgs A;
  int r = fill_args(tree, P, st, pts, dist, upstream, n, batch_capacity, ws, ws_bytes, A);
  if (r) return r;
  if (n <= 0) return NG_OK;
  A.level_sums = level_sums;
  A.grad_Z = grad_Z;
  A.grad_dec = grad_dec;
  A.dec_touched = dec_touched;
  A.psi_out = psi_out;
  A.status = status;
  return launch_batch(tree, A, (cudaStream_t)stream);
}

int ng_train_flush(const ng_train_params* P, int64_t step, const double* adam_c, double lr, void* stream) {
  if (P->corner_count <= 0 || step < 1) return NG_OK;
  k_train_flush<<<tr_grid(P->corner_count * 32, 256), 256, 0, (cudaStream_t)stream>>>(
      P->Z, P->Zm, P->Zv, P->Zlast, P->corner_count, step, lr, adam_c);
  NG_CHECK_LAUNCH("k_train_flush");
  return NG_OK;
}

// RAII holder of ng_train_epoch's side stream: on destruction (every return
// path) the caller's stream waits for the side stream's queued work, then the
// stream and events are released (the driver frees them once that work ends).
struct SideStream {
  cudaStream_t caller;
  cudaStream_t side = nullptr;
  cudaEvent_t e_loc[2] = {nullptr, nullptr}, e_done[2] = {nullptr, nullptr}, e_start = nullptr, e_join = nullptr;
  explicit SideStream(cudaStream_t s) : caller(s) {}
  int create() {
    int r = cuda_status(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking), "train side stream");
    for (int k = 0; k < 2 && !r; ++k) {
      r = cuda_status(cudaEventCreateWithFlags(&e_loc[k], cudaEventDisableTiming), "train event");
      if (!r) r = cuda_status(cudaEventCreateWithFlags(&e_done[k], cudaEventDisableTiming), "train event");
    }
    if (!r) r = cuda_status(cudaEventCreateWithFlags(&e_start, cudaEventDisableTiming), "train event");
    if (!r) r = cuda_status(cudaEventCreateWithFlags(&e_join, cudaEventDisableTiming), "train event");
    if (!r) r = cuda_status(cudaEventRecord(e_start, caller), "train record");
    if (!r) r = cuda_status(cudaStreamWaitEvent(side, e_start, 0), "train wait");
    return r;
  }
  ~SideStream() {
    if (side && e_join && cudaEventRecord(e_join, side) == cudaSuccess) cudaStreamWaitEvent(caller, e_join, 0);
    for (cudaEvent_t e : {e_loc[0], e_loc[1], e_done[0], e_done[1], e_start, e_join})
      if (e) cudaEventDestroy(e);
    if (side) cudaStreamDestroy(side);
  }
};

int ng_train_epoch(const ng_octree* tree, const ng_train_params* P, const double* pts, const double* dist,
                   int64_t n, int64_t batch_size, int32_t active_mask, int32_t update_decoders, double lr,
                   int64_t step0, const double* adam_c, int32_t flush_every, void* ws, size_t ws_bytes,
                   double* level_sums, int64_t* status, void* stream) {
  if (batch_size < 1) {
    set_error("batch_size must be positive");
    return NG_ERR_CONFIG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  // Batch b+1's point location depends only on the points and the octree,
  // so it runs on a side stream in the other workspace buffer while batch
  // b's step runs (a buffer is reused once the step two batches back has
  // left its corner counters at zero). NG_TRAIN_OVERLAP=0: one stream.
  static const int overlap_env = (env_int("NG_TRAIN_OVERLAP", 1) != 0 && env_int("NG_TRAIN_EVENTS", 0) != 1) ? 1 : 0;
  const size_t half = ws_bytes / 2;
  const int64_t nb = (n + batch_size - 1) / batch_size;
  auto args_for = [&](int64_t bi, TrainArgs& A) -> int {
    const int64_t s0 = bi * batch_size;
    const int64_t cnt = (n - s0 < batch_size) ? n - s0 : batch_size;
    ng_train_step st;
    st.active_mask = active_mask;
    st.update_decoders = update_decoders;
    st.mode = 0;
    st.pad = 0;
    st.denom = (double)cnt;
    st.lr = lr;
    st.step = step0 + bi + 1;
    st.adam_c = adam_c;
    st.batch_index = s0;
    char* wsb = (char*)ws + (overlap_env ? (size_t)(bi & 1) * half : 0);
    int r = fill_args(tree, P, &st, pts + 3 * s0, dist + s0, nullptr, cnt, batch_size, wsb,
                      overlap_env ? half : ws_bytes, A);
    if (r) return r;
    A.level_sums = level_sums;
    A.grad_Z = nullptr;
    A.grad_dec = nullptr;
    A.dec_touched = nullptr;
    A.psi_out = nullptr;
    A.status = status;
    return NG_OK;
  };
  // The side stream and its events belong to this call (on the caller's
  // current device, so concurrent epochs on other streams or devices never
  // share them); created per epoch (~10 us against ~100 ms) and released
  // when the call returns, by which point -- on every exit path -- the
  // caller's stream has been made to wait for everything queued on it.
  SideStream ss(s);
  cudaStream_t side = nullptr;
  cudaEvent_t *e_loc = ss.e_loc, *e_done = ss.e_done;
  if (overlap_env) {  // the side stream starts after everything already queued on the caller's stream
    if (int r0 = ss.create()) return r0;
    side = ss.side;
  }
  int64_t step = step0;
  if (nb > 0) {
    TrainArgs A;
    int r = args_for(0, A);
    if (r) return r;
    if ((r = launch_batch(tree, A, s, overlap_env ? 1 : 3))) return r;
    if (!overlap_env) {
      ++step;
      if (flush_every > 0 && 1 % flush_every == 0 && (r = ng_train_flush(P, step, adam_c, lr, s))) return r;
    }
  }
  for (int64_t bi = overlap_env ? 0 : 1; bi < nb; ++bi) {
    TrainArgs A;
    int r = args_for(bi, A);
    if (r) return r;
    if (overlap_env) {
      if (bi + 1 < nb) {  // locate the next batch on the side stream
        TrainArgs An;
        if ((r = args_for(bi + 1, An))) return r;
        if (bi >= 1 && (r = cuda_status(cudaStreamWaitEvent(side, e_done[(bi + 1) & 1], 0), "train wait"))) return r;
        if ((r = launch_batch(tree, An, side, 1))) return r;
        if ((r = cuda_status(cudaEventRecord(e_loc[(bi + 1) & 1], side), "train record"))) return r;
      }
      if (bi >= 1 && (r = cuda_status(cudaStreamWaitEvent(s, e_loc[bi & 1], 0), "train wait"))) return r;
      if ((r = launch_batch(tree, A, s, 2))) return r;
      if ((r = cuda_status(cudaEventRecord(e_done[bi & 1], s), "train record"))) return r;
    } else {
      if ((r = launch_batch(tree, A, s, 3))) return r;
    }
    ++step;
    if (flush_every > 0 && (bi + 1) % flush_every == 0 && (r = ng_train_flush(P, step, adam_c, lr, s))) return r;
  }
  return ng_train_flush(P, step, adam_c, lr, s);
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
  st.lr = 0.0;
  st.step = 0;
  st.adam_c = nullptr;
  st.batch_index = 0;
  TrainArgs A;
  int r = fill_args(tree, P, &st, pts, nullptr, nullptr, n, n, ws, ws_bytes, A);
  if (r) return r;
  A.psi_out = psi;
  A.pre_out = pre;
  A.inp_out = inp;
  cudaStream_t s = (cudaStream_t)stream;
  if ((r = launch_batch(tree, A, s))) return r;
  const TrainLayout Ly = train_layout(n, tree->max_level, P->n_decoders, P->corner_count, P->dec_stride);
  const char* b = (const char*)ws;
  // records are laid out [p][level][8] with LM = level
  if ((r = cuda_status(cudaMemcpyAsync(ids, b + Ly.rec_id, sizeof(int32_t) * n * level * 8,
                                       cudaMemcpyDeviceToDevice, s), "export ids")))
    return r;
  return cuda_status(cudaMemcpyAsync(weights, b + Ly.rec_w, sizeof(double) * n * level * 8,
                                     cudaMemcpyDeviceToDevice, s), "export weights");
}

/* Debug (NG_TRAIN_EVENTS=1): mean device ms per batch of each training
 * kernel (locate, rowprep, gather, dec, reduce, update) since the last call; resets. */
int ng_train_profile(double* host_out6) {
  for (int k = 0; k < 6; ++k) {
    host_out6[k] = g_phase_batches ? g_phase_ms[k] / (double)g_phase_batches : 0.0;
    g_phase_ms[k] = 0.0;
  }
  g_phase_batches = 0;
  return NG_OK;
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
