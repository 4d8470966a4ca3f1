// Presummed feature grids for the sphere tracer.
//
// sum_features (field.py:154-169) at a point x inside a level-G voxel V is
// z_L(x) = sum_{l <= L} psi_l(x), psi_l the trilinear interpolation of level
// l's corner features over the level-l ancestor of V. A trilinear function
// restricted to a sub-box is the trilinear interpolation of its own values
// at the sub-box corners, and every ancestor cell contains V, so
//
//     z_L(x) = sum_j w_j^V(x) * S_L(c_j),   S_L(c) = sum_{l <= L} psi_l(c),
//
// with c_j the corners of V and w^V the level-G trilinear weights. S_L is
// a per-corner table on the level-G corner ids; with it one evaluation reads
// 8 corner rows per output level instead of 8 per level 1..L. This is a
// reassociation of the reference's sum, not an approximation: S is built in
// float64 from the fp32 features and stored as fp32 (the render path's
// feature precision), so the result differs from the level-by-level sum only
// by rounding (well inside the 1e-4 SDF bar).
//
// Corners shared by several level-G voxels are computed once, from the
// voxel with the smallest index that references them, so S is
// deterministic.
#include "common.cuh"

namespace ng {

static inline int pgrid(int64_t n, int nt) { return (int)((n + nt - 1) / nt); }

__global__ void k_presum_owner(const __grid_constant__ ng_octree tree, int G, int64_t offset, int* owner) {
  const int tl = G + tree.n_virtual;
  const int64_t nv = tree.count[tl];
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nv * 8) return;
  const int id = tree.corners[tl][e];
  atomicMin(owner + (id - offset), (int)(e >> 3));
}

// Warp per (voxel, corner) slot, lane = channel.
__global__ void k_presum(const __grid_constant__ ng_octree tree, const float* __restrict__ Z, int G, int out_mask,
                         int64_t offset, int64_t n_corners, const int* __restrict__ owner, float* __restrict__ S) {
  const int lane = threadIdx.x & 31;
  const int tl = G + tree.n_virtual;
  const int64_t nv = tree.count[tl];
  const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (e >= nv * 8) return;
  const int64_t v = e >> 3;
  const int j = (int)(e & 7);
  const int id = __ldg(tree.corners[tl] + e);
  if (__ldg(owner + (id - offset)) != (int)v) return;
  const uint64_t code = __ldg(tree.codes[tl] + v);
  // corner lattice coordinates at level G (exact integers)
  const int cg[3] = {(int)compact3(code) + (j & 1), (int)compact3(code >> 1) + ((j >> 1) & 1),
                     (int)compact3(code >> 2) + ((j >> 2) & 1)};
  double z = 0.0;
  int slot = 0;
  for (int l = 1; l <= G; ++l) {
    const int sh = G - l;
    // the level-l ancestor of voxel v (exists: parent closure, octree.py:183-187)
    const int vc[3] = {(int)compact3(code) >> sh, (int)compact3(code >> 1) >> sh, (int)compact3(code >> 2) >> sh};
    const int64_t idx = rank_lookup(tree.bitmap[l + tree.n_virtual], tree.rank[l + tree.n_virtual],
                                    morton(vc[0], vc[1], vc[2]));
    const int* cid = tree.corners[l + tree.n_virtual] + 8 * idx;
    // local coordinates of the corner point inside the ancestor cell: exact
    // dyadic values in [0, 1] (corner at cg / 2^sh in level-l cell units)
    const double inv = 1.0 / (double)(1 << sh);
    double u[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) u[a] = (double)cg[a] * inv - (double)vc[a];
    double psi = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double wx = (q & 1) ? u[0] : 1.0 - u[0];
      const double wy = ((q >> 1) & 1) ? u[1] : 1.0 - u[1];
      const double wz = ((q >> 2) & 1) ? u[2] : 1.0 - u[2];
      psi += (wx * wy * wz) * (double)__ldg(Z + 32 * (int64_t)__ldg(cid + q) + lane);
    }
    z += psi;
    if ((out_mask >> (l - 1)) & 1) {
      S[((int64_t)slot * n_corners + (id - offset)) * 32 + lane] = (float)z;
      ++slot;
    }
  }
}

}  // namespace ng

using namespace ng;

extern "C" int ng_field_presum(const ng_octree* tree, const float* Z, int32_t level, int32_t out_mask,
                               int64_t offset, int64_t n_corners, float* S, int32_t* owner_scratch, void* stream) {
  if (level < 1 || level > tree->max_level || out_mask <= 0 || (out_mask >> level) != 0) {
    set_error("presum: level %d / output mask 0x%x invalid", level, out_mask);
    return NG_ERR_STRUCTURAL;
  }
  const int tl = level + tree->n_virtual;
  const int64_t nv = tree->count[tl];
  if (nv <= 0 || n_corners <= 0) return NG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  int r = cuda_status(cudaMemsetAsync(owner_scratch, 0x7f, sizeof(int32_t) * n_corners, s), "presum owner");
  if (r) return r;
  k_presum_owner<<<pgrid(nv * 8, 256), 256, 0, s>>>(*tree, level, offset, owner_scratch);
  NG_CHECK_LAUNCH("k_presum_owner");
  k_presum<<<pgrid(nv * 8 * 32, 256), 256, 0, s>>>(*tree, Z, level, out_mask, offset, n_corners, owner_scratch, S);
  NG_CHECK_LAUNCH("k_presum");
  return NG_OK;
}
