// blocks.cuh -- additive-Schwarz blocks of general shape ("elementwise and
// patchwise"): a block is anchored at a cell (elementwise: the DOFs supported on that cell)
// or at a grid vertex (patchwise: the union of the DOFs of the 2^d cells around the vertex).
// The block's DOF list is translation invariant: DOF l of the block at anchor A is local DOF
// loc[l] of member cell A + mo[mem[l]] (Table 1 sizes (2p+1)^d for tensor
// patches).  Setup assembles A_i = P_i^T A_q P_i (Eq. AdditiveSchwarz) from the cell
// matrices of the assembly cells around the anchor; the smoother applies
// x += omega sum_i P_i A_i^{-1} P_i^T r with one warp per block (patch sizes up to 729).
#pragma once
#include <cstdint>

#include "cellop.cuh"

namespace fcm {

constexpr int kBlkNone = INT32_MIN;   // anchor whose block has no free DOF (skipped)
constexpr int kBlkWb = INT32_MIN + 1;  // individual patch applied as a low-rank correction (patch_wb.cuh)

struct BlockAsmArgs {
  int nx, ny, nz, dim;          // owned cell grid (anchor coordinates are relative to it)
  int lo[3], ne[3];             // cell arrays (kind, cut_idx) cover [lo, lo + ne) per axis
  int mb;                       // block size
  int ldK;                      // element matrix leading dimension (fine m)
  int na[3];                    // anchor grid extents
  int nasm, aoff;               // assembly cells per axis and their first offset
  const int64_t* anchors;       // block -> anchor index (x fastest over na)
  const uint8_t* virt;          // 1: treat every assembly cell as uncut physical (type block)
  const int16_t* amap;          // [nasm^d][mb] local index in the assembly cell, -1 none
  const int8_t* dirich;         // [nblocks][mb] 1: DOF absent or Dirichlet (identity row)
  const uint8_t* kind;
  const int32_t* cut_idx;
  const double* Kref;
  const double* cutK;
  double alpha;
  double* out;                  // [nblocks][mb][mb]
};

__global__ void k_assemble_blocks(BlockAsmArgs a) {
  const int64_t blk = blockIdx.x;
  const int64_t A = a.anchors[blk];
  const int ax = (int)(A % a.na[0]), ay = (int)((A / a.na[0]) % a.na[1]), az = (int)(A / ((int64_t)a.na[0] * a.na[1]));
  const int mb = a.mb;
  double* out = a.out + blk * (int64_t)mb * mb;
  const int8_t* dir = a.dirich + blk * mb;
  const int ncz = a.dim == 3 ? a.nasm : 1, ncy = a.dim >= 2 ? a.nasm : 1;
  const int nas = a.nasm * ncy * ncz;
  for (int64_t e = threadIdx.x; e < (int64_t)mb * mb; e += blockDim.x) {
    const int i = (int)(e / mb), j = (int)(e % mb);
    double s = 0.0;
    if (dir[i] || dir[j]) {
      s = (i == j) ? 1.0 : 0.0;
    } else {
      for (int d = 0; d < nas; ++d) {
        const int ii = a.amap[d * mb + i], jj = a.amap[d * mb + j];
        if (ii < 0 || jj < 0) continue;
        const int cx = ax + a.aoff + d % a.nasm;
        const int cy = a.dim >= 2 ? ay + a.aoff + (d / a.nasm) % a.nasm : 0;
        const int cz = a.dim == 3 ? az + a.aoff + d / (a.nasm * a.nasm) : 0;
        if (cx < a.lo[0] || cy < a.lo[1] || cz < a.lo[2] || cx >= a.lo[0] + a.ne[0] ||
            cy >= a.lo[1] + a.ne[1] || cz >= a.lo[2] + a.ne[2])
          continue;
        const int64_t c = ((int64_t)(cz - a.lo[2]) * a.ne[1] + (cy - a.lo[1])) * a.ne[0] + (cx - a.lo[0]);
        double v;
        if (a.virt[blk]) {
          v = a.Kref[(int64_t)ii * a.ldK + jj];
        } else {
          const uint8_t k = a.kind[c];
          if (k == 2) v = a.cutK[(int64_t)a.cut_idx[c] * a.ldK * a.ldK + (int64_t)ii * a.ldK + jj];
          else v = a.Kref[(int64_t)ii * a.ldK + jj] * (k == 1 ? a.alpha : 1.0);
        }
        s += v;
      }
    }
    out[e] = s;
  }
}

// One smoother application over general (patch) blocks: one warp per anchor.
struct BlockOp {
  int colour;                 // deterministic mode: only anchors of this colour (v mod 3 per axis), -1 all
  int nx, ny, nz;               // cells
  int na[3];                    // anchors
  int64_t nanchor;
  int mb;
  int nmem;
  int mo[8][3];                 // member cell offsets
  const int8_t* mem;            // [mb]
  const int16_t* loc;           // [mb]
  // level table (dof index of local DOF a of a cell), as in CellOp
  int m;                        // level element size
  const int64_t* base;
  const int32_t* stride;
  const int16_t* cmin;
  const int16_t* cmax;
  const int32_t* blk;           // per anchor: >= 0 individual, < 0 type (slot | alpha << 12), kBlkNone
  const double* type_inv;       // [ntypes][mb*mb]
  const double* irr_inv;        // [n_irr][mb*mb]
  double inv_alpha;
  const double* in;
  double* out;
  double coef;
};

// smem: [Tab][per warp: xs[mb] doubles][per warp: ids[mb] ints]
__global__ void __launch_bounds__(256) k_block_smooth(BlockOp op) {
  extern __shared__ __align__(16) unsigned char smem[];
  Tab& T = *reinterpret_cast<Tab*>(smem);
  const int wpb = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mb = op.mb;
  double* xs = reinterpret_cast<double*>(smem + sizeof(Tab)) + (size_t)w * mb;
  int* ids = reinterpret_cast<int*>(reinterpret_cast<double*>(smem + sizeof(Tab)) + (size_t)wpb * mb) + (size_t)w * mb;
  for (int a = threadIdx.x; a < op.m; a += blockDim.x) {
    T.g[a] = make_int4((int32_t)op.base[a], op.stride[a * 3 + 1], op.stride[a * 3 + 2], 0);
    T.lo[a] = make_int4(op.cmin[a * 3 + 0], op.cmin[a * 3 + 1], op.cmin[a * 3 + 2], 0);
    T.hi[a] = make_int4(op.cmax[a * 3 + 0], op.cmax[a * 3 + 1], op.cmax[a * 3 + 2], 0);
  }
  __syncthreads();
  for (int64_t A = (int64_t)blockIdx.x * wpb + w; A < op.nanchor; A += (int64_t)gridDim.x * wpb) {
    const int32_t bq = op.blk[A];
    if (bq == kBlkNone || bq >= 0) continue;   // warp-uniform; individual blocks: k_patch_irr
    const int ax = (int)(A % op.na[0]), ay = (int)((A / op.na[0]) % op.na[1]);
    const int az = (int)(A / ((int64_t)op.na[0] * op.na[1]));
    if (op.colour >= 0 && (ax % 3) + 3 * (ay % 3) + 9 * (az % 3) != op.colour) continue;   // deterministic mode
    for (int l = lane; l < mb; l += 32) {
      const int k = op.mem[l], a = op.loc[l];
      const int cx = ax + op.mo[k][0], cy = ay + op.mo[k][1], cz = az + op.mo[k][2];
      bool ok = cx >= 0 && cy >= 0 && cz >= 0 && cx < op.nx && cy < op.ny && cz < op.nz;
      ok = ok && dof_free(T, a, cx, cy, cz);
      const int idx = ok ? dof_index(T, a, cx, cy, cz) : -1;
      ids[l] = idx;
      xs[l] = ok ? __ldg(op.in + idx) : 0.0;
    }
    __syncwarp();
    const double* Mat;
    double scale = 1.0;
    if (bq >= 0) {
      Mat = op.irr_inv + (size_t)bq * mb * mb;
    } else {
      const int t = -bq - 1;
      Mat = op.type_inv + (size_t)(t & 0xfff) * mb * mb;
      scale = (t >> 12) ? op.inv_alpha : 1.0;
    }
    // symmetric inverse streamed column by column: lanes read consecutive rows (coalesced)
    for (int l = lane; l < mb; l += 32) {
      double acc0 = 0.0, acc1 = 0.0;
      const double* col = Mat + l;
      int b = 0;
      for (; b + 2 <= mb; b += 2) {
        acc0 = fma(__ldg(col + (size_t)b * mb), xs[b], acc0);
        acc1 = fma(__ldg(col + (size_t)(b + 1) * mb), xs[b + 1], acc1);
      }
      if (b < mb) acc0 = fma(__ldg(col + (size_t)b * mb), xs[b], acc0);
      const int id = ids[l];
      if (id >= 0) atomicAdd(op.out + id, op.coef * scale * (acc0 + acc1));
    }
    __syncwarp();
  }
}

}  // namespace fcm
