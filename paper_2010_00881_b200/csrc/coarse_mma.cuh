// coarse_mma.cuh -- the tiled coarse PCG (coarse_tiled.cuh: bricks in shared memory,
// Chronopoulos-Gear CG, one grid barrier per iteration) with the smoother and the operator
// applied CELL-CENTRIC instead of vertex-centric (3D scalar p = 1 level, AS preconditioner):
//  * regular cells (one shared matrix per group: a Schwarz type inverse, or K_ref) in groups
//    of up to 8 x-consecutive cells -> Y = A [v_c1 .. v_c8] as two fp64 MMAs (m8n8k4),
//  * individual cells (irregular Schwarz blocks / cut cells) one thread per cell, their
//    packed matrices streamed from L1/L2 in 32-cell SoA chunks (host-built per brick),
//  * then every vertex sums its 2^d cell contributions Y[corner][cell] in a fixed order.
// Each cell's 8 products are formed once per phase (the vertex-centric form re-reads every
// matrix row per corner), the shared-memory traffic per iteration roughly halves, and the
// shared memory no longer holds individual matrices (room for Y).  Same iterates and the same
// determinism as k_coarse_tiled (bit-identical redundant halo values: every product depends
// only on its own cell's data and is formed by the same code on every CTA).
#pragma once
#include "cellmma.cuh"
#include "coarse_tiled.cuh"

namespace fcm {

constexpr int kMmaOpSlot = 255;   // group slot of the operator groups (K_ref)

__host__ __device__ constexpr size_t mma_tiled_smem_bytes(int E2, int EC, int T, int ntypes, int max_groups) {
  return (size_t)(3 * E2 + 2 * T + 8 * EC + (ntypes + 1) * 64) * 8 + (size_t)(E2 + 3 * EC + 2 * max_groups) * 4 + 64;
}

__global__ void __launch_bounds__(kTiledThreads, 1) k_coarse_mma(TiledArgs a) {
  constexpr int PK = 36;   // packed 8x8
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double red[96];
  __shared__ double tot[3];
  __shared__ int n_gsm, n_gop;
  const int e0 = a.e[0], e1 = a.e[1], e01 = a.e[0] * a.e[1];
  const int t0 = a.tile[0], t1 = a.tile[1], t2 = a.tile[2];
  const int ec0 = a.ec[0], ec1 = a.ec[1], ec01 = ec0 * ec1;
  const int E2 = e0 * e1 * a.e[2], EC = ec01 * a.ec[2], nT = t0 * t1 * t2;
  double* r = reinterpret_cast<double*>(smem);
  double* sv = r + E2;
  double* u = sv + E2;
  double* p = u + E2;
  double* x = p + nT;
  double* Y = x + nT;                  // [8][EC] corner-major
  double* Afr = Y + 8 * EC;            // [ntypes + 1][2][32]: type slots, then K_ref
  int* gidx = reinterpret_cast<int*>(Afr + (a.ntypes + 1) * 64);
  int* csm = gidx + E2;                // per cell: -1 none, -2 individual, else slot | scale bit
  int* cop = csm + EC;                 // per cell: -1 none, -2 cut, else 0 | scale bit (alpha)
  int* cvb = cop + EC;                 // per cell: E2 index of corner 0
  int* gsm = cvb + EC;                 // smoother groups
  int* gop = gsm + a.max_groups;       // operator groups
  const int bt = blockIdx.x;
  const int tix = bt % a.ntile[0], tiy = (bt / a.ntile[0]) % a.ntile[1], tiz = bt / (a.ntile[0] * a.ntile[1]);
  const int o0 = a.blo[0] + tix * t0 - 2, o1 = a.blo[1] + tiy * t1 - 2, o2 = a.blo[2] + tiz * t2 - 2;
  // ---- one-time staging -------------------------------------------------------------------
  if (threadIdx.x == 0) { n_gsm = 0; n_gop = 0; }
  for (int t = threadIdx.x; t < (a.ntypes + 1) * 64; t += blockDim.x) {
    const int sl = t / 64, kt = (t / 32) & 1, lane = t & 31;
    const int row = lane >> 2, col = kt * 4 + (lane & 3);
    Afr[t] = sl < a.ntypes ? a.type_inv[(size_t)sl * 64 + row * 8 + col] : a.Kref[row * a.ldK + col];
  }
  for (int t = threadIdx.x; t < 8 * EC; t += blockDim.x) Y[t] = 0.0;
  for (int t = threadIdx.x; t < EC; t += blockDim.x) {
    const int lx = t % ec0, ly = (t / ec0) % ec1, lz = t / ec01;
    const int cx = o0 + lx, cy = o1 + ly, cz = o2 + lz;
    int sm = -1, op = -1;
    if (cx >= 0 && cy >= 0 && cz >= 0 && cx < a.n[0] && cy < a.n[1] && cz < a.n[2]) {
      const int c = (cz * a.n[1] + cy) * a.n[0] + cx;
      const int k = a.kind[c];
      op = k == 2 ? -2 : (k == 1 ? kScaleBit : 0);
      const int bq = a.blk[c];
      if (bq >= 0) sm = -2;
      else { const int tt = -bq - 1; sm = (tt & 0xfff) | ((tt >> 12) ? kScaleBit : 0); }
    }
    csm[t] = sm;
    cop[t] = op;
    cvb[t] = (lz * e1 + ly) * e0 + lx;
  }
  for (int t = threadIdx.x; t < E2; t += blockDim.x) {
    const int v0 = o0 + t % e0, v1 = o1 + (t / e0) % e1, v2 = o2 + t / e01;
    int g = -1;
    if (v0 >= a.vlo[0][0] && v0 <= a.vhi[0][0] && v1 >= a.vlo[0][1] && v1 <= a.vhi[0][1] &&
        v2 >= a.vlo[0][2] && v2 <= a.vhi[0][2]) {
      const int s0 = a.vhi[0][0] - a.vlo[0][0] + 1, s1 = a.vhi[0][1] - a.vlo[0][1] + 1;
      g = (int)a.voff[0] + (v0 - a.vlo[0][0]) + s0 * ((v1 - a.vlo[0][1]) + s1 * (v2 - a.vlo[0][2]));
    }
    gidx[t] = g;
    r[t] = g >= 0 ? a.b[g] : 0.0;
    sv[t] = 0.0;
    u[t] = 0.0;
  }
  for (int t = threadIdx.x; t < nT; t += blockDim.x) { p[t] = 0.0; x[t] = 0.0; }
  __syncthreads();
  // regular groups: runs of <= 8 x-consecutive cells with one matrix, one x-row per thread
  // smoother: the whole cell box; operator: the cells touching the brick ([1, tile+1] per axis)
  for (int row = threadIdx.x; row < ec1 * a.ec[2]; row += blockDim.x) {
    const int ly = row % ec1, lz = row / ec1;
    int start = -1, cnt = 0, slot = -1;
    for (int lx = 0; lx <= ec0; ++lx) {
      const int c = lz * ec01 + ly * ec0 + lx;
      const int code = lx < ec0 ? csm[c] : -1;
      const int sl = code >= 0 ? (code & 0xfff) : -1;
      if (cnt > 0 && (sl != slot || cnt == 8)) {
        gsm[atomicAdd(&n_gsm, 1)] = start | ((cnt - 1) << 13) | (slot << 16);
        cnt = 0;
      }
      if (sl >= 0) {
        if (cnt == 0) { start = c; slot = sl; }
        ++cnt;
      }
    }
    if (ly >= 1 && ly <= t1 + 1 && lz >= 1 && lz <= t2 + 1) {
      cnt = 0;
      for (int lx = 1; lx <= t0 + 2; ++lx) {
        const int c = lz * ec01 + ly * ec0 + lx;
        const bool reg = lx <= t0 + 1 && cop[c] >= 0;
        if (cnt > 0 && (!reg || cnt == 8)) {
          gop[atomicAdd(&n_gop, 1)] = start | ((cnt - 1) << 13) | (kMmaOpSlot << 16);
          cnt = 0;
        }
        if (reg) {
          if (cnt == 0) start = c;
          ++cnt;
        }
      }
    }
  }
  __syncthreads();
  const int ngsm = n_gsm, ngop = n_gop;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int ism0 = a.ism_off[bt], ism1 = a.ism_off[bt + 1];
  const int iop0 = a.iop_off[bt], iop1 = a.iop_off[bt + 1];
  const double sc_sm = a.inv_alpha, sc_op = a.alpha;
  // corner offsets in E2 (corner k: x = k&1, y = (k>>1)&1, z = k>>2)
  auto corner = [&](int k) { return (k & 1) + ((k >> 1) & 1) * e0 + (k >> 2) * e01; };

  // Y[corner][cell] = s_c Mat_c v_c for every cell of the groups and of the individual list
  auto cell_products = [&](const double* __restrict__ v, const int* grp, int ng, const int* codes,
                           double scale_flag, const int32_t* __restrict__ icell,
                           const double* __restrict__ imat, int i0, int i1) {
    for (int g = warp; g < ng; g += nwarp) {
      const int d = grp[g];
      const int start = d & 0x1fff, cnt = ((d >> 13) & 7) + 1, slot = d >> 16;
      const double* A = Afr + (slot == kMmaOpSlot ? a.ntypes : slot) * 64;
      const int n = lane >> 2, kq = lane & 3;
      double b0 = 0.0, b1 = 0.0;
      if (n < cnt) {
        const int vb = cvb[start + n];
        b0 = v[vb + corner(kq)];
        b1 = v[vb + corner(4 + kq)];
      }
      double d0 = 0.0, d1 = 0.0;
      dmma_8x8x4(d0, d1, A[lane], b0, d0, d1);
      dmma_8x8x4(d0, d1, A[32 + lane], b1, d0, d1);
      const int row = lane >> 2, n0 = 2 * kq, n1 = n0 + 1;
      if (n0 < cnt) {
        const int c = start + n0;
        Y[row * EC + c] = ((codes[c] & kScaleBit) ? scale_flag : 1.0) * d0;
      }
      if (n1 < cnt) {
        const int c = start + n1;
        Y[row * EC + c] = ((codes[c] & kScaleBit) ? scale_flag : 1.0) * d1;
      }
    }
    for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
      const int c = __ldg(icell + i);
      if (c < 0) continue;
      const double* M = imat + ((size_t)(i >> 5) * PK) * 32 + (i & 31);
      const int vb = cvb[c];
      double vc[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) vc[k] = v[vb + corner(k)];
      double y[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) y[k] = 0.0;
#pragma unroll
      for (int ra = 0; ra < 8; ++ra)
#pragma unroll
        for (int cb = 0; cb <= ra; ++cb) {
          const double m = __ldg(M + (ra * (ra + 1) / 2 + cb) * 32);
          y[ra] = fma(m, vc[cb], y[ra]);
          if (cb != ra) y[cb] = fma(m, vc[ra], y[cb]);
        }
#pragma unroll
      for (int k = 0; k < 8; ++k) Y[k * EC + c] = y[k];
    }
  };
  // vertex sum over the 2^d cells around E2 entry (lx, ly, lz), corner order kc = 0..7
  auto vertex_sum = [&](int lx, int ly, int lz) {
    double acc = 0.0;
#pragma unroll
    for (int kc = 0; kc < 8; ++kc) {
      const int ox = kc & 1, oy = (kc >> 1) & 1, oz = kc >> 2;
      acc += Y[kc * EC + (lz - oz) * ec01 + (ly - oy) * ec0 + (lx - ox)];
    }
    return acc;
  };
  const int g1x = t0 + 2, g1y = t1 + 2, nE1 = g1x * g1y * (t2 + 2);
  auto smooth_E1 = [&]() {   // u = M r on E1
    cell_products(r, gsm, ngsm, csm, sc_sm, a.ism_cell, a.ism_mat, ism0, ism1);
    __syncthreads();
    for (int q = threadIdx.x; q < nE1; q += blockDim.x) {
      const int lx = q % g1x + 1, ly = (q / g1x) % g1y + 1, lz = q / (g1x * g1y) + 1;
      const int l = (lz * e1 + ly) * e0 + lx;
      u[l] = gidx[l] >= 0 ? vertex_sum(lx, ly, lz) : 0.0;
    }
  };
  auto t_local = [&](int q) {
    const int lx = q % t0 + 2, ly = (q / t0) % t1 + 2, lz = q / (t0 * t1) + 2;
    return (lz * e1 + ly) * e0 + lx;
  };
  auto apply_T = [&](double* wout, double& gg, double& dl, double& rh) {   // w = A u on T
    cell_products(u, gop, ngop, cop, sc_op, a.iop_cell, a.iop_mat, iop0, iop1);
    __syncthreads();
    gg = 0.0; dl = 0.0; rh = 0.0;
    for (int q = threadIdx.x; q < nT; q += blockDim.x) {
      const int lx = q % t0 + 2, ly = (q / t0) % t1 + 2, lz = q / (t0 * t1) + 2;
      const int l = (lz * e1 + ly) * e0 + lx;
      const int gi = gidx[l];
      if (gi < 0) continue;
      const double w = vertex_sum(lx, ly, lz);
      __stcg(wout + gi, w);
      const double ri = r[l], ui = u[l];
      gg = fma(ri, ui, gg);
      dl = fma(w, ui, dl);
      rh = fma(ri, ri, rh);
    }
  };

  const unsigned cnt0 = t_ld_relaxed(&a.ctl->base);
  unsigned gen = 0;
  double g_loc, d_loc, r_loc;
  smooth_E1();
  __syncthreads();
  apply_T(a.wpub[0], g_loc, d_loc, r_loc);
  double wl[4];
  auto preload_w = [&](const double* wv) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int t = k * blockDim.x + threadIdx.x;
      const int gi = t < E2 ? gidx[t] : -1;
      wl[k] = gi >= 0 ? __ldcg(wv + gi) : 0.0;
    }
  };
  tiled_arrive_wait(g_loc, d_loc, r_loc, a.part, a.ctl, cnt0 + (gen + 1) * gridDim.x, gen + 1, red);
  ++gen;
  preload_w(a.wpub[0]);
  tiled_totals(a.part, gen, tot);
  __syncthreads();
  double gamma = tot[0], delta = tot[1];
  const double rho0 = tot[2];
  double rho = rho0;
  double gamma_old = 1.0, alpha_old = 1.0;
  int it = 0;
  while (rho0 > 0.0 && !(rho < a.rtol2 * rho0) && it < a.maxit) {
    double beta, alpha;
    if (it == 0) {
      beta = 0.0;
      alpha = gamma / delta;
    } else {
      beta = gamma / gamma_old;
      alpha = gamma / (delta - beta * gamma / alpha_old);
    }
    if (!(alpha > 0.0) || !(gamma > 0.0)) break;   // breakdown (not SPD): keep x_it
    const unsigned long long tp0 = a.prof ? t_now() : 0ull;
    const double* wv = a.wpub[it & 1];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int t = k * blockDim.x + threadIdx.x;
      if (t < E2 && gidx[t] >= 0) {
        const double s_ = fma(beta, sv[t], wl[k]);
        sv[t] = s_;
        r[t] = fma(-alpha, s_, r[t]);
      }
    }
    for (int t = 4 * blockDim.x + threadIdx.x; t < E2; t += blockDim.x) {
      const int gi = gidx[t];
      if (gi < 0) continue;
      const double s_ = fma(beta, sv[t], __ldcg(wv + gi));
      sv[t] = s_;
      r[t] = fma(-alpha, s_, r[t]);
    }
    for (int q = threadIdx.x; q < nT; q += blockDim.x) {
      const double pv = fma(beta, p[q], u[t_local(q)]);
      p[q] = pv;
      x[q] = fma(alpha, pv, x[q]);
    }
    ++it;
    gamma_old = gamma;
    alpha_old = alpha;
    __syncthreads();
    const unsigned long long tp1 = a.prof ? t_now() : 0ull;
    smooth_E1();
    __syncthreads();
    const unsigned long long tp2 = a.prof ? t_now() : 0ull;
    apply_T(a.wpub[it & 1], g_loc, d_loc, r_loc);
    __syncthreads();
    const unsigned long long tp3 = a.prof ? t_now() : 0ull;
    tiled_arrive_wait(g_loc, d_loc, r_loc, a.part, a.ctl, cnt0 + (gen + 1) * gridDim.x, gen + 1, red);
    ++gen;
    preload_w(a.wpub[it & 1]);
    tiled_totals(a.part, gen, tot);
    __syncthreads();
    if (a.prof && threadIdx.x == 0) {
      const unsigned long long tp4 = t_now();
      unsigned long long* pr = a.prof + 4 * blockIdx.x;
      pr[0] += tp1 - tp0; pr[1] += tp2 - tp1; pr[2] += tp3 - tp2; pr[3] += tp4 - tp3;
    }
    gamma = tot[0];
    delta = tot[1];
    rho = tot[2];
  }
  for (int q = threadIdx.x; q < nT; q += blockDim.x) {
    const int gi = gidx[t_local(q)];
    if (gi >= 0) a.x[gi] = x[q];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.iters[0] = it;
    a.iters[1] += it;
    a.ctl->base = cnt0 + gen * gridDim.x;
  }
}

}  // namespace fcm
