// 3D linear elasticity on cubic Kuhn cells in lattice-edge flux form (cfg3, cfg5).
//
// Replaces the element loop of reference fem.py:397-411 (+ the Dirichlet
// elimination fem.py:274-291) for d = 3 on the structured Kuhn mesh of
// ops3d.cu.  For a tetrahedron with path axes (a, b, c) every P1 gradient is a
// difference of unit axis vectors / h, so with D^x, D^y, D^z the raw
// differences of u along the tet's x-, y- and z-directed path edges, and
// s = w mu / h^2, l = w lam / h^2 (w = |T| times the ersatz weight of the tet),
//   sigma_aa = l (D^x_x + D^y_y + D^z_z) + 2 s D^a_a,  sigma_ab = s (D^a_b + D^b_a),
// and the tet adds the column sigma e_a to the flux of its a-directed edge
// (the edge's start node receives -flux, its end node +flux).  Every path edge
// is an edge of the cube, so all fluxes live on the lattice's axis edges:
// each lattice edge sums the fluxes of the six tets that share it, and a node's
// result is the divergence
//   y(P) = sum_a F(P - e_a -> P) - F(P -> P + e_a).
// Per cell and right-hand side this is ~156 fp64 instructions (edge
// differences 24, stresses 72, edge sums 45, divergence 15) against ~260 for
// the corner-scatter form (march3s<ElastC>): no edge difference and no flux is
// formed twice.
//
// Execution: a CTA of 8 warps covers 31 node columns (lanes 1..31; lane 0 is
// a halo column) and 8 node rows (warp 0 is a halo row) and marches along z.
// Thread (i, j) owns the lattice edges leaving node (i, j) in +x, +y, +z.  At
// step kc it evaluates cell (i, j, kc) (between planes kc and kc+1), routes
// the cell's twelve edge fluxes to the owning threads -- itself (plane kc, and
// plane kc+1 as pending sums), lane+1 (shuffles), the warp above (one
// parity-double-buffered shared exchange, one CTA barrier per plane) -- and
// then emits node (i, j, kc).  Every node is summed by one thread in a fixed
// order (deterministic, independent of the launch geometry).
//
// Staging: each plane's 9 rows of u (33 nodes x 24 B) and material words are
// brought into a 4-slot shared ring by bulk copies (cp.async.bulk, TMA engine)
// completing on one mbarrier per slot, three planes ahead; one lane per warp
// issues its row.  Dirichlet-masked inputs are zeroed in the staged copy (the
// masked rows are the clamped face only, so a warp vote skips the fix-up
// everywhere else).
#pragma once

namespace lsg {
namespace d3 {

constexpr int kEStrip = 31;          // owned node columns per warp (lane 0 is halo)
constexpr int kEWarps = 8;           // node rows per CTA (warp 0 is halo)
constexpr int kEThreads = kEWarps * 32;
constexpr int kERows = kEWarps + 1;  // staged rows per plane
constexpr int kESlots = 4;           // plane ring, three planes in flight
constexpr int kEUSlot = 100;         // doubles per staged row: 33 nodes x 3 (+ 8-byte phase), 16-B multiple
constexpr int kEWSlot = 40;          // words per staged row: 33 (+ up to 3 phase), 16-B multiple
#ifndef KE_MINB
#define KE_MINB 2
#endif
constexpr int kEX = 12;              // doubles per lane handed to the warp above each step

struct ETab {
  double s, s2, l, pad;
};

struct ESmem {
  double u[kESlots][kERows][kEUSlot];
  uint32_t wd[kESlots][kERows][kEWSlot];
  double xchg[2][kEWarps][kEX][32];
  double carry[9][kEThreads];  // per thread: x/y-edge flux sums from the cell below, z-edge flux below
  ETab tab[8];
  uint64_t bar[kESlots];
  double scratch[3 * kEWarps];
};

// The six stress components of one tet from its x-, y-, z-edge differences.
__device__ __forceinline__ void kuhn_sigma(const double *Dx, const double *Dy, const double *Dz,
                                           const ETab &t, double (&sg)[6]) {
  const double lt = t.l * (Dx[0] + Dy[1] + Dz[2]);
  sg[0] = fma(t.s2, Dx[0], lt);     // xx
  sg[1] = fma(t.s2, Dy[1], lt);     // yy
  sg[2] = fma(t.s2, Dz[2], lt);     // zz
  sg[3] = t.s * (Dx[1] + Dy[0]);    // xy
  sg[4] = t.s * (Dx[2] + Dz[0]);    // xz
  sg[5] = t.s * (Dy[2] + Dz[1]);    // yz
}
// the flux columns of a stress: x-edge (xx, xy, xz), y-edge (xy, yy, yz), z-edge (xz, yz, zz)
__device__ __forceinline__ double fxc(const double (&s)[6], int q) { return q == 0 ? s[0] : q == 1 ? s[3] : s[4]; }
__device__ __forceinline__ double fyc(const double (&s)[6], int q) { return q == 0 ? s[3] : q == 1 ? s[1] : s[5]; }
__device__ __forceinline__ double fzc(const double (&s)[6], int q) { return q == 0 ? s[4] : q == 1 ? s[5] : s[2]; }

template <int ACT>
__global__ void __launch_bounds__(kEThreads, KE_MINB) kuhn_edge(ElastC ph, Geo g, MArgs a) {
  static_assert(ACT == APPLY || ACT == RESID || ACT == PCGQ, "kuhn_edge modes");
  constexpr int NP = Traits<ACT>::NP;
  constexpr int NPA = NP > 0 ? NP : 1;
  constexpr int kSlotD = kERows * kEUSlot;  // doubles per ring slot
  constexpr int kSlotW = kERows * kEWSlot;  // words per ring slot
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ESmem &S = *reinterpret_cast<ESmem *>(smem_raw);

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nzseg = a.nzseg;
  const int zseg = blockIdx.z % nzseg, rhs = blockIdx.z / nzseg;
  const int nk = gridDim.z / nzseg;  // right-hand sides in the batch
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const int64_t nxp = nx + 1;
  const int64_t plane = nxp * (ny + 1);
  const int64_t nn = plane * (nz + 1);

  if (threadIdx.x < 8) {  // per-tet coefficients by n_in (0..4); index 7 (invalid cell) is zero
    const int n = threadIdx.x;
    const double wt = n <= 4 ? fma((double)n, ph.w1, ph.w0) : 0.0;
    ETab t;
    t.s = wt * ph.cs;
    t.s2 = 2.0 * t.s;
    t.l = wt * ph.cl;
    t.pad = 0.0;
    S.tab[n] = t;
  }
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < kESlots; ++s) mbar_init(&S.bar[s], kERows);
    mbar_init_fence();
  }
  if constexpr (ACT == PCGQ) pdl_wait();  // launched with launch_pdl (common.cuh)
  if constexpr (ACT == RESID || ACT == PCGQ) {
    if (a.scal[rhs].done != 0.0) return;
  }
  __syncthreads();

  const int strip = blockIdx.x;
  const int i = strip * kEStrip - 1 + lane;
  const int j0 = (int)blockIdx.y * (kEWarps - 1) - 1;
  const int jw = j0 + w;
  const bool top = (w == kEWarps - 1);
  const bool col_ok = (strip < a.nstrips) && i >= 0 && i <= nx;
  const bool node_ok = col_ok && jw >= 0 && jw <= ny;
  const bool own = node_ok && lane >= 1 && w >= 1;
  const int lo = min(max(strip * kEStrip - 1, 0), nx);
  const int hi = min(max(strip * kEStrip + kEStrip, 0), nx);
  const int nwin = hi - lo + 1;
  const int iw = min(max(i, lo), hi) - lo;       // own node in the staged window
  const int iwr = min(max(i + 1, lo), hi) - lo;  // right neighbour
  const int K0 = zseg * a.seg;
  const int K1 = min(K0 + a.seg, nz + 1);
  const int kstart = max(K0 - 1, 0);
  const int kend = min(K1, nz);
  const size_t voff = (size_t)rhs * (size_t)nn * 3;
  const double *src = a.x + voff;

  // Per-row constants.  Staged row r of plane kk holds the window of node
  // row jr(r) starting at node n0 = kk*plane + jr*(nx+1) + lo; its first
  // double sits (address of u(n0)) mod 16 / 8 into the slot, its first word
  // (address of word(n0)) mod 16 / 4 into the word slot.
  const uint32_t p1 = (uint32_t)plane & 1u, p3 = (uint32_t)plane & 3u;
  const uint32_t ub = (uint32_t)(reinterpret_cast<uintptr_t>(src) >> 3) & 1u;
  const uint32_t wbb = (uint32_t)(reinterpret_cast<uintptr_t>(a.words) >> 2) & 3u;
  auto jrow = [&](int r) { return min(max(j0 + r, 0), ny); };
  const int64_t rn0 = (int64_t)jrow(w) * nxp + lo, rn1 = (int64_t)jrow(w + 1) * nxp + lo;
  const uint32_t uph0 = (ub ^ (uint32_t)rn0) & 1u, uph1 = (ub ^ (uint32_t)rn1) & 1u;
  const uint32_t wph0 = (wbb + (uint32_t)rn0) & 3u, wph1 = (wbb + (uint32_t)rn1) & 3u;
  // doubles offset of (row, lane node / right node) within a slot, phase excluded
  const int o00 = w * kEUSlot + iw * 3, o01 = w * kEUSlot + iwr * 3;
  const int o10 = (w + 1) * kEUSlot + iw * 3, o11 = (w + 1) * kEUSlot + iwr * 3;
  const int64_t own_node = (int64_t)jw * nxp + i;  // + kk*plane

  const double *U = &S.u[0][0][0];
  const uint32_t *W = &S.wd[0][0][0];
  auto slot_of = [&](int kk) { return (uint32_t)(kk - kstart) & (kESlots - 1); };
  auto parity_of = [&](int kk) { return (unsigned)((uint32_t)(kk - kstart) >> 2) & 1u; };
  // double offset of row w (r = 0) / w+1 (r = 1) of plane kk: slot + phase
  auto ubase = [&](int kk, int r) -> int {
    return (int)slot_of(kk) * kSlotD + (int)((r ? uph1 : uph0) ^ ((uint32_t)kk & p1));
  };
  auto wword = [&](int kk, int r, int idx) -> uint32_t {
    const int wb = (int)slot_of(kk) * kSlotW + (w + r) * kEWSlot +
                   (int)(((r ? wph1 : wph0) + (uint32_t)kk * p3) & 3u);
    return W[wb + idx];
  };

  // stage rows w (and w+1 for the top warp) of plane kk: lane 0 issues bulk
  // copies; windows at either end of the array (only possible on planes 0 and
  // nz) take a checked path with plain loads when a copy would leave the array
  auto issue = [&](int kk) {
    if (kk > kend) return;
    const uint32_t slot = slot_of(kk);
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      if (rr == 1 && !top) break;
      const int64_t n0 = (int64_t)kk * plane + (rr ? rn1 : rn0);
      const char *us = reinterpret_cast<const char *>(src + n0 * 3);
      const char *ua = reinterpret_cast<const char *>(reinterpret_cast<uintptr_t>(us) & ~(uintptr_t)15);
      const unsigned ubytes = (unsigned)(((us - ua) + nwin * 24 + 15) & ~15);
      const char *ws = reinterpret_cast<const char *>(a.words + n0);
      const char *wa = reinterpret_cast<const char *>(reinterpret_cast<uintptr_t>(ws) & ~(uintptr_t)15);
      const unsigned wbytes = (unsigned)(((ws - wa) + nwin * 4 + 15) & ~15);
      double *ud = S.u[slot][w + rr];
      uint32_t *wd = S.wd[slot][w + rr];
      bool bulk = true;
      if (kk == 0 || kk == nz) {
        const char *xlo = reinterpret_cast<const char *>(a.x);
        const char *xhi = reinterpret_cast<const char *>(a.x + (size_t)nk * (size_t)nn * 3);
        const char *wlo = reinterpret_cast<const char *>(a.words);
        const char *whi = reinterpret_cast<const char *>(a.words + nn);
        bulk = ua >= xlo && ua + ubytes <= xhi && wa >= wlo && wa + wbytes <= whi;
      }
      if (bulk) {
        if (lane == 0) {
          fence_proxy_async_smem();
          mbar_arrive_tx(&S.bar[slot], ubytes + wbytes);
          bulk_g2s(ud, ua, ubytes, &S.bar[slot]);
          bulk_g2s(wd, wa, wbytes, &S.bar[slot]);
        }
      } else {
        const int uph = (int)((us - ua) >> 3), wph = (int)((ws - wa) >> 2);
        const double *u0 = reinterpret_cast<const double *>(us);
        const uint32_t *w0 = reinterpret_cast<const uint32_t *>(ws);
        for (int c = lane; c < nwin * 3; c += 32) ud[uph + c] = __ldg(u0 + c);
        for (int c = lane; c < nwin; c += 32) wd[wph + c] = __ldg(w0 + c);
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.bar[slot]);
      }
    }
  };
  // wait for plane kk and zero its Dirichlet-masked inputs in this warp's row(s)
  auto land = [&](int kk) {
    if (kk > kend) return;
    mbar_wait(&S.bar[slot_of(kk)], parity_of(kk));
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      if (rr == 1 && !top) break;
      const uint32_t m = (wword(kk, rr, iw) >> 19) & 7u;
      const uint32_t mr = lane == 31 ? ((wword(kk, rr, iwr) >> 19) & 7u) : 0u;
      if (__any_sync(0xffffffffu, (m | mr) != 0u)) {
        double *ur = const_cast<double *>(U) + ubase(kk, rr);
        const int oo = rr ? o10 : o00, orr = rr ? o11 : o01;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          if ((m >> q) & 1u) ur[oo + q] = 0.0;
          if ((mr >> q) & 1u) ur[orr + q] = 0.0;
        }
      }
      __syncwarp();
    }
  };

  // Carried between steps in shared memory (everything else is re-read
  // from the staged planes): this node's x/y-edge flux sums from the cell
  // below (ax, ay) and the z-edge flux of the node below (azb).
  auto CAX = [&](int q) -> double & { return S.carry[q][threadIdx.x]; };
  auto CAY = [&](int q) -> double & { return S.carry[3 + q][threadIdx.x]; };
  auto CAZ = [&](int q) -> double & { return S.carry[6 + q][threadIdx.x]; };
  double part[NPA];
#pragma unroll
  for (int t = 0; t < NPA; ++t) part[t] = 0.0;

  // y(kk) of this node: raw input for masked dofs, the operator elsewhere
  auto emit = [&](int kk, uint32_t wv, const double *own_in, const double *yv) {
    const int64_t node = (int64_t)kk * plane + own_node;
    const uint32_t m = (wv >> 19) & 7u;
    double raw[3] = {own_in[0], own_in[1], own_in[2]};
    if (m) {  // zeroed in the stage: the raw input from memory
#pragma unroll
      for (int q = 0; q < 3; ++q)
        if ((m >> q) & 1u) raw[q] = __ldg(a.x + voff + node * 3 + q);
    }
    double out[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) out[q] = ((m >> q) & 1u) ? raw[q] : yv[q];
    double *yo = a.y + voff + node * 3;
    if constexpr (ACT == APPLY) {
#pragma unroll
      for (int q = 0; q < 3; ++q) yo[q] = out[q];
    } else if constexpr (ACT == PCGQ) {
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        yo[q] = out[q];
        part[0] += raw[q] * out[q];
      }
    } else {  // RESID
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const double bv = __ldg(a.b + voff + node * 3 + q);
        const double dg = __ldg(a.dinv + node * 3 + q);
        const double r = bv - out[q];
        yo[q] = r;
        part[0] += bv * bv;
        part[1] += r * r;
        part[2] += r * (r * dg);
      }
    }
  };

  const int wm1 = w > 0 ? w - 1 : 0;  // warp 0 (halo row, never emits) reads its own slot

  // One step: cell kc between planes kc and kc+1 (both staged); emits plane kc.
  // One barrier.
  auto step = [&](int kc) {
    issue(kc + 3);
    const double *c0 = U + ubase(kc, 0), *c1 = U + ubase(kc, 1);
    const double *n0 = U + ubase(kc + 1, 0), *n1 = U + ubase(kc + 1, 1);
    const uint32_t wv = node_ok ? wword(kc, 0, iw) : 0u;
    const uint32_t nb = ElastC::valid(wv) ? wv : 0x3ffffu;  // no cell: every tet reads entry 7 (zero)
    auto T = [&](int m) -> const ETab & { return S.tab[(nb >> (3 * m)) & 7u]; };
    // Tets in the cycle order m0 m1 m4 m5 m3 m2: consecutive tets share an
    // edge, so each edge difference is formed once and lives briefly (register
    // pressure); corners are read from the stage when first needed.
    auto ld = [&](const double *base, int o, double (&v)[3]) {
#pragma unroll
      for (int q = 0; q < 3; ++q) v[q] = base[o + q];
    };
    auto df = [&](const double (&p)[3], const double (&m)[3], double (&d)[3]) {
#pragma unroll
      for (int q = 0; q < 3; ++q) d[q] = p[q] - m[q];
    };
    double a0[3], a1[3], a3[3], b3[3];
    ld(c0, o00, a0); ld(c0, o01, a1); ld(c1, o11, a3); ld(n1, o11, b3);
    double own_in[3] = {a0[0], a0[1], a0[2]};
    double X00[3], Y10[3], Z11[3];
    df(a1, a0, X00); df(a3, a1, Y10); df(b3, a3, Z11);
    double s0[6], s1[6], s2[6], s3[6], s4[6], s5[6];
    kuhn_sigma(X00, Y10, Z11, T(0), s0);  // (x,y,z)
    double b1[3], Y11[3], Z10[3];
    ld(n0, o01, b1);
    df(b3, b1, Y11); df(b1, a1, Z10);
    kuhn_sigma(X00, Y11, Z10, T(1), s1);  // (x,z,y)
    double b0[3], X01[3], Z00[3];
    ld(n0, o00, b0);
    df(b1, b0, X01); df(b0, a0, Z00);
    kuhn_sigma(X01, Y11, Z00, T(4), s4);  // (z,x,y)
    double fy10[3], fz10[3], fy11[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      fy10[q] = __shfl_up_sync(0xffffffffu, fyc(s0, q), 1);
      fz10[q] = __shfl_up_sync(0xffffffffu, fzc(s1, q), 1);
      fy11[q] = __shfl_up_sync(0xffffffffu, fyc(s1, q) + fyc(s4, q), 1);
    }
    double b2[3], X11[3], Y01[3];
    ld(n1, o10, b2);
    df(b3, b2, X11); df(b2, b0, Y01);
    kuhn_sigma(X11, Y01, Z00, T(5), s5);  // (z,y,x)
    double a2[3], Y00[3], Z01[3];
    ld(c1, o10, a2);
    df(a2, a0, Y00); df(b2, a2, Z01);
    kuhn_sigma(X11, Y00, Z01, T(3), s3);  // (y,z,x)
    double X10[3];
    df(a3, a2, X10);
    kuhn_sigma(X10, Y00, Z11, T(2), s2);  // (y,x,z)
    const int par = kc & 1;
    double *xw = &S.xchg[par][w][0][0];
    const double *xr = &S.xchg[par][wm1][0][0];
    double ay[3], azp[3], axp[3], fz01[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      ay[q] = (CAY(q) + (fyc(s2, q) + fyc(s3, q))) + fy10[q];
      CAY(q) = fyc(s5, q) + fy11[q];
      azp[q] = (fzc(s4, q) + fzc(s5, q)) + fz10[q];
      axp[q] = CAX(q) + (fxc(s0, q) + fxc(s1, q));
      // FZ01 of this cell + FZ11 of the cell at i-1: both go to (i, j+1)
      fz01[q] = fzc(s3, q) + __shfl_up_sync(0xffffffffu, fzc(s0, q) + fzc(s2, q), 1);
    }
    if (!top) {
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        xw[q * 32 + lane] = fxc(s2, q);                     // FX10 -> row j+1, plane kc
        xw[(3 + q) * 32 + lane] = fxc(s3, q) + fxc(s5, q);  // FX11 -> row j+1, plane kc+1
        xw[(6 + q) * 32 + lane] = fz01[q];                  // FZ01 + FZ11(i-1) -> row j+1
        xw[(9 + q) * 32 + lane] = ay[q];                    // complete y-edge flux
      }
    }
    land(kc + 2);
    __syncthreads();
    double yv[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const double ax = axp[q] + xr[q * 32 + lane];
      CAX(q) = fxc(s4, q) + xr[(3 + q) * 32 + lane];
      const double az = azp[q] + xr[(6 + q) * 32 + lane];
      const double axl = __shfl_up_sync(0xffffffffu, ax, 1);
      yv[q] = ((axl - ax) + (xr[(9 + q) * 32 + lane] - ay[q])) + (CAZ(q) - az);
      CAZ(q) = az;
    }
    if (own && kc >= K0) emit(kc, wv, own_in, yv);
  };

  // prologue: planes kstart .. kstart+2 in flight, kstart and kstart+1 landed
  issue(kstart);
  issue(kstart + 1);
  issue(kstart + 2);
  land(kstart);
  land(kstart + 1);
#pragma unroll
  for (int q = 0; q < 3; ++q) CAX(q) = CAY(q) = CAZ(q) = 0.0;
  __syncthreads();

#pragma unroll 1
  for (int kc = kstart; kc < kend; ++kc) step(kc);

  if (K1 == nz + 1 && nz >= K0) {  // plane nz: no cell above, no z-edge above
    const int par = kend & 1;
    if (!top) {
#pragma unroll
      for (int q = 0; q < 3; ++q) S.xchg[par][w][9 + q][lane] = CAY(q);
    }
    __syncthreads();
    double yv[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const double axl = __shfl_up_sync(0xffffffffu, CAX(q), 1);
      yv[q] = ((axl - CAX(q)) + (S.xchg[par][wm1][9 + q][lane] - CAY(q))) + CAZ(q);
    }
    if (own) {
      const double *c0 = U + ubase(nz, 0);
      const double in[3] = {c0[o00], c0[o00 + 1], c0[o00 + 2]};
      emit(nz, wword(nz, 0, iw), in, yv);
    }
  }

  if constexpr (NP > 0) {
    const int nblk = gridDim.x * gridDim.y * nzseg;
    const int blk = ((int)zseg * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    double tot[NPA];
    const size_t pbase = (size_t)rhs * (size_t)nblk * NP;
    if (block_partial_and_total<NP, Traits<ACT>::MAXMASK>(part, a.partials + pbase, a.counters + rhs, blk,
                                                          nblk, S.scratch, tot)) {
      if (threadIdx.x == 0) finalize<ACT>(a, rhs, tot);
    }
  }
}

}  // namespace d3
}  // namespace lsg
