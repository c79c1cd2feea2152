// 3D z-marching kernel with an asynchronous shared-memory staging pipeline.
//
// Same decomposition as described in ops3d.cu (CTA = 8 warps = 8 node rows
// incl. one halo row, 30 owned columns per warp, marching along z).  The
// global loads of planes k+1 and k+2 are in flight as 16-byte cp.async
// (LDGSTS) copies into a 3-slot ring while plane k is computed, so no
// registers are spent on prefetching and no warp waits on a load it issued in
// the same step.  The row above (y+1) is read from the staged plane and its
// operator input recomputed locally; the only cross-warp exchange is the
// y-contribution hand-off, through a parity-double-buffered shared buffer:
// one barrier per plane.  Plane states ping-pong between two register sets.
#pragma once

namespace lsg {
namespace d3 {

// Node vectors are interleaved [node][3], so the 32 nodes of a warp row are
// one contiguous window of <= 768 bytes per source array.  It is staged
// verbatim with 16-byte copies into a 784-byte slot (the window starts 0 or 8
// bytes into its first 16-byte chunk); lanes then read their node at a
// 3-double stride (conflict-free for 64-bit shared loads).
// Source arrays per row: APPLY/STATS: input; RESID: x, dinv; PCGQ: p;
// SHAPE: KB states.
constexpr int kRowSlot = 98;  // doubles: 49 chunks of 16 bytes

template <class PH, int ACT>
struct Stage {
  static constexpr int NS = (ACT == RESID) ? 2 : PH::NIN / 3;  // APPLY/PCGQ/STATS: 1
  static constexpr int NOUT = PH::NOUT;
  static constexpr size_t doubles = (size_t)3 * (kWarps + 1) * NS * kRowSlot;
  static constexpr size_t words = (size_t)3 * (kWarps + 1) * 32;
  static constexpr size_t xchg = (size_t)2 * kWarps * 2 * NOUT * 32;  // double-buffered
  static constexpr size_t bytes = doubles * 8 + xchg * 8 + words * 4;
};

#ifndef LSG_M3_MINB
#define LSG_M3_MINB 2
#endif

template <class PH, int ACT>
__global__ void __launch_bounds__(kThreads, LSG_M3_MINB) march3s(PH ph, Geo g, MArgs a) {
  constexpr int NIN = PH::NIN, NOUT = PH::NOUT;
  constexpr int NP = Traits<ACT>::NP;
  constexpr int NPA = NP > 0 ? NP : 1;
  constexpr int NS = Stage<PH, ACT>::NS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *stage = reinterpret_cast<double *>(smem_raw);               // [3][kWarps+1][NS][kRowSlot]
  double *xchg = stage + Stage<PH, ACT>::doubles;                      // [2][kWarps][2*NOUT][32]
  uint32_t *stw = reinterpret_cast<uint32_t *>(xchg + Stage<PH, ACT>::xchg);  // [3][kWarps+1][32]
  __shared__ double scratch[NPA * kWarps];
  __shared__ double wtab[24];  // per-tet weights (physics with kTable)
  if constexpr (ACT == PCGQ) pdl_wait();  // launched with launch_pdl (see common.cuh)
  if constexpr (PH::kTable) ph.fill_table(wtab, threadIdx.x);
  auto SR = [&](int slot, int row, int s) -> double * {
    return stage + (((size_t)slot * (kWarps + 1) + row) * NS + s) * kRowSlot;
  };
  auto SW = [&](int slot, int row, int l) -> uint32_t & {
    return stw[((size_t)slot * (kWarps + 1) + row) * 32 + l];
  };
  auto SC = [&](int par, int wr, int t, int l) -> double & {
    return xchg[(((size_t)par * kWarps + wr) * 2 * NOUT + t) * 32 + l];
  };

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nzseg = a.nzseg;
  const int zseg = blockIdx.z % nzseg, rhs = blockIdx.z / nzseg;
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const int64_t nxp = nx + 1, nyp = ny + 1;
  const int64_t plane = nxp * nyp;
  const int64_t nn = plane * (nz + 1);

  const int i = (int)blockIdx.x * kStrip - 1 + lane;
  const int jw = (int)blockIdx.y * (kWarps - 1) - 1 + w;
  const int jx = jw + 1;
  const bool top = (w == kWarps - 1);
  const bool col_ok = ((int)blockIdx.x < a.nstrips) && i >= 0 && i <= nx;
  const bool node_ok = col_ok && jw >= 0 && jw <= ny;
  const bool up_ok = col_ok && jx >= 0 && jx <= ny;  // the row above exists
  const bool own = node_ok && lane >= 1 && lane <= kStrip && w >= 1;
  const int ic = min(max(i, 0), nx);
  const int jc = min(max(jw, 0), ny), jxc = min(max(jx, 0), ny);
  const int K0 = zseg * a.seg;
  const int K1 = min(K0 + a.seg, nz + 1);
  const size_t voff = (ACT == SHAPE) ? 0 : (size_t)rhs * (size_t)nn * 3;

  if constexpr (ACT == RESID || ACT == PCGQ) {
    if (a.scal[rhs].done != 0.0) return;
  }

  double part[NPA];
#pragma unroll
  for (int t = 0; t < NPA; ++t) part[t] = 0.0;

  const int kstart = max(K0 - 1, 0);
  const int kend = min(K1, nz);

  // source arrays staged per row
  const double *src[NS];
  if constexpr (ACT == RESID) {
    src[0] = a.x + voff; src[1] = a.dinv;
  } else if constexpr (ACT == SHAPE) {
#pragma unroll
    for (int f = 0; f < NS; ++f) src[f] = a.x + (size_t)f * nn * 3;
  } else {
    src[0] = a.x + voff;
  }
  // 8-byte phase of each base pointer: node n of array s starts at an odd
  // multiple of 8 bytes iff bit s of spm differs from the parity of n
  uint32_t spm = 0;
#pragma unroll
  for (int s = 0; s < NS; ++s) spm |= (uint32_t)((reinterpret_cast<uintptr_t>(src[s]) >> 3) & 1u) << s;
  // column window of this strip: nodes lo..hi (clamped); lane reads node ic
  const int lo = min(max((int)blockIdx.x * kStrip - 1, 0), nx);
  const int hi = min(max((int)blockIdx.x * kStrip + kStrip, 0), nx);
  const int li3 = (ic - lo) * 3;
  const int wbytes = (hi - lo + 1) * 24;
  const int64_t rown = (int64_t)jc * nxp + lo, rowu = (int64_t)jxc * nxp + lo;
  const int64_t node_in_plane = (int64_t)jw * nxp + i;  // this lane's node within a plane

  // stage the window of node row n0.. (one plane) into ring slot `slot`
  auto stage_row = [&](int64_t n0, int slot, int srow) {
    cp_async4(&SW(slot, srow, lane), a.words + n0 + (ic - lo));
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const char *S = reinterpret_cast<const char *>(src[s] + n0 * 3);
      const char *A = reinterpret_cast<const char *>(reinterpret_cast<uintptr_t>(S) & ~(uintptr_t)15);
      char *dst = reinterpret_cast<char *>(SR(slot, srow, s));
      if (A + 16 * (kRowSlot / 2) <= reinterpret_cast<const char *>(src[s] + nn * 3)) {
        // 49 chunks cover the window whatever its phase (it may over-read
        // up to 16 bytes past the window, never past the array)
        cp_async16(dst + 16 * lane, A + 16 * lane);
        if (lane < kRowSlot / 2 - 32) cp_async16(dst + 512 + 16 * lane, A + 512 + 16 * lane);
      } else {  // the array's last row: exact chunks
        const char *E = S + wbytes;
        for (int c = lane; c < kRowSlot / 2; c += 32) {
          const char *gp = A + 16 * c;
          if (gp < E) {
            if (gp < S) cp_async8(dst + 16 * c + 8, gp + 8);
            else if (gp + 16 > E) cp_async8(dst + 16 * c, gp);
            else cp_async16(dst + 16 * c, gp);
          }
        }
      }
    }
  };
  auto issue = [&](int kk, int slot) {
    if (kk <= kend) {
      const int64_t kp = (int64_t)kk * plane;
      stage_row(kp + rown, slot, w);
      if (top) stage_row(kp + rowu, slot, w + 1);
    }
    cp_async_commit();
  };

  // operator input (masked), raw value, inverse diagonal of a staged row
  auto prepare = [&](int kk, int slot, int srow, int64_t rowoff, bool ok, bool write_own, double *in,
                     double *raw, double *dg, uint32_t &wc) {
    wc = ok ? SW(slot, srow, lane) : 0u;
    const uint32_t ph = ((uint32_t)kk & (uint32_t)plane & 1u) ^ ((uint32_t)rowoff & 1u);
    auto V = [&](int s, int q) -> double {
      return SR(slot, srow, s)[(int)(ph ^ ((spm >> s) & 1u)) + li3 + q];
    };
    if constexpr (ACT == SHAPE) {
#pragma unroll
      for (int t = 0; t < NIN; ++t) in[t] = V(t / 3, t % 3);
    } else {
      const uint32_t m = PH::mask(wc);
      double v[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) v[q] = V(0, q);
      if constexpr (ACT == RESID) {
#pragma unroll
        for (int q = 0; q < 3; ++q) dg[q] = V(1, q);
      }
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        raw[q] = v[q];
        in[q] = ((m >> q) & 1u) ? 0.0 : v[q];
      }
    }
  };

  auto emit = [&](int kk, uint32_t wc, const double *accv, const double *raw, const double *dg) {
    const int64_t node = (int64_t)kk * plane + node_in_plane;
    if constexpr (ACT == SHAPE) {
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        double o = accv[q];
        if (a.accumulate) o += a.y[node * 3 + q];
        a.y[node * 3 + q] = o;
        if (!a.accumulate) a.y2[node * 3 + q] = accv[3 + q];
      }
    } else {
      const uint32_t m = PH::mask(wc);
      double yv[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) yv[q] = ((m >> q) & 1u) ? raw[q] : accv[q];
      if constexpr (ACT == APPLY) {
#pragma unroll
        for (int q = 0; q < 3; ++q) __stcs(a.y + voff + node * 3 + q, yv[q]);  // not re-read here: keep x in L2
      } else if constexpr (ACT == RESID) {
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const double bv = __ldg(a.b + voff + node * 3 + q);
          const double r = bv - yv[q];
          a.y[voff + node * 3 + q] = r;
          part[0] += bv * bv;
          part[1] += r * r;
          part[2] += r * (r * dg[q]);
        }
      } else if constexpr (ACT == PCGQ) {
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          a.y[voff + node * 3 + q] = yv[q];
          part[0] += raw[q] * yv[q];
        }
      } else if constexpr (ACT == STATS) {
        double sp = 0.0;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const double vv = __ldg(a.x2 + node * 3 + q);
          part[0] += raw[q] * yv[q];
          part[1] += vv * raw[q];
          sp += fabs(raw[q]) * g.ih[q];
        }
        part[2] = fmax(part[2], sp);
      }
    }
  };

  // Marching state of one plane: own-row input, its x-neighbour (lane+1),
  // the row above and its x-neighbour; raw values / inverse diagonal / word
  // for the emission of this plane's node.
  struct PlaneState {
    double in[NIN], rt[NIN], iy[NIN], iyr[NIN], raw[3], dg[3];
    uint32_t wc;
  };
  auto load_plane = [&](int kk, int slot, bool write_own, PlaneState &s) {
    double raw_t[3], dg_t[3];
    uint32_t wt;
    prepare(kk, slot, w, rown, node_ok, write_own, s.in, s.raw, s.dg, s.wc);
    prepare(kk, slot, w + 1, rowu, up_ok, false, s.iy, raw_t, dg_t, wt);
#pragma unroll
    for (int t = 0; t < NIN; ++t) {
      s.rt[t] = __shfl_down_sync(0xffffffffu, s.in[t], 1);
      s.iyr[t] = __shfl_down_sync(0xffffffffu, s.iy[t], 1);
    }
  };
  const int wm1 = w > 0 ? w - 1 : 0;  // warp 0 (halo row, never emits) reads its own slot

  // One step: cells (., ., kk-1) from planes kk-1 (c) and kk (n); emits plane
  // kk-1.  Lane 0 and warp 0 are halo: their sums are never emitted, so the
  // shuffle / exchange edges need no zero-fill.  One barrier per plane: it
  // publishes this step's y-contributions (exchange double-buffered by
  // parity) and the staged plane kk+1.
  auto step = [&](int kk, int sl, int sl2, PlaneState &c, PlaneState &n, double *acc_c,
                  double *acc_n) {
    issue(kk + 2, sl2);  // slot of plane kk-1, fully read before the last barrier
    load_plane(kk, sl, own && kk >= K0 && kk < K1, n);
    double U[8][NIN];
#pragma unroll
    for (int t = 0; t < NIN; ++t) {
      U[0][t] = c.in[t];  U[1][t] = c.rt[t];  U[2][t] = c.iy[t];  U[3][t] = c.iyr[t];
      U[4][t] = n.in[t];  U[5][t] = n.rt[t];  U[6][t] = n.iy[t];  U[7][t] = n.iyr[t];
    }
    double C[8][NOUT];
    if constexpr (ACT == SHAPE) {
      ph.cell(U, c.wc, own && (kk - 1) >= K0, C, part);
    } else {
      if constexpr (PH::kTable) ph.cell(U, c.wc, i, jw, kk - 1, C, wtab);
      else ph.cell(U, c.wc, i, jw, kk - 1, C);
    }
    double T[4][NOUT];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int t = 0; t < NOUT; ++t) T[q][t] = C[2 * q][t] + __shfl_up_sync(0xffffffffu, C[2 * q + 1][t], 1);
    const int par = kk & 1;
#pragma unroll
    for (int t = 0; t < NOUT; ++t) {
      SC(par, w, t, lane) = T[1][t];
      SC(par, w, NOUT + t, lane) = T[3][t];
    }
    cp_async_wait<1>();  // plane kk+1 has landed (kk+2 may still be in flight)
    __syncthreads();
#pragma unroll
    for (int t = 0; t < NOUT; ++t) {
      acc_c[t] += T[0][t] + SC(par, wm1, t, lane);
      acc_n[t] = T[2][t] + SC(par, wm1, NOUT + t, lane);
    }
    if (own && (kk - 1) >= K0) emit(kk - 1, c.wc, acc_c, c.raw, c.dg);
  };

  PlaneState P0, P1;
  double acc0[NOUT], acc1[NOUT];
  auto nxt3 = [](int s) { return s == 2 ? 0 : s + 1; };
  int sl = kstart % 3;
  issue(kstart, sl);
  issue(kstart + 1, nxt3(sl));
  cp_async_wait<1>();
  __syncthreads();
  issue(kstart + 2, nxt3(nxt3(sl)));
  load_plane(kstart, sl, own && kstart >= K0, P0);
#pragma unroll
  for (int t = 0; t < NOUT; ++t) acc0[t] = 0.0;
  cp_async_wait<1>();  // plane kstart+1 has landed
  __syncthreads();     // ... for every thread

  // two steps per trip with the roles of the plane states swapped: no
  // register copies between steps
  bool last_in_1 = false;
  for (int kk = kstart + 1; kk <= kend; kk += 2) {
    sl = nxt3(sl);  // slot of plane kk
    step(kk, sl, nxt3(nxt3(sl)), P0, P1, acc0, acc1);
    if (kk == kend) { last_in_1 = true; break; }
    sl = nxt3(sl);
    step(kk + 1, sl, nxt3(nxt3(sl)), P1, P0, acc1, acc0);
  }
  cp_async_wait<0>();
  if (K1 == nz + 1 && own && nz >= K0) {  // plane nz: the last state written
    if (last_in_1) emit(nz, P1.wc, acc1, P1.raw, P1.dg);
    else emit(nz, P0.wc, acc0, P0.raw, P0.dg);
  }

  if constexpr (NP > 0) {
    const int nblk = gridDim.x * gridDim.y * nzseg;
    const int blk = ((int)zseg * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    double tot[NPA];
    const size_t pbase = (size_t)rhs * (size_t)nblk * NP;
    if (block_partial_and_total<NP, Traits<ACT>::MAXMASK>(part, a.partials + pbase,
                                                          a.counters + rhs, blk, nblk, scratch, tot)) {
      if (threadIdx.x == 0) finalize<ACT>(a, rhs, tot);
    }
  }
}

}  // namespace d3
}  // namespace lsg
