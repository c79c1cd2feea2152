// Lean z-marching stencil for the cubic-cell elasticity operator (ElastC):
// the cfg3 / cfg5 hot kernel (q = A p of the 3D PCG, and the standalone apply).
//
// Same decomposition, exchange pattern and summation order as march3s
// (march3s.cuh: CTA = kWarps node rows x 30 owned columns marching along z, so
// both kernels give bitwise-identical results), with the per-step overhead
// stripped:
//   * a 4-slot staging ring and a 4x unrolled step, so every shared-memory
//     address is `register + immediate` (slot, exchange parity and the
//     ping-pong plane states are compile-time);
//   * global addresses are per-thread pointers advanced by one plane per step
//     (no 64-bit index arithmetic in the loop);
//   * Dirichlet inputs are zeroed once in the staged plane by the warp that
//     staged the row (a branch only Dirichlet nodes take), so all four in-plane
//     corner columns are plain 64-bit shared loads: no input shuffles, no
//     selects; a masked output dof re-reads its input from memory (rare);
//   * planes are prefetched three steps ahead.
// Reference operation: fem.py:397-411 (elasticity form) with fem.py:274-291
// (Dirichlet elimination) applied matrix-free.
#pragma once

#include <type_traits>

namespace lsg {
namespace d3 {
namespace e3 {
#ifndef LSG_M3E_RELOAD
#define LSG_M3E_RELOAD 0
#endif
#ifndef LSG_M3E_TAB2
#define LSG_M3E_TAB2 1
#endif
#ifndef LSG_M3E_MINB
#define LSG_M3E_MINB 2
#endif

constexpr int kSlots = 4;
constexpr int kRowB = 800;  // staged row: 50 chunks of 16 bytes (33 nodes of 24 bytes + 8 phase)
constexpr int kRows = kWarps + 1;
constexpr int kSlotB = kRows * kRowB;
constexpr int kWordRowB = 128;
constexpr int kWSlotB = kRows * kWordRowB;
constexpr int kWordOff = kSlots * kSlotB;
constexpr int kXchgParB = kWarps * 6 * 32 * 8;  // [warp][6][32] doubles per parity
constexpr int kXchgOff = kWordOff + kSlots * kWSlotB;
constexpr int kBytes = kXchgOff + 2 * kXchgParB;
constexpr uint32_t kDir = 7u << 19;  // Dirichlet bits of the material word

// 16-byte async copy of which only the first `nbytes` (0..16) are read from
// memory; the rest of the chunk is zero-filled
__device__ __forceinline__ void cp_async16_part(void *smem_dst, const void *gmem, int nbytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gmem), "r"(nbytes));
}

// shared-memory load the compiler may not repeat (it otherwise re-reads the
// previous plane from the ring instead of keeping it in registers: 12 more
// 64-bit shared loads per step on a kernel whose shared-memory pipe is loaded)
__device__ __forceinline__ double lds_once(const unsigned char *p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}

struct PS {
  double in[3], rt[3], iy[3], iyr[3];
  uint32_t wc;
};

}  // namespace e3

template <int ACT>
__global__ void __launch_bounds__(kThreads, LSG_M3E_MINB) march3e(ElastC ph, Geo g, MArgs a) {
  using namespace e3;
  static_assert(ACT == APPLY || ACT == PCGQ, "march3e: apply and PCG stencil only");
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double scratch[kWarps];
#if LSG_M3E_TAB2
  __shared__ double2 wtab[8];
#else
  __shared__ double wtab[24];
#endif
  if constexpr (ACT == PCGQ) pdl_wait();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nzseg = a.nzseg;
  const int zseg = blockIdx.z % nzseg, rhs = blockIdx.z / nzseg;
  if constexpr (ACT == PCGQ) {
    if (a.scal[rhs].done != 0.0) return;
  }
#if LSG_M3E_TAB2
  ph.fill_table2(wtab, threadIdx.x);
#else
  ph.fill_table(wtab, threadIdx.x);
#endif
  // finite contents everywhere a halo lane may read before (or beyond what) a copy lands
  for (int o = threadIdx.x * 16; o < kXchgOff; o += kThreads * 16)
    *reinterpret_cast<int4 *>(smem + o) = make_int4(0, 0, 0, 0);

  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const int nxp = nx + 1;
  const int64_t plane = (int64_t)nxp * (ny + 1);
  const int64_t nn = plane * (nz + 1);
  const int i = (int)blockIdx.x * kStrip - 1 + lane;
  const int jw = (int)blockIdx.y * (kWarps - 1) - 1 + w;
  const bool top = (w == kWarps - 1);
  const bool node_ok = i >= 0 && i <= nx && jw >= 0 && jw <= ny;
  const bool own = node_ok && lane >= 1 && lane <= kStrip && w >= 1;
  const int ic = min(max(i, 0), nx);
  const int jc = min(max(jw, 0), ny), jxc = min(max(jw + 1, 0), ny);
  const int K0 = zseg * a.seg;
  const int K1 = min(K0 + a.seg, nz + 1);
  const int kstart = max(K0 - 1, 0);
  const int kend = min(K1, nz);
  const int lo = min(max((int)blockIdx.x * kStrip - 1, 0), nx);
  const int li = ic - lo;
  // planes below this one may be staged with whole 16-byte chunks (the
  // over-read stays inside the array); the array's last plane is staged exactly
  const int kfast = plane >= 40 ? nz : -1;

  const size_t voff = (size_t)rhs * (size_t)nn * 3;
  const char *src = reinterpret_cast<const char *>(a.x + voff);
  const char *srcE = src + (size_t)nn * 24;
  const int64_t planeB = plane * 24;
  const int64_t row0 = ((int64_t)kstart * plane + (int64_t)jc * nxp + lo) * 24;  // own row, plane kstart
  const int64_t upB = (int64_t)(jxc - jc) * nxp * 24;                             // row above (0 when clamped)
  const char *sl = src + row0 + 16 * lane;                                        // this lane's chunk, issue plane
  const uint32_t *wl = a.words + ((int64_t)kstart * plane + (int64_t)jc * nxp + ic);
  const int64_t wup = (int64_t)(jxc - jc) * nxp;
  double *yp = a.y + voff + ((int64_t)kstart * plane + (int64_t)jc * nxp + ic) * 3;  // emission plane

  // shared-memory byte offsets (slot / parity / component added as immediates)
  const uint32_t c_own = (uint32_t)(w * kRowB + li * 24);
  const uint32_t xup8 = (uint32_t)(upB & 8);
  const uint32_t pxor = (uint32_t)(planeB & 8);
  uint32_t phc = (uint32_t)(reinterpret_cast<uintptr_t>(src + row0) & 8);  // phase of the plane read next
  const uint32_t sdst = (uint32_t)(w * kRowB + 16 * lane);
  const uint32_t swd = (uint32_t)(kWordOff + w * kWordRowB + 4 * lane);
  const int wm1 = w > 0 ? w - 1 : 0;  // warp 0 (halo row, never emits) reads its own slot
  const uint32_t sc_wr = (uint32_t)(kXchgOff + (w * 3 * 32 + lane) * 16);
  const uint32_t sc_rd = (uint32_t)(kXchgOff + (wm1 * 3 * 32 + lane) * 16);

  double part = 0.0;
  int kiss = kstart;  // next plane to stage

  auto issue = [&](auto slot_tag) {
    constexpr int SLOT = decltype(slot_tag)::value;
    if (kiss <= kend) {
      unsigned char *dw = smem + (swd + SLOT * kWSlotB);
      unsigned char *dd = smem + (sdst + SLOT * kSlotB);
      cp_async4(dw, wl);
      if (top) cp_async4(dw + kWordRowB, wl + wup);
      if (kiss < kfast) {
        const char *A = reinterpret_cast<const char *>(reinterpret_cast<uintptr_t>(sl) & ~(uintptr_t)15);
        cp_async16(dd, A);
        if (lane < kRowB / 16 - 32) cp_async16(dd + 512, A + 512);
        if (top) {
          const char *B = reinterpret_cast<const char *>(reinterpret_cast<uintptr_t>(sl + upB) & ~(uintptr_t)15);
          cp_async16(dd + kRowB, B);
          if (lane < kRowB / 16 - 32) cp_async16(dd + kRowB + 512, B + 512);
        }
      } else {  // the array's last plane: never read past its end
        const char *A = reinterpret_cast<const char *>(reinterpret_cast<uintptr_t>(sl) & ~(uintptr_t)15);
        auto left = [&](const char *p) { return (int)min((int64_t)16, max((int64_t)0, (int64_t)(srcE - p))); };
        cp_async16_part(dd, A, left(A));
        if (lane < kRowB / 16 - 32) cp_async16_part(dd + 512, A + 512, left(A + 512));
        if (top) {
          const char *B = reinterpret_cast<const char *>(reinterpret_cast<uintptr_t>(sl + upB) & ~(uintptr_t)15);
          cp_async16_part(dd + kRowB, B, left(B));
          if (lane < kRowB / 16 - 32) cp_async16_part(dd + kRowB + 512, B + 512, left(B + 512));
        }
      }
    }
    sl += planeB;
    wl += plane;
    ++kiss;
    cp_async_commit();
  };

  // After this thread's copies of the plane in SLOT have landed: zero the
  // Dirichlet inputs of the row(s) this warp staged (phase php) and return the
  // material word of the own node.
  auto mask_plane = [&](auto slot_tag, uint32_t php) -> uint32_t {
    constexpr int SLOT = decltype(slot_tag)::value;
    __syncwarp();
    const uint32_t wd = *reinterpret_cast<const uint32_t *>(smem + (swd + SLOT * kWSlotB));
    if (wd & kDir) {
      double *p = reinterpret_cast<double *>(smem + (c_own + SLOT * kSlotB + php));
#pragma unroll
      for (int q = 0; q < 3; ++q)
        if ((wd >> (19 + q)) & 1u) p[q] = 0.0;
    }
    if (top) {
      const uint32_t wu = *reinterpret_cast<const uint32_t *>(smem + (swd + kWordRowB + SLOT * kWSlotB));
      if (wu & kDir) {
        double *p = reinterpret_cast<double *>(smem + (c_own + kRowB + SLOT * kSlotB + (php ^ xup8)));
#pragma unroll
        for (int q = 0; q < 3; ++q)
          if ((wu >> (19 + q)) & 1u) p[q] = 0.0;
      }
    }
    return node_ok ? wd : 0u;
  };

  auto load_plane = [&](auto slot_tag, PS &s) {
    constexpr int SLOT = decltype(slot_tag)::value;
    const unsigned char *ro = smem + (c_own + SLOT * kSlotB + phc);
    const unsigned char *ru = smem + (c_own + kRowB + SLOT * kSlotB + (phc ^ xup8));
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      s.in[q] = lds_once(ro + 8 * q);
      s.rt[q] = lds_once(ro + 24 + 8 * q);
      s.iy[q] = lds_once(ru + 8 * q);
      s.iyr[q] = lds_once(ru + 24 + 8 * q);
    }
    phc ^= pxor;
  };

  // writes plane (pointed to by yp) from acc; a Dirichlet dof returns its input
  auto emit = [&](const PS &s, const double *acc) {
    double yv[3] = {acc[0], acc[1], acc[2]};
    if (s.wc & kDir) {
      const double *xr = reinterpret_cast<const double *>(src) + (yp - (a.y + voff));
#pragma unroll
      for (int q = 0; q < 3; ++q)
        if ((s.wc >> (19 + q)) & 1u) {
          yv[q] = __ldg(xr + q);
          if constexpr (ACT == PCGQ) part = fma(yv[q], yv[q], part);
        }
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      yp[q] = yv[q];
      if constexpr (ACT == PCGQ) part = fma(s.in[q], yv[q], part);
    }
  };

  // One step: cells of layer kk-1 from planes kk-1 (c, registers) and kk (n,
  // read from SLOT); emits plane kk-1.  Lane 0 and warp 0 are halo: their sums
  // are never emitted.  One barrier per plane publishes the y-contributions
  // (exchange double-buffered by parity) and the staged, masked plane kk+1.
  auto step = [&](auto slot_tag, int kk, PS &c, PS &n, double *acc_c, double *acc_n) {
    constexpr int SLOT = decltype(slot_tag)::value;
    constexpr int PAR = SLOT & 1;
#if LSG_M3E_RELOAD
    issue(std::integral_constant<int, (SLOT + 2) & 3>{});  // slot of plane kk-2: read before the last barrier
    phc ^= pxor;  // back to plane kk-1
    load_plane(std::integral_constant<int, (SLOT + 3) & 3>{}, c);
#else
    issue(std::integral_constant<int, (SLOT + 3) & 3>{});  // slot of plane kk-1: read before the last barrier
#endif
    load_plane(slot_tag, n);
    double U[8][3];
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      U[0][t] = c.in[t];  U[1][t] = c.rt[t];  U[2][t] = c.iy[t];  U[3][t] = c.iyr[t];
      U[4][t] = n.in[t];  U[5][t] = n.rt[t];  U[6][t] = n.iy[t];  U[7][t] = n.iyr[t];
    }
    double C[8][3];
    ph.cell_prog(U, c.wc, C, wtab);
    double T[4][3];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int t = 0; t < 3; ++t) T[q][t] = C[2 * q][t] + __shfl_up_sync(0xffffffffu, C[2 * q + 1][t], 1);
    {
      double2 *sc = reinterpret_cast<double2 *>(smem + (sc_wr + PAR * kXchgParB));
      sc[0] = make_double2(T[1][0], T[1][1]);
      sc[32] = make_double2(T[1][2], T[3][0]);
      sc[64] = make_double2(T[3][1], T[3][2]);
    }
    uint32_t wnext = 0u;
    cp_async_wait<LSG_M3E_RELOAD ? 1 : 2>();  // plane kk+1 has landed (later planes may still be in flight)
    if (kk < kend) wnext = mask_plane(std::integral_constant<int, (SLOT + 1) & 3>{}, phc);
    __syncthreads();
    {
      const double2 *sc = reinterpret_cast<const double2 *>(smem + (sc_rd + PAR * kXchgParB));
      const double2 v0 = sc[0], v1 = sc[32], v2 = sc[64];
      acc_c[0] += T[0][0] + v0.x;
      acc_c[1] += T[0][1] + v0.y;
      acc_c[2] += T[0][2] + v1.x;
      acc_n[0] = T[2][0] + v1.y;
      acc_n[1] = T[2][1] + v2.x;
      acc_n[2] = T[2][2] + v2.y;
    }
    if (own && kk > K0) emit(c, acc_c);
    yp += plane * 3;
    c.wc = wnext;  // c becomes the state of plane kk+1
  };

  using S0 = std::integral_constant<int, 0>;
  using S1 = std::integral_constant<int, 1>;
  using S2 = std::integral_constant<int, 2>;
  using S3 = std::integral_constant<int, 3>;

  PS P0, P1;
  double acc0[3] = {0.0, 0.0, 0.0}, acc1[3];
  __syncthreads();  // table and zero fill
  issue(S0{});
  issue(S1{});
  issue(S2{});
  if (!LSG_M3E_RELOAD) issue(S3{});
  cp_async_wait<LSG_M3E_RELOAD ? 2 : 3>();
  P0.wc = mask_plane(S0{}, phc);
  __syncthreads();
  load_plane(S0{}, P0);
  cp_async_wait<LSG_M3E_RELOAD ? 1 : 2>();
  P1.wc = (kstart < kend) ? mask_plane(S1{}, phc) : 0u;
  __syncthreads();

  // four steps per trip: slots, exchange parity and the roles of the two plane
  // states are compile-time
  bool last_in_1 = false;
  for (int kk = kstart + 1; kk <= kend; kk += 4) {
    step(S1{}, kk, P0, P1, acc0, acc1);
    if (kk == kend) { last_in_1 = true; break; }
    step(S2{}, kk + 1, P1, P0, acc1, acc0);
    if (kk + 1 == kend) break;
    step(S3{}, kk + 2, P0, P1, acc0, acc1);
    if (kk + 2 == kend) { last_in_1 = true; break; }
    step(S0{}, kk + 3, P1, P0, acc1, acc0);
  }
  cp_async_wait<0>();
  if (K1 == nz + 1 && own && nz >= K0) {  // plane nz: the last state written
    if (last_in_1) emit(P1, acc1);
    else emit(P0, acc0);
  }

  if constexpr (ACT == PCGQ) {
    const int nblk = gridDim.x * gridDim.y * nzseg;
    const int blk = ((int)zseg * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    double pv[1] = {part}, tot[1];
    const size_t pbase = (size_t)rhs * (size_t)nblk;
    if (block_partial_and_total<1, 0u>(pv, a.partials + pbase, a.counters + rhs, blk, nblk, scratch, tot)) {
      if (threadIdx.x == 0) finalize<ACT>(a, rhs, tot);
    }
  }
}

}  // namespace d3
}  // namespace lsg
