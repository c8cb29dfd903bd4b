// ATOMIC assembly (north_star (iii), the alternative to the TILED owner-
// computes gather): element loads scattered into a global nodal load array
// with warp-aggregated atomics, then a node-update kernel.  Two launches per
// step, no halo duplication, but the summation order of each node's load
// depends on atomic arrival order: results are repeatable only to rounding
// (tolerance-only, like the reference's fastmath-free numba path is not).
// Kept as the measured alternative of "deterministic CSR gather or
// warp-aggregated atomics, selected by measurement".
//
//   k_atomic_elem : one thread per element (elements sorted by their smallest
//                   new node id, so a warp touches neighbouring nodes): corner
//                   temperatures and k(T) gathered from HBM/L2, kbar_e, the
//                   G-form element load (A = D G D^T, as fh_tiled.cu), then per
//                   corner: lanes adding to the same node are grouped with
//                   __match_any_sync, the group's values are summed in lane
//                   order through shuffles and its lowest lane issues one
//                   red.global.add into F.
//   k_atomic_node : per node, T' = T + dt (F - kb T + qb + qm + q_ext + src
//                   [+ Robin]) / C (the TILED node law), F reset to 0 for the
//                   next step, runaway check.  Dirichlet nodes keep their values.
#include "fh_atomic.h"

namespace fh {

template <bool LIN, typename S>
__device__ __forceinline__ S ipa(const Curve<S> &c, S x) {
  if (!LIN) return interp(c, x);
  S r = c.slope[0] * (x - c.x[0]) + c.y[0];
  r = (x >= c.x[1]) ? c.y[1] : r;
  return (x <= c.x[0]) ? c.y[0] : r;
}

__device__ __forceinline__ float afast_exp(float x) { return __expf(x); }
__device__ __forceinline__ double afast_exp(double x) { return exp(x); }

// group-sum of v over the lanes holding the same key, added once by the group's lowest lane
template <typename S>
__device__ __forceinline__ void warp_aggregated_add(S *F, int key, S v) {
  const unsigned grp = __match_any_sync(0xffffffffu, key);
  S total = S(0);
  for (unsigned m = grp; m; m &= m - 1) total += __shfl_sync(grp, v, __ffs(m) - 1);
  if (key >= 0 && (int)(threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(F + key, total);
}

template <typename S, int N, bool LIN>
__global__ void __launch_bounds__(256) k_atomic_elem(const __grid_constant__ TiledArgs<S> g, const int32_t *__restrict__ conn,
                                                     const S *__restrict__ G, int64_t n, S *__restrict__ F) {
  if (g.flag->step < g.step_no) return;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool valid = i < n;
  const int64_t ii = valid ? i : n - 1;
  int nd[N];
  if (N == 8) {
    const int4 a = __ldg(reinterpret_cast<const int4 *>(conn + 8 * ii));
    const int4 b = __ldg(reinterpret_cast<const int4 *>(conn + 8 * ii) + 1);
    nd[0] = a.x; nd[1] = a.y; nd[2] = a.z; nd[3] = a.w;
    nd[4 % N] = b.x; nd[5 % N] = b.y; nd[6 % N] = b.z; nd[7 % N] = b.w;
  } else {
    const int4 a = __ldg(reinterpret_cast<const int4 *>(conn + 4 * ii));
    nd[0] = a.x; nd[1 % N] = a.y; nd[2 % N] = a.z; nd[3 % N] = a.w;
  }
  S T[N], K[N];
  const Curve<S> &kc = g.mats.m[0].k;
#pragma unroll
  for (int b = 0; b < N; ++b) {
    T[b] = __ldg(g.Tin + nd[b]);
    K[b] = ipa<LIN>(kc, T[b]);
  }
  const S g00 = __ldg(G + ii), g01 = __ldg(G + n + ii), g02 = __ldg(G + 2 * n + ii), g11 = __ldg(G + 3 * n + ii),
          g12 = __ldg(G + 4 * n + ii), g22 = __ldg(G + 5 * n + ii);
  S c[N];
  if (N == 8) {
    const S kb = (((K[0] + K[1]) + (K[2 % N] + K[3 % N])) + ((K[4 % N] + K[5 % N]) + (K[6 % N] + K[7 % N]))) * S(0.125);
    const S gx = ((T[1] - T[0]) + (T[2 % N] - T[3 % N])) + ((T[5 % N] - T[4 % N]) + (T[6 % N] - T[7 % N]));
    const S gy = ((T[3 % N] - T[0]) + (T[2 % N] - T[1])) + ((T[7 % N] - T[4 % N]) + (T[6 % N] - T[5 % N]));
    const S gz = ((T[4 % N] - T[0]) + (T[5 % N] - T[1])) + ((T[6 % N] - T[2 % N]) + (T[7 % N] - T[3 % N]));
    const S u = kb * (g00 * gx + g01 * gy + g02 * gz);
    const S v = kb * (g01 * gx + g11 * gy + g12 * gz);
    const S w2 = kb * (g02 * gx + g12 * gy + g22 * gz);
    const S a = u + v, b2 = u - v;
    c[0] = -a - w2; c[1] = b2 - w2; c[2 % N] = a - w2; c[3 % N] = -b2 - w2;
    c[4 % N] = -a + w2; c[5 % N] = b2 + w2; c[6 % N] = a + w2; c[7 % N] = -b2 + w2;
  } else {
    const S kb = ((K[0] + K[1]) + (K[2 % N] + K[3 % N])) * S(0.25);
    const S d1 = T[1] - T[0], d2 = T[2 % N] - T[0], d3 = T[3 % N] - T[0];
    c[1] = kb * (g00 * d1 + g01 * d2 + g02 * d3);
    c[2 % N] = kb * (g01 * d1 + g11 * d2 + g12 * d3);
    c[3 % N] = kb * (g02 * d1 + g12 * d2 + g22 * d3);
    c[0] = -((c[1] + c[2 % N]) + c[3 % N]);
  }
#pragma unroll
  for (int a = 0; a < N; ++a) warp_aggregated_add(F, valid ? nd[a] : -1, -c[a]);
}

template <typename S, bool LIN>
__global__ void __launch_bounds__(256) k_atomic_node(const __grid_constant__ TiledArgs<S> g, S *__restrict__ F,
                                                     const uint8_t *__restrict__ cls, int64_t V,
                                                     const S *__restrict__ hA, const S *__restrict__ hAT) {
  if (g.flag->step < g.step_no) return;
  const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  bool bad = false;
  if (n < V) {
    const S f = F[n];
    F[n] = S(0);
    const uint8_t cl = cls[n];
    if (cl != 2) {
      const Mat<S> &m = g.mats.m[0];
      const S x = g.Tin[n];
      S v, px = 0, py = 0, pz = 0;
      if (g.n_src) {
        px = g.xyzv[4 * n];
        py = g.xyzv[4 * n + 1];
        pz = g.xyzv[4 * n + 2];
        v = g.xyzv[4 * n + 3];
      } else {
        v = g.vol[n];
      }
      const S cap = ipa<LIN>(m.rho, x) * ipa<LIN>(m.c, x) * v;
      const S kb = m.td_perf ? ipa<LIN>(m.wb, x) * m.cb * v : m.wbcb * v;
      S rate = (((f - kb * x) + kb * m.Ta) + m.Qm * v) + (g.q_ext ? g.q_ext[n] : S(0));
      for (int k = 0; k < g.n_src; ++k) {
        const SourceT<S> &s = g.src[k];
        const S dx = px - s.cx, dy = py - s.cy, dz = pz - s.cz;
        const S r2 = (dx * dx + dy * dy) + dz * dz;
        const S q = k < g.n_gauss ? s.amp * afast_exp(-r2 * s.inv2s2)
                                  : (r2 > S(0) ? min(s.cap, s.inv4pi_amp / r2) : s.cap);
        rate += q * v;
      }
      if (cl == 1) rate += hAT[n] - hA[n] * x;  // Robin (rate - hA T) + hA T_inf, as fh_tiled.cu
      const S xn = x + g.dt * rate / cap;
      g.Tout[n] = xn;
      if (g.F_out) g.F_out[n] = f;
      bad = !(fabs(xn) <= g.runaway_limit);
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicMin(&g.flag->step, g.step_no);
}

template <typename S>
void atomic_step(const TiledArgs<S> &g, const AtomicState &a, S *F, cudaStream_t s) {
  const bool lin = g.lin != 0;
  auto blocks = [](int64_t n) { return (unsigned)((n + 255) / 256); };
  if (a.n_tet) {
    if (lin) k_atomic_elem<S, 4, true><<<blocks(a.n_tet), 256, 0, s>>>(g, a.tet_conn, (const S *)a.tet_G, a.n_tet, F);
    else k_atomic_elem<S, 4, false><<<blocks(a.n_tet), 256, 0, s>>>(g, a.tet_conn, (const S *)a.tet_G, a.n_tet, F);
  }
  if (a.n_hex) {
    if (lin) k_atomic_elem<S, 8, true><<<blocks(a.n_hex), 256, 0, s>>>(g, a.hex_conn, (const S *)a.hex_G, a.n_hex, F);
    else k_atomic_elem<S, 8, false><<<blocks(a.n_hex), 256, 0, s>>>(g, a.hex_conn, (const S *)a.hex_G, a.n_hex, F);
  }
  const S *hA = (const S *)a.hA, *hAT = (const S *)a.hAT;
  if (lin) k_atomic_node<S, true><<<blocks(a.V), 256, 0, s>>>(g, F, a.cls, a.V, hA, hAT);
  else k_atomic_node<S, false><<<blocks(a.V), 256, 0, s>>>(g, F, a.cls, a.V, hA, hAT);
  FH_CUDA(cudaGetLastError());
}
template void atomic_step<float>(const TiledArgs<float> &, const AtomicState &, float *, cudaStream_t);
template void atomic_step<double>(const TiledArgs<double> &, const AtomicState &, double *, cudaStream_t);

// G (6 per element, original element order) -> SoA [6][n] in the sorted order,
// hexes pre-scaled by 1/64, the conductivity factor folded in
template <typename S>
__global__ void k_pack_soa(const int32_t *__restrict__ elem, int64_t n, const double *__restrict__ G, double scale,
                           const double *__restrict__ kf, S *__restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t e = elem[i];
  const double f = kf ? kf[e] : 1.0;
#pragma unroll
  for (int c = 0; c < 6; ++c) out[c * n + i] = (S)(G[6 * e + c] * scale * f);
}

template <typename S>
void atomic_pack(const int32_t *elem, int64_t n, const double *G, double scale, const double *kf, S *out,
                 cudaStream_t s) {
  if (n <= 0) return;
  k_pack_soa<S><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(elem, n, G, scale, kf, out);
  FH_CUDA(cudaGetLastError());
}
template void atomic_pack<float>(const int32_t *, int64_t, const double *, double, const double *, float *,
                                 cudaStream_t);
template void atomic_pack<double>(const int32_t *, int64_t, const double *, double, const double *, double *,
                                  cudaStream_t);

}  // namespace fh
