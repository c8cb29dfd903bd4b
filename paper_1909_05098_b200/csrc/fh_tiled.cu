// TILED mode: the whole explicit step (north_star (ii)-(iv)) as ONE kernel.
//
// One CTA per tile ("part") of <= max_part_nodes nodes (fh_partition.cpp):
//   1. zero the tile's nodal load accumulators in shared memory;
//   2. stream the tile's element slots in batches of 256 (one thread per
//      element): gather the corner temperatures, evaluate k(T) per corner
//      (TD) for kbar_e, form the element load from the 6-value metric tensor
//      G (A = D G D^T):  g = D^T (T - T_0),  f = G g,
//      c_a = kbar * D_a . f  -- then add -c_a into the shared accumulator of
//      every corner the tile owns, phase by phase (a barrier per phase, so the
//      per-node summation order is fixed: deterministic without atomics);
//   3. for every owned non-Dirichlet node, the lumped update
//      T' = T + dt (F - kb T + qb + qm + q_ext [+ Robin]) / C with C, kb from
//      rho(T) c(T) and w_b(T), written to the other temperature buffer, plus
//      the runaway check.
// Global memory traffic per step: the slot stream (conn, G, factor) once, the
// nodal streams (T, v, [q, xyz]) once, T' once; halo temperatures come from L2.
#include <cstdio>

#include "fh_tiled.cuh"

namespace fh {

constexpr unsigned long long kNone = ~0ull;

template <typename S>
__device__ __forceinline__ S ldg(const S *p) {
  return __ldg(p);
}
// products that must not be contracted into an FMA (keeps T == Ta a bitwise
// fixed point: kb*T and qb = kb*Ta round identically)
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }

template <typename S>
__device__ __forceinline__ S kbar_of(const TiledArgs<S> &g, const Curve<S> &kc, const S *Tn, int n, S kf) {
  S s = S(0);
#pragma unroll
  for (int b = 0; b < 8; ++b)
    if (b < n) s += interp(kc, Tn[b]);
  return s / S(n) * kf;
}

// ---- element loads ---------------------------------------------------------

template <typename S, bool TD>
__device__ __forceinline__ void hex_loads(const TiledArgs<S> &g, int s, int32_t nd[8], S c[8]) {
  const int4 *cp = reinterpret_cast<const int4 *>(g.hex_conn + 8 * (size_t)s);
  const int4 c0 = __ldg(cp), c1 = __ldg(cp + 1);
  nd[0] = c0.x; nd[1] = c0.y; nd[2] = c0.z; nd[3] = c0.w;
  nd[4] = c1.x; nd[5] = c1.y; nd[6] = c1.z; nd[7] = c1.w;
  S T[8];
#pragma unroll
  for (int b = 0; b < 8; ++b) T[b] = ldg(g.Tin + nd[b]);
  const S *G = g.hex_G + 6 * (size_t)s;
  const S g00 = ldg(G), g01 = ldg(G + 1), g02 = ldg(G + 2), g11 = ldg(G + 3), g12 = ldg(G + 4), g22 = ldg(G + 5);
  S kb;
  if (TD) {
    const Curve<S> &kc = g.mats.m[g.hex_region ? g.hex_region[s] : 0].k;
    kb = kbar_of(g, kc, T, 8, g.hex_kf ? ldg(g.hex_kf + s) : S(1));
  } else {
    kb = ldg(g.hex_kf + s);  // frozen kbar
  }
  S d[8];
#pragma unroll
  for (int b = 0; b < 8; ++b) d[b] = T[b] - T[0];
  // g = sum_b s_b d_b  (signs of element.py HEX_VERTEX_SIGNS; the 1/8 of
  // D = S/8 on both sides is folded into G as 1/64)
  const S gx = ((d[1] - d[0]) + (d[2] - d[3])) + ((d[5] - d[4]) + (d[6] - d[7]));
  const S gy = ((d[3] - d[0]) + (d[2] - d[1])) + ((d[7] - d[4]) + (d[6] - d[5]));
  const S gz = ((d[4] - d[0]) + (d[5] - d[1])) + ((d[6] - d[2]) + (d[7] - d[3]));
  const S u = kb * (g00 * gx + g01 * gy + g02 * gz);
  const S v = kb * (g01 * gx + g11 * gy + g12 * gz);
  const S w = kb * (g02 * gx + g12 * gy + g22 * gz);
  const S a = u + v, b2 = u - v;
  c[0] = -a - w; c[1] = b2 - w; c[2] = a - w; c[3] = -b2 - w;
  c[4] = -a + w; c[5] = b2 + w; c[6] = a + w; c[7] = -b2 + w;
}

template <typename S, bool TD>
__device__ __forceinline__ void tet_loads(const TiledArgs<S> &g, int s, int32_t nd[4], S c[4]) {
  const int4 cc = __ldg(reinterpret_cast<const int4 *>(g.tet_conn + 4 * (size_t)s));
  nd[0] = cc.x; nd[1] = cc.y; nd[2] = cc.z; nd[3] = cc.w;
  S T[4];
#pragma unroll
  for (int b = 0; b < 4; ++b) T[b] = ldg(g.Tin + nd[b]);
  const S *G = g.tet_G + 6 * (size_t)s;
  const S g00 = ldg(G), g01 = ldg(G + 1), g02 = ldg(G + 2), g11 = ldg(G + 3), g12 = ldg(G + 4), g22 = ldg(G + 5);
  S kb;
  if (TD) {
    const Curve<S> &kc = g.mats.m[g.tet_region ? g.tet_region[s] : 0].k;
    kb = kbar_of(g, kc, T, 4, g.tet_kf ? ldg(g.tet_kf + s) : S(1));
  } else {
    kb = ldg(g.tet_kf + s);
  }
  const S d1 = T[1] - T[0], d2 = T[2] - T[0], d3 = T[3] - T[0];
  c[1] = kb * (g00 * d1 + g01 * d2 + g02 * d3);
  c[2] = kb * (g01 * d1 + g11 * d2 + g12 * d3);
  c[3] = kb * (g02 * d1 + g12 * d2 + g22 * d3);
  c[0] = -((c[1] + c[2]) + c[3]);
}

// add -c[a] into the owned corners, one phase per barrier
template <typename S, int N, bool UNIQ>
__device__ __forceinline__ void accumulate(S *acc, const int32_t nd[N], const S c[N], int n0, int nfree,
                                           bool valid, const uint8_t *rank, int n_phase) {
  int loc[N];
#pragma unroll
  for (int a = 0; a < N; ++a) {
    loc[a] = nd[a] - n0;
    if (!valid || (unsigned)loc[a] >= (unsigned)nfree) loc[a] = -1;
  }
  if (UNIQ) {
#pragma unroll
    for (int a = 0; a < N; ++a) {
      if (loc[a] >= 0) acc[loc[a]] -= c[a];
      __syncthreads();
    }
  } else {
    uint8_t r[N];
#pragma unroll
    for (int a = 0; a < N; ++a) r[a] = valid ? rank[a] : 0xff;
    for (int ph = 0; ph < n_phase; ++ph) {
#pragma unroll
      for (int a = 0; a < N; ++a)
        if (r[a] == ph && loc[a] >= 0) acc[loc[a]] -= c[a];
      __syncthreads();
    }
  }
}

template <typename S>
__device__ __forceinline__ S sources_at(const TiledArgs<S> &g, const S *xyz) {
  const S x = xyz[0], y = xyz[1], z = xyz[2];
  S q = S(0);
  for (int k = 0; k < g.n_src; ++k) {
    const SourceT<S> &s = g.src[k];
    if (!s.active) continue;
    const S dx = x - s.cx, dy = y - s.cy, dz = z - s.cz;
    const S r2 = (dx * dx + dy * dy) + dz * dz;
    if (s.kind == FH_SOURCE_GAUSSIAN) {
      q += s.amp * exp(-r2 * s.inv2s2);
    } else {
      q += r2 > S(0) ? min(s.cap, s.inv4pi_amp / r2) : s.cap;
    }
  }
  return q;
}

template <typename S, bool TD, bool UNIQ>
__global__ void __launch_bounds__(kTileThreads) k_tiled_step(const __grid_constant__ TiledArgs<S> g) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S *acc = reinterpret_cast<S *>(smem_raw);
  __shared__ int s_bad;
  if (g.flag->step != kNone) return;
  const int p = g.part_list ? g.part_list[g.part_begin + blockIdx.x] : g.part_begin + (int)blockIdx.x;
  const int n0 = g.part_node_start[p];
  const int nfree = g.part_n_free[p];
  const int tid = threadIdx.x;
  if (tid == 0) s_bad = 0;
  for (int i = tid; i < nfree; i += kTileThreads) acc[i] = S(0);
  __syncthreads();

  // tets
  {
    const int s0 = g.part_tet_start[p], s1 = g.part_tet_start[p + 1];
    for (int b = s0; b < s1; b += kTileThreads) {
      const int s = b + tid;
      const bool valid = s < s1;
      int32_t nd[4] = {0, 0, 0, 0};
      S c[4] = {S(0), S(0), S(0), S(0)};
      if (valid) tet_loads<S, TD>(g, s, nd, c);
      uint8_t rk[4] = {0xff, 0xff, 0xff, 0xff};
      if (!UNIQ && valid) {
        const uint32_t w = __ldg(reinterpret_cast<const uint32_t *>(g.tet_rank) + s);
        rk[0] = w & 0xff; rk[1] = (w >> 8) & 0xff; rk[2] = (w >> 16) & 0xff; rk[3] = w >> 24;
      }
      accumulate<S, 4, UNIQ>(acc, nd, c, n0, nfree, valid, rk, g.max_phase_tet);
    }
  }
  // hexes
  {
    const int s0 = g.part_hex_start[p], s1 = g.part_hex_start[p + 1];
    for (int b = s0; b < s1; b += kTileThreads) {
      const int s = b + tid;
      const bool valid = s < s1;
      int32_t nd[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      S c[8];
#pragma unroll
      for (int a = 0; a < 8; ++a) c[a] = S(0);
      if (valid) hex_loads<S, TD>(g, s, nd, c);
      uint8_t rk[8];
#pragma unroll
      for (int a = 0; a < 8; ++a) rk[a] = 0xff;
      if (!UNIQ && valid) {
        const uint2 w = __ldg(reinterpret_cast<const uint2 *>(g.hex_rank) + s);
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          rk[a] = (w.x >> (8 * a)) & 0xff;
          rk[a + 4] = (w.y >> (8 * a)) & 0xff;
        }
      }
      accumulate<S, 8, UNIQ>(acc, nd, c, n0, nfree, valid, rk, g.max_phase_hex);
    }
  }
  __syncthreads();

  // lumped nodal update of the owned free nodes
  bool bad = false;
  const int rstart = g.part_robin_start[p];
  for (int loc = tid; loc < nfree; loc += kTileThreads) {
    const int n = n0 + loc;
    const S x = g.Tin[n];
    const S v = g.vol[n];
    const Mat<S> &m = g.mats.m[g.node_region ? g.node_region[n] : 0];
    S cap, kb;
    if (TD) {
      cap = interp(m.rho, x) * interp(m.c, x) * v;
      kb = m.td_perf ? interp(m.wb, x) * m.cb * v : m.wbcb * v;
    } else {
      cap = g.cap_frozen[n];
      kb = m.td_perf ? g.kb_frozen[n] : m.wbcb * v;
    }
    S rate = ((acc[loc] - mul_rn(kb, x)) + mul_rn(kb, m.Ta)) + m.Qm * v;
    if (g.q_ext) rate += g.q_ext[n];
    if (g.n_src) rate += sources_at(g, g.xyz + 3 * (size_t)n) * v;
    if (loc >= rstart) {
      const int rb = g.part_robin_base[p] + (loc - rstart);
      rate += g.robin_hAT[rb] - g.robin_hA[rb] * x;
    }
    const S xn = x + g.dt * rate / cap;
    g.Tout[n] = xn;
    bad |= !(fabs(xn) <= g.runaway_limit);  // also catches NaN
  }
  if (__any_sync(0xffffffffu, bad) && (tid & 31) == 0) s_bad = 1;
  __syncthreads();
  if (tid == 0 && s_bad) atomicMin(&g.flag->step, g.step_no);
}

template <typename S>
static void launch_step(const TiledArgs<S> &g, int n_parts, bool td, bool uniq, size_t smem, cudaStream_t s) {
  if (n_parts <= 0) return;
  auto kern = td ? (uniq ? k_tiled_step<S, true, true> : k_tiled_step<S, true, false>)
                 : (uniq ? k_tiled_step<S, false, true> : k_tiled_step<S, false, false>);
  static size_t configured[2][2] = {{0, 0}, {0, 0}};
  size_t &cfg = configured[td][uniq];
  if (smem > cfg) {
    FH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cfg = smem;
  }
  kern<<<n_parts, kTileThreads, smem, s>>>(g);
  FH_CUDA(cudaGetLastError());
}

void tiled_step(const TiledArgs<float> &g, int n_parts, bool td, bool uniq, size_t smem, cudaStream_t s) {
  launch_step(g, n_parts, td, uniq, smem, s);
}
void tiled_step(const TiledArgs<double> &g, int n_parts, bool td, bool uniq, size_t smem, cudaStream_t s) {
  launch_step(g, n_parts, td, uniq, smem, s);
}

// ---- TI freeze ---------------------------------------------------------------
template <typename S, int N>
__global__ void k_freeze_slots(const TiledArgs<S> g, const int32_t *__restrict__ conn, const uint8_t *region,
                               int64_t n_slots, const S *__restrict__ kf, S *__restrict__ kbar) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= n_slots) return;
  const Curve<S> &kc = g.mats.m[region ? region[s] : 0].k;
  S T[8];
#pragma unroll
  for (int b = 0; b < 8; ++b) T[b] = b < N ? g.Tin[conn[N * s + b]] : S(0);
  kbar[s] = kbar_of(g, kc, T, N, kf ? kf[s] : S(1));
}

template <typename S>
__global__ void k_freeze_nodes(const TiledArgs<S> g, int64_t V, S *__restrict__ cap, S *__restrict__ kb) {
  const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (n >= V) return;
  const Mat<S> &m = g.mats.m[g.node_region ? g.node_region[n] : 0];
  const S x = g.Tin[n], v = g.vol[n];
  cap[n] = interp(m.rho, x) * interp(m.c, x) * v;
  kb[n] = m.td_perf ? interp(m.wb, x) * m.cb * v : m.wbcb * v;
}

template <typename S>
void tiled_freeze(const TiledArgs<S> &g, int64_t nt, int64_t nh, int64_t V, const S *kf_tet, const S *kf_hex,
                  S *kbar_tet, S *kbar_hex, S *cap, S *kb, cudaStream_t s) {
  if (nt) k_freeze_slots<S, 4><<<(unsigned)((nt + 255) / 256), 256, 0, s>>>(g, g.tet_conn, g.tet_region, nt, kf_tet, kbar_tet);
  if (nh) k_freeze_slots<S, 8><<<(unsigned)((nh + 255) / 256), 256, 0, s>>>(g, g.hex_conn, g.hex_region, nh, kf_hex, kbar_hex);
  if (V) k_freeze_nodes<S><<<(unsigned)((V + 255) / 256), 256, 0, s>>>(g, V, cap, kb);
  FH_CUDA(cudaGetLastError());
}

template void tiled_freeze<float>(const TiledArgs<float> &, int64_t, int64_t, int64_t, const float *, const float *,
                                  float *, float *, float *, float *, cudaStream_t);
template void tiled_freeze<double>(const TiledArgs<double> &, int64_t, int64_t, int64_t, const double *,
                                   const double *, double *, double *, double *, double *, cudaStream_t);

template <typename S>
__global__ void k_probes_t(const S *__restrict__ T, const int32_t *__restrict__ probes, int64_t np,
                           double *__restrict__ out, const FailFlag *flag) {
  if (flag && flag->step != kNone) return;
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q < np) out[q] = (double)T[probes[q]];
}

template <typename S>
void gather_probes_t(const S *T, const int32_t *probes, int64_t np, double *out, const FailFlag *flag,
                     cudaStream_t s) {
  if (np <= 0) return;
  k_probes_t<S><<<(unsigned)((np + 127) / 128), 128, 0, s>>>(T, probes, np, out, flag);
  FH_CUDA(cudaGetLastError());
}
template void gather_probes_t<float>(const float *, const int32_t *, int64_t, double *, const FailFlag *, cudaStream_t);
template void gather_probes_t<double>(const double *, const int32_t *, int64_t, double *, const FailFlag *,
                                      cudaStream_t);

}  // namespace fh
