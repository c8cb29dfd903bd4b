// Device helpers of the EXACT step shared by the two-launch path (fh_exact.cu)
// and the resident small-mesh path (fh_resident.cu).  Both units compile with
// -fmad=false and every product / sum is an explicit _rn intrinsic, so the
// two paths produce the same bits (the reference's operation order,
// kernels.py:61-142, solver.py:354-365).
#pragma once
#include "fh_exact.h"

namespace fh {

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dvd(double a, double b) { return __ddiv_rn(a, b); }

constexpr unsigned long long kNoFail = ~0ull;

__device__ __forceinline__ int64_t eoff(const ExactArgs &g, int64_t e) {
  if (g.conn_offs) return g.conn_offs[e];
  return e < g.n_tet ? 4 * e : 4 * g.n_tet + 8 * (e - g.n_tet);
}
__device__ __forceinline__ int64_t moff(const ExactArgs &g, int64_t e) {
  if (g.mat_offs) return g.mat_offs[e];
  return e < g.n_tet ? 16 * e : 16 * g.n_tet + 64 * (e - g.n_tet);
}
__device__ __forceinline__ int64_t elem_of_pos(const ExactArgs &g, int64_t p) {
  if (g.elem_of) return g.elem_of[p];
  return p < 4 * g.n_tet ? p / 4 : g.n_tet + (p - 4 * g.n_tet) / 8;
}

__device__ __forceinline__ double source_density(const fh_source &s, double x, double y, double z, double t) {
  if (!(s.t0 <= t && t < s.t1)) return 0.0;
  const double d0 = x - (s.x0[0] + s.vel[0] * t), d1 = y - (s.x0[1] + s.vel[1] * t),
               d2 = z - (s.x0[2] + s.vel[2] * t);
  const double r2 = (d0 * d0 + d1 * d1) + d2 * d2;
  if (s.kind == FH_SOURCE_GAUSSIAN) return s.amp * exp(-r2 / (2.0 * s.sigma * s.sigma));
  double q = s.cap;
  if (r2 > 0.0) q = fmin(q, s.amp / (4.0 * 3.14159265358979323846 * r2));
  return q;
}

// per-node operands of the lumped update (read once per node; the resident
// path keeps them in shared memory for a whole launch)
struct NodeIn {
  double v, cap, kb, qb, qm, qr, qs, hA, hAT, dirv, x, y, z;
  int region, robin, dir;
};

__device__ __forceinline__ NodeIn load_node(const ExactArgs &g, int64_t i, int td) {
  NodeIn n;
  n.v = g.node_vol[i];
  n.region = g.node_region ? g.node_region[i] : 0;
  const Mat<double> &m = g.mats.m[n.region];
  n.cap = td ? 0.0 : g.cap[i];
  n.kb = (td && m.td_perf) ? 0.0 : g.kb[i];
  n.qb = (td && m.td_perf) ? 0.0 : g.qb[i];
  n.qm = g.qm[i];
  n.qr = g.qr[i];
  n.qs = g.q_static ? g.q_static[i] : 0.0;
  n.x = n.y = n.z = 0.0;
  if (g.n_src) {
    n.x = g.xyz[3 * i];
    n.y = g.xyz[3 * i + 1];
    n.z = g.xyz[3 * i + 2];
  }
  const int32_t rs = g.robin_slot ? g.robin_slot[i] : -1;
  n.robin = rs >= 0;
  n.hA = rs >= 0 ? g.robin_hA[rs] : 0.0;
  n.hAT = rs >= 0 ? g.robin_hAT[rs] : 0.0;
  const int32_t ds = g.dir_slot ? g.dir_slot[i] : -1;
  n.dir = ds >= 0;
  n.dirv = ds >= 0 ? g.dir_vals[ds] : 0.0;
  return n;
}

// the lumped update of a node with net conduction inflow F from temperature x
// (kernels.py:137-142 + the extensions), then the Dirichlet overwrite
// (solver.py:364-365); returns the new temperature
__device__ __forceinline__ double exact_update_in(const ExactArgs &g, const NodeIn &n, double F, double x, double dt,
                                                  double t_start, int td) {
  const Mat<double> &m = g.mats.m[n.region];
  double cap, kb, qb;
  if (td) {
    cap = mul(mul(interp_rn(m.rho, x), interp_rn(m.c, x)), n.v);
    if (m.td_perf) {
      kb = mul(mul(interp_rn(m.wb, x), m.cb), n.v);
      qb = mul(kb, m.Ta);
    } else {
      kb = n.kb;
      qb = n.qb;
    }
  } else {
    cap = n.cap;
    kb = n.kb;
    qb = n.qb;
  }
  double rate = add(add(add(sub(F, mul(kb, x)), qb), n.qm), n.qr);
  if (g.q_static) rate = add(rate, n.qs);
  if (g.n_src) {
    double q = 0.0;
    for (int s = 0; s < g.n_src; ++s) q += source_density(g.src[s], n.x, n.y, n.z, t_start);
    rate = add(rate, mul(q, n.v));
  }
  if (n.robin) rate = add(sub(rate, mul(n.hA, x)), n.hAT);
  double xn = add(x, dvd(mul(dt, rate), cap));
  if (n.dir) xn = n.dirv;
  return xn;
}

__device__ __forceinline__ double exact_update(const ExactArgs &g, int64_t i, double F, double x, double dt,
                                               double t_start, int td) {
  return exact_update_in(g, load_node(g, i, td), F, x, dt, t_start, td);
}

}  // namespace fh
