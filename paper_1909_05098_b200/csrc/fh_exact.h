// EXACT-mode kernel arguments and launchers (fh_exact.cu).
#pragma once
#include "fh_internal.h"

namespace fh {

constexpr int kMaxSources = 8;

struct ExactArgs {
  int64_t V, E, n_tet;
  int64_t chunk_size;
  const int32_t *conn;       // flat connectivity, tets then hexes (reference conn_data)
  const int64_t *conn_offs;  // E+1 (null: tets-then-hexes layout, 4/8 nodes)
  const int64_t *mat_offs;   // E+1 (null: same layout, 16/64 entries)
  const double *mat;         // row-major A per element
  const double *row_abs;
  const int32_t *csr_offs;   // V+1: incident conn positions per node, ascending
  const int32_t *csr_pos;
  const int32_t *elem_of;    // element of each conn position (null: from the layout)
  const double *node_vol;
  const int32_t *elem_region, *node_region;
  const double *kfactor;
  MatSet<double> mats;
  double *kbar, *cap, *kb, *qb;  // kb/qb: constant lumps (or frozen TD-perfusion)
  const double *qm, *qr, *q_static;
  double *contrib, *F;
  const int32_t *dir_slot;
  const double *dir_vals;
  const int32_t *robin_slot;
  const double *robin_hA, *robin_hAT;
  const double *xyz;
  int n_src;
  fh_source src[kMaxSources];
  double runaway_limit;
  FailFlag *flag;
};

void exact_props(const ExactArgs &g, const double *T, cudaStream_t s);
void exact_step(const ExactArgs &g, double *T, double dt, double t_start, int64_t step_no, bool td,
                cudaStream_t s);
void exact_scatter(const ExactArgs &g, const double *kbar, const double *T, double *out, cudaStream_t s);
void exact_critical(const ExactArgs &g, const double *T, double *kbar_scratch, double *lam, cudaStream_t s);
void gather_probes(const double *T, const int32_t *probes, int64_t np, double *out, const FailFlag *flag,
                   cudaStream_t s);

void op_curve(const Curve<double> &c, const double *T, int64_t n, double *out, cudaStream_t s);
void op_capacity(const Curve<double> &r, const Curve<double> &c, const double *T, const double *v, int64_t n,
                 double *out, cudaStream_t s);
void op_mean(const int32_t *conn, const int64_t *offs, int64_t E, const double *nodal, double *out,
             cudaStream_t s);
void op_update(double *T, const double *F, const double *C, const double *kb, const double *qb, const double *qm,
               const double *qr, int64_t n, double dt, cudaStream_t s);

}  // namespace fh
