// TILED mode: one fused kernel per explicit step (fh_tiled.cu).
#pragma once
#include "fh_exact.h"

namespace fh {

constexpr int kTileThreads = 256;  // == partition batch size

template <typename S>
struct SourceT {
  int kind;
  S amp, inv2s2, cap, inv4pi_amp;
  S cx, cy, cz;  // centre at the step-start time (host-evaluated per step)
  int active;
};

template <typename S>
struct TiledArgs {
  // part tables
  const int32_t *part_list;  // parts processed by this launch: part_list[part_begin + blockIdx.x]
  int32_t part_begin;
  const int32_t *part_node_start, *part_n_free, *part_robin_start, *part_robin_base;
  const int32_t *part_tet_start, *part_hex_start;
  // slots
  const int32_t *tet_conn, *hex_conn;   // new node ids, 4 / 8 per slot
  const S *tet_G, *hex_G;               // 6 per slot (hex pre-scaled by 1/64)
  const S *tet_kf, *hex_kf;             // per-slot conductivity factor, or frozen kbar (TI), or null
  const uint8_t *tet_rank, *hex_rank;   // phases (ranked mode) or null (corner-unique)
  const uint8_t *tet_region, *hex_region;
  int max_phase_tet, max_phase_hex;
  // nodes (new numbering)
  const S *Tin;
  S *Tout;
  const S *vol;
  const S *cap_frozen, *kb_frozen;  // TI
  const S *q_ext;                   // heat loads + static sources (W) or null
  const S *xyz;                     // 3 per node, for time-dependent sources
  const uint8_t *node_region;
  const S *robin_hA, *robin_hAT;
  MatSet<S> mats;
  int n_src;
  SourceT<S> src[kMaxSources];
  S dt, runaway_limit;
  int frozen_kbar;  // TI: *_kf hold kbar
  FailFlag *flag;
  unsigned long long step_no;
};

void tiled_step(const TiledArgs<float> &g, int n_parts, bool td, bool corner_unique, size_t smem,
                cudaStream_t s);
void tiled_step(const TiledArgs<double> &g, int n_parts, bool td, bool corner_unique, size_t smem,
                cudaStream_t s);

// TI freeze: per-slot kbar (into kbar_tet / kbar_hex, using the factor
// arrays kf_tet / kf_hex if given) and per-node capacity / perfusion from Tin.
template <typename S>
void tiled_freeze(const TiledArgs<S> &g, int64_t n_tet_slots, int64_t n_hex_slots, int64_t n_nodes,
                  const S *kf_tet, const S *kf_hex, S *kbar_tet, S *kbar_hex, S *cap, S *kb, cudaStream_t s);

template <typename S>
void gather_probes_t(const S *T, const int32_t *probes, int64_t np, double *out, const FailFlag *flag,
                     cudaStream_t s);

}  // namespace fh
