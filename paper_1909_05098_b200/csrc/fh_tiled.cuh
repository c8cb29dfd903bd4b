// TILED mode: one fused kernel per explicit step (fh_tiled.cu).
#pragma once
#include "fh_exact.h"

namespace fh {

#ifndef FH_TILE_THREADS
#define FH_TILE_THREADS 256
#endif
constexpr int kTileThreads = FH_TILE_THREADS;  // threads per tile CTA
constexpr int kSPT = 1;            // element slots per thread per batch (2 measured slower: smem)
constexpr int kBatch = kTileThreads * kSPT;  // == partition batch size B
constexpr int kMaxStages = 4;      // TMA ring depth limit (batches in flight per CTA)

template <typename S>
struct SourceT {
  int kind;
  S amp, inv2s2, cap, inv4pi_amp;
  S cx, cy, cz;  // centre at the step-start time (host-evaluated per step)
  int active;
};

// Slot streams of a part are stored in batches of kTileThreads slots, every
// part's range starting on a batch boundary:
//   rec    [batch] { conn16 [B][N] uint16 tile-local node index (owned | halo),
//                    G [6][B] metric tensor components (hex pre-scaled by 1/64) }
//   kf     [slot]      conductivity factor (TD) or frozen kbar (TI), optional
//   rank   [slot][N]   accumulation phase per corner (ranked mode only)
template <typename S>
struct TiledArgs {
  const int32_t *part_list;  // parts processed by this launch: part_list[part_begin + blockIdx.x]
  int32_t part_begin;
  const int32_t *part_node_start, *part_n_free, *part_robin_start, *part_robin_base;
  const int32_t *part_tet_start, *part_tet_count, *part_hex_start, *part_hex_count;
  const int32_t *part_halo_start, *halo_nodes;
  // per-batch records [conn16 block | G block] (RecBytes), null when the kind is absent
  const unsigned char *tet_rec, *hex_rec;
  const S *tet_kf, *hex_kf;
  const uint8_t *tet_rank, *hex_rank;  // null: corner-unique (phase == corner)
  const uint8_t *tet_phase, *hex_phase;  // colored mode: phase per slot
  const uint8_t *tet_bnph, *hex_bnph;    // colored mode: phases per batch (index slot / B)
  const uint8_t *tet_region, *hex_region;
  int max_phase_tet, max_phase_hex;
  // smem carve-up (bytes) and ring depth
  int smem_T, smem_acc, stage_bytes, n_stages;
  // nodes (new numbering)
  const S *Tin;
  S *Tout;
  S *F_out;  // optional: net conduction inflow of the updated nodes (ExplicitEngine.step's state.inflow)
  const S *vol;
  const S *cap_frozen, *kb_frozen;  // TI
  const S *q_ext;                   // heat loads + static sources (W) or null
  const S *xyzv;                    // (x, y, z, v) per node, for time-dependent sources
  const uint8_t *node_region;
  const int8_t *part_mat;  // with node_region: the tile's single material, or -1
  const int8_t *part_region;  // with slot regions: the region all the tile's slots share, or -1
  const S *robin_hA, *robin_hAT;
  MatSet<S> mats;   // one-knot curves normalised to two knots (see normalise_curves)
  int lin;          // every curve has <= 2 knots: branch-free interpolation kernels
  S lin_lo, lin_hi; // lin: intersection of the knot ranges of material 0's sloped laws (open interval)
  int tet_rows;     // tet accumulator rows (1 or 4; tet-only meshes), see Partition::tet_rows
  int n_gauss;      // active sources, Gaussians first: src[0, n_gauss) Gaussian, [n_gauss, n_src) RF
  int n_src;
  SourceT<S> src[kMaxSources];
  S dt, runaway_limit;
  FailFlag *flag;
  unsigned long long step_no;
  int64_t n_nodes;  // length of Tin / Tout (bounds checks of the checked build)
  int lean;         // 1: the LEAN batch loops (records packed with paired G; see setup_tiled)
  int max_tile_batches;  // most 256-slot batches in one tile (LEAN tiles: <= kTileThreads)
  int max_local;    // owned + halo nodes a tile may stage (shared-memory capacity)
};

// one batch record of the connectivity + metric stream in HBM, laid out like
// the head of the stage: conn16 [B][N] (uint16) | G [6][B] (hex pre-scaled by
// 1/64, conductivity factor folded in when temperature-dependent)
template <typename S>
constexpr int RecBytes(int N) {
  return kBatch * N * 2 + 6 * kBatch * (int)sizeof(S);
}

// bytes of one staged batch: conn16 [B][N] | G [6][B] | kf [B] | region [B] | rank [B][N] | phase [B]
template <typename S>
inline int StageBytes(int N, bool has_kf, bool has_rank, bool has_phase = false, bool has_region = false) {
  int b = kBatch * N * 2 + 6 * kBatch * (int)sizeof(S);
  if (has_kf) b += kBatch * (int)sizeof(S);
  if (has_region) b += kBatch;
  if (has_rank) b += kBatch * N;
  if (has_phase) b += kBatch;
  return (b + 15) & ~15;
}

template <typename S>
void tiled_step(const TiledArgs<S> &g, int n_parts, bool td, int mode, size_t smem, cudaStream_t s);
// resident step CTAs per SM of the kernel tiled_step would launch
template <typename S>
int tiled_occupancy(const TiledArgs<S> &g, bool td, int mode, size_t smem);

// accumulation mode of the step kernel (see fh_tiled.cu): 0 ranked phases,
// 1 corner phases, 2 corner slots (the last two need corner-unique tiles)
enum TileMode {
  kModeRanked = 0,
  kModeCornerPhase = 1,
  kModeCornerSlot = 2,    // removed (measured slower); rejected by fh_create
  kModeColored = 3,
  kModeSharedAtomic = 4,
  kModeCornerPhase2 = 5,
  kModeCornerPhase4 = 6   // removed (measured slower); rejected by fh_create
};

// TI freeze: per-slot kbar (global-id connectivity conn4/conn8) and per-node
// capacity / perfusion from Tin.
template <typename S>
void tiled_freeze(const TiledArgs<S> &g, const int32_t *tet_conn, const int32_t *hex_conn, int64_t n_tet_slots,
                  int64_t n_hex_slots, int64_t n_nodes, const S *kf_tet, const S *kf_hex, S *kbar_tet,
                  S *kbar_hex, S *cap, S *kb, cudaStream_t s);

template <typename S>
void gather_probes_t(const S *T, const int32_t *probes, int64_t np, double *out, const FailFlag *flag,
                     cudaStream_t s);

}  // namespace fh
