// Host-side bookkeeping for the fused step: node renumbering, tiles
// ("parts") of nodes, the element slots of every part and the deterministic
// accumulation phases.  Integer work only; floating-point precompute runs on
// the device (fh_precompute.cu).
//
// Layout produced:
//  * domains: the node set is cut into n_domains pieces (slabs along an axis,
//    or recursive coordinate bisection).  Multi-GPU engines own a contiguous
//    range of domains; the tile decomposition never depends on the GPU count,
//    so results are bitwise identical for 1, 2, 4 or 8 GPUs.
//  * parts: each domain is cut by recursive coordinate bisection into parts of
//    <= target nodes.  New node ids are part-major; inside a part nodes are
//    ordered free | robin | dirichlet (original id order inside each class),
//    so "updated by this part" is one range check and Dirichlet nodes are never
//    touched by the step kernel.
//  * slots: every element is listed in each part that owns one of its
//    non-Dirichlet nodes (owner computes; halo elements are recomputed by
//    each owner instead of exchanging partial loads).  Slots of a part are
//    tets then hexes, ascending original element id.
//  * phases: inside a batch of `batch` slots the contribution of corner a of
//    slot s is added in phase rank(s, a) = number of earlier slots of the
//    batch that touch the same node.  Phases are separated by barriers, so
//    every node's sum has a fixed order: deterministic, no atomics.  When each
//    node meets every corner index at most once per batch (structured hex
//    grids) the phase is simply the corner index and no rank bytes are stored.
#include <algorithm>
#include <type_traits>
#include <cmath>
#include <cstring>
#include <numeric>

#include "fh_internal.h"

namespace fh {

void build_node_csr(int64_t V, int64_t n_tet, const int64_t *tets, int64_t n_hex, const int64_t *hexes,
                    std::vector<int32_t> &offs, std::vector<int32_t> &pos) {
  const int64_t nconn = 4 * n_tet + 8 * n_hex;
  offs.assign(V + 1, 0);
  for (int64_t p = 0; p < 4 * n_tet; ++p) offs[tets[p] + 1]++;
  for (int64_t p = 0; p < 8 * n_hex; ++p) offs[hexes[p] + 1]++;
  for (int64_t i = 0; i < V; ++i) offs[i + 1] += offs[i];
  pos.resize(nconn);
  std::vector<int32_t> fill(offs.begin(), offs.end() - 1);
  for (int64_t p = 0; p < 4 * n_tet; ++p) pos[fill[tets[p]]++] = (int32_t)p;
  for (int64_t p = 0; p < 8 * n_hex; ++p) pos[fill[hexes[p]]++] = (int32_t)(4 * n_tet + p);
}

namespace {

struct Rcb {
  const double *xyz;
  // split idx[lo,hi) into `parts` pieces of near-equal size; appends piece
  // boundaries (as offsets into idx) in leaf order.
  void split(std::vector<int64_t> &idx, int64_t lo, int64_t hi, int parts, std::vector<int64_t> &bounds,
             int forced_axis) {
    if (parts <= 1 || hi - lo <= 1) {
      bounds.push_back(hi);
      return;
    }
    int axis = forced_axis;
    if (axis < 0) {
      double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
      for (int64_t q = lo; q < hi; ++q)
        for (int d = 0; d < 3; ++d) {
          const double v = xyz[3 * idx[q] + d];
          mn[d] = std::min(mn[d], v);
          mx[d] = std::max(mx[d], v);
        }
      axis = 0;
      // longest extent; ties go to the highest axis (z first) so that cubes
      // split into z-slabs first, then y, then x
      for (int d = 1; d < 3; ++d)
        if (mx[d] - mn[d] >= mx[axis] - mn[axis]) axis = d;
    }
    const int left_parts = parts / 2;
    const int64_t mid = lo + (int64_t)((double)(hi - lo) * left_parts / parts);
    const double *x = xyz;
    auto less = [x, axis](int64_t a, int64_t b) {
      const double va = x[3 * a + axis], vb = x[3 * b + axis];
      return va < vb || (va == vb && a < b);
    };
    std::nth_element(idx.begin() + lo, idx.begin() + mid, idx.begin() + hi, less);
    split(idx, lo, mid, left_parts, bounds, forced_axis);
    split(idx, mid, hi, parts - left_parts, bounds, forced_axis);
  }
};

template <int N>
void build_slots(int64_t n_elem, const int64_t *conn_old, int64_t elem_offset, const Partition &P,
                 const std::vector<int32_t> &part_of_new, const std::vector<uint8_t> &updatable_new,
                 std::vector<std::vector<int32_t>> &per_part) {
  for (int64_t e = 0; e < n_elem; ++e) {
    int32_t seen[N];
    int ns = 0;
    for (int a = 0; a < N; ++a) {
      const int64_t nn = P.new_of_old[conn_old[N * e + a]];
      if (!updatable_new[nn]) continue;
      const int32_t p = part_of_new[nn];
      bool dup = false;
      for (int k = 0; k < ns; ++k) dup |= (seen[k] == p);
      if (!dup) seen[ns++] = p;
    }
    for (int k = 0; k < ns; ++k) per_part[seen[k]].push_back((int32_t)(e + elem_offset));
  }
}

}  // namespace

void build_partition(const PartitionInput &in, Partition &P) {
  const int64_t V = in.V;
  P = Partition{};
  P.batch = in.batch;
  const int target = std::max(64, in.target_part_nodes);
  const int ndom = std::max(1, in.n_domains);
  std::vector<int64_t> idx(V);
  std::iota(idx.begin(), idx.end(), 0);
  Rcb rcb{in.xyz};
  // 1. domains
  std::vector<int64_t> dom_bounds;
  if (ndom > 1 && in.slab_axis >= 0) {
    const int ax = in.slab_axis;
    const double *x = in.xyz;
    std::stable_sort(idx.begin(), idx.end(), [x, ax](int64_t a, int64_t b) { return x[3 * a + ax] < x[3 * b + ax]; });
    for (int d = 1; d <= ndom; ++d) dom_bounds.push_back((int64_t)((double)V * d / ndom));
  } else {
    rcb.split(idx, 0, V, ndom, dom_bounds, -1);
  }
  // 2. parts inside each domain
  std::vector<int64_t> part_bounds;
  P.domain_part_start.assign(1, 0);
  int64_t lo = 0;
  for (int d = 0; d < ndom; ++d) {
    const int64_t hi = dom_bounds[d];
    const int parts = (int)std::max<int64_t>(1, (hi - lo + target - 1) / target);
    rcb.split(idx, lo, hi, parts, part_bounds, -1);
    P.domain_part_start.push_back((int32_t)part_bounds.size());
    lo = hi;
  }
  P.n_parts = (int)part_bounds.size();
  P.part_domain.resize(P.n_parts);
  for (int d = 0; d < ndom; ++d)
    for (int p = P.domain_part_start[d]; p < P.domain_part_start[d + 1]; ++p) P.part_domain[p] = d;
  // 3. order inside parts: class (free, robin, dirichlet), then original id
  P.new_of_old.assign(V, -1);
  P.old_of_new.resize(V);
  P.part_node_start.assign(P.n_parts + 1, 0);
  P.part_n_free.resize(P.n_parts);
  P.part_robin_start.resize(P.n_parts);
  std::vector<int32_t> part_of_new(V);
  int64_t start = 0, next = 0;
  P.max_part_nodes = 0;
  for (int p = 0; p < P.n_parts; ++p) {
    const int64_t end = part_bounds[p];
    auto cls = in.node_class;
    std::sort(idx.begin() + start, idx.begin() + end, [cls](int64_t a, int64_t b) {
      const int ca = cls ? cls[a] : 0, cb = cls ? cls[b] : 0;
      return ca < cb || (ca == cb && a < b);
    });
    int n_free = 0, n_plain = 0;
    for (int64_t q = start; q < end; ++q) {
      const int c = in.node_class ? in.node_class[idx[q]] : 0;
      if (c < 2) ++n_free;
      if (c == 0) ++n_plain;
      P.new_of_old[idx[q]] = next;
      P.old_of_new[next] = idx[q];
      part_of_new[next] = p;
      ++next;
    }
    P.part_node_start[p + 1] = (int32_t)next;
    P.part_n_free[p] = n_free;
    P.part_robin_start[p] = n_plain;
    P.max_part_nodes = std::max<int>(P.max_part_nodes, (int)(end - start));
    start = end;
  }
  std::vector<uint8_t> updatable_new(V);
  for (int64_t n = 0; n < V; ++n) updatable_new[n] = !(in.node_class && in.node_class[P.old_of_new[n]] == 2);
  // 4. slots (each part's tet / hex slot range starts on a multiple of 4
  //    slots so that the per-batch bulk copies are 16-byte aligned)
  std::vector<std::vector<int32_t>> tet_pp(P.n_parts), hex_pp(P.n_parts);
  build_slots<4>(in.n_tet, in.tets, 0, P, part_of_new, updatable_new, tet_pp);
  build_slots<8>(in.n_hex, in.hexes, in.n_tet, P, part_of_new, updatable_new, hex_pp);
  std::vector<std::vector<uint8_t>> tet_color_pp, hex_color_pp, tet_rows_pp;
  // order the slots of a part by their smallest corner id (new numbering), so
  // that neighbouring threads of a batch touch neighbouring nodes: the
  // shared-memory gathers and accumulations are then bank-conflict free
  // (element id order of a structured cube steps by a whole z-plane).
  {
    auto key = [&](int N, int32_t e) {
      const int64_t *c = N == 4 ? in.tets + 4 * (int64_t)e : in.hexes + 8 * ((int64_t)e - in.n_tet);
      int64_t m = P.new_of_old[c[0]];
      for (int a = 1; a < N; ++a) m = std::min<int64_t>(m, P.new_of_old[c[a]]);
      return m;
    };
    std::vector<std::pair<int64_t, int32_t>> tmp;
    auto sort_part = [&](std::vector<int32_t> &v, int N) {
      tmp.clear();
      for (int32_t e : v) tmp.emplace_back(key(N, e), e);
      std::sort(tmp.begin(), tmp.end());
      for (size_t q = 0; q < v.size(); ++q) v[q] = tmp[q].second;
    };
    for (int p = 0; p < P.n_parts; ++p) {
      sort_part(tet_pp[p], 4);
      sort_part(hex_pp[p], 8);
    }
    // greedy colouring of each tile's slots: two slots of one colour never
    // share a node the tile updates.  A stable sort by colour makes every
    // batch span few colours -> few accumulation phases (kColored mode).
    // With R accumulator rows a class may touch a node up to R times: the
    // r-th write of a class to a node goes to row r (tets only, R = 1 or 4).
    // Classes then grow R-fold, so a 256-slot batch spans fewer of them.
    const int R_tet = std::max(1, std::min(4, in.tet_rows));
    std::vector<uint64_t> used((size_t)P.max_part_nodes * 4, 0);  // used[loc * 4 + r]: colours written >= r + 1 times
    struct Ct {
      int col;
      int32_t e;
      uint8_t rows;  // 2 bits per corner
    };
    std::vector<Ct> ct;
    P.colored_ok = true;
    P.max_colors = 0;
    auto colour_part = [&](std::vector<int32_t> &v, int N, int p) {
      const int64_t n0 = P.part_node_start[p], nf = P.part_n_free[p];
      const int R = N == 4 ? R_tet : 1;
      ct.clear();
      for (int32_t e : v) {
        const int64_t *c = N == 4 ? in.tets + 4 * (int64_t)e : in.hexes + 8 * ((int64_t)e - in.n_tet);
        uint64_t m = 0;  // colours in which some corner is already full
        for (int a = 0; a < N; ++a) {
          const int64_t loc = P.new_of_old[c[a]] - n0;
          if (loc >= 0 && loc < nf) m |= used[(size_t)loc * 4 + (R - 1)];
        }
        if (~m == 0) {
          P.colored_ok = false;
          ct.push_back({63, e, 0});
          continue;
        }
        const int col = __builtin_ctzll(~m);
        const uint64_t bit = 1ull << col;
        P.max_colors = std::max(P.max_colors, col + 1);
        uint8_t rows = 0;
        for (int a = 0; a < N; ++a) {
          const int64_t loc = P.new_of_old[c[a]] - n0;
          if (loc < 0 || loc >= nf) continue;
          int r = 0;
          while (used[(size_t)loc * 4 + r] & bit) ++r;  // r < R: the class is not full at this node
          used[(size_t)loc * 4 + r] |= bit;
          if (N == 4) rows |= (uint8_t)(r << (2 * a));
        }
        ct.push_back({col, e, rows});
      }
      for (int32_t e : v) {  // reset the masks of this tile
        const int64_t *c = N == 4 ? in.tets + 4 * (int64_t)e : in.hexes + 8 * ((int64_t)e - in.n_tet);
        for (int a = 0; a < N; ++a) {
          const int64_t loc = P.new_of_old[c[a]] - n0;
          if (loc >= 0 && loc < nf)
            for (int r = 0; r < 4; ++r) used[(size_t)loc * 4 + r] = 0;
        }
      }
      std::stable_sort(ct.begin(), ct.end(), [](const Ct &x, const Ct &y) { return x.col < y.col; });
      for (size_t q = 0; q < v.size(); ++q) v[q] = ct[q].e;
      return ct;
    };
    // Hexes that are corner-unique inside every tile use corner phases and
    // keep the min-corner order (neighbouring threads touch neighbouring
    // nodes); a colour sort would interleave them and double the shared-memory
    // wavefronts (measured: 0.426 -> 0.48 ms/step on cfg4).
    bool hex_unique = true;
    {
      std::vector<uint8_t> mask(P.max_part_nodes, 0);
      for (int p = 0; p < P.n_parts && hex_unique; ++p) {
        const int64_t n0 = P.part_node_start[p], nf = P.part_n_free[p];
        for (int32_t e : hex_pp[p]) {
          const int64_t *c = in.hexes + 8 * ((int64_t)e - in.n_tet);
          for (int a = 0; a < 8; ++a) {
            const int64_t loc = P.new_of_old[c[a]] - n0;
            if (loc < 0 || loc >= nf) continue;
            if (mask[loc] & (1u << a)) hex_unique = false;
            mask[loc] |= (uint8_t)(1u << a);
          }
        }
        for (int32_t e : hex_pp[p]) {
          const int64_t *c = in.hexes + 8 * ((int64_t)e - in.n_tet);
          for (int a = 0; a < 8; ++a) {
            const int64_t loc = P.new_of_old[c[a]] - n0;
            if (loc >= 0 && loc < nf) mask[loc] = 0;
          }
        }
      }
    }
    P.hex_colored = !hex_unique || in.hex_color == 1;
    P.tet_color.clear();
    P.hex_color.clear();
    tet_color_pp.assign(P.n_parts, {});
    hex_color_pp.assign(P.n_parts, {});
    tet_rows_pp.assign(P.n_parts, {});
    for (int p = 0; p < P.n_parts; ++p) {
      for (auto &x : colour_part(tet_pp[p], 4, p)) {
        tet_color_pp[p].push_back((uint8_t)x.col);
        tet_rows_pp[p].push_back(x.rows);
      }
      if (P.hex_colored)
        for (auto &x : colour_part(hex_pp[p], 8, p)) hex_color_pp[p].push_back((uint8_t)x.col);
      else
        hex_color_pp[p].assign(hex_pp[p].size(), 0);
    }
    P.tet_rows = P.colored_ok ? R_tet : 1;
  }
  // 4b. node order inside each tile by first touch: scanning the tile's
  //     batches corner by corner (corner a of every slot of the batch, then
  //     corner a + 1), each node gets the next id of its class the first time
  //     it is met.  Neighbouring threads then gather neighbouring shared-memory
  //     words for every corner, whatever the slot order (colour or min
  //     corner), so the gathers and accumulations stay bank-conflict free.
  //     The class ranges (free | robin | dirichlet) are kept.
  if (in.first_touch) {
    const size_t Bt = (size_t)std::max(1, in.batch);
    std::vector<int32_t> touch(P.max_part_nodes);
    std::vector<int32_t> loc;
    std::vector<int64_t> olds;
    for (int p = 0; p < P.n_parts; ++p) {
      const int64_t n0 = P.part_node_start[p], nn = P.part_node_start[p + 1] - n0;
      std::fill(touch.begin(), touch.begin() + nn, -1);
      int32_t k = 0;
      auto scan = [&](const std::vector<int32_t> &v, int N) {
        for (size_t b = 0; b < v.size(); b += Bt) {
          const size_t be = std::min(v.size(), b + Bt);
          for (int a = 0; a < N; ++a)
            for (size_t q = b; q < be; ++q) {
              const int32_t e = v[q];
              const int64_t *c = N == 4 ? in.tets + 4 * (int64_t)e : in.hexes + 8 * ((int64_t)e - in.n_tet);
              const int64_t l = P.new_of_old[c[a]] - n0;
              if (l >= 0 && l < nn && touch[l] < 0) touch[l] = k++;
            }
        }
      };
      scan(tet_pp[p], 4);
      scan(hex_pp[p], 8);
      for (int64_t i = 0; i < nn; ++i)
        if (touch[i] < 0) touch[i] = k++;
      const int64_t rs = P.part_robin_start[p], nf = P.part_n_free[p];
      auto cls_of = [rs, nf](int64_t i) { return i < rs ? 0 : (i < nf ? 1 : 2); };
      loc.resize(nn);
      std::iota(loc.begin(), loc.end(), 0);
      std::sort(loc.begin(), loc.end(), [&](int32_t x, int32_t y) {
        const int cx = cls_of(x), cy = cls_of(y);
        return cx < cy || (cx == cy && touch[x] < touch[y]);
      });
      olds.resize(nn);
      for (int64_t j = 0; j < nn; ++j) olds[j] = P.old_of_new[n0 + loc[j]];
      for (int64_t j = 0; j < nn; ++j) {
        P.old_of_new[n0 + j] = olds[j];
        P.new_of_old[olds[j]] = n0 + j;
      }
    }
  }
  P.part_tet_start.assign(P.n_parts + 1, 0);
  P.part_hex_start.assign(P.n_parts + 1, 0);
  P.part_tet_count.assign(P.n_parts, 0);
  P.part_hex_count.assign(P.n_parts, 0);
  const int64_t Bp = std::max(4, in.batch);
  auto pad4 = [Bp](int64_t n) { return (n + Bp - 1) / Bp * Bp; };  // batch-aligned part ranges
  for (int p = 0; p < P.n_parts; ++p) {
    P.part_tet_count[p] = (int32_t)tet_pp[p].size();
    P.part_hex_count[p] = (int32_t)hex_pp[p].size();
    P.part_tet_start[p + 1] = P.part_tet_start[p] + (int32_t)pad4(tet_pp[p].size());
    P.part_hex_start[p + 1] = P.part_hex_start[p] + (int32_t)pad4(hex_pp[p].size());
  }
  P.tet_slot_elem.assign(P.part_tet_start.back(), -1);
  P.hex_slot_elem.assign(P.part_hex_start.back(), -1);
  P.tet_color.assign(P.part_tet_start.back(), 0xff);
  P.hex_color.assign(P.part_hex_start.back(), 0xff);
  std::vector<uint8_t> tet_rowbits(P.part_tet_start.back(), 0);
  for (int p = 0; p < P.n_parts; ++p) {
    if (P.tet_rows > 1 && p < (int)tet_rows_pp.size())
      std::copy(tet_rows_pp[p].begin(), tet_rows_pp[p].end(), tet_rowbits.begin() + P.part_tet_start[p]);
    std::copy(tet_pp[p].begin(), tet_pp[p].end(), P.tet_slot_elem.begin() + P.part_tet_start[p]);
    std::copy(hex_pp[p].begin(), hex_pp[p].end(), P.hex_slot_elem.begin() + P.part_hex_start[p]);
    std::copy(tet_color_pp[p].begin(), tet_color_pp[p].end(), P.tet_color.begin() + P.part_tet_start[p]);
    std::copy(hex_color_pp[p].begin(), hex_color_pp[p].end(), P.hex_color.begin() + P.part_hex_start[p]);
  }
  tet_pp.clear();
  hex_pp.clear();
  P.tet_conn.assign(4 * P.tet_slot_elem.size(), 0);
  for (size_t s = 0; s < P.tet_slot_elem.size(); ++s)
    if (P.tet_slot_elem[s] >= 0)
      for (int a = 0; a < 4; ++a)
        P.tet_conn[4 * s + a] = (int32_t)P.new_of_old[in.tets[4 * (int64_t)P.tet_slot_elem[s] + a]];
  P.hex_conn.assign(8 * P.hex_slot_elem.size(), 0);
  for (size_t s = 0; s < P.hex_slot_elem.size(); ++s)
    if (P.hex_slot_elem[s] >= 0) {
      const int64_t h = P.hex_slot_elem[s] - in.n_tet;
      for (int a = 0; a < 8; ++a) P.hex_conn[8 * s + a] = (int32_t)P.new_of_old[in.hexes[8 * h + a]];
    }
  // 5. halo lists and tile-local 16-bit connectivity: local index of node n in
  //    part p is n - n0 for owned nodes, nn + rank in the sorted halo list else
  P.part_halo_start.assign(P.n_parts + 1, 0);
  P.halo_nodes.clear();
  P.tet_conn16.assign(P.tet_conn.size(), 0);
  P.hex_conn16.assign(P.hex_conn.size(), 0);
  P.max_local_nodes = 0;
  P.max_part_free = 0;
  {
    std::vector<int32_t> halo, hrank, hord;
    const int32_t B0 = std::max(1, in.batch);
    for (int p = 0; p < P.n_parts; ++p) {
      const int32_t n0 = P.part_node_start[p], nn = P.part_node_start[p + 1] - n0;
      halo.clear();
      auto collect = [&](const std::vector<int32_t> &conn, int N, int32_t s0, int32_t cnt) {
        for (int64_t q = (int64_t)N * s0; q < (int64_t)N * (s0 + cnt); ++q) {
          const int32_t n = conn[q];
          if (n < n0 || n >= n0 + nn) halo.push_back(n);
        }
      };
      collect(P.tet_conn, 4, P.part_tet_start[p], P.part_tet_count[p]);
      collect(P.hex_conn, 8, P.part_hex_start[p], P.part_hex_count[p]);
      std::sort(halo.begin(), halo.end());
      halo.erase(std::unique(halo.begin(), halo.end()), halo.end());
      // staging order of the halo (sT[nn + i] = T[hord[i]]): first touch, like the owned nodes
      hrank.assign(halo.size(), -1);
      {
        int32_t k = 0;
        auto scan = [&](const std::vector<int32_t> &conn, int N, int32_t s0, int32_t cnt) {
          for (int32_t b = 0; b < cnt; b += B0) {
            const int32_t be = std::min(cnt, b + B0);
            for (int a = 0; a < N; ++a)
              for (int32_t q = b; q < be; ++q) {
                const int32_t n = conn[(size_t)N * (s0 + q) + a];
                if (n >= n0 && n < n0 + nn) continue;
                const size_t h = std::lower_bound(halo.begin(), halo.end(), n) - halo.begin();
                if (hrank[h] < 0) hrank[h] = k++;
              }
          }
        };
        if (in.first_touch) {
          scan(P.tet_conn, 4, P.part_tet_start[p], P.part_tet_count[p]);
          scan(P.hex_conn, 8, P.part_hex_start[p], P.part_hex_count[p]);
        } else {
          for (size_t h = 0; h < halo.size(); ++h) hrank[h] = (int32_t)h;
        }
      }
      hord.resize(halo.size());
      for (size_t h = 0; h < halo.size(); ++h) hord[hrank[h]] = halo[h];
      const int64_t nloc = (int64_t)nn + (int64_t)halo.size();
      if (nloc >= 0xfffe) fail(FH_ERR_CONFIG, "tile has too many local nodes; lower part_nodes");
      P.max_local_nodes = std::max<int>(P.max_local_nodes, (int)nloc);
      P.max_part_free = std::max<int>(P.max_part_free, P.part_n_free[p]);
      auto local = [&](int32_t n) -> uint16_t {
        if (n >= n0 && n < n0 + nn) return (uint16_t)(n - n0);
        return (uint16_t)(nn + hrank[std::lower_bound(halo.begin(), halo.end(), n) - halo.begin()]);
      };
      if (P.tet_rows > 1 && nloc + 1 >= (1 << 14))
        fail(FH_ERR_CONFIG, "tile has too many local nodes for row-tagged tet slots; lower part_nodes");
      for (int64_t q = 4 * (int64_t)P.part_tet_start[p]; q < 4 * (int64_t)(P.part_tet_start[p] + P.part_tet_count[p]); ++q)
        P.tet_conn16[q] = (uint16_t)(local(P.tet_conn[q]) | (((tet_rowbits[q / 4] >> (2 * (q % 4))) & 3) << 14));
      for (int64_t q = 8 * (int64_t)P.part_hex_start[p]; q < 8 * (int64_t)(P.part_hex_start[p] + P.part_hex_count[p]); ++q)
        P.hex_conn16[q] = local(P.hex_conn[q]);
      // padding slots up to the batch boundary point every corner at the
      // dummy staged node nloc (T = k = 0, never updated): the LEAN loops read
      // them like real slots and need no per-thread validity test
      for (int64_t q = 4 * (int64_t)(P.part_tet_start[p] + P.part_tet_count[p]); q < 4 * (int64_t)P.part_tet_start[p + 1]; ++q)
        P.tet_conn16[q] = (uint16_t)nloc;
      for (int64_t q = 8 * (int64_t)(P.part_hex_start[p] + P.part_hex_count[p]); q < 8 * (int64_t)P.part_hex_start[p + 1]; ++q)
        P.hex_conn16[q] = (uint16_t)nloc;
      P.halo_nodes.insert(P.halo_nodes.end(), hord.begin(), hord.end());
      P.part_halo_start[p + 1] = (int32_t)P.halo_nodes.size();
    }
  }
  // 6. phases per batch
  const int B = in.batch;
  std::vector<uint8_t> count(P.max_part_nodes, 0);
  std::vector<uint16_t> cornermask(P.max_part_nodes, 0);
  bool unique = true;
  P.tet_rank.assign(P.tet_conn.size(), 0xff);
  P.hex_rank.assign(P.hex_conn.size(), 0xff);
  // corner uniqueness is checked over a whole part: the kernel can then give
  // every (node, corner) pair its own accumulator slot (no phases at all)
  auto do_kind = [&](int N, const std::vector<int32_t> &starts, const std::vector<int32_t> &counts,
                     const std::vector<int32_t> &conn, std::vector<uint8_t> &rank, int &max_phase) {
    max_phase = 0;
    for (int p = 0; p < P.n_parts; ++p) {
      const int32_t n0 = P.part_node_start[p], nf = P.part_n_free[p];
      const int32_t s_end = starts[p] + counts[p];
      for (int32_t s = starts[p]; s < s_end; ++s)
        for (int a = 0; a < N; ++a) {
          const int32_t loc = conn[(size_t)N * s + a] - n0;
          if (loc >= 0 && loc < nf) {
            if ((cornermask[loc] & (1u << a)) && N == 8) unique = false;  // hexes only: tets use colours
            cornermask[loc] |= (uint16_t)(1u << a);
          }
        }
      for (int32_t s = starts[p]; s < s_end; ++s)
        for (int a = 0; a < N; ++a) {
          const int32_t loc = conn[(size_t)N * s + a] - n0;
          if (loc >= 0 && loc < nf) cornermask[loc] = 0;
        }
      for (int32_t b = starts[p]; b < s_end; b += B) {
        const int32_t be = std::min(s_end, b + B);
        for (int32_t s = b; s < be; ++s)
          for (int a = 0; a < N; ++a) {
            const int32_t loc = conn[(size_t)N * s + a] - n0;
            uint8_t r = 0xff;
            if (loc >= 0 && loc < nf) {
              if (count[loc] == 0xfe) fail(FH_ERR_CONFIG, "more than 254 elements share a node inside one batch");
              r = count[loc]++;
              max_phase = std::max<int>(max_phase, r + 1);
            }
            rank[(size_t)N * s + a] = r;
          }
        for (int32_t s = b; s < be; ++s)
          for (int a = 0; a < N; ++a) {
            const int32_t loc = conn[(size_t)N * s + a] - n0;
            if (loc >= 0 && loc < nf) count[loc] = 0;
          }
      }
    }
  };
  do_kind(4, P.part_tet_start, P.part_tet_count, P.tet_conn, P.tet_rank, P.max_phase_tet);
  do_kind(8, P.part_hex_start, P.part_hex_count, P.hex_conn, P.hex_rank, P.max_phase_hex);
  P.corner_unique = unique;
  // 7. colour phases: phase of a slot = index of its colour among the colours
  //    of its batch (colours are sorted, so each batch holds a contiguous run)
  auto colour_phases = [&](const std::vector<int32_t> &starts, const std::vector<int32_t> &counts,
                           const std::vector<uint8_t> &color, std::vector<uint8_t> &phase,
                           std::vector<uint8_t> &batch_nph, int &max_nph) {
    phase.assign(color.size(), 0);
    batch_nph.assign(color.size() / B + 1, 0);
    max_nph = 0;
    for (int p = 0; p < P.n_parts; ++p) {
      const int32_t s_end = starts[p] + counts[p];
      for (int32_t b = starts[p]; b < s_end; b += B) {
        const int32_t be = std::min(s_end, b + B);
        int ph = 0;
        for (int32_t s = b; s < be; ++s) {
          if (s > b && color[s] != color[s - 1]) ++ph;
          phase[s] = (uint8_t)ph;
        }
        batch_nph[b / B] = (uint8_t)(ph + 1);
        max_nph = std::max(max_nph, ph + 1);
      }
    }
  };
  if (P.colored_ok) {
    colour_phases(P.part_tet_start, P.part_tet_count, P.tet_color, P.tet_phase, P.tet_batch_nph, P.max_nph_tet);
    colour_phases(P.part_hex_start, P.part_hex_count, P.hex_color, P.hex_phase, P.hex_batch_nph, P.max_nph_hex);
  }
}

}  // namespace fh

namespace fh {

// See fh_internal.h.  Every rank runs this on the same partition, so the
// send list of r towards q is, element for element, the recv list of q from r.
void build_exchange(const Partition &P, const uint8_t *is_dir, int n_domains, int world, int rank, Exchange &X) {
  const int D = std::max(1, n_domains);
  if (world < 1 || D % world != 0) fail(FH_ERR_CONFIG, "n_domains must be a multiple of the rank count");
  X = Exchange{};
  X.rank = rank;
  X.world = world;
  auto dom_lo = [&](int r) { return r * (D / world); };
  X.part_lo = P.domain_part_start[dom_lo(rank)];
  X.part_hi = P.domain_part_start[dom_lo(rank + 1)];
  X.node_lo = P.part_node_start[X.part_lo];
  X.node_hi = P.part_node_start[X.part_hi];
  // rank owning a new node id
  std::vector<int64_t> rank_node_start(world + 1);
  for (int r = 0; r <= world; ++r) rank_node_start[r] = P.part_node_start[P.domain_part_start[dom_lo(r)]];
  auto owner = [&](int64_t n) {
    return (int)(std::upper_bound(rank_node_start.begin(), rank_node_start.end(), n) - rank_node_start.begin()) - 1;
  };
  // recv: remote, non-Dirichlet halo nodes of my parts; send: my nodes in the
  // halo of any other rank's parts
  std::vector<std::vector<int32_t>> recv(world), send(world);
  std::vector<uint8_t> boundary(P.n_parts, 0);
  for (int p = 0; p < P.n_parts; ++p) {
    const int pr = owner(P.part_node_start[p]);
    for (int32_t q = P.part_halo_start[p]; q < P.part_halo_start[p + 1]; ++q) {
      const int32_t n = P.halo_nodes[q];
      if (is_dir && is_dir[n]) continue;
      const int nr = owner(n);
      if (nr == pr) continue;
      if (pr == rank) {
        recv[nr].push_back(n);
        boundary[p] = 1;
      } else if (nr == rank) {
        send[pr].push_back(n);
      }
    }
  }
  // parts owning a sent node are boundary parts too
  std::vector<int32_t> part_of(X.node_hi - X.node_lo);
  for (int p = X.part_lo; p < X.part_hi; ++p)
    for (int32_t n = P.part_node_start[p]; n < P.part_node_start[p + 1]; ++n) part_of[n - X.node_lo] = p;
  X.send_offs.assign(1, 0);
  X.recv_offs.assign(1, 0);
  for (int r = 0; r < world; ++r) {
    if (r == rank) continue;
    auto &s = send[r], &v = recv[r];
    std::sort(s.begin(), s.end());
    s.erase(std::unique(s.begin(), s.end()), s.end());
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    if (s.empty() && v.empty()) continue;
    X.peers.push_back(r);
    for (int32_t n : s) boundary[part_of[n - X.node_lo]] = 1;
    X.send_nodes.insert(X.send_nodes.end(), s.begin(), s.end());
    X.recv_nodes.insert(X.recv_nodes.end(), v.begin(), v.end());
    X.send_offs.push_back((int64_t)X.send_nodes.size());
    X.recv_offs.push_back((int64_t)X.recv_nodes.size());
  }
  for (int p = X.part_lo; p < X.part_hi; ++p)
    if (boundary[p]) X.part_order.push_back(p);
  X.n_boundary = (int)X.part_order.size();
  for (int p = X.part_lo; p < X.part_hi; ++p)
    if (!boundary[p]) X.part_order.push_back(p);
}

// Rank-local view (multi-GPU engines): only the rank's parts, their slots and
// the nodes they read.  Local node ids are the owned range [node_lo, node_hi)
// shifted to 0, then the foreign nodes the parts' halos reference (sorted by
// new id: received halo nodes and other ranks' Dirichlet nodes).  Slot and
// batch arrays are the rank's contiguous slice (part ranges start on batch
// boundaries).  The exchange lists are mapped to local ids in place.
void localize_partition(const Partition &P, Exchange &X, Partition &L) {
  const int p0 = X.part_lo, p1 = X.part_hi, np = p1 - p0;
  const int64_t node_lo = X.node_lo, n_own = X.node_hi - X.node_lo;
  std::vector<int32_t> foreign;
  for (int32_t q = P.part_halo_start[p0]; q < P.part_halo_start[p1]; ++q) {
    const int32_t n = P.halo_nodes[q];
    if (n < node_lo || n >= node_lo + n_own) foreign.push_back(n);  // nodes of other ranks' parts
  }
  std::sort(foreign.begin(), foreign.end());
  foreign.erase(std::unique(foreign.begin(), foreign.end()), foreign.end());
  const int64_t V = (int64_t)P.new_of_old.size();
  const int64_t n_local = n_own + (int64_t)foreign.size();
  auto local_of = [&](int64_t n) -> int64_t {
    if (n >= node_lo && n < node_lo + n_own) return n - node_lo;
    auto it = std::lower_bound(foreign.begin(), foreign.end(), (int32_t)n);
    if (it == foreign.end() || *it != n)
      fail(FH_ERR_DEVICE, "localize_partition: node " + std::to_string(n) + " outside the rank's view [" +
                              std::to_string(node_lo) + ", +" + std::to_string(n_own) + ")");
    return n_own + (it - foreign.begin());
  };
  L = Partition{};
  L.n_parts = np;
  L.new_of_old.assign(V, -1);
  L.old_of_new.resize(n_local);
  for (int64_t l = 0; l < n_local; ++l) {
    const int64_t n = l < n_own ? node_lo + l : foreign[l - n_own];
    L.old_of_new[l] = P.old_of_new[n];
    L.new_of_old[P.old_of_new[n]] = l;
  }
  auto slice = [](const auto &v, int64_t lo, int64_t hi) { return std::decay_t<decltype(v)>(v.begin() + lo, v.begin() + hi); };
  L.part_node_start.resize(np + 1);
  L.part_tet_start.resize(np + 1);
  L.part_hex_start.resize(np + 1);
  L.part_halo_start.resize(np + 1);
  const int32_t ts0 = P.part_tet_start[p0], ts1 = P.part_tet_start[p1];
  const int32_t hs0 = P.part_hex_start[p0], hs1 = P.part_hex_start[p1];
  const int32_t h0 = P.part_halo_start[p0];
  for (int k = 0; k <= np; ++k) {
    L.part_node_start[k] = (int32_t)(P.part_node_start[p0 + k] - node_lo);
    L.part_tet_start[k] = P.part_tet_start[p0 + k] - ts0;
    L.part_hex_start[k] = P.part_hex_start[p0 + k] - hs0;
    L.part_halo_start[k] = P.part_halo_start[p0 + k] - h0;
  }
  L.part_n_free = slice(P.part_n_free, p0, p1);
  L.part_robin_start = slice(P.part_robin_start, p0, p1);
  L.part_tet_count = slice(P.part_tet_count, p0, p1);
  L.part_hex_count = slice(P.part_hex_count, p0, p1);
  L.part_domain = slice(P.part_domain, p0, p1);
  L.halo_nodes.resize(P.part_halo_start[p1] - h0);
  for (size_t q = 0; q < L.halo_nodes.size(); ++q) L.halo_nodes[q] = (int32_t)local_of(P.halo_nodes[h0 + q]);
  L.tet_conn16 = slice(P.tet_conn16, 4 * (int64_t)ts0, 4 * (int64_t)ts1);
  L.hex_conn16 = slice(P.hex_conn16, 8 * (int64_t)hs0, 8 * (int64_t)hs1);
  L.tet_slot_elem = slice(P.tet_slot_elem, ts0, ts1);
  L.hex_slot_elem = slice(P.hex_slot_elem, hs0, hs1);
  // per-slot corner ids (padding slots hold node 0: local node 0 then)
  auto map_conn = [&](const std::vector<int32_t> &c, const std::vector<int32_t> &slot_elem, int N, int64_t s_lo,
                      int64_t s_hi, std::vector<int32_t> &out) {
    out.resize(N * (s_hi - s_lo));
    for (int64_t sl = s_lo; sl < s_hi; ++sl)
      for (int a = 0; a < N; ++a)
        out[N * (sl - s_lo) + a] = slot_elem[sl] < 0 ? 0 : (int32_t)local_of(c[N * sl + a]);
  };
  if (!P.tet_conn.empty()) map_conn(P.tet_conn, P.tet_slot_elem, 4, ts0, ts1, L.tet_conn);
  if (!P.hex_conn.empty()) map_conn(P.hex_conn, P.hex_slot_elem, 8, hs0, hs1, L.hex_conn);
  if (!P.tet_rank.empty()) L.tet_rank = slice(P.tet_rank, 4 * (int64_t)ts0, 4 * (int64_t)ts1);
  if (!P.hex_rank.empty()) L.hex_rank = slice(P.hex_rank, 8 * (int64_t)hs0, 8 * (int64_t)hs1);
  if (!P.tet_color.empty()) L.tet_color = slice(P.tet_color, ts0, ts1);
  if (!P.hex_color.empty()) L.hex_color = slice(P.hex_color, hs0, hs1);
  if (!P.tet_phase.empty()) L.tet_phase = slice(P.tet_phase, ts0, ts1);
  if (!P.hex_phase.empty()) L.hex_phase = slice(P.hex_phase, hs0, hs1);
  if (!P.tet_batch_nph.empty()) L.tet_batch_nph = slice(P.tet_batch_nph, ts0 / P.batch, ts1 / P.batch);
  if (!P.hex_batch_nph.empty()) L.hex_batch_nph = slice(P.hex_batch_nph, hs0 / P.batch, hs1 / P.batch);
  L.corner_unique = P.corner_unique;
  L.max_phase_tet = P.max_phase_tet;
  L.max_phase_hex = P.max_phase_hex;
  L.max_part_nodes = P.max_part_nodes;
  L.max_local_nodes = P.max_local_nodes;
  L.max_part_free = P.max_part_free;
  L.colored_ok = P.colored_ok;
  L.hex_colored = P.hex_colored;
  L.max_colors = P.max_colors;
  L.max_nph_tet = P.max_nph_tet;
  L.max_nph_hex = P.max_nph_hex;
  L.tet_rows = P.tet_rows;
  L.batch = P.batch;
  L.domain_part_start = {0, np};
  // exchange lists and part order in local terms
  for (auto &n : X.send_nodes) n = (int32_t)local_of(n);
  for (auto &n : X.recv_nodes) n = (int32_t)local_of(n);
  for (auto &p : X.part_order) p -= p0;
  X.node_lo = 0;
  X.node_hi = n_own;
  X.part_lo = 0;
  X.part_hi = np;
}

}  // namespace fh
