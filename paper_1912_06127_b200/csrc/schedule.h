// p2TDVP half-step programs (reconstructed from
// PAPER.md:414-432 §III.A, :470-488 §III.B, :722-739 App. A/B).
// Host-only; one source of truth for the single-process executor, the NCCL
// per-rank executor and the tdvp_plan() test entry point.
#pragma once
#include <set>
#include <string>
#include <utility>
#include <vector>

enum OpKind {
  OP_PAIR = 1, OP_BACK = 2, OP_SEND_R = 3, OP_RECV_L = 4, OP_SEND_L = 5, OP_RECV_R = 6,
  // one-site interior operations of the p1TDVP programs (reading R-P1TDVP):
  // SITE_R j: forward site j by dt/2 (skipped if full = 1: evolved by dt at the
  // end of half 1), split bond j, beta_{j+1}, bond j backward by dt/2, absorb
  // into site j+1; SITE_L j: the mirror onto bond j-1 / site j-1; FWD j: site j
  // forward by dt (full = 1) or dt/2
  OP_SITE_R = 7, OP_SITE_L = 8, OP_FWD = 9
};
enum { BUILD_BETA = 1, BUILD_GAMMA = 2 };

struct SchedOp {
  int kind, j, full, build;
};

// Contiguous segments (SURVEY O-3): p = 1, or p even with
// 2 <= p <= L/2; remainder sites alternate to segment 0, p-1, 0, ...
inline bool plan_partition(int L, int p, std::vector<std::pair<int, int>>& out, std::string& err) {
  out.clear();
  if (L < 2) { err = "L must be >= 2"; return false; }
  if (p != 1 && (p % 2 != 0 || p < 2 || p > L / 2)) {
    err = "n_segments must be 1 or even with 2 <= p <= L/2 (PAPER.md:470)";
    return false;
  }
  std::vector<int> sizes(p, L / p);
  int rem = L % p;
  for (int i = 0; rem > 0; ++i, --rem) sizes[(i % 2 == 0) ? 0 : p - 1] += 1;
  int s = 0;
  for (int q = 0; q < p; ++q) {
    if (p > 1 && sizes[q] < 2) { err = "segment shorter than two sites"; return false; }
    out.emplace_back(s, s + sizes[q] - 1);
    s += sizes[q];
  }
  return true;
}

// Half 1: q sweeps LEFT iff q = p/2 - 1 (mod 2): the central segments sweep
// away from the centre, neighbours alternate; half 2
// reverses.  p = 1: RIGHT then LEFT.  true = RIGHT.
inline bool sweeps_right(int p, int h, int q) {
  bool right = (p == 1) ? true : !((q % 2) == ((p / 2 - 1) % 2));
  return (h == 1) ? right : !right;
}

inline std::vector<SchedOp> segment_program(int L, int p, int h, int q, const std::pair<int, int>& se,
                                            const std::set<int>& merged) {
  std::vector<SchedOp> ops;
  const int s = se.first, e = se.second;
  auto is_merged = [&](int j) { return h == 2 && merged.count(j) > 0; };
  if (sweeps_right(p, h, q)) {
    if (q > 0) {
      if (!is_merged(s - 1)) ops.push_back({OP_RECV_L, s - 1, 0, 0});
      ops.push_back({OP_BACK, s, 0, 0});
    }
    for (int j = s; j < e; ++j) {
      if (!is_merged(j)) {
        const int full = (h == 1 && j + 1 == L - 1) ? 1 : 0;
        ops.push_back({OP_PAIR, j, full, full ? BUILD_GAMMA : BUILD_BETA});
      }
      if (!(j + 1 == e && e == L - 1)) ops.push_back({OP_BACK, j + 1, 0, 0});
    }
    if (q < p - 1) {
      ops.push_back({OP_RECV_R, e, 0, 0});
      ops.push_back({OP_PAIR, e, h == 1 ? 1 : 0, BUILD_BETA | BUILD_GAMMA});
      ops.push_back({OP_SEND_R, e, 0, 0});
    }
  } else {
    if (q < p - 1) {
      if (!is_merged(e)) {
        ops.push_back({OP_PAIR, e, 0, BUILD_BETA | BUILD_GAMMA});
        ops.push_back({OP_SEND_R, e, 0, 0});
      }
      ops.push_back({OP_BACK, e, 0, 0});
    }
    for (int j = e - 1; j >= s; --j) {
      if (!is_merged(j)) {
        const int full = (h == 1 && j == 0) ? 1 : 0;
        ops.push_back({OP_PAIR, j, full, full ? BUILD_BETA : BUILD_GAMMA});
      }
      if (!(j == s && s == 0)) ops.push_back({OP_BACK, j, 0, 0});
    }
    if (q > 0) {
      ops.push_back({OP_SEND_L, s, 0, 0});
      ops.push_back({OP_RECV_L, s - 1, 0, 0});
    }
  }
  return ops;
}

// Pairs evolved by the full dt at the end of half 1 (skipped in half 2; O-9).
inline std::set<int> merged_pairs(int L, int p, const std::vector<std::pair<int, int>>& bounds) {
  std::set<int> m;
  for (int q = 0; q < p; ++q)
    for (const SchedOp& op : segment_program(L, p, 1, q, bounds[q], {}))
      if (op.kind == OP_PAIR && op.full) m.insert(op.j);
  return m;
}

// p1TDVP half-step programs (reading R-P1TDVP; oracle/tdvp1.py _half1): the
// App. A programs with the boundary phases unchanged (two-site Lambda^-1-merged
// boundary pairs, D-phase backward steps, merged full-dt boundary pairs) and
// one-site segment interiors.  merged: boundary pairs evolved by dt in half 1;
// msites: chain-end sites evolved by dt in half 1 (both skipped in half 2).
inline std::vector<SchedOp> segment_program1(int L, int p, int h, int q, const std::pair<int, int>& se,
                                             const std::set<int>& merged, const std::set<int>& msites) {
  std::vector<SchedOp> ops;
  const int s = se.first, e = se.second;
  auto is_merged = [&](int j) { return h == 2 && merged.count(j) > 0; };
  auto site_done = [&](int j) { return h == 2 && msites.count(j) > 0; };
  if (sweeps_right(p, h, q)) {
    if (q > 0) {
      if (!is_merged(s - 1)) ops.push_back({OP_RECV_L, s - 1, 0, 0});
      ops.push_back({OP_BACK, s, 0, 0});
    }
    for (int j = s; j < e; ++j) ops.push_back({OP_SITE_R, j, site_done(j) ? 1 : 0, BUILD_BETA});
    if (e == L - 1 && !site_done(L - 1)) ops.push_back({OP_FWD, L - 1, h == 1 ? 1 : 0, 0});
    if (q < p - 1) {
      ops.push_back({OP_RECV_R, e, 0, 0});
      ops.push_back({OP_PAIR, e, h == 1 ? 1 : 0, BUILD_BETA | BUILD_GAMMA});
      ops.push_back({OP_SEND_R, e, 0, 0});
    }
  } else {
    if (q < p - 1) {
      if (!is_merged(e)) {
        ops.push_back({OP_PAIR, e, 0, BUILD_BETA | BUILD_GAMMA});
        ops.push_back({OP_SEND_R, e, 0, 0});
      }
      ops.push_back({OP_BACK, e, 0, 0});
    }
    for (int j = e; j > s; --j) ops.push_back({OP_SITE_L, j, site_done(j) ? 1 : 0, BUILD_GAMMA});
    if (s == 0 && !site_done(0)) ops.push_back({OP_FWD, 0, h == 1 ? 1 : 0, 0});
    if (q > 0) {
      ops.push_back({OP_SEND_L, s, 0, 0});
      ops.push_back({OP_RECV_L, s - 1, 0, 0});
    }
  }
  return ops;
}

// the boundary pairs and chain-end sites a p1TDVP half 1 evolves by dt
inline void merged1(int L, int p, const std::vector<std::pair<int, int>>& bounds, std::set<int>& pairs,
                    std::set<int>& sites) {
  pairs.clear();
  sites.clear();
  for (int q = 0; q < p; ++q)
    for (const SchedOp& op : segment_program1(L, p, 1, q, bounds[q], {}, {})) {
      if (op.kind == OP_PAIR && op.full) pairs.insert(op.j);
      if (op.kind == OP_FWD && op.full) sites.insert(op.j);
    }
}
