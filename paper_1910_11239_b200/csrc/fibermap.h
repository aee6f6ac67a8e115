// fibermap.h - bank-conflict-free thread -> (subdomain, fiber) maps for the
// FDM solve kernel (fdm2.cuh), built on the host once per kernel shape.
//
// Each contraction pass of fdm2 gives every thread one fiber of one of the
// CTA's G subdomain tensors.  Any bijection threads <-> (g, f) computes the
// same result, but the shared-memory bank pattern depends on it: a warp's
// 8-byte accesses are served per half-warp (16 lanes, 16 eight-byte banks)
// and its 16-byte accesses per quarter-warp (8 lanes, 8 bank groups).  The
// natural order (g = tid / F) leaves conflicts in the dense 48-byte cell rows
// of the bulk staging (m = 12: 3 chunks per row) and in the strided
// direction-(d-1) pass: ncu, cfg 5: 36M of 316M shared wavefronts.
//
// The builder below assigns (g, f) to threads so that every half-warp sees
// 16 distinct 8-byte bank residues and every quarter-warp 8 distinct 16-byte
// bank groups (randomised greedy over the residue classes, fixed seeds, so
// the maps are deterministic; it keeps the natural order when that is not
// worse).  Pass kinds: 0 = direction 0 (first and last pass: dense rows and
// the padded tensor row), 1 = directions 1 .. d-2, 2 = the fused direction
// d-1 pass.  Entry = g << 16 | f.
#pragma once
#include <algorithm>
#include <cstdint>
#include <vector>

namespace dgb {

struct FiberItem {
  uint32_t code;    // g << 16 | f
  int a;            // 8-byte bank residue (mod 16) of the fiber base
  int b[2];         // 16-byte bank group (mod 8) of the dense rows h = 0, 1 (-1: none)
};

// wavefronts of one pass under a thread order (8-byte half-warps and, when
// the items carry dense residues, 16-byte quarter-warps)
inline long fibermap_cost(const std::vector<FiberItem>& order, int nb) {
  long w = 0;
  const int n = (int)order.size();
  for (int h0 = 0; h0 < n; h0 += 16) {
    int cnt[16] = {0};
    int mx = 0;
    for (int i = h0; i < std::min(n, h0 + 16); ++i) mx = std::max(mx, ++cnt[order[i].a]);
    w += mx;
  }
  for (int h = 0; h < nb; ++h)
    for (int q0 = 0; q0 < n; q0 += 8) {
      int cnt[8] = {0};
      int mx = 0;
      for (int i = q0; i < std::min(n, q0 + 8); ++i) mx = std::max(mx, ++cnt[order[i].b[h]]);
      w += mx;
    }
  return w;
}

// randomised greedy: fill half-warps residue by residue, each lane taking an
// item of an unused 8-byte residue whose dense groups are unused in its
// quarter; restarts with other seeds, keeps the cheapest order
inline std::vector<uint32_t> fibermap_build(const std::vector<FiberItem>& items, int nb) {
  const int n = (int)items.size();
  std::vector<FiberItem> best = items;
  long best_cost = fibermap_cost(items, nb);
  uint64_t state = 0x9e3779b97f4a7c15ull;
  auto rnd = [&]() {
    state ^= state << 13;
    state ^= state >> 7;
    state ^= state << 17;
    return state;
  };
  long ideal = 0;
  for (int h0 = 0; h0 < n; h0 += 16) ideal += 1;
  for (int q0 = 0; q0 < n; q0 += 8) ideal += nb;
  for (int attempt = 0; attempt < 400 && best_cost > ideal; ++attempt) {
    std::vector<FiberItem> pool = items;
    for (int i = n - 1; i > 0; --i) std::swap(pool[i], pool[rnd() % (i + 1)]);
    std::vector<FiberItem> out;
    out.reserve(n);
    std::vector<char> used(n, 0);
    while ((int)out.size() < n) {
      // one half-warp: distinct a; its two quarters: distinct b[h]
      bool ua[16] = {false};
      bool ub[2][2][8] = {};
      const int start = (int)out.size();
      for (int lane = 0; lane < 16 && (int)out.size() < n; ++lane) {
        const int q = lane / 8;
        int pick = -1;
        for (int pass = 0; pass < 2 && pick < 0; ++pass)
          for (int i = 0; i < n; ++i) {
            if (used[i]) continue;
            const FiberItem& it = pool[i];
            if (ua[it.a]) continue;
            bool ok = true;
            for (int h = 0; h < nb && pass == 0; ++h) ok = ok && !ub[q][h][it.b[h]];
            if (ok) { pick = i; break; }
          }
        if (pick < 0)  // nothing fits: any remaining item
          for (int i = 0; i < n; ++i)
            if (!used[i]) { pick = i; break; }
        used[pick] = 1;
        const FiberItem& it = pool[pick];
        ua[it.a] = true;
        for (int h = 0; h < nb; ++h) ub[q][h][it.b[h]] = true;
        out.push_back(it);
      }
      (void)start;
    }
    const long c = fibermap_cost(out, nb);
    if (c < best_cost) {
      best_cost = c;
      best = out;
    }
  }
  std::vector<uint32_t> codes(n);
  for (int i = 0; i < n; ++i) codes[i] = best[i].code;
  return codes;
}

}  // namespace dgb
