// Host-side domain decomposition: split choice, partition construction and worker
// assignment (src/schwarz.cpp:16-128). Integer work on the host; results are bit-exact
// with the reference (pinned field by field against it in tests/test_partition.py).
#include "partition.hpp"

#include <algorithm>
#include <cmath>
#include <string>

namespace ffb {

// enumerate_splits, schwarz.cpp:16-30
std::vector<Split> enumerate_splits(int W, int H, int n_parts) {
  if (n_parts < 1) fail("schwarz.enumerate_splits: n_parts must be >= 1");
  std::vector<Split> out;
  for (int px = 1; px <= n_parts; ++px) {
    if (n_parts % px != 0) continue;
    const int py = n_parts / px;
    const double cw = double(W) / px, ch = double(H) / py;
    out.push_back({px, py, (cw * ch) / (2.0 * (cw + ch))});
  }
  return out;
}

// choose_split, schwarz.cpp:32-44: max ratio, ties (relative 1e-9) prefer px >= py
Split choose_split(int W, int H, int n_parts) {
  const auto all = enumerate_splits(W, H, n_parts);
  Split best = all.front();
  for (const auto& s : all) {
    const double tol = 1e-9 * std::max(1.0, best.ratio);
    if (s.ratio > best.ratio + tol)
      best = s;
    else if (std::abs(s.ratio - best.ratio) <= tol && s.px >= s.py && best.px < best.py)
      best = s;
  }
  return best;
}

// assign_workers, schwarz.cpp:46-52
std::vector<int> assign_workers(int n_workers, int n_parts) {
  if (n_workers < 1 || n_parts < 1) fail("schwarz.assign_workers: counts must be >= 1");
  std::vector<int> a(n_workers);
  for (int w = 0; w < n_workers; ++w) a[w] = w % n_parts;
  return a;
}

// build_partition, schwarz.cpp:54-128
Partition build_partition(int W, int H, int px, int py, int ov) {
  if (px < 1 || py < 1) fail("schwarz.build_partition: part counts must be >= 1");
  if (ov < 1 && px * py > 1) fail("schwarz.build_partition: overlap must be >= 1");
  Partition P;
  P.W = W, P.H = H, P.px = px, P.py = py, P.ov = ov;
  P.xs.resize(px + 1);
  P.ys.resize(py + 1);
  for (int i = 0; i <= px; ++i) P.xs[i] = static_cast<int>(static_cast<long long>(i) * W / px);
  for (int j = 0; j <= py; ++j) P.ys[j] = static_cast<int>(static_cast<long long>(j) * H / py);
  const int np = px * py;
  P.parts.resize(np);
  for (int j = 0; j < py; ++j)
    for (int i = 0; i < px; ++i) {
      Part& s = P.parts[j * px + i];
      s.core = {P.xs[i], P.ys[j], P.xs[i + 1], P.ys[j + 1]};
      if (np > 1 && (s.core.w() <= 2 * ov || s.core.h() <= 2 * ov))
        fail("schwarz.build_partition: core " + std::to_string(s.core.w()) + "x" +
             std::to_string(s.core.h()) + " not larger than twice the overlap " +
             std::to_string(ov));
      s.ext = {std::max(0, s.core.x0 - ov), std::max(0, s.core.y0 - ov),
               std::min(W, s.core.x1 + ov), std::min(H, s.core.y1 + ov)};
    }
  auto owner = [&](int x, int y) {
    const int i = int(std::upper_bound(P.xs.begin(), P.xs.end(), x) - P.xs.begin()) - 1;
    const int j = int(std::upper_bound(P.ys.begin(), P.ys.end(), y) - P.ys.begin()) - 1;
    return j * px + i;
  };
  for (int p = 0; p < np; ++p) {
    Part& s = P.parts[p];
    const Rect& e = s.ext;
    // artificial ring of ext, row-major (ascending vertex id)
    std::vector<std::pair<int, int>> owned;
    for (int y = e.y0; y < e.y1; ++y) {
      const bool edge_row = y == e.y0 || y == e.y1 - 1;
      for (int x = e.x0; x < e.x1; ++x) {
        if (!edge_row && x != e.x0 && x != e.x1 - 1) continue;
        const bool art = (x == e.x0 && e.x0 > 0) || (x == e.x1 - 1 && e.x1 < W) ||
                         (y == e.y0 && e.y0 > 0) || (y == e.y1 - 1 && e.y1 < H);
        if (!art) continue;
        const int v = y * W + x;
        s.boundary.push_back(v);
        owned.emplace_back(owner(x, y), v);
      }
    }
    for (int q = 0; q < np; ++q) {
      if (q == p) continue;
      Neighbor nb;
      nb.part = q;
      for (const auto& [o, v] : owned)
        if (o == q) nb.gamma.push_back(v);
      if (nb.gamma.empty()) continue;
      const Rect& f = P.parts[q].ext;
      nb.band = {std::max(e.x0, f.x0), std::max(e.y0, f.y0), std::min(e.x1, f.x1),
                 std::min(e.y1, f.y1)};
      s.neighbors.push_back(std::move(nb));
    }
  }
  return P;
}

std::vector<int> flatten(const Partition& P) {
  std::vector<int> out = {P.W, P.H, P.px, P.py, P.ov, static_cast<int>(P.parts.size())};
  for (const auto& s : P.parts) {
    const int h[10] = {s.core.x0, s.core.y0, s.core.x1, s.core.y1, s.ext.x0, s.ext.y0,
                       s.ext.x1,  s.ext.y1,  static_cast<int>(s.boundary.size()),
                       static_cast<int>(s.neighbors.size())};
    out.insert(out.end(), h, h + 10);
  }
  for (const auto& s : P.parts) {
    out.insert(out.end(), s.boundary.begin(), s.boundary.end());
    for (const auto& nb : s.neighbors) {
      const int h[6] = {nb.part, nb.band.x0, nb.band.y0, nb.band.x1, nb.band.y1,
                        static_cast<int>(nb.gamma.size())};
      out.insert(out.end(), h, h + 6);
      out.insert(out.end(), nb.gamma.begin(), nb.gamma.end());
    }
  }
  return out;
}

Rect free_rect(const Partition& P, int p) {
  // ext minus the artificial Dirichlet ring (the `boundary` vertices of schwarz.cpp:93-112)
  const Rect& e = P.parts[p].ext;
  return {e.x0 + (e.x0 > 0 ? 1 : 0), e.y0 + (e.y0 > 0 ? 1 : 0), e.x1 - (e.x1 < P.W ? 1 : 0),
          e.y1 - (e.y1 < P.H ? 1 : 0)};
}

}  // namespace ffb
