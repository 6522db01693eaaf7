// Reverse Cuthill-McKee ordering of a SparseSystem's free-vertex graph, expanded to scalar
// unknowns: the symbolic step of the linsolve boundary's direct solve (rcm_order,
// linsolve.hpp:22-24, linsolve.cpp:37-83). Host integer work, bit-exact with the reference:
//   * block adjacency from each vertex's first-component row, consecutive duplicates and the
//     vertex itself dropped (linsolve.cpp:20-33);
//   * each BFS starts at the unvisited vertex of minimum degree (smallest id on ties) and
//     visits unvisited neighbours by (degree, id); the concatenated order is reversed.
#include <algorithm>
#include <string>
#include <vector>

#include "partition.hpp"

namespace ffb {

std::vector<int> rcm_order(int n, int nc, const int* row_ptr, const int* cols) {
  if (nc <= 0 || n % nc != 0) fail("linsolve.rcm_order: system size not a multiple of components");
  const int nb = n / nc;
  std::vector<int> adj_ptr(nb + 1, 0), adj;
  adj.reserve(row_ptr[n] / std::max(nc, 1) + 1);
  for (int b = 0; b < nb; ++b) {
    int last = -1;
    for (int q = row_ptr[b * nc]; q < row_ptr[b * nc + 1]; ++q) {
      const int k = cols[q] / nc;
      if (k != b && k != last) adj.push_back(k);
      last = k;
    }
    adj_ptr[b + 1] = static_cast<int>(adj.size());
  }
  std::vector<int> degree(nb);
  for (int b = 0; b < nb; ++b) degree[b] = adj_ptr[b + 1] - adj_ptr[b];
  std::vector<char> visited(nb, 0);
  std::vector<int> order, nbrs;
  order.reserve(nb);
  int scanned = 0;
  while (static_cast<int>(order.size()) < nb) {
    int start = -1;
    for (int b = scanned; b < nb; ++b)
      if (!visited[b] && (start < 0 || degree[b] < degree[start])) start = b;
    while (scanned < nb && visited[scanned]) ++scanned;
    visited[start] = 1;
    size_t head = order.size();
    order.push_back(start);
    while (head < order.size()) {
      const int v = order[head++];
      nbrs.clear();
      for (int q = adj_ptr[v]; q < adj_ptr[v + 1]; ++q)
        if (!visited[adj[q]]) nbrs.push_back(adj[q]);
      std::sort(nbrs.begin(), nbrs.end(), [&](int a, int b) {
        return degree[a] != degree[b] ? degree[a] < degree[b] : a < b;
      });
      for (int w : nbrs) {
        visited[w] = 1;
        order.push_back(w);
      }
    }
  }
  std::vector<int> perm(n);
  for (int i = 0; i < nb; ++i)
    for (int c = 0; c < nc; ++c) perm[i * nc + c] = order[nb - 1 - i] * nc + c;
  return perm;
}

}  // namespace ffb
