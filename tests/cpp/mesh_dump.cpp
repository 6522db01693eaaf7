// Writes every array of build_pixel_mesh(W, H) and the P1 gradients of every triangle to a
// binary file. tests/test_abi.py compiles it twice — against include/flowfem_b200.hpp and
// against the reference's own mesh.hpp + mesh.cpp — and compares the two dumps byte for byte.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "flowfem/mesh.hpp"

template <class T>
void put(std::FILE* f, const std::vector<T>& v) {
  const long long n = static_cast<long long>(v.size());
  std::fwrite(&n, sizeof n, 1, f);
  if (n) std::fwrite(v.data(), sizeof(T), v.size(), f);
}

int main(int argc, char** argv) {
  if (argc < 4) return 2;
  const flowfem::TriMesh m = flowfem::build_pixel_mesh(std::atoi(argv[1]), std::atoi(argv[2]));
  std::FILE* f = std::fopen(argv[3], "wb");
  if (!f) return 3;
  const int hdr[4] = {m.width, m.height, m.n_vertices, m.n_triangles};
  std::fwrite(hdr, sizeof hdr, 1, f);
  put(f, m.tri);
  put(f, m.area);
  put(f, m.hK);
  std::vector<int> ev;
  std::vector<double> eg;
  for (const auto& e : m.edges) {
    ev.insert(ev.end(), {e.v0, e.v1, e.t0, e.t1});
    eg.insert(eg.end(), {e.length, e.nx, e.ny});
  }
  put(f, ev);
  put(f, eg);
  put(f, m.tri_edges);
  put(f, m.lumped);
  put(f, m.v2t_ptr);
  put(f, m.v2t);
  put(f, m.v2v_ptr);
  put(f, m.v2v);
  std::vector<double> g;
  for (int t = 0; t < m.n_triangles; ++t) {
    double gx[3], gy[3];
    flowfem::p1_gradients(m, t, gx, gy);
    g.insert(g.end(), gx, gx + 3);
    g.insert(g.end(), gy, gy + 3);
  }
  put(f, g);
  std::fclose(f);
  return 0;
}
