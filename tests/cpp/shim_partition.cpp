// Host-only check of the C++ layer (include/flowfem_b200.hpp): the decomposition entry points
// through the C-ABI, with the reference's known answers (test_schwarz.cpp:46-147).
#include <cstdio>
#include <stdexcept>

#include "flowfem_b200.hpp"

int main() {
  namespace ff = flowfem;
  const auto s = ff::choose_split(96, 80, 4);
  if (s.parts_x != 2 || s.parts_y != 2) return 1;
  const auto all = ff::enumerate_splits(640, 480, 12);
  if (all.size() != 6) return 2;
  if (ff::choose_split(640, 480, 12).parts_x != 4) return 3;
  const auto P = ff::build_partition(97, 83, 3, 4, 4);
  if (P.parts.size() != 12) return 4;
  for (const auto& p : P.parts) {
    size_t g = 0;
    for (const auto& nb : p.neighbors) g += nb.gamma.size();
    if (g != p.boundary.size()) return 5;
  }
  try {
    ff::build_partition(20, 20, 2, 1, 5);
    return 6;
  } catch (const std::runtime_error& e) {
    if (std::string(e.what()).find("schwarz.build_partition: core 10x20") != 0) return 7;
  }
  if (ff::assign_workers(7, 3)[6] != 0) return 8;
  // host-side parts of the linsolve and I/O layers (linsolve.cpp:37-83, image_io, metrics)
  {
    ff::SparseSystem sys;  // 1-D chain of 4 vertices, 1 component: RCM from vertex 0 reversed
    sys.n = 4;
    sys.components = 1;
    sys.row_ptr = {0, 2, 5, 8, 10};
    sys.cols = {0, 1, 0, 1, 2, 1, 2, 3, 2, 3};
    sys.vals.assign(10, 1.0);
    const auto perm = ff::rcm_order(sys);
    if (perm.size() != 4 || perm[0] != 3 || perm[3] != 0) return 9;
    ff::Image img(3, 2);
    for (size_t i = 0; i < img.data.size(); ++i) img.data[i] = i / 5.0;
    ff::save_pgm("shim_tmp.pgm", img);
    const ff::Image back = ff::load_image("shim_tmp.pgm");
    if (back.width != 3 || back.height != 2 || back.data[5] != 1.0 || back.data[1] != 51 / 255.0)
      return 10;
    ff::FloField f;
    f.width = 2, f.height = 1, f.u = {1.5f, -2.0f}, f.v = {0.25f, 3.0f};
    ff::write_flo("shim_tmp.flo", f);
    const ff::FloField g = ff::read_flo("shim_tmp.flo");
    if (g.width != 2 || g.u[1] != -2.0f || g.v[0] != 0.25f) return 11;
    std::remove("shim_tmp.pgm");
    std::remove("shim_tmp.flo");
  }
  std::printf("shim ok\n");
  return 0;
}
