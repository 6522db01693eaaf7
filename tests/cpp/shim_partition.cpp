// Host-only check of the C++ layer (include/flowfem_b200.hpp): the decomposition entry points
// through the C-ABI, with the reference's known answers (test_schwarz.cpp:46-147).
#include <cstdio>
#include <stdexcept>

#include "flowfem_b200.hpp"

int main() {
  namespace ff = flowfem_b200;
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
  std::printf("shim ok\n");
  return 0;
}
