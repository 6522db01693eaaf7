// Host-side domain decomposition types (include/flowfem/schwarz.hpp:11-57 of the reference).
#pragma once

#include <string>
#include <vector>

namespace ffb {

[[noreturn]] void fail(const std::string& msg);

struct Split {
  int px, py;
  double ratio;
};
struct Rect {
  int x0 = 0, y0 = 0, x1 = 0, y1 = 0;
  int w() const { return x1 - x0; }
  int h() const { return y1 - y0; }
};
struct Neighbor {
  int part;
  Rect band;
  std::vector<int> gamma;
};
struct Part {
  Rect core, ext;
  std::vector<Neighbor> neighbors;
  std::vector<int> boundary;
};
struct Partition {
  int W = 0, H = 0, px = 1, py = 1, ov = 0;
  std::vector<int> xs, ys;
  std::vector<Part> parts;
};

std::vector<Split> enumerate_splits(int W, int H, int n_parts);
Split choose_split(int W, int H, int n_parts);
// rcm_order (linsolve.cpp:37-83) of a CSR system with nc components per vertex (rcm.cpp)
std::vector<int> rcm_order(int n, int nc, const int* row_ptr, const int* cols);
// file I/O (io.cpp): image_io.cpp:19-160, metrics.cpp:22-64
std::vector<double> load_image(const std::string& path, int& W, int& H);
void save_pgm(const std::string& path, int W, int H, const double* img);
void read_flo(const std::string& path, int& W, int& H, std::vector<float>& u,
              std::vector<float>& v);
void write_flo(const std::string& path, int W, int H, const float* u, const float* v);
std::vector<int> assign_workers(int n_workers, int n_parts);
Partition build_partition(int W, int H, int px, int py, int ov);
std::vector<int> flatten(const Partition& P);
Rect free_rect(const Partition& P, int p);

}  // namespace ffb
