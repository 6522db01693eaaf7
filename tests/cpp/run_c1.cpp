// A C++ caller of the reference API compiled against include/flowfem_b200.hpp (the drop-in)
// and linked with libflowfem_b200.so: reads a frame pair (raw fp64, H x W each), runs
// flowfem::run_on_frames with the converged-pass protocol of config c1 (3 adaptive passes,
// 2x2 subdomains, overlap 4, sigma 1) and writes u1, u2, mt and alpha (raw fp64).
//   run_c1 W H frames.bin out.bin
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

#include "flowfem/pipeline.hpp"

int main(int argc, char** argv) {
  if (argc < 5) return 2;
  const int W = std::atoi(argv[1]), H = std::atoi(argv[2]);
  flowfem::Image f0(W, H), f1(W, H);
  std::FILE* in = std::fopen(argv[3], "rb");
  if (!in || std::fread(f0.data.data(), sizeof(double), f0.size(), in) != f0.size() ||
      std::fread(f1.data.data(), sizeof(double), f1.size(), in) != f1.size())
    return 3;
  std::fclose(in);
  flowfem::RunConfig cfg;
  cfg.sigma = 1.0;
  cfg.parts = 4;
  cfg.overlap = 4;
  cfg.adapt_iters = 3;
  cfg.cg_tolerance = 1e-10;
  cfg.protocol = "converged";
  try {
    const flowfem::RunResult r = flowfem::run_on_frames(f0, f1, cfg);
    std::FILE* out = std::fopen(argv[4], "wb");
    std::fwrite(r.flow.u1.data(), sizeof(double), r.flow.u1.size(), out);
    std::fwrite(r.flow.u2.data(), sizeof(double), r.flow.u2.size(), out);
    std::fwrite(r.flow.mt.data(), sizeof(double), r.flow.mt.size(), out);
    std::fwrite(r.reg.alpha.data(), sizeof(double), r.reg.alpha.size(), out);
    std::fclose(out);
    // the reference's error convention through the drop-in
    flowfem::Image tiny(1, 1);
    try {
      flowfem::run_on_frames(tiny, tiny, cfg);
      return 4;
    } catch (const std::runtime_error& e) {
      std::printf("%s\n", e.what());
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "run_c1: %s\n", e.what());
    return 1;
  }
  std::printf("run_c1 ok\n");
  return 0;
}
