// TEST INFRASTRUCTURE (oracle) — not product code.
//
// Replacement for the reference's libpng-backed image_io translation unit
// (/root/reference/proj/src/image_io.cpp:136-182), which cannot be compiled in
// this image because libpng is absent. The hot path never touches file I/O:
// frames enter the solver as in-memory fp64 arrays. These three
// symbols only have to exist so that pipeline.cpp links.
#include <stdexcept>
#include <string>

#include "flowfem/imaging.hpp"

namespace flowfem {

Image load_image(const std::string& path) {
  throw std::runtime_error("imaging.load_image: file I/O is not built in the oracle (" + path +
                           ")");
}

void save_pgm(const std::string&, const Image&) {}

void save_png_rgb(const std::string&, const RgbImage&) {}

}  // namespace flowfem
