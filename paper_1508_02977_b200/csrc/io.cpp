// File I/O around the solver: the reference's image loaders with [0,1]
// normalisation (load_image / load_pgm / load_png, src/image_io.cpp:19-145), save_pgm
// (:147-160) and the Middlebury .flo reader/writer (read_flo / write_flo,
// src/metrics.cpp:22-64). Host code: these are file formats, the arithmetic they feed runs
// on the device. PNG is decoded here on top of zlib (non-interlaced images; the same
// transforms the reference asks libpng for: palette -> RGB, gray < 8 bit expanded to 8 bit,
// alpha stripped, RGB -> 0.299 R + 0.587 G + 0.114 B, divided by 255 or 65535).
#include <zlib.h>

#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "partition.hpp"

namespace ffb {

namespace {

[[noreturn]] void img_fail(const std::string& msg) { fail("imaging.load_image: " + msg); }

int read_pnm_int(std::istream& in) {
  int c = in.get();
  while (c != EOF) {  // whitespace and '#' comments
    if (c == '#') {
      while (c != EOF && c != '\n') c = in.get();
    } else if (!std::isspace(c)) {
      break;
    }
    c = in.get();
  }
  if (c == EOF || !std::isdigit(c)) img_fail("malformed PGM header");
  long long v = 0;
  while (c != EOF && std::isdigit(c)) {
    v = v * 10 + (c - '0');
    if (v > 1000000000LL) img_fail("malformed PGM header");
    c = in.get();
  }
  return static_cast<int>(v);
}

std::vector<double> load_pgm(const std::string& path, int& W, int& H) {
  std::ifstream in(path, std::ios::binary);
  char magic[2];
  in.read(magic, 2);
  if (!in || magic[0] != 'P' || magic[1] != '5') img_fail("not a binary PGM: " + path);
  const int w = read_pnm_int(in), h = read_pnm_int(in), maxval = read_pnm_int(in);
  if (w <= 0 || h <= 0 || maxval <= 0 || maxval > 65535)
    img_fail("bad PGM dimensions in " + path);
  const size_t n = static_cast<size_t>(w) * h;
  std::vector<double> img(n);
  const int bpp = maxval < 256 ? 1 : 2;
  std::vector<unsigned char> buf(bpp * n);
  in.read(reinterpret_cast<char*>(buf.data()), static_cast<std::streamsize>(buf.size()));
  if (!in) img_fail("truncated PGM data in " + path);
  for (size_t i = 0; i < n; ++i) {
    const unsigned v = bpp == 1 ? buf[i] : (unsigned(buf[2 * i]) << 8) | buf[2 * i + 1];
    img[i] = v / double(maxval);
  }
  W = w, H = h;
  return img;
}

uint32_t be32(const unsigned char* p) {
  return (uint32_t(p[0]) << 24) | (uint32_t(p[1]) << 16) | (uint32_t(p[2]) << 8) | p[3];
}

int paeth(int a, int b, int c) {
  const int p = a + b - c, pa = std::abs(p - a), pb = std::abs(p - b), pc = std::abs(p - c);
  return (pa <= pb && pa <= pc) ? a : (pb <= pc ? b : c);
}

std::vector<double> load_png(const std::string& path, int& W, int& H) {
  std::ifstream in(path, std::ios::binary);
  if (!in) img_fail("cannot open " + path);
  std::vector<unsigned char> file((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  static const unsigned char sig[8] = {0x89, 'P', 'N', 'G', 0x0d, 0x0a, 0x1a, 0x0a};
  if (file.size() < 8 || std::memcmp(file.data(), sig, 8) != 0) img_fail("bad PNG signature in " + path);
  uint32_t w = 0, h = 0;
  int depth = 0, color = -1, interlace = 0;
  std::vector<unsigned char> idat, plte, trns;
  size_t pos = 8;
  bool have_ihdr = false, have_iend = false;
  while (pos + 12 <= file.size()) {
    const uint32_t len = be32(&file[pos]);
    if (pos + 12 + static_cast<size_t>(len) > file.size()) img_fail("truncated PNG chunk in " + path);
    const std::string type(reinterpret_cast<const char*>(&file[pos + 4]), 4);
    const unsigned char* d = &file[pos + 8];
    if (type == "IHDR" && len >= 13) {
      w = be32(d), h = be32(d + 4), depth = d[8], color = d[9], interlace = d[12];
      have_ihdr = true;
    } else if (type == "PLTE") {
      plte.assign(d, d + len);
    } else if (type == "tRNS") {
      trns.assign(d, d + len);
    } else if (type == "IDAT") {
      idat.insert(idat.end(), d, d + len);
    } else if (type == "IEND") {
      have_iend = true;
      break;
    }
    pos += 12 + len;
  }
  if (!have_ihdr || !have_iend) img_fail("libpng error reading " + path);
  if (w == 0 || h == 0 || w > 100000 || h > 100000) img_fail("bad PNG dimensions in " + path);
  if (interlace) img_fail("interlaced PNG is not supported: " + path);
  int samples;  // per pixel in the stored stream
  switch (color) {
    case 0: samples = 1; break;
    case 2: samples = 3; break;
    case 3: samples = 1; break;
    case 4: samples = 2; break;
    case 6: samples = 4; break;
    default: img_fail("libpng error reading " + path);
  }
  const bool ok_depth = (color == 0 && (depth == 1 || depth == 2 || depth == 4 || depth == 8 || depth == 16)) ||
                        (color == 3 && (depth == 1 || depth == 2 || depth == 4 || depth == 8)) ||
                        ((color == 2 || color == 4 || color == 6) && (depth == 8 || depth == 16));
  if (!ok_depth) img_fail("libpng error reading " + path);
  const size_t bits_pp = static_cast<size_t>(samples) * depth;
  const size_t rowbytes = (bits_pp * w + 7) / 8;
  const size_t bpp = std::max<size_t>(1, bits_pp / 8);  // filter byte distance
  std::vector<unsigned char> raw((rowbytes + 1) * h);
  uLongf out_len = static_cast<uLongf>(raw.size());
  if (uncompress(raw.data(), &out_len, idat.data(), static_cast<uLong>(idat.size())) != Z_OK ||
      out_len != raw.size())
    img_fail("libpng error reading " + path);
  // unfilter in place (PNG filter types 0-4)
  std::vector<unsigned char> prev(rowbytes, 0), cur(rowbytes);
  std::vector<unsigned char> pix(rowbytes * h);
  for (uint32_t y = 0; y < h; ++y) {
    const unsigned char ft = raw[y * (rowbytes + 1)];
    const unsigned char* src = &raw[y * (rowbytes + 1) + 1];
    for (size_t i = 0; i < rowbytes; ++i) {
      const int a = i >= bpp ? cur[i - bpp] : 0, b = prev[i], c = i >= bpp ? prev[i - bpp] : 0;
      int v = src[i];
      switch (ft) {
        case 0: break;
        case 1: v += a; break;
        case 2: v += b; break;
        case 3: v += (a + b) >> 1; break;
        case 4: v += paeth(a, b, c); break;
        default: img_fail("libpng error reading " + path);
      }
      cur[i] = static_cast<unsigned char>(v);
    }
    std::memcpy(&pix[y * rowbytes], cur.data(), rowbytes);
    prev.swap(cur);
  }
  auto sample = [&](uint32_t y, size_t idx) -> unsigned {  // idx-th sample of row y
    const unsigned char* row = &pix[y * rowbytes];
    if (depth == 16) return (unsigned(row[2 * idx]) << 8) | row[2 * idx + 1];
    if (depth == 8) return row[idx];
    const size_t bit = idx * depth;
    return (row[bit / 8] >> (8 - depth - bit % 8)) & ((1u << depth) - 1);
  };
  std::vector<double> img(static_cast<size_t>(w) * h);
  const double scale = depth == 16 ? 65535.0 : 255.0;
  for (uint32_t y = 0; y < h; ++y)
    for (uint32_t x = 0; x < w; ++x) {
      double v;
      if (color == 3) {  // palette -> RGB
        const unsigned k = sample(y, x);
        if (3 * k + 2 >= plte.size()) img_fail("libpng error reading " + path);
        const double r = plte[3 * k] / scale, g = plte[3 * k + 1] / scale, b = plte[3 * k + 2] / scale;
        v = 0.299 * r + 0.587 * g + 0.114 * b;
      } else if (color == 2 || color == 6) {
        const double r = sample(y, x * samples) / scale, g = sample(y, x * samples + 1) / scale,
                     b = sample(y, x * samples + 2) / scale;
        v = 0.299 * r + 0.587 * g + 0.114 * b;
      } else {  // gray (+alpha); < 8 bit expanded to the 8-bit range
        unsigned s = sample(y, x * samples);
        if (depth < 8) s = s * 255u / ((1u << depth) - 1);
        v = s / scale;
      }
      img[static_cast<size_t>(y) * w + x] = v;
    }
  W = static_cast<int>(w), H = static_cast<int>(h);
  return img;
}

const float kFloMagic = 202021.25f;  // metrics.hpp:25

}  // namespace

// load_image (image_io.cpp:136-145): dispatch on the signature
std::vector<double> load_image(const std::string& path, int& W, int& H) {
  std::ifstream probe(path, std::ios::binary);
  if (!probe) img_fail("cannot open " + path);
  unsigned char s[2] = {0, 0};
  probe.read(reinterpret_cast<char*>(s), 2);
  probe.close();
  if (s[0] == 'P' && s[1] == '5') return load_pgm(path, W, H);
  if (s[0] == 0x89 && s[1] == 'P') return load_png(path, W, H);
  img_fail("unrecognized format (want PGM P5 or PNG): " + path);
}

// save_pgm (image_io.cpp:147-160): clamp to [0,1], 8-bit, round half up
void save_pgm(const std::string& path, int W, int H, const double* img) {
  std::ofstream out(path, std::ios::binary);
  if (!out) fail("imaging.save_pgm: cannot open " + path);
  out << "P5\n" << W << " " << H << "\n255\n";
  const size_t n = static_cast<size_t>(W) * H;
  std::vector<unsigned char> buf(n);
  for (size_t i = 0; i < n; ++i) {
    double v = img[i];
    v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    buf[i] = static_cast<unsigned char>(v * 255.0 + 0.5);
  }
  out.write(reinterpret_cast<const char*>(buf.data()), static_cast<std::streamsize>(n));
  if (!out) fail("imaging.save_pgm: write failed for " + path);
}

// read_flo (metrics.cpp:22-45): magic, int32 w, h, then rows of interleaved (u, v) float32
void read_flo(const std::string& path, int& W, int& H, std::vector<float>& u,
              std::vector<float>& v) {
  std::ifstream in(path, std::ios::binary);
  if (!in) fail("metrics.read_flo: cannot open " + path);
  float magic = 0.0f;
  int32_t w = 0, h = 0;
  in.read(reinterpret_cast<char*>(&magic), 4);
  in.read(reinterpret_cast<char*>(&w), 4);
  in.read(reinterpret_cast<char*>(&h), 4);
  if (!in || magic != kFloMagic) fail("metrics.read_flo: bad magic in " + path);
  if (w <= 0 || h <= 0 || w > 100000 || h > 100000)
    fail("metrics.read_flo: implausible dimensions in " + path);
  const size_t n = static_cast<size_t>(w) * h;
  u.assign(n, 0.0f), v.assign(n, 0.0f);
  std::vector<float> row(static_cast<size_t>(w) * 2);
  for (int y = 0; y < h; ++y) {
    in.read(reinterpret_cast<char*>(row.data()), static_cast<std::streamsize>(row.size() * 4));
    if (!in) fail("metrics.read_flo: truncated data in " + path);
    for (int x = 0; x < w; ++x) {
      u[static_cast<size_t>(y) * w + x] = row[2 * x];
      v[static_cast<size_t>(y) * w + x] = row[2 * x + 1];
    }
  }
  W = w, H = h;
}

// write_flo (metrics.cpp:47-64)
void write_flo(const std::string& path, int W, int H, const float* u, const float* v) {
  std::ofstream out(path, std::ios::binary);
  if (!out) fail("metrics.write_flo: cannot open " + path);
  const int32_t w = W, h = H;
  out.write(reinterpret_cast<const char*>(&kFloMagic), 4);
  out.write(reinterpret_cast<const char*>(&w), 4);
  out.write(reinterpret_cast<const char*>(&h), 4);
  std::vector<float> row(static_cast<size_t>(W) * 2);
  for (int y = 0; y < H; ++y) {
    for (int x = 0; x < W; ++x) {
      row[2 * x] = u[static_cast<size_t>(y) * W + x];
      row[2 * x + 1] = v[static_cast<size_t>(y) * W + x];
    }
    out.write(reinterpret_cast<const char*>(row.data()), static_cast<std::streamsize>(row.size() * 4));
  }
  if (!out) fail("metrics.write_flo: write failed for " + path);
}

}  // namespace ffb
