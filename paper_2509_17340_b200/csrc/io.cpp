// Wire / on-disk formats around the plan path:
//   * the reference's text cloud frame "# amppi-cloud v1" (io.cpp:24-66),
//     %.17g per coordinate, so a double survives the round trip exactly;
//   * a binary variant "# amppi-cloud-bin v1" (header line, frame id and point
//     count as little-endian u64, then n x 3 float64) that loads with one read
//     straight into a caller (e.g. pinned) buffer;
//   * the debug dumps partition.csv (io.cpp:68-76) and anchors.csv
//     (io.cpp:78-99) in the reference's row order and number format.
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/amppi_b200.h"

namespace {

const char kTextHeader[] = "# amppi-cloud v1";
const char kBinHeader[] = "# amppi-cloud-bin v1\n";

struct File {
  FILE* f;
  explicit File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
  ~File() {
    if (f) std::fclose(f);
  }
};

bool read_line(FILE* f, std::string& line) {
  line.clear();
  int c;
  while ((c = std::fgetc(f)) != EOF) {
    if (c == '\n') return true;
    line.push_back(static_cast<char>(c));
  }
  return !line.empty();
}

void put(FILE* f, double v, char sep) { std::fprintf(f, "%.17g%c", v, sep); }

}  // namespace

extern "C" {

int amppi_cloud_read(const char* path, double* xyz, int64_t cap, int64_t* n_points, uint64_t* frame_id) {
  if (!path || !n_points) return AMPPI_INVALID_ARGUMENT;
  File in(path, "rb");
  if (!in.f) return AMPPI_INVALID_ARGUMENT;
  std::string line;
  if (!read_line(in.f, line)) return AMPPI_INVALID_ARGUMENT;
  if (line + "\n" == kBinHeader) {
    uint64_t id = 0, n = 0;
    if (std::fread(&id, sizeof(id), 1, in.f) != 1 || std::fread(&n, sizeof(n), 1, in.f) != 1)
      return AMPPI_INVALID_ARGUMENT;
    *n_points = static_cast<int64_t>(n);
    if (frame_id) *frame_id = id;
    const int64_t take = std::min<int64_t>(static_cast<int64_t>(n), cap);
    if (xyz && take > 0 && std::fread(xyz, sizeof(double) * 3, static_cast<size_t>(take), in.f) !=
                               static_cast<size_t>(take))
      return AMPPI_INVALID_ARGUMENT;
    return AMPPI_OK;
  }
  // read_cloud_frame (io.cpp:38-56): header, "frame <id>", then "x y z" lines
  if (line.rfind(kTextHeader, 0) != 0) return AMPPI_INVALID_ARGUMENT;
  if (!read_line(in.f, line) || line.rfind("frame ", 0) != 0) return AMPPI_INVALID_ARGUMENT;
  if (frame_id) *frame_id = std::strtoull(line.c_str() + 6, nullptr, 10);
  int64_t n = 0;
  while (read_line(in.f, line)) {
    if (line.empty()) continue;
    const char* s = line.c_str();
    char* end = nullptr;
    double v[3];
    for (int a = 0; a < 3; ++a) {
      errno = 0;
      v[a] = std::strtod(s, &end);
      if (end == s) return AMPPI_INVALID_ARGUMENT;  // malformed cloud point line
      s = end;
    }
    if (xyz && n < cap)
      for (int a = 0; a < 3; ++a) xyz[3 * n + a] = v[a];
    ++n;
  }
  *n_points = n;
  return AMPPI_OK;
}

int amppi_cloud_write(const char* path, const double* xyz, int64_t n_points, uint64_t frame_id, int32_t binary) {
  if (!path || (n_points > 0 && !xyz) || n_points < 0) return AMPPI_INVALID_ARGUMENT;
  File out(path, "wb");
  if (!out.f) return AMPPI_INVALID_ARGUMENT;
  if (binary) {
    const uint64_t id = frame_id, n = static_cast<uint64_t>(n_points);
    std::fwrite(kBinHeader, 1, sizeof(kBinHeader) - 1, out.f);
    std::fwrite(&id, sizeof(id), 1, out.f);
    std::fwrite(&n, sizeof(n), 1, out.f);
    if (n_points > 0) std::fwrite(xyz, sizeof(double) * 3, static_cast<size_t>(n_points), out.f);
    return std::ferror(out.f) ? AMPPI_INVALID_ARGUMENT : AMPPI_OK;
  }
  // write_cloud_frame (io.cpp:24-35)
  std::fprintf(out.f, "%s\nframe %llu\n", kTextHeader, static_cast<unsigned long long>(frame_id));
  for (int64_t i = 0; i < n_points; ++i) {
    put(out.f, xyz[3 * i], ' ');
    put(out.f, xyz[3 * i + 1], ' ');
    put(out.f, xyz[3 * i + 2], '\n');
  }
  return std::ferror(out.f) ? AMPPI_INVALID_ARGUMENT : AMPPI_OK;
}

int amppi_partition_csv(const char* path, const double* ranges) {  // write_partition_csv (io.cpp:68-76)
  if (!path || !ranges) return AMPPI_INVALID_ARGUMENT;
  File out(path, "wb");
  if (!out.f) return AMPPI_INVALID_ARGUMENT;
  std::fprintf(out.f, "i,j,range\n");
  for (int i = 0; i < 120; ++i)
    for (int j = 0; j < 60; ++j) {
      std::fprintf(out.f, "%d,%d,", i, j);
      put(out.f, ranges[i * 60 + j], '\n');
    }
  return std::ferror(out.f) ? AMPPI_INVALID_ARGUMENT : AMPPI_OK;
}

int amppi_anchors_csv(const char* path, int32_t step, int32_t n_anchors, const double* refined,
                      const double* guide_coeffs, double horizon, int32_t samples) {
  // write_anchors_csv (io.cpp:78-99): per anchor its refined endpoint, then
  // `samples` points of eval_guide at horizon * s / samples (guidance.cpp:96-101)
  if (!path || n_anchors < 0 || (n_anchors > 0 && !refined)) return AMPPI_INVALID_ARGUMENT;
  File out(path, "wb");
  if (!out.f) return AMPPI_INVALID_ARGUMENT;
  std::fprintf(out.f, "step,anchor,x,y,z\n");
  auto row = [&](int a, double x, double y, double z) {
    std::fprintf(out.f, "%d,%d,", step, a);
    put(out.f, x, ',');
    put(out.f, y, ',');
    put(out.f, z, '\n');
  };
  for (int a = 0; a < n_anchors; ++a) {
    row(a, refined[3 * a], refined[3 * a + 1], refined[3 * a + 2]);
    if (!guide_coeffs) continue;
    const double* c = guide_coeffs + 18 * a;  // [axis][power]
    for (int s = 1; s <= samples; ++s) {
      double t = horizon * s / samples;
      t = t < 0.0 ? 0.0 : (t > horizon ? horizon : t);
      double p[3];
      for (int ax = 0; ax < 3; ++ax) {
        double o = c[6 * ax + 5];
        for (int k = 4; k >= 0; --k) o = o * t + c[6 * ax + k];
        p[ax] = o;
      }
      row(a, p[0], p[1], p[2]);
    }
  }
  return std::ferror(out.f) ? AMPPI_INVALID_ARGUMENT : AMPPI_OK;
}

}  // extern "C"
