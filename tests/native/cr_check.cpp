// Host check of the product's correctly-rounded sin/cos/atan2
// (paper_2509_17340_b200/csrc/cr_math.cuh) against glibc libm, which the
// reference links.  Prints one JSON line with mismatch counts.
// Built and run by tests/test_cr_math.py with g++ -O2 -ffp-contract=off.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <initializer_list>
#include <numbers>

#include "../../paper_2509_17340_b200/csrc/cr_math.cuh"

namespace {
std::uint64_t state = 0x243F6A8885A308D3ull;
std::uint64_t next() {
  std::uint64_t z = (state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
double uni(double lo, double hi) { return lo + (hi - lo) * (static_cast<double>(next() >> 11) * 0x1.0p-53); }
}  // namespace

int main(int argc, char** argv) {
  const long n = argc > 1 ? std::atol(argv[1]) : 1000000;
  constexpr double kPi = std::numbers::pi;
  long bad_sin = 0, bad_cos = 0, bad_atan2 = 0, bad_atan2_struct = 0, bad_struct_trig = 0;
  long n_struct = 0, n_struct_trig = 0;
  for (long i = 0; i < n; ++i) {
    const double x = uni(-7.0, 7.0);
    if (crm::sin_cr(x) != std::sin(x)) ++bad_sin;
    if (crm::cos_cr(x) != std::cos(x)) ++bad_cos;
    const double a = uni(-20.0, 20.0), b = uni(-20.0, 20.0);
    if (crm::atan2_cr(a, b) != std::atan2(a, b)) ++bad_atan2;
  }
  // structured: angles on the 3 degree / 18 degree lattices, as the anchor
  // sampler and cell_direction produce them (guidance.cpp:16-38)
  const double spacing = 18.0 * kPi / 180.0;
  for (int k = -40; k <= 40; ++k) {
    for (double off : {0.0, 0.5, -0.5, 1.5, -1.5, 1.0, -1.0, 2.0, -2.0}) {
      const double ang = k * (3.0 * kPi / 180.0) + off * spacing;
      ++n_struct_trig;
      if (crm::sin_cr(ang) != std::sin(ang) || crm::cos_cr(ang) != std::cos(ang)) ++bad_struct_trig;
      for (double r : {0.3, 1.0, 5.0, 9.7}) {
        const double ce = std::cos(0.1 * k);
        const double px = r * ce * std::cos(ang), py = r * ce * std::sin(ang);
        ++n_struct;
        if (crm::atan2_cr(py, px) != std::atan2(py, px)) ++bad_atan2_struct;
      }
    }
  }
  std::printf(
      "{\"n\": %ld, \"sin\": %ld, \"cos\": %ld, \"atan2\": %ld, \"struct_trig_n\": %ld, \"struct_trig\": %ld, "
      "\"struct_atan2_n\": %ld, \"struct_atan2\": %ld}\n",
      n, bad_sin, bad_cos, bad_atan2, n_struct_trig, bad_struct_trig, n_struct, bad_atan2_struct);
  return 0;
}
