// Drop-in check through the C++ shim: reads a system exported by
// tests/test_cpp_shim.py (raw little-endian doubles), runs the reference-shaped
// calls (apply_S, deflated_solve) and writes the results back.
#include <cstdio>
#include <fstream>
#include <iostream>
#include <vector>

#include "smpm_b200.hpp"

static std::vector<double> load(const std::string& path, size_t n) {
  std::vector<double> v(n);
  std::ifstream f(path, std::ios::binary);
  f.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(n * sizeof(double)));
  if (!f) throw std::runtime_error("cannot read " + path);
  return v;
}
static void save(const std::string& path, const std::vector<double>& v) {
  std::ofstream f(path, std::ios::binary);
  f.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(double)));
}

int main(int argc, char** argv) {
  if (argc < 5) return 2;
  const std::string dir = argv[1];
  const int n = std::atoi(argv[2]), mx = std::atoi(argv[3]), mz = std::atoi(argv[4]);
  const size_t w = static_cast<size_t>(n) * mz, k = 2 * w * (mx - 1);
  smpm_b200::Device dev(0);
  smpm_b200::System sys(dev, n, mx, mz);
  auto gw = load(dir + "/G_W.bin", w * w), gi = load(dir + "/G_I.bin", 4 * w * w), ge = load(dir + "/G_E.bin", w * w);
  sys.set_couplings(gw.data(), gi.data(), ge.data());
  sys.set_nullspace(load(dir + "/u_S.bin", k));
  sys.finalize();
  const auto b = load(dir + "/b_S.bin", k);
  save(dir + "/Sb.bin", smpm_b200::apply_S(sys, b));
  const auto r = smpm_b200::deflated_solve(sys, b, 1e-10, 50, 50);
  save(dir + "/x_S.bin", r.x_S);
  std::printf("%d %d %.3e %lld\n", r.report.iterations, r.report.converged ? 1 : 0, r.report.final_rel_residual,
              static_cast<long long>(r.krylov_s_applies));
  try {
    smpm_b200::apply_S(sys, std::vector<double>(k + 1));
    return 3;  // must have thrown std::invalid_argument
  } catch (const std::invalid_argument&) {
  }
  return 0;
}
