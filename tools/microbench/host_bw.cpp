// Host memory bandwidth with T threads: each copies its slice of a 4 GB
// buffer (read + write) and expands an upper triangle into a full matrix
// (the work a symmetric-K host path would add).  g++ -O3 -pthread host_bw.cpp
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

int main() {
  const size_t n = size_t(1) << 29;  // doubles (4 GB)
  std::vector<double> a(n, 1.0), b(n, 0.0);
  for (int t : {1, 4, 8, 16, 32}) {
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int k = 0; k < t; ++k)
      th.emplace_back([&, k] {
        const size_t lo = n * k / t, hi = n * (k + 1) / t;
        std::memcpy(&b[lo], &a[lo], (hi - lo) * 8);
      });
    for (auto& x : th) x.join();
    const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::printf("memcpy %2d threads: %.1f GB/s (read+write %.1f)\n", t, n * 8 / dt / 1e9, 2 * n * 8 / dt / 1e9);
  }
  // expansion: packed upper triangle of 75x75 -> full, per element
  const int d = 75, tri = d * (d + 1) / 2;
  const size_t ne = n / (d * d);
  for (int t : {8, 16, 32}) {
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int k = 0; k < t; ++k)
      th.emplace_back([&, k] {
        for (size_t e = ne * k / t; e < ne * (k + 1) / t; ++e) {
          const double* src = &a[e * tri];
          double* dst = &b[e * d * d];
          int o = 0;
          for (int i = 0; i < d; ++i)
            for (int j = i; j < d; ++j, ++o) dst[i * d + j] = dst[j * d + i] = src[o];
        }
      });
    for (auto& x : th) x.join();
    const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::printf("expand %2d threads: %.1f GB/s of full K written\n", t, ne * d * d * 8 / dt / 1e9);
  }
  return 0;
}
