// rngstream.h — host-side restatement of the reference's RngStream
// (src/rng.cpp:12-61): key = mix64(seed + phi), next_u64 = mix64(key + phi *
// ++counter), labelled split via FNV-1a.  Used by the fit driver so the
// initial factors are the reference's own (kruskal.cpp:33-45 draws them from
// RngStream(seed).split("init")), and to derive the Philox keys of the
// estimator and gradient streams from the same seed.
#pragma once
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string_view>

namespace gcpb {

class HostRngStream {
 public:
  explicit HostRngStream(uint64_t seed) : key_(mix(seed + kGolden)) {}
  HostRngStream split(std::string_view label) const {
    uint64_t h = 0xcbf29ce484222325ull;
    for (char c : label) {
      h ^= static_cast<unsigned char>(c);
      h *= 0x100000001b3ull;
    }
    return HostRngStream(mix(key_ ^ mix(h + kGolden)), 0);
  }
  HostRngStream split(uint64_t label) const {  // rng.cpp:35-37
    return HostRngStream(mix(key_ ^ mix(label + kGolden)), 0);
  }
  static HostRngStream from_key(uint64_t key) { return HostRngStream(key, 0); }
  static HostRngStream from_state(uint64_t key, uint64_t counter, bool has_cached, double cached) {
    HostRngStream s(key, 0);
    s.counter_ = counter;
    s.has_cached_normal_ = has_cached;
    s.cached_normal_ = cached;
    return s;
  }
  uint64_t next_u64() { return mix(key_ + kGolden * ++counter_); }
  double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  uint64_t key() const { return key_; }
  uint64_t counter() const { return counter_; }
  void set_counter(uint64_t c) { counter_ = c; }
  bool has_cached_normal() const { return has_cached_normal_; }
  double cached_normal() const { return cached_normal_; }
  static uint64_t hash(uint64_t key, uint64_t counter) { return mix(key + kGolden * counter); }

  // rng.cpp:49-61
  uint64_t next_below(uint64_t n) {
    if (n == 0) throw std::invalid_argument("RngStream::next_below: n must be positive");
    const uint64_t threshold = (0 - n) % n;
    for (;;) {
      const uint64_t r = next_u64();
      if (r >= threshold) return r % n;
    }
  }
  // Box-Muller with the second value cached (rng.cpp:75-90).
  double next_normal(double mean, double stddev) {
    if (has_cached_normal_) {
      has_cached_normal_ = false;
      return mean + stddev * cached_normal_;
    }
    double u1;
    do {
      u1 = next_double();
    } while (u1 <= 0.0);
    const double u2 = next_double();
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = 2.0 * 3.141592653589793 * u2;
    cached_normal_ = radius * std::sin(angle);
    has_cached_normal_ = true;
    return mean + stddev * radius * std::cos(angle);
  }
  // Geometric skips, or the rounded normal approximation above 5e7
  // expected successes (rng.cpp:97-128).
  int64_t next_binomial(int64_t n, double p) {
    if (n < 0) throw std::invalid_argument("RngStream::next_binomial: n must be nonnegative");
    if (n == 0 || p <= 0.0) return 0;
    if (p >= 1.0) return n;
    if (p > 0.5) return n - next_binomial(n, 1.0 - p);
    const double expected = static_cast<double>(n) * p;
    if (expected > 5e7) {
      const double sd = std::sqrt(expected * (1.0 - p));
      double draw = std::round(next_normal(expected, sd));
      if (draw < 0.0) draw = 0.0;
      if (draw > static_cast<double>(n)) draw = static_cast<double>(n);
      return static_cast<int64_t>(draw);
    }
    const double log_q = std::log1p(-p);
    int64_t count = 0;
    double position = 0.0;
    for (;;) {
      double u;
      do {
        u = next_double();
      } while (u <= 0.0);
      position += std::floor(std::log(u) / log_q) + 1.0;
      if (position > static_cast<double>(n)) return count;
      ++count;
    }
  }

 private:
  HostRngStream(uint64_t key, int) : key_(key) {}
  static constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;
  static uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  uint64_t key_ = 0;
  uint64_t counter_ = 0;
  bool has_cached_normal_ = false;
  double cached_normal_ = 0.0;
};

}  // namespace gcpb
