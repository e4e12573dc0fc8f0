// rngstream.h — host-side restatement of the reference's RngStream
// (src/rng.cpp:12-61): key = mix64(seed + phi), next_u64 = mix64(key + phi *
// ++counter), labelled split via FNV-1a.  Used by the fit driver so the
// initial factors are the reference's own (kruskal.cpp:33-45 draws them from
// RngStream(seed).split("init")), and to derive the Philox keys of the
// estimator and gradient streams from the same seed.
#pragma once
#include <cstdint>
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
  uint64_t next_u64() { return mix(key_ + kGolden * ++counter_); }
  double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  uint64_t key() const { return key_; }

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
};

}  // namespace gcpb
