// sfi/distribution.hpp — score distributions over prefix positions (reference:
// proj/include/sfi/distribution.hpp:23-58, proj/src/distribution.cpp). Same
// types and signatures. normalize() runs on the B200 (one-row Selector stage
// kernel, stages in selector.cu); the predicates and the two reductions used
// by callers' checks (dot, squared_norm) are host code with the reference's
// sequential order.
#pragma once

#include <cstdint>
#include <span>
#include <vector>

namespace __attribute__((visibility("default"))) sfi {

using Pos = std::int32_t;      // 1-based absolute prefix position
using TokenId = std::int32_t;

struct ScoreDistribution {
  std::vector<Pos> support;  // strictly increasing
  std::vector<double> mass;  // aligned with support
  std::size_t size() const { return support.size(); }
};

bool validate_distribution(const ScoreDistribution& d);
ScoreDistribution normalize(std::span<const Pos> support, std::span<const double> weights);
double dot(const ScoreDistribution& a, const ScoreDistribution& b);
double squared_norm(const ScoreDistribution& d);
bool same_support(const ScoreDistribution& a, const ScoreDistribution& b);

}  // namespace sfi
