// Drop-in for the configuration half of proj/include/spotlight/ranking_loss.hpp
// (ranking_loss.hpp:15-24). The loss itself (partition_topk's sampling, the
// pairwise soft-code loss and its gradient) runs inside train_hasher on the
// B200 (paper_2508_19740_b200/csrc/trainer.cu); the standalone per-matrix
// ranking_loss / ranking_loss_grad helpers of the reference are not part of
// this API (SURVEY §8 f4 covers training, not the loss as a library call).
#pragma once

#include <cstddef>
#include <cstdint>
#include <optional>

namespace spotlight {

// Pairwise ranking objective configuration. k = floor(n * (1 - maskout)) is
// the per-query count of reference top scores; max_top / max_oth /
// query_subsample bound the sampled pair set for long sequences.
struct RankingLossConfig {
    double beta = 1.0;
    double alpha = 3.0;
    double maskout = 0.98;
    std::optional<std::uint32_t> max_top;
    std::optional<std::uint32_t> max_oth;
    std::optional<std::uint32_t> query_subsample;
    /// Throws DimensionError with the reference's messages (ranking_loss.cpp:13-28).
    void validate(std::size_t n_keys) const;
};

}  // namespace spotlight
