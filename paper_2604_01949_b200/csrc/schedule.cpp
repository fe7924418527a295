#include "schedule.hpp"

#include <algorithm>
#include <numeric>
#include <string>

#include "format.hpp"

namespace rfl {

void LoaderCfg::validate() const {
    if (f < 1) invalid("loader config: fetch_block_rows must be >= 1");
    if (B < f)
        invalid("loader config: buffer_capacity_rows " + std::to_string(B) + " < fetch_block_rows " +
                std::to_string(f));
    if (b < 1 || b > B) invalid("loader config: batch_rows must satisfy 1 <= b <= B");
    if (world < 1 || rank >= world) invalid("loader config: rank must satisfy 0 <= rank < world");
}

std::vector<uint64_t> plan_epoch_ids(uint64_t n_obs, const LoaderCfg& cfg, uint64_t epoch) {
    if (n_obs == 0) invalid("plan_epoch: n_obs must be >= 1");
    cfg.validate();
    std::vector<uint64_t> ids((n_obs + cfg.f - 1) / cfg.f);
    std::iota(ids.begin(), ids.end(), uint64_t{0});
    // Shuffling ids == shuffling the RowRange vector: the swap sequence
    // depends only on the length (rng.hpp:73-81).
    Rng(cfg.seed).stream(2 * epoch).shuffle(ids.data(), ids.size());
    return ids;
}

EpochReplay::EpochReplay(uint64_t n_obs, const LoaderCfg& cfg, uint64_t epoch)
    : n_obs_(n_obs), cfg_(cfg), smp_(0) {
    const std::vector<uint64_t> all = plan_epoch_ids(n_obs, cfg, epoch);
    plan_.reserve(all.size() / cfg.world + 1);
    for (uint64_t i = cfg.rank; i < all.size(); i += cfg.world) plan_.push_back(all[i]);
    smp_ = Rng(cfg.seed).stream(2 * epoch + 1);  // loader.cpp:18-19
    if (cfg.world > 1) smp_ = smp_.stream(cfg.rank);
    buf_.reserve(cfg.B + cfg.f);
    if (cfg.even_batches && cfg.world > 1)
        for (uint32_t k = 0; k < cfg.world; ++k)
            max_batches_ = std::min(max_batches_, rank_batch_count(all, n_obs, cfg, k));
}

uint64_t rank_batch_count(const std::vector<uint64_t>& all_ids, uint64_t n_obs, const LoaderCfg& cfg, uint32_t rank) {
    uint64_t rows = 0;
    for (uint64_t i = rank; i < all_ids.size(); i += cfg.world) {
        const uint64_t s = all_ids[i] * cfg.f;
        rows += (s + cfg.f < n_obs ? s + cfg.f : n_obs) - s;
    }
    return rows / cfg.b + (!cfg.drop_last && rows % cfg.b ? 1 : 0);
}

void EpochReplay::consume(std::vector<uint64_t>& consumed) {
    const uint64_t id = plan_[next_block_++];
    const uint64_t s = id * cfg_.f;
    const uint64_t e = s + cfg_.f < n_obs_ ? s + cfg_.f : n_obs_;
    for (uint64_t g = s; g < e; ++g) buf_.push_back(g);
    if (buf_.size() > peak_) peak_ = buf_.size();
    consumed.push_back(id);
}

bool EpochReplay::next(std::vector<uint64_t>& gidx, std::vector<uint64_t>& consumed) {
    gidx.clear();
    consumed.clear();
    if (done_) return false;
    if (batch_index_ >= max_batches_) {  // even_batches: this rank stops with the shortest one
        done_ = true;
        return false;
    }
    const uint64_t nb = plan_.size();
    if (!filled_) {  // loader.cpp:261-266
        while (buf_.size() < cfg_.B && next_block_ < nb) consume(consumed);
        filled_ = true;
    }
    const uint64_t refill_below = cfg_.B - cfg_.f;
    while (gidx.size() < cfg_.b) {  // loader.cpp:281-294
        if (buf_.empty()) {
            if (next_block_ >= nb) break;
            consume(consumed);
            continue;
        }
        const uint64_t j = smp_.bounded(buf_.size());
        gidx.push_back(buf_[j]);
        buf_[j] = buf_.back();
        buf_.pop_back();
        while (buf_.size() < refill_below && next_block_ < nb) consume(consumed);
    }
    if (gidx.empty() || (gidx.size() < cfg_.b && cfg_.drop_last)) {  // :296-299
        done_ = true;
        gidx.clear();
        return false;
    }
    ++batch_index_;
    return true;
}

ShufflePlan plan_shuffle(uint64_t total_rows, uint64_t block_rows, uint64_t buffer_rows, uint64_t seed) {
    if (block_rows == 0) invalid("plan_shuffle: block_rows must be >= 1");
    if (buffer_rows < block_rows)
        invalid("plan_shuffle: buffer_rows " + std::to_string(buffer_rows) + " < block_rows " +
                std::to_string(block_rows));
    ShufflePlan p;
    p.seed = seed;
    p.block_rows = block_rows;
    p.buffer_rows = buffer_rows;
    p.total_rows = total_rows;
    std::vector<uint64_t> ids(p.block_count());
    std::iota(ids.begin(), ids.end(), uint64_t{0});
    Rng(seed).stream(0).shuffle(ids.data(), ids.size());
    std::vector<uint64_t> round;
    uint64_t rows_in_round = 0;
    for (const uint64_t id : ids) {
        const uint64_t rows = p.block_end(id) - p.block_start(id);
        if (!round.empty() && rows_in_round + rows > buffer_rows) {
            p.rounds.push_back(std::move(round));
            round.clear();
            rows_in_round = 0;
        }
        round.push_back(id);
        rows_in_round += rows;
    }
    if (!round.empty()) p.rounds.push_back(std::move(round));
    return p;
}

std::vector<uint64_t> round_permutation(uint64_t seed, uint64_t round, uint64_t round_rows) {
    std::vector<uint64_t> perm(round_rows);
    std::iota(perm.begin(), perm.end(), uint64_t{0});
    Rng(seed).stream(1 + round).shuffle(perm.data(), perm.size());
    return perm;
}

}  // namespace rfl
