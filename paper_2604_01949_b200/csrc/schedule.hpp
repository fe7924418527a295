// Host-side schedules.  Every random decision of the loader and the
// pre-shuffler depends only on the seeded RNG and on buffer *occupancy*, never
// on data, so the host replays them on row ids and the GPU moves the bytes.
#pragma once
#include <cstdint>
#include <vector>

#include "rng.hpp"

namespace rfl {

// LoaderConfig (reference loader.hpp:12-22) + per-rank partition.
struct LoaderCfg {
    uint64_t f = 1024;      // fetch_block_rows
    uint64_t B = 16384;     // buffer_capacity_rows
    uint64_t b = 256;       // batch_rows
    uint64_t seed = 0;
    uint32_t prefetch_depth = 0;
    bool drop_last = false;
    bool cache_bypass = false;
    uint32_t rank = 0;
    uint32_t world = 1;
    // new: every rank of `world` ends the epoch after the smallest per-rank batch
    // count (rank-sharded epochs can differ by a batch; a DDP step per batch would
    // otherwise hang at epoch end).  world == 1: no effect.
    bool even_batches = false;
    void validate() const;  // loader.cpp:159-168 (+ rank < world)
};

// plan_epoch (loader.cpp:170-181): ids of the f-row blocks of [0, n_obs) in
// seeded order (Rng(seed).stream(2e)); block id i covers [i*f, min(n,(i+1)*f)).
std::vector<uint64_t> plan_epoch_ids(uint64_t n_obs, const LoaderCfg& cfg, uint64_t epoch);

// BatchIterator::next (loader.cpp:257-306 with refill :219-226, consume
// :206-217, swap-with-last take :105-117/:145-154) replayed on row ids.
// Rank k of W works on plan positions i == k (mod W) with sampler
// stream(2e+1) (W == 1, identical to the reference) or stream(2e+1).stream(k).
class EpochReplay {
public:
    EpochReplay(uint64_t n_obs, const LoaderCfg& cfg, uint64_t epoch);
    // Next batch's global indices; `consumed` receives the ids of the blocks
    // pulled into the buffer during this call, in fetch order.  Returns false
    // at end of epoch (idempotent).
    bool next(std::vector<uint64_t>& gidx, std::vector<uint64_t>& consumed);
    uint64_t peak_buffer_rows() const { return peak_; }
    uint64_t blocks_fetched() const { return next_block_; }
    uint64_t batch_index() const { return batch_index_; }
    const std::vector<uint64_t>& plan() const { return plan_; }
    uint64_t block_rows(uint64_t id) const {
        const uint64_t s = id * cfg_.f;
        return (s + cfg_.f < n_obs_ ? s + cfg_.f : n_obs_) - s;
    }

private:
    void consume(std::vector<uint64_t>& consumed);
    uint64_t n_obs_;
    LoaderCfg cfg_;
    std::vector<uint64_t> plan_;  // this rank's block ids in fetch order
    Rng smp_;
    std::vector<uint64_t> buf_;
    uint64_t next_block_ = 0, peak_ = 0, batch_index_ = 0;
    uint64_t max_batches_ = ~uint64_t{0};  // even_batches: the minimum over ranks
    bool filled_ = false, done_ = false;
};

// Batches rank `rank` yields in one epoch (rows of its plan positions / b,
// rounded up unless drop_last): every batch but the last holds exactly b rows.
uint64_t rank_batch_count(const std::vector<uint64_t>& all_ids, uint64_t n_obs, const LoaderCfg& cfg, uint32_t rank);

// plan_shuffle (preshuffle.cpp:150-181)
struct ShufflePlan {
    uint64_t seed = 0, block_rows = 1, buffer_rows = 1, total_rows = 0;
    std::vector<std::vector<uint64_t>> rounds;
    uint64_t block_count() const { return block_rows ? (total_rows + block_rows - 1) / block_rows : 0; }
    uint64_t block_start(uint64_t id) const { return id * block_rows; }
    uint64_t block_end(uint64_t id) const {
        const uint64_t e = (id + 1) * block_rows;
        return e < total_rows ? e : total_rows;
    }
};
ShufflePlan plan_shuffle(uint64_t total_rows, uint64_t block_rows, uint64_t buffer_rows, uint64_t seed);

// Round r's permutation (preshuffle.cpp:336-338): output row k of the round is
// assembly row perm[k]; perm = iota(round_rows) shuffled by Rng(seed).stream(1+r).
std::vector<uint64_t> round_permutation(uint64_t seed, uint64_t round, uint64_t round_rows);

}  // namespace rfl
