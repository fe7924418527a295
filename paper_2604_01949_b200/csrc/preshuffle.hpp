// GPU pre-shuffle writer: run_shuffle (reference preshuffle.cpp:185-378) with
// the round gather, permutation and chunk-record packing on the device.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace rfl {

struct ShuffleArgs {
    std::vector<std::string> inputs;
    std::string out_path;
    uint64_t c = 1, m = 1, seed = 0;
    uint64_t out_chunk_rows = 1024, out_cps = 128;
    int32_t out_idt = -1;  // -1: first input's index dtype
    int32_t device = 0;
    bool outer = true;
    uint32_t rank = 0, world = 1;
};

struct ShuffleResult {
    uint64_t peak_resident_rows = 0, rows_written = 0, rounds = 0, input_bytes = 0, h2d_bytes = 0, d2h_bytes = 0;
    double gpu_ms = 0.0;
};

ShuffleResult run_shuffle_gpu(const ShuffleArgs& a);

}  // namespace rfl
