// Synthetic store generators (product side).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "format.hpp"

namespace rfl {

// SynthConfig (reference include/riffle/synth.hpp:15-27)
struct SynthCfg {
    uint64_t n_obs = 0, n_var = 0;
    Layout layout = Layout::dense;
    VDtype value_dtype = VDtype::f32;
    IDtype index_dtype = IDtype::u32;
    double density = 0.01;
    uint64_t seed = 0;
    uint64_t chunk_rows = 1024, chunks_per_shard = 128;
    Codec codec = Codec::none;
    unsigned threads = 0;
    // one_hot > 0 (dense u8 only, not in the reference): procedural one-hot rows of
    // `one_hot` channel planes x n_var / one_hot positions -- position p of row i
    // has its 1 in channel mix64(seed ^ mix64(i) ^ p) % one_hot (SURVEY §8d
    // config 4, "4 x 1024 one-hot").  The store is an ordinary dense u8 store.
    unsigned one_hot = 0;
    // counts (csr f32/i32 only, not in the reference): procedural counts-like rows
    // (SURVEY §8d config 2): h = mix64(seed ^ mix64(row)); nnz = 2,000 + h % 2,001
    // (capped at n_var); one column per stratum of n_var / nnz (stratified jitter,
    // strictly increasing); value = 1 + mix64(h ^ (k + 2^32)) % 64.
    bool counts = false;
};

// synth_store (reference src/synth.cpp:60-144), byte-identical output.
Manifest synth_store(const std::string& path, const SynthCfg& c);

// The counts store's record of rows [r0, r0 + rows) (SynthCfg::counts).
void counts_record(const SynthCfg& c, uint64_t r0, uint64_t rows, std::vector<uint8_t>& rec, unsigned threads);

// encode_csr_record (store.cpp:52-64) of rows [r0, r1) of an in-memory CSR.
void encode_csr_rows(const uint64_t* indptr, const uint64_t* indices, const uint8_t* data, size_t vs, IDtype idt,
                     uint64_t r0, uint64_t r1, std::vector<uint8_t>& rec);

}  // namespace rfl
