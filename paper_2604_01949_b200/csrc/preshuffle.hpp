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
    uint32_t out_codec = 0;  // Codec of the output store and its provenance sidecar
};

struct ShuffleResult {
    uint64_t peak_resident_rows = 0, rows_written = 0, rounds = 0, input_bytes = 0, h2d_bytes = 0, d2h_bytes = 0;
    double gpu_ms = 0.0;
    double send_ms = 0.0;     // multi-GPU send-side pack kernels
    uint64_t peer_bytes = 0;  // message bytes addressed to other ranks
};

ShuffleResult run_shuffle_gpu(const ShuffleArgs& a);

// Multi-GPU rank API (one process per GPU; the caller runs the control plane):
// per round  stage -> [sizes all-gathered] -> recv buffer + IPC handles ->
// send (pack kernel writes into the owners' receive buffers) -> [barrier] ->
// emit (owner packs its complete chunks and writes its shards).
struct RankShuffle;
RankShuffle* rank_shuffle_create(const ShuffleArgs& a, uint64_t* n_rounds);
void rank_shuffle_stage(RankShuffle* h, uint64_t round, uint64_t* send_bytes);
void rank_shuffle_recv(RankShuffle* h, uint64_t bytes, void** ptr, void* ipc_handle, int* changed);
void rank_shuffle_send(RankShuffle* h, uint64_t round, void* const* dst);
void rank_shuffle_emit(RankShuffle* h, uint64_t round, const uint64_t* recv_bytes);
ShuffleResult rank_shuffle_finish(RankShuffle* h);
void rank_shuffle_destroy(RankShuffle* h);

}  // namespace rfl
