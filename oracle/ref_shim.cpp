// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A flat C-ABI shim over the *unmodified* reference C++ library
// (/root/reference/proj/core, compiled in place by oracle/Makefile into
// oracle/_ref/libriffle_ref.so).  Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load it.
//
// Every entry point forwards to the reference's own public API:
//   Rng                   core/include/riffle/rng.hpp:26-90
//   plan_epoch            core/src/loader.cpp:170-181
//   BatchIterator::next   core/src/loader.cpp:257-306
//   to_dense              core/src/block.cpp:135-146
//   StoreReader::read_rows core/src/store.cpp:590-620
//   synth_store           core/src/synth.cpp:59-143
//   plan_shuffle          core/src/preshuffle.cpp:150-181
//   run_shuffle           core/src/preshuffle.cpp:185-378
//   run_throughput        core/src/metrics.cpp:99-136
#include <atomic>
#include <chrono>
#include <cstring>
#include <memory>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "riffle/block.hpp"
#include "riffle/collection.hpp"
#include "riffle/error.hpp"
#include "riffle/loader.hpp"
#include "riffle/metrics.hpp"
#include "riffle/preshuffle.hpp"
#include "riffle/rng.hpp"
#include "riffle/store.hpp"
#include "riffle/synth.hpp"

using namespace riffle;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const InvalidArgument*>(&e)) return 1;
    if (dynamic_cast<const CorruptStore*>(&e)) return 2;
    if (dynamic_cast<const IoError*>(&e)) return 3;
    return 9;
}

struct Iter {
    std::shared_ptr<const StoreReader> store;
    std::optional<BatchIterator> it;
    std::optional<MiniBatch> cur;
};

LoaderConfig make_cfg(uint64_t f, uint64_t B, uint64_t b, uint64_t seed, uint32_t depth,
                      int drop_last) {
    LoaderConfig c;
    c.fetch_block_rows = f;
    c.buffer_capacity_rows = B;
    c.batch_rows = b;
    c.seed = seed;
    c.prefetch_depth = depth;
    c.drop_last = drop_last != 0;
    return c;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- Rng -------------------------------------------------------------------
void ref_rng_next(uint64_t seed, uint64_t tag, int use_tag, uint64_t n, uint64_t* out) {
    Rng r = use_tag ? Rng(seed).stream(tag) : Rng(seed);
    for (uint64_t i = 0; i < n; ++i) out[i] = r.next();
}
void ref_rng_bounded(uint64_t seed, uint64_t tag, int use_tag, uint64_t bound, uint64_t n,
                     uint64_t* out) {
    Rng r = use_tag ? Rng(seed).stream(tag) : Rng(seed);
    for (uint64_t i = 0; i < n; ++i) out[i] = r.bounded(bound);
}
void ref_rng_shuffle_iota(uint64_t seed, uint64_t tag, uint64_t n, uint64_t* out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = i;
    Rng(seed).stream(tag).shuffle(std::span<uint64_t>(out, n));
}

// ---- plan_epoch --------------------------------------------------------------
int ref_plan_epoch(uint64_t n_obs, uint64_t f, uint64_t B, uint64_t b, uint64_t seed,
                   uint64_t epoch, uint64_t* starts, uint64_t* ends) {
    try {
        const EpochPlan p = plan_epoch(n_obs, make_cfg(f, B, b, seed, 0, 0), epoch);
        for (size_t i = 0; i < p.blocks.size(); ++i) {
            starts[i] = p.blocks[i].start;
            ends[i] = p.blocks[i].end;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---- synth_store ---------------------------------------------------------------
int ref_synth(const char* path, uint64_t n_obs, uint64_t n_var, int layout, int vdtype,
              int idtype, double density, uint64_t seed, uint64_t chunk_rows, uint64_t cps, int codec) {
    try {
        SynthConfig c;
        c.n_obs = n_obs;
        c.n_var = n_var;
        c.layout = static_cast<Layout>(layout);
        c.value_dtype = static_cast<ValueDtype>(vdtype);
        c.index_dtype = static_cast<IndexDtype>(idtype);
        c.density = density;
        c.seed = seed;
        c.chunk_rows = chunk_rows;
        c.chunks_per_shard = cps;
        c.codec = static_cast<Codec>(codec);
        synth_store(path, c);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---- BatchIterator -----------------------------------------------------------
void* ref_iter_open(const char* path, uint64_t f, uint64_t B, uint64_t b, uint64_t seed,
                    uint32_t depth, int drop_last, uint64_t epoch, int cache_bypass) {
    try {
        auto* h = new Iter;
        h->store = std::make_shared<const StoreReader>(path);
        LoaderConfig cfg = make_cfg(f, B, b, seed, depth, drop_last);
        cfg.cache_bypass = cache_bypass != 0;
        h->it.emplace(open_epoch(h->store, cfg, epoch));
        return h;
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

// Returns 1 with a batch, 0 at end of epoch, <0 on error.
int ref_iter_next(void* hv, uint64_t* n_rows, uint64_t* nnz) {
    auto* h = static_cast<Iter*>(hv);
    try {
        h->cur = h->it->next();
        if (!h->cur) return 0;
        *n_rows = h->cur->global_indices.size();
        if (const auto* c = std::get_if<CsrBlock>(&h->cur->block))
            *nnz = c->nnz();
        else
            *nnz = std::get<DenseBlock>(h->cur->block).values.size();
        return 1;
    } catch (const std::exception& e) {
        return -fail(e);
    }
}

void ref_iter_gidx(void* hv, uint64_t* out) {
    auto* h = static_cast<Iter*>(hv);
    std::memcpy(out, h->cur->global_indices.data(), h->cur->global_indices.size() * 8);
}

void ref_iter_csr(void* hv, uint64_t* indptr, uint64_t* indices, void* data) {
    auto* h = static_cast<Iter*>(hv);
    const auto& c = std::get<CsrBlock>(h->cur->block);
    std::memcpy(indptr, c.indptr.data(), c.indptr.size() * 8);
    std::memcpy(indices, c.indices.data(), c.indices.size() * 8);
    std::memcpy(data, c.data.data(), c.data.size());
}

void ref_iter_dense(void* hv, void* values) {
    auto* h = static_cast<Iter*>(hv);
    const auto& d = std::get<DenseBlock>(h->cur->block);
    std::memcpy(values, d.values.data(), d.values.size());
}

// to_dense of the current CSR batch (block.cpp:135-146).
int ref_iter_to_dense(void* hv, void* out) {
    auto* h = static_cast<Iter*>(hv);
    try {
        const DenseBlock d = to_dense(std::get<CsrBlock>(h->cur->block));
        std::memcpy(out, d.values.data(), d.values.size());
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

void ref_iter_counters(void* hv, uint64_t* blocks_fetched, uint64_t* peak, uint64_t* read_ops,
                       uint64_t* bytes_read, uint64_t* chunks_decoded) {
    auto* h = static_cast<Iter*>(hv);
    *blocks_fetched = h->it->counters().blocks_fetched;
    *peak = h->it->peak_buffer_rows();
    *read_ops = h->it->counters().io.read_ops;
    *bytes_read = h->it->counters().io.bytes_read;
    *chunks_decoded = h->it->counters().io.chunks_decoded;
}

void ref_iter_close(void* hv) { delete static_cast<Iter*>(hv); }

// ---- store reads -------------------------------------------------------------
// Two-call protocol: call with indptr==nullptr to learn (rows, nnz), then fill.
int ref_read_rows_csr(const char* path, const uint64_t* starts, const uint64_t* ends,
                      uint64_t n_ranges, uint64_t* rows_out, uint64_t* nnz_out,
                      uint64_t* indptr, uint64_t* indices, void* data) {
    try {
        StoreReader r(path);
        std::vector<RowRange> ranges(n_ranges);
        for (uint64_t i = 0; i < n_ranges; ++i) ranges[i] = {starts[i], ends[i]};
        const CsrBlock c = r.read_rows_csr(ranges);
        *rows_out = c.n_rows;
        *nnz_out = c.nnz();
        if (indptr) {
            std::memcpy(indptr, c.indptr.data(), c.indptr.size() * 8);
            std::memcpy(indices, c.indices.data(), c.indices.size() * 8);
            std::memcpy(data, c.data.data(), c.data.size());
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_read_rows_dense(const char* path, const uint64_t* starts, const uint64_t* ends,
                        uint64_t n_ranges, void* values) {
    try {
        StoreReader r(path);
        std::vector<RowRange> ranges(n_ranges);
        for (uint64_t i = 0; i < n_ranges; ++i) ranges[i] = {starts[i], ends[i]};
        const DenseBlock d = r.read_rows_dense(ranges);
        std::memcpy(values, d.values.data(), d.values.size());
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---- preshuffle ----------------------------------------------------------------
// Flattened rounds: out_round_len[r] blocks each, ids concatenated in out_ids.
int ref_plan_shuffle(uint64_t total_rows, uint64_t c, uint64_t m, uint64_t seed,
                     uint64_t* n_rounds, uint64_t* out_round_len, uint64_t* out_ids) {
    try {
        const ShufflePlan p = plan_shuffle(total_rows, c, m, seed);
        *n_rounds = p.rounds.size();
        uint64_t k = 0;
        for (size_t r = 0; r < p.rounds.size(); ++r) {
            if (out_round_len) out_round_len[r] = p.rounds[r].size();
            for (auto id : p.rounds[r]) {
                if (out_ids) out_ids[k] = id;
                ++k;
            }
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_run_shuffle(const char* const* in_paths, uint64_t n_in, int outer_join, uint64_t c,
                    uint64_t m, uint64_t seed, const char* out_path, uint64_t out_chunk_rows,
                    uint64_t out_cps, int out_idt, int out_codec, uint64_t* peak_resident, uint64_t* rounds) {
    try {
        DatasetCollection coll(outer_join ? JoinMode::outer : JoinMode::inner);
        for (uint64_t i = 0; i < n_in; ++i) coll.add(std::make_shared<const StoreReader>(in_paths[i]));
        const ShufflePlan plan = plan_shuffle(coll.total_rows(), c, m, seed);
        ShuffleOutputConfig oc;
        oc.chunk_rows = out_chunk_rows;
        oc.chunks_per_shard = out_cps;
        if (out_idt >= 0) oc.index_dtype = static_cast<IndexDtype>(out_idt);
        oc.codec = static_cast<Codec>(out_codec);
        ShuffleRunStats st;
        run_shuffle(coll, plan, out_path, oc, &st);
        if (peak_resident) *peak_resident = st.peak_resident_rows;
        if (rounds) *rounds = st.rounds_executed;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---- CPU baseline timing --------------------------------------------------------
// n_threads concurrent iterators (epochs epoch0 .. epoch0+n_threads-1), each
// draining up to max_batches batches (0 = whole epoch), optional to_dense per
// batch.  Mirrors metrics.cpp:36-48,99-136 (steady_clock around whole drains).
// Returns aggregate rows/s; rows_out = rows emitted.
double ref_throughput(const char* path, uint64_t f, uint64_t B, uint64_t b, uint64_t seed,
                      uint32_t depth, uint64_t epoch0, uint32_t n_threads, uint64_t max_batches,
                      int densify, uint64_t* rows_out, double* wall_out) {
    try {
        auto store = std::make_shared<const StoreReader>(path);
        std::atomic<uint64_t> rows{0};
        std::atomic<int> err{0};
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> ts;
        for (uint32_t t = 0; t < n_threads; ++t) {
            ts.emplace_back([&, t] {
                try {
                    auto it = open_epoch(store, make_cfg(f, B, b, seed, depth, 0), epoch0 + t);
                    uint64_t nb = 0;
                    while (auto batch = it.next()) {
                        if (densify) {
                            const DenseBlock d = to_dense(std::get<CsrBlock>(batch->block));
                            if (d.values.empty()) err = 1;
                        }
                        rows += batch->global_indices.size();
                        if (max_batches && ++nb >= max_batches) break;
                    }
                } catch (...) {
                    err = 1;
                }
            });
        }
        for (auto& th : ts) th.join();
        const double wall =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (err) {
            g_err = "worker failed";
            return -1;
        }
        *rows_out = rows;
        *wall_out = wall;
        return static_cast<double>(rows) / wall;
    } catch (const std::exception& e) {
        fail(e);
        return -1;
    }
}

}  // extern "C"
