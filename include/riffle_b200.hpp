// riffle_b200.hpp — the C++ host side of the drop-in: the reference's loader /
// pre-shuffle API (proj/core/include/riffle/{loader,preshuffle,collection,
// store,block,error}.hpp) restated over the flat C ABI of riffle_b200.h, so a
// riffle program swaps `riffle::` for `riffle_b200::` and gets batches
// assembled by the sm_100a kernels.  Header-only, C++20; link
// libriffle_b200.so.  Same names, argument meaning and error behaviour:
//
//   reference                                  here
//   LoaderConfig{...}.validate()   loader.hpp:12-22     LoaderConfig (+ rank/world)
//   plan_epoch                     loader.hpp:32-33     plan_epoch
//   BatchIterator{ctor,next,...}   loader.hpp:58-78     BatchIterator (next() -> host MiniBatch;
//                                                       next_device() -> zero-copy device views)
//   open_epoch                     loader.hpp:80-81     open_epoch
//   plan_shuffle / ShufflePlan     preshuffle.hpp:19-40 plan_shuffle / ShufflePlan
//   DatasetCollection(JoinMode)    collection.hpp:37-91 DatasetCollection (store list + join mode)
//   run_shuffle                    preshuffle.hpp:85-88 run_shuffle (GPU writer, byte-identical)
//   Error/InvalidArgument/CorruptStore/IoError  error.hpp:9-32   same hierarchy (+ DeviceError)
#pragma once

#include <cstddef>
#include <cstdint>
#include <cstring>
#include <filesystem>
#include <memory>
#include <new>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <variant>
#include <vector>

#include "riffle_b200.h"

namespace riffle_b200 {

// ---------------------------------------------------------------- errors ---
class Error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class InvalidArgument : public Error {
public:
    using Error::Error;
};
class CorruptStore : public Error {
public:
    using Error::Error;
};
class IoError : public Error {
public:
    using Error::Error;
};
class DeviceError : public Error {  // CUDA / NCCL failures (new: the reference has no device)
public:
    using Error::Error;
};

inline void check(rfl_status st) {
    if (st == RFL_OK || st == RFL_END) return;
    const std::string msg = rfl_last_error();
    switch (st) {
        case RFL_EINVAL: throw InvalidArgument(msg);
        case RFL_ECORRUPT: throw CorruptStore(msg);
        case RFL_EIO: throw IoError(msg);
        case RFL_ENOMEM: throw std::bad_alloc();  // what the reference would have let propagate
        default: throw DeviceError(msg);
    }
}

// ----------------------------------------------------------- store types ---
enum class Layout : std::uint32_t { dense = RFL_LAYOUT_DENSE, csr = RFL_LAYOUT_CSR };
enum class ValueDtype : std::uint32_t { f32 = RFL_F32, f64 = RFL_F64, i32 = RFL_I32, u8 = RFL_U8 };
enum class IndexDtype : std::uint32_t { u32 = RFL_IDX_U32, u64 = RFL_IDX_U64 };
enum class Codec : std::uint32_t { none = 0, deflate = 1 };  // dtype.hpp:16 (zlib raw DEFLATE per record)

[[nodiscard]] inline std::size_t value_size(ValueDtype d) noexcept {
    switch (d) {
        case ValueDtype::f64: return 8;
        case ValueDtype::u8: return 1;
        default: return 4;
    }
}

struct RowRange {  // read_plan.hpp
    std::uint64_t start = 0;
    std::uint64_t end = 0;
    [[nodiscard]] std::uint64_t rows() const noexcept { return end - start; }
    bool operator==(const RowRange&) const = default;
};

struct StoreManifest {  // manifest.hpp:16-54 (the fields the hot path reads)
    Layout layout = Layout::dense;
    std::uint64_t n_obs = 0;
    std::uint64_t n_var = 0;
    ValueDtype value_dtype = ValueDtype::f32;
    std::optional<IndexDtype> index_dtype;
    std::uint64_t chunk_rows = 0;
    std::uint64_t chunks_per_shard = 0;
    Codec codec = Codec::none;
    bool has_provenance = false;
};

struct IoStats {  // store.hpp:18-42 (payload accounting)
    std::uint64_t read_ops = 0;
    std::uint64_t bytes_read = 0;
    std::uint64_t chunks_decoded = 0;
};

/// StoreReader (store.hpp:136-170): manifest + shard footers on the host.
/// Const and shareable between iterators.
class StoreReader {
public:
    explicit StoreReader(const std::filesystem::path& root) : root_(root) {
        rfl_store* s = nullptr;
        check(rfl_store_open(root.c_str(), &s));
        h_.reset(s);
        rfl_store_info i{};
        check(rfl_store_get_info(s, &i));
        man_.layout = static_cast<Layout>(i.layout);
        man_.n_obs = i.n_obs;
        man_.n_var = i.n_var;
        man_.value_dtype = static_cast<ValueDtype>(i.value_dtype);
        if (man_.layout == Layout::csr) man_.index_dtype = static_cast<IndexDtype>(i.index_dtype);
        man_.chunk_rows = i.chunk_rows;
        man_.chunks_per_shard = i.chunks_per_shard;
        man_.codec = static_cast<Codec>(i.codec);
        man_.has_provenance = i.has_provenance != 0;
    }
    [[nodiscard]] const StoreManifest& manifest() const noexcept { return man_; }
    [[nodiscard]] const std::filesystem::path& root() const noexcept { return root_; }
    /// Raw (undecoded) chunk record bytes (SURVEY §8b's "missing lower-level API").
    [[nodiscard]] std::vector<std::byte> read_record(std::uint64_t chunk) const {
        std::uint64_t n = 0;
        check(rfl_store_record_size(h_.get(), chunk, &n));
        std::vector<std::byte> out(n);
        check(rfl_store_read_record(h_.get(), chunk, out.data(), n));
        return out;
    }
    [[nodiscard]] rfl_store* handle() const noexcept { return h_.get(); }

private:
    struct Close {
        void operator()(rfl_store* s) const noexcept { rfl_store_close(s); }
    };
    std::filesystem::path root_;
    std::unique_ptr<rfl_store, Close> h_;
    StoreManifest man_;
};

// ----------------------------------------------------------------- blocks --
struct DenseBlock {  // block.hpp:23-56
    std::size_t n_rows = 0;
    std::size_t n_var = 0;
    ValueDtype dtype = ValueDtype::f32;
    std::vector<std::byte> values;
    [[nodiscard]] std::size_t row_bytes() const noexcept { return n_var * value_size(dtype); }
    bool operator==(const DenseBlock&) const = default;
};
struct CsrBlock {  // block.hpp:58-97: indices widened to u64 in memory
    std::size_t n_rows = 0;
    std::size_t n_var = 0;
    ValueDtype dtype = ValueDtype::f32;
    std::vector<std::uint64_t> indptr{0};
    std::vector<std::uint64_t> indices;
    std::vector<std::byte> data;
    bool operator==(const CsrBlock&) const = default;
};
using RowBlock = std::variant<DenseBlock, CsrBlock>;

// ----------------------------------------------------------------- loader --
struct LoaderConfig {  // loader.hpp:12-22
    std::uint64_t fetch_block_rows = 1024;
    std::uint64_t buffer_capacity_rows = 16384;
    std::uint64_t batch_rows = 256;
    std::uint64_t seed = 0;
    std::uint32_t prefetch_depth = 0;
    bool drop_last = false;
    bool cache_bypass = false;
    std::uint32_t rank = 0;   // rank k of `world` takes plan positions i == k (mod world)
    std::uint32_t world = 1;  // world == 1 is exactly the reference
    bool even_batches = false;  // new: every rank stops after the smallest per-rank batch count

    [[nodiscard]] rfl_loader_config c() const noexcept {
        return {fetch_block_rows, buffer_capacity_rows, batch_rows, seed, prefetch_depth,
                drop_last ? 1u : 0u, cache_bypass ? 1u : 0u, rank, world, even_batches ? 1u : 0u};
    }
    void validate() const {  // loader.cpp:159-168
        const rfl_loader_config cc = c();
        check(rfl_loader_config_validate(&cc));
    }
};

struct EpochPlan {  // loader.hpp:27-30
    std::vector<RowRange> blocks;
    std::uint64_t epoch_index = 0;
};

[[nodiscard]] inline EpochPlan plan_epoch(std::uint64_t n_obs, const LoaderConfig& config,
                                          std::uint64_t epoch_index) {
    if (n_obs == 0) throw InvalidArgument("plan_epoch: n_obs must be >= 1");  // loader.cpp:171-172
    config.validate();
    const std::uint64_t f = config.fetch_block_rows;
    const std::uint64_t nb = (n_obs + f - 1) / f;
    std::vector<std::uint64_t> s(nb), e(nb);
    const rfl_loader_config cc = config.c();
    check(rfl_plan_epoch(n_obs, &cc, epoch_index, s.data(), e.data()));
    EpochPlan p;
    p.epoch_index = epoch_index;
    p.blocks.reserve(nb);
    for (std::uint64_t i = 0; i < nb; ++i) p.blocks.push_back({s[i], e[i]});
    return p;
}

struct MiniBatch {  // loader.hpp:35-40
    RowBlock block;
    std::vector<std::uint64_t> global_indices;
    std::uint64_t epoch_index = 0;
    std::uint64_t batch_index = 0;
};

struct LoaderCounters {  // loader.hpp:42-45 (+ device staging counters)
    std::uint64_t blocks_fetched = 0;
    IoStats io;
    std::uint64_t h2d_bytes = 0;
    std::uint64_t kernels_launched = 0;
};

enum class Staging : std::uint32_t {
    resident = RFL_STAGE_RESIDENT,            // every chunk record in HBM
    stream_pinned = RFL_STAGE_STREAM_PINNED,  // records in pinned host RAM, blocks copied per fetch
    stream_file = RFL_STAGE_STREAM_FILE,      // read-ahead from the files (O_DIRECT with cache_bypass)
    resident_coded = RFL_STAGE_RESIDENT_CODED,  // re-encoded staging image in HBM (dense output reads it directly)
};
enum class Output : std::uint32_t { csr = RFL_OUT_CSR, dense = RFL_OUT_DENSE };
enum class OutDtype : std::uint32_t { native = RFL_NATIVE, f32 = RFL_F32, bf16 = RFL_BF16 };
enum class Transform : std::uint32_t { none = RFL_XF_NONE, normalize_log1p = RFL_XF_NORMALIZE_LOG1P };

/// Where and how batches are assembled.  The defaults reproduce the reference's
/// MiniBatch exactly: CSR stores -> CSR batches, dense stores -> dense batches.
struct DeviceOptions {
    int device = 0;
    Staging staging = Staging::resident;
    std::optional<Output> output;  // default: the store's layout
    OutDtype out_dtype = OutDtype::native;
    Transform transform = Transform::none;
    float target_sum = 1e4f;
    std::uint32_t out_slots = 2;
    void* stream = nullptr;  // cudaStream_t; nullptr = loader-owned
    std::uint32_t batches_per_launch = 1;  // batches assembled per launch (see rfl_device_config)
};

/// Device image of a store, shared by the iterators over it (loader.hpp:55-57).
class DeviceStore {
public:
    DeviceStore(std::shared_ptr<const StoreReader> store, int device, Staging staging)
        : store_(std::move(store)), device_(device), staging_(staging) {
        rfl_dstore* d = nullptr;
        check(rfl_dstore_create(store_->handle(), device, static_cast<std::uint32_t>(staging), &d));
        h_.reset(d);
    }
    [[nodiscard]] const StoreReader& store() const noexcept { return *store_; }
    [[nodiscard]] rfl_dstore* handle() const noexcept { return h_.get(); }
    [[nodiscard]] int device() const noexcept { return device_; }
    [[nodiscard]] Staging staging() const noexcept { return staging_; }

private:
    struct Destroy {
        void operator()(rfl_dstore* d) const noexcept { rfl_dstore_destroy(d); }
    };
    std::shared_ptr<const StoreReader> store_;
    int device_;
    Staging staging_;
    std::unique_ptr<rfl_dstore, Destroy> h_;
};

/// One batch on the device (valid for out_slots further next calls).
struct DeviceBatch {
    rfl_batch raw{};
    [[nodiscard]] std::uint64_t n_rows() const noexcept { return raw.n_rows; }
    [[nodiscard]] const std::uint64_t* host_global_indices() const noexcept { return raw.h_gidx; }
};

/// BatchIterator (loader.hpp:58-78): the same batch stream as the reference for
/// (store bytes, config, epoch) — bit-identical — assembled on the GPU.
class BatchIterator {
public:
    BatchIterator(std::shared_ptr<const StoreReader> store, LoaderConfig config, std::uint64_t epoch_index,
                  DeviceOptions opts = {})
        : BatchIterator(std::make_shared<DeviceStore>(store, opts.device, opts.staging), config, epoch_index,
                        opts) {}
    BatchIterator(std::shared_ptr<DeviceStore> ds, LoaderConfig config, std::uint64_t epoch_index,
                  DeviceOptions opts = {})
        : ds_(std::move(ds)), config_(config), epoch_(epoch_index) {
        const StoreManifest& m = ds_->store().manifest();
        const Output out = opts.output.value_or(m.layout == Layout::csr ? Output::csr : Output::dense);
        rfl_device_config dc{static_cast<std::uint32_t>(out), static_cast<std::uint32_t>(opts.out_dtype),
                             static_cast<std::uint32_t>(opts.transform), opts.target_sum, opts.out_slots, 0u,
                             opts.stream, opts.batches_per_launch, 0u};
        const rfl_loader_config cc = config_.c();
        rfl_loader* l = nullptr;
        check(rfl_loader_create(ds_->handle(), &cc, epoch_index, &dc, &l));
        h_.reset(l);
    }

    /// Next batch on the device, or nullopt at end of epoch (idempotent).
    std::optional<DeviceBatch> next_device() {
        DeviceBatch b;
        const rfl_status st = rfl_loader_next(h_.get(), &b.raw);
        if (st == RFL_END) return std::nullopt;
        check(st);
        refresh_counters();
        return b;
    }

    /// Next batch as the reference's host MiniBatch (device -> host copy;
    /// indices widened to u64 like CsrBlock), or nullopt at end of epoch.
    std::optional<MiniBatch> next() {
        std::optional<DeviceBatch> d = next_device();
        if (!d) return std::nullopt;
        return download(*d);
    }

    static MiniBatch download(const DeviceBatch& d) {
        const rfl_batch& b = d.raw;
        MiniBatch mb;
        mb.epoch_index = b.epoch_index;
        mb.batch_index = b.batch_index;
        mb.global_indices.resize(b.n_rows);
        static constexpr std::size_t esz[] = {4, 8, 4, 1, 2};
        if (b.layout == RFL_LAYOUT_CSR) {
            CsrBlock c;
            c.n_rows = b.n_rows;
            c.n_var = b.n_var;
            c.dtype = static_cast<ValueDtype>(b.dtype);
            c.indptr.resize(b.n_rows + 1);
            c.indices.resize(b.nnz);
            c.data.resize(b.nnz * esz[b.dtype]);
            std::vector<std::uint32_t> narrow(b.index_dtype == RFL_IDX_U32 ? b.nnz : 0);
            void* idx = b.index_dtype == RFL_IDX_U32 ? static_cast<void*>(narrow.data())
                                                     : static_cast<void*>(c.indices.data());
            check(rfl_batch_download(&b, c.indptr.data(), idx, c.data.data(), mb.global_indices.data()));
            for (std::size_t k = 0; k < narrow.size(); ++k) c.indices[k] = narrow[k];
            mb.block = std::move(c);
        } else {
            if (b.dtype == RFL_BF16) throw InvalidArgument("download: bf16 batches have no riffle host dtype");
            DenseBlock dn;
            dn.n_rows = b.n_rows;
            dn.n_var = b.n_var;
            dn.dtype = static_cast<ValueDtype>(b.dtype);
            dn.values.resize(b.n_rows * b.n_var * esz[b.dtype]);
            check(rfl_batch_download(&b, nullptr, nullptr, dn.values.data(), mb.global_indices.data()));
            mb.block = std::move(dn);
        }
        return mb;
    }

    [[nodiscard]] const LoaderCounters& counters() const noexcept { return counters_; }
    [[nodiscard]] std::uint64_t peak_buffer_rows() const noexcept { return peak_; }
    [[nodiscard]] std::uint64_t epoch_index() const noexcept { return epoch_; }
    [[nodiscard]] const LoaderConfig& config() const noexcept { return config_; }

private:
    void refresh_counters() {
        rfl_loader_counters c{};
        check(rfl_loader_counters_get(h_.get(), &c));
        counters_.blocks_fetched = c.blocks_fetched;
        counters_.io = {c.read_ops, c.bytes_read, c.chunks_decoded};
        counters_.h2d_bytes = c.h2d_bytes;
        counters_.kernels_launched = c.kernels_launched;
        peak_ = c.peak_buffer_rows;
    }
    struct Destroy {
        void operator()(rfl_loader* l) const noexcept { rfl_loader_destroy(l); }
    };
    std::shared_ptr<DeviceStore> ds_;
    LoaderConfig config_;
    std::uint64_t epoch_;
    std::unique_ptr<rfl_loader, Destroy> h_;
    LoaderCounters counters_;
    std::uint64_t peak_ = 0;
};

[[nodiscard]] inline BatchIterator open_epoch(std::shared_ptr<const StoreReader> store, const LoaderConfig& config,
                                              std::uint64_t epoch_index, DeviceOptions opts = {}) {
    return BatchIterator(std::move(store), config, epoch_index, std::move(opts));
}

// ------------------------------------------------------------- preshuffle --
struct ShufflePlan {  // preshuffle.hpp:19-34
    std::uint64_t seed = 0;
    std::uint64_t block_rows = 1;
    std::uint64_t buffer_rows = 1;
    std::uint64_t total_rows = 0;
    std::vector<std::vector<std::uint64_t>> rounds;
    [[nodiscard]] std::uint64_t block_count() const noexcept {
        return block_rows == 0 ? 0 : (total_rows + block_rows - 1) / block_rows;
    }
    [[nodiscard]] RowRange block_range(std::uint64_t id) const noexcept {
        const std::uint64_t s = id * block_rows, e = s + block_rows;
        return {s, e < total_rows ? e : total_rows};
    }
};

[[nodiscard]] inline ShufflePlan plan_shuffle(std::uint64_t total_rows, std::uint64_t block_rows,
                                              std::uint64_t buffer_rows, std::uint64_t seed) {
    std::uint64_t nr = 0;
    check(rfl_plan_shuffle(total_rows, block_rows, buffer_rows, seed, &nr, nullptr, nullptr));
    std::vector<std::uint64_t> len(nr), ids(block_rows ? (total_rows + block_rows - 1) / block_rows : 0);
    check(rfl_plan_shuffle(total_rows, block_rows, buffer_rows, seed, &nr, len.data(), ids.data()));
    ShufflePlan p{seed, block_rows, buffer_rows, total_rows, {}};
    std::size_t pos = 0;
    for (std::uint64_t r = 0; r < nr; ++r) {
        p.rounds.emplace_back(ids.begin() + static_cast<std::ptrdiff_t>(pos),
                              ids.begin() + static_cast<std::ptrdiff_t>(pos + len[r]));
        pos += len[r];
    }
    return p;
}

struct ShuffleOutputConfig {  // preshuffle.hpp:44-50
    std::uint64_t chunk_rows = 1024;
    std::uint64_t chunks_per_shard = 128;
    Codec codec = Codec::none;
    std::optional<IndexDtype> index_dtype;
};

struct ShuffleRunStats {  // preshuffle.hpp:69-77
    std::uint64_t peak_resident_rows = 0;
    std::uint64_t rows_written = 0;
    std::uint64_t rounds_executed = 0;
    IoStats input_io;
    std::uint64_t h2d_bytes = 0;
    std::uint64_t d2h_bytes = 0;
    double gpu_ms = 0.0;
};

enum class JoinMode { inner, outer };  // collection.hpp:15-27

/// DatasetCollection (collection.hpp:37-91): an ordered list of member stores
/// on a unified var axis (inner = intersection in first-member order, outer =
/// union in first-seen order); the GPU writer reprojects non-identity members.
class DatasetCollection {
public:
    explicit DatasetCollection(JoinMode mode) : mode_(mode) {}
    void add(std::shared_ptr<const StoreReader> store) {
        if (!members_.empty()) {  // collection.cpp:10-24
            const StoreManifest& f = members_.front()->manifest();
            const StoreManifest& m = store->manifest();
            if (m.layout != f.layout) throw InvalidArgument("collection: store layout does not match collection layout");
            if (m.value_dtype != f.value_dtype)
                throw InvalidArgument("collection: store value_dtype does not match collection value_dtype");
        }
        members_.push_back(std::move(store));
    }
    [[nodiscard]] std::size_t size() const noexcept { return members_.size(); }
    [[nodiscard]] const StoreReader& store(std::size_t i) const { return *members_.at(i); }
    [[nodiscard]] JoinMode join_mode() const noexcept { return mode_; }
    [[nodiscard]] std::uint64_t total_rows() const noexcept {
        std::uint64_t n = 0;
        for (const auto& m : members_) n += m->manifest().n_obs;
        return n;
    }

private:
    JoinMode mode_;
    std::vector<std::shared_ptr<const StoreReader>> members_;
};

/// run_shuffle (preshuffle.hpp:85-88): the output store and provenance sidecar
/// are byte-identical to the reference's; returns the output manifest.
inline StoreManifest run_shuffle(const DatasetCollection& collection, const ShufflePlan& plan,
                                 const std::filesystem::path& out_path, const ShuffleOutputConfig& out_config,
                                 ShuffleRunStats* stats = nullptr, int device = 0) {
    if (collection.size() == 0) throw InvalidArgument("run_shuffle: empty collection");
    if (plan.total_rows != collection.total_rows())
        throw InvalidArgument("run_shuffle: plan covers " + std::to_string(plan.total_rows) +
                              " rows, collection holds " + std::to_string(collection.total_rows()));
    std::vector<std::string> paths;
    std::vector<const char*> argv;
    for (std::size_t i = 0; i < collection.size(); ++i) paths.push_back(collection.store(i).root().string());
    for (const auto& p : paths) argv.push_back(p.c_str());
    const rfl_shuffle_config cfg{plan.block_rows,
                                 plan.buffer_rows,
                                 plan.seed,
                                 out_config.chunk_rows,
                                 out_config.chunks_per_shard,
                                 out_config.index_dtype ? static_cast<std::int32_t>(*out_config.index_dtype) : -1,
                                 device,
                                 collection.join_mode() == JoinMode::outer ? 1u : 0u,
                                 0u,
                                 1u,
                                 static_cast<std::uint32_t>(out_config.codec)};
    rfl_shuffle_stats st{};
    check(rfl_run_shuffle(argv.data(), argv.size(), out_path.c_str(), &cfg, &st));
    if (stats) {
        stats->peak_resident_rows = st.peak_resident_rows;
        stats->rows_written = st.rows_written;
        stats->rounds_executed = st.rounds_executed;
        stats->input_io.bytes_read = st.input_bytes_read;
        stats->h2d_bytes = st.h2d_bytes;
        stats->d2h_bytes = st.d2h_bytes;
        stats->gpu_ms = st.gpu_ms;
    }
    return StoreReader(out_path).manifest();
}

}  // namespace riffle_b200
