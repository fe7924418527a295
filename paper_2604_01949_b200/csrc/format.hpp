// riffle on-disk store format, host side.  The format is the contract between
// the reference and this build, so every byte written here matches the
// reference writer:
//   manifest.json         manifest.hpp:16-54, manifest.cpp:49-97 (nlohmann ordered dump(2))
//   shards/s%08d.bin      shard.hpp:13-67, shard.cpp:18-103 (records, footer, SHRDIDX1)
//   CSR chunk record      store.cpp:52-64 ([rows u32][nnz u64][indptr][indices][data])
//   dense chunk record    store.cpp:31-33 (row-major values)
#pragma once
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

namespace rfl {

// ---- errors (error.hpp:9-32) ------------------------------------------------
enum Code : int { kOk = 0, kInvalid = 1, kCorrupt = 2, kIo = 3, kCuda = 4, kNccl = 5, kEnd = 6, kNoMem = 7 };
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void invalid(const std::string& m) { throw Error(kInvalid, m); }
[[noreturn]] inline void corrupt(const std::string& m) { throw Error(kCorrupt, m); }
[[noreturn]] inline void ioerr(const std::string& m) { throw Error(kIo, m); }

// ---- dtypes (dtype.hpp:10-40) -------------------------------------------------
enum class Layout : uint8_t { dense = 0, csr = 1 };
enum class VDtype : uint8_t { f32 = 0, f64 = 1, i32 = 2, u8 = 3 };
enum class IDtype : uint8_t { u32 = 0, u64 = 1 };
enum class Codec : uint8_t { none = 0, deflate = 1 };

constexpr size_t value_size(VDtype d) {
    return d == VDtype::f64 ? 8 : d == VDtype::u8 ? 1 : 4;
}
constexpr size_t index_size(IDtype d) { return d == IDtype::u32 ? 4 : 8; }
const char* to_string(Layout l);
const char* to_string(VDtype d);
const char* to_string(IDtype d);
const char* to_string(Codec c);

// ---- manifest -------------------------------------------------------------------
struct Manifest {
    uint32_t format_version = 1;
    Layout layout = Layout::dense;
    uint64_t n_obs = 0;
    uint64_t n_var = 0;
    VDtype value_dtype = VDtype::f32;
    std::optional<IDtype> index_dtype;
    uint64_t chunk_rows = 1;
    uint64_t chunks_per_shard = 1;
    Codec codec = Codec::none;
    std::vector<std::string> var_names;
    bool has_provenance = false;

    uint64_t chunk_count() const { return (n_obs + chunk_rows - 1) / chunk_rows; }
    uint64_t shard_count() const { return (chunk_count() + chunks_per_shard - 1) / chunks_per_shard; }
    uint64_t rows_in_chunk(uint64_t c) const {
        const uint64_t s = c * chunk_rows;
        return n_obs - s < chunk_rows ? n_obs - s : chunk_rows;
    }
    void validate() const;                      // manifest.cpp:34-47
    std::string serialize() const;              // manifest.cpp:49-63 (dump(2) + "\n")
    static Manifest parse(const std::string&);  // manifest.cpp:65-97
};

std::string shard_file_name(uint64_t shard_index);  // manifest.cpp:99-103
std::string json_escape(const std::string& s);      // nlohmann dump string escaping

// ---- low-level file I/O (file_io.hpp:23-127) ------------------------------------
class File {
public:
    File() = default;
    File(const File&) = delete;
    File& operator=(const File&) = delete;
    File(File&& o) noexcept : fd_(o.fd_) { o.fd_ = -1; }
    File& operator=(File&& o) noexcept;
    ~File();
    static File open_read(const std::string& p);
    static File try_open_direct(const std::string& p);
    static File create_write(const std::string& p);
    bool valid() const { return fd_ >= 0; }
    uint64_t size() const;
    void pread_exact(uint64_t off, void* dst, uint64_t n) const;
    // read up to n bytes at off; end of file is fine once `need` bytes are in
    void pread_upto(uint64_t off, void* dst, uint64_t n, uint64_t need) const;
    void write_all(const void* src, uint64_t n);
    void pwrite_all(uint64_t off, const void* src, uint64_t n) const;

private:
    int fd_ = -1;
};

std::string read_text_file(const std::string& p);
void write_text_file(const std::string& p, const std::string& text);
void make_dirs(const std::string& p);
bool path_exists(const std::string& p);
bool dir_nonempty(const std::string& p);

// ---- shards ------------------------------------------------------------------------
struct Slot {
    uint64_t off = ~0ull;
    uint64_t len = ~0ull;
    bool empty() const { return off == ~0ull; }
};
// ShardFooter::read (shard.cpp:18-54): magic, size, slot bounds, prefix occupancy.
std::vector<Slot> read_footer(const File& f, const std::string& path, uint64_t slots);

// ---- records generated on demand ------------------------------------------------------
// A store that is never materialised (the bench's 240 GB BASELINE config 2 does
// not fit the box's disk): every record is generated from its chunk id by a
// procedural generator, byte-identical to the file the same synth config writes.
struct RecordSource {
    virtual ~RecordSource() = default;
    virtual uint64_t record_bytes(uint64_t chunk) const = 0;
    virtual void record(uint64_t chunk, std::vector<uint8_t>& out) const = 0;
};
// "procedural:counts?n_obs=..&n_var=..&seed=..&chunk_rows=..&chunks_per_shard=..[&value_dtype=f32|i32]"
// (SynthCfg::counts, synth.hpp); fills the manifest (synth.cpp).
std::shared_ptr<const RecordSource> make_record_source(const std::string& spec, Manifest& man);

// ---- a finished store, host side ------------------------------------------------------
// Thread-safe lazily-opened fds/footers, like StoreReader::Impl (store.cpp:301-368).
class HostStore {
public:
    explicit HostStore(std::string root);  // a store directory, or a "procedural:..." spec
    bool procedural() const { return src_ != nullptr; }
    const Manifest& manifest() const { return man_; }
    const std::string& root() const { return root_; }
    Slot record_slot(uint64_t chunk) const;  // throws CorruptStore on empty slot
    uint64_t shard_bytes(uint64_t shard) const;  // file size of a shard
    bool direct_ok(uint64_t shard) const;        // the shard opens with O_DIRECT
    // IoStats::bytes_read of a shard's first footer load through this store
    // (StoreReader::footer, store.cpp:318-328): the footer bytes once, then 0.
    // Readers sharing the store share the charge, as they share the reference's footer cache.
    uint64_t charge_footer(uint64_t shard) const;
    void read_record(uint64_t chunk, void* dst, uint64_t cap) const;
    // pread an arbitrary byte range of one shard (coalesced runs, store.cpp:427-447)
    void read_shard_bytes(uint64_t shard, uint64_t off, void* dst, uint64_t n, bool direct) const;
    // Bytes [off, off+n) of a shard into a 4 KiB-aligned dst holding at least
    // aligned_span(off, n) bytes; returns where they start inside dst.  With
    // direct, an O_DIRECT read of the 4 KiB-aligned superset (no page-cache
    // copy, file_io.hpp:50-56), else a plain pread to dst.
    uint64_t read_shard_span(uint64_t shard, uint64_t off, void* dst, uint64_t n, bool direct) const;
    static uint64_t aligned_span(uint64_t off, uint64_t n) {
        return ((off + n + 4095) & ~4095ull) - (off & ~4095ull);
    }

private:
    const File& fd(uint64_t shard, bool direct) const;
    std::string root_;
    Manifest man_;
    mutable std::mutex mu_;
    mutable std::unordered_map<uint64_t, File> fds_, dfds_;
    mutable std::unordered_map<uint64_t, std::vector<Slot>> footers_;
    mutable std::vector<uint8_t> footer_charged_;
    // procedural store: the generator and every record's (offset in its shard, length)
    std::shared_ptr<const RecordSource> src_;
    std::vector<Slot> src_slots_;
    void gen_range(uint64_t shard, uint64_t off, uint8_t* dst, uint64_t n) const;
};

// ---- CSR record header accessors (store.cpp:52-64,81-122) ---------------------------
constexpr uint64_t kCsrHeaderBytes = 12;
inline uint32_t rd32(const uint8_t* p) { uint32_t v; std::memcpy(&v, p, 4); return v; }
inline uint64_t rd64(const uint8_t* p) { uint64_t v; std::memcpy(&v, p, 8); return v; }
inline void wr32(uint8_t* p, uint32_t v) { std::memcpy(p, &v, 4); }
inline void wr64(uint8_t* p, uint64_t v) { std::memcpy(p, &v, 8); }

// ---- append-only writer of pre-encoded records (StoreWriter, store.cpp:140-297) ----
// Records are handed over already encoded (codec none); shards finalize as they fill.
class RecordWriter {
public:
    RecordWriter(std::string root, Manifest man, bool defer_manifest, const char* shard_dir = "shards",
                 bool write_manifest_file = true);
    // append_record / append_record_at take DECODED records and apply the
    // manifest's codec (codec_encode, store.cpp:200); append_encoded takes
    // records already encoded with it.
    void append_record(const void* rec, uint64_t nbytes, uint64_t rows);
    void append_encoded(const void* enc, uint64_t nbytes, uint64_t rows, int64_t chunk = -1);
    // Sparse writing for multi-rank writers that own a subset of the shards:
    // chunk ids must increase and fill each owned shard from slot 0.
    void append_record_at(uint64_t chunk, const void* rec, uint64_t nbytes, uint64_t rows);
    // Two-step form for streamed records: reserve the next slot (chunk < 0:
    // consecutive), then write its bytes in any number of parts with
    // write_part(p, offset in record, ...) before the next reserve/finish.
    struct Placement {
        const File* file = nullptr;
        uint64_t off = 0;  // file offset of the record's first byte
    };
    Placement reserve_record(uint64_t nbytes, uint64_t rows, int64_t chunk = -1);
    static void write_part(const Placement& p, uint64_t rel, const void* src, uint64_t n);
    // finish(): flush shard footer, write manifest (n_obs = rows appended, or
    // n_obs_override when several ranks wrote the store)
    Manifest finish(int64_t n_obs_override = -1);
    Codec codec() const { return man_.codec; }
    uint64_t rows() const { return man_.n_obs; }

private:
    void open_shard();
    void close_shard();
    std::string root_, shard_dir_;
    Manifest man_;
    bool write_manifest_file_;
    std::optional<File> shard_;
    std::vector<Slot> slots_;
    uint64_t shard_bytes_ = 0, chunk_in_shard_ = 0, chunks_emitted_ = 0;
    bool finished_ = false;
};

}  // namespace rfl
