// Device-side store images and the GPU BatchIterator engine.
//
// The reference loop (loader.cpp:257-306) interleaves fetch, decode, buffer
// maintenance and per-row copies on one thread.  Here the host only replays
// the occupancy-driven schedule (schedule.hpp) and moves raw chunk records;
// all payload bytes are moved by the sm_100a kernels (kernels.cuh).
#pragma once
#include <cuda_runtime.h>

#include <array>
#include <condition_variable>
#include <cstdint>
#include <exception>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "format.hpp"
#include "kernels.cuh"
#include "schedule.hpp"

namespace rfl {

// Record placement in store images: 16-B aligned records, 256 B of tail padding
// for 16-B over-reads.
constexpr uint64_t kRecAlign = 16;
constexpr uint64_t kRecPad = 256;
// Staging images are page-locked in pieces of this size (one registration per
// piece, staging.cpp); a host->device copy never crosses a piece boundary.
constexpr uint64_t kPinPiece = 1ull << 30;

// n / d for the per-row loops of a group (tens of thousands of rows per call):
// a shift for powers of two, else Lemire's multiply-high (exact for 32-bit n
// and d), else the hardware divide
struct FastDiv {
    uint64_t d = 1, m = 0;
    unsigned sh = 0;
    bool pow2 = true;
    FastDiv() = default;
    explicit FastDiv(uint64_t dv) : d(dv ? dv : 1) {
        pow2 = (d & (d - 1)) == 0;
        while ((1ull << sh) < d) ++sh;
        m = d <= 0xFFFFFFFFull ? ~0ull / d + 1 : 0;
    }
    uint64_t div(uint64_t n) const {
        if (pow2) return n >> sh;
        if (m && n <= 0xFFFFFFFFull) return static_cast<uint64_t>((static_cast<unsigned __int128>(m) * n) >> 64);
        return n / d;
    }
};
inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

// resident: verbatim records in HBM; stream_pinned: staging image in pinned host
// memory, each fetched block copied H2D; stream_file: records read from the
// shard files per fetch; resident_coded: the (re-encoded) staging image held in
// HBM, each fetched block expanded device-to-device (a store whose verbatim
// image exceeds HBM but whose staging image fits).
enum Staging : uint32_t { kResident = 0, kStreamPinned = 1, kStreamFile = 2, kResidentCoded = 3 };
enum StageMode : uint32_t { kStageVerbatim = 0, kStageIdx16 = 1, kStageDelta = 2, kStageOneHot = 3 };

// Per-record staging encoding (staging.cpp): kind (D8Kind), staged bytes, bytes
// of the expanded record, top-byte dictionary + escape count of coded values.
struct StagePlan {
    uint8_t kind = 0;  // D8Kind, | kD8Packed when the column deltas are bit-packed
    std::array<uint8_t, 4> dict{0, 0, 0, 0};
    uint64_t n_esc = 0, bytes = 0, exp = 0;
    uint64_t pbytes = 0;    // packed delta bits, bytes (kD8Packed)
    uint64_t pbytes_v = 0;  // packed value bits, bytes (kD8IntP)
};
StagePlan plan_csr_stage(const uint8_t* rec, uint64_t vs, bool allow_delta, bool code_values, bool vfloat = true,
                         bool pack_deltas = false);
void encode_csr_stage(const uint8_t* rec, uint64_t vs, const StagePlan& p, uint8_t* dst);
bool one_hot_record(const uint8_t* rec, uint64_t rows, uint64_t n_var);
void encode_one_hot(const uint8_t* rec, uint64_t rows, uint64_t n_var, uint8_t* dst);

void cuda_ok(cudaError_t e, const char* what);

struct DeviceGuard {  // sets and restores the current device
    int prev = 0;
    explicit DeviceGuard(int dev);
    ~DeviceGuard();
};

// decode_record + CsrBlock::validate (store.cpp:81-122, block.cpp:110-133) on a
// raw CSR record, throwing CorruptStore with the reference's text (wrapped as
// process_shard does, store.cpp:455-457) for the first error in its order.
void full_check_csr_record(const Manifest& m, uint64_t chunk, const uint8_t* rec, uint64_t len);
void check_dense_record(const Manifest& m, uint64_t chunk, uint64_t len);
// Cheap pass (header, length, indptr; optionally per-row nnz); false -> run the full check.
bool check_csr_record(const Manifest& m, uint64_t chunk, const uint8_t* rec, uint64_t len, uint32_t* row_nnz);
// CsrBlock::validate's column checks (every id < n_var, strictly increasing per
// row) on a u32 record whose header and indptr passed; false -> full check.
bool columns_ok(const Manifest& m, uint64_t chunk, const uint8_t* rec);
// decode_record (store.cpp:81-122) of a stored record: decoded bytes (inflated for
// Codec::deflate), checked as the reference checks them; CorruptStore errors are
// wrapped "chunk q in shard s: ..." as process_shard does (store.cpp:455-457).
std::vector<uint8_t> decode_record_checked(const Manifest& m, uint64_t chunk, const uint8_t* enc, uint64_t n);
// Decoded CSR record bytes from the record's header: 12 + (rows+1)*is + nnz*(is+vs).
uint64_t csr_record_bytes(const Manifest& m, uint64_t rows, uint64_t nnz);
// Codec::deflate store: every record's decoded length (dense: rows x row bytes;
// CSR: from the inflated header) and, for CSR with row_nnz, per-row nnz from the
// inflated indptr; header / indptr checks as check_csr_record, errors as the
// reference reports them.  Parallel over records.
void deflate_record_lengths(const HostStore& hs, std::vector<uint64_t>& rec_len, uint32_t* row_nnz);

// One output slot of an iterator: batch buffers on the device + pinned row
// references.  Kept by the DStore between iterators (open_epoch per epoch must
// not pay cudaMalloc / cudaHostAlloc, which also serialise the device).
struct OutBuffers {
    void *gidx = nullptr, *indptr = nullptr, *indices = nullptr, *data = nullptr, *scratch = nullptr;
    RowRef* d_refs = nullptr;
    RowRef* h_refs = nullptr;
    uint64_t* h_gidx = nullptr;
    uint64_t* h_prefix = nullptr;  // CSR output: the batch indptr, planned on the host
    uint64_t cap_rows = 0, cap_nnz = 0, data_bytes = 0;
    cudaEvent_t done = nullptr;
    cudaEvent_t tk[3] = {nullptr, nullptr, nullptr};  // time_kernels: before decode, before assembly, after
    bool timed = false;                               // tk holds an unharvested batch
    bool used = false;
    uint32_t key = 0;  // output kind the buffers were sized for (output mode, dtype, transform)
    void free_all();
};

// A store image: every chunk record at a 16-B aligned offset of a virtual
// image, either resident in HBM, in pinned host memory, or left in the files.
class DStore {
public:
    DStore(std::shared_ptr<HostStore> hs, int device, uint32_t staging);
    ~DStore();
    const Manifest& manifest() const { return hs_->manifest(); }
    const HostStore& host() const { return *hs_; }
    int device() const { return device_; }
    uint32_t staging() const { return staging_; }
    const uint8_t* d_arena() const { return d_arena_; }
    const uint8_t* h_image() const { return h_image_; }
    // the pinned image is device-addressable at its host address (every registered
    // piece): the staging pull kernel reads it in place; else copy-engine transfers
    bool pull_ok() const;
    const std::vector<uint64_t>& rec_off() const { return rec_off_; }
    const std::vector<uint64_t>& rec_len() const { return rec_len_; }    // decoded record bytes
    const std::vector<uint64_t>& slot_len() const { return slot_len_; }  // stored (encoded) bytes
    const std::vector<uint64_t>& slot_off() const { return slot_off_; }  // file offset in its shard
    bool deflate() const { return manifest().codec == Codec::deflate; }
    // layout of the staged image (stream_pinned: possibly narrowed, see idx16()); == rec_* otherwise
    const std::vector<uint64_t>& img_off() const { return img_off_; }
    const std::vector<uint64_t>& img_len() const { return img_len_; }
    bool idx16() const { return idx16_; }
    // delta staging (kernels.cuh d8_*): img_* describe the staged delta records,
    // exp_len the idx16 records they expand to in a slot
    bool d8() const { return d8_; }
    uint32_t d8_kind(uint64_t q) const { return d8_rec_[q]; }  // D8Kind of staged record q
    // every staged record is a delta record with 4-byte values and every row has <=
    // kD8FusedMaxNnz entries: dense output can densify the staged records directly
    bool d8_fused() const { return d8_fused_; }
    const std::vector<uint64_t>& exp_len() const { return exp_len_; }
    uint64_t image_bytes() const { return image_bytes_; }
    uint64_t staged_bytes() const { return staged_bytes_; }  // staging image (0: verbatim)
    uint64_t row_nnz(uint64_t row) const { return row_nnz_.empty() ? 0 : row_nnz_[row]; }
    // staged bytes of the largest f-row block (+ its idx16 expansion unless !expanded)
    uint64_t max_block_bytes(uint64_t f, bool expanded = true) const;
    ArenaView view(const uint8_t* base) const;

    // streaming slot pool (shared by the iterators over this store)
    struct SlotRef {
        uint8_t* ptr = nullptr;
        cudaEvent_t released = nullptr;  // recorded after the last kernel reading it (null: never used)
        uint64_t bytes = 0;
        uint64_t owner = 0;           // id of the loader that recorded `released` (on its compute stream) ...
        uint64_t seq = 0;             // ... after its batch `seq`
    };
    SlotRef acquire_slot(uint64_t bytes);
    // grow the pool (slot geometry `bytes`) until it holds >= n free slots, so a
    // steady-state epoch never allocates (cudaMalloc stalls the device)
    void reserve_slots(uint64_t bytes, uint64_t n);
    void release_slot(const SlotRef& s);
    // release events: a loader records ONE event per group on its compute stream and
    // every slot freed by that group points at it (SlotRef::released); the events
    // live as long as the store, handed out / back per loader
    std::vector<cudaEvent_t> take_events(size_t n);
    void give_events(std::vector<cudaEvent_t>&& ev);
    // output-buffer pool shared by the iterators over this store
    OutBuffers take_out(uint32_t key);
    void give_out(OutBuffers&& b);
    // pinned read-ahead buffers of stream_file iterators, kept the same way
    uint8_t* take_pinned(uint64_t bytes);
    void give_pinned(uint8_t* p, uint64_t bytes);

private:
    void open_image();
    void load_records(bool to_device);
    void deflate_layout();
    void load_records_deflate(bool to_device);
    void validate_records(const uint8_t* base);
    uint32_t stage_mode() const;
    bool build_staged_image(uint32_t mode);
    void read_checked(uint64_t q, uint8_t* dst, std::vector<uint8_t>& scratch, bool validate) const;
    void free_host_image();
    std::shared_ptr<HostStore> hs_;
    int device_;
    uint32_t staging_;
    std::vector<uint64_t> rec_off_, rec_len_, slot_len_, slot_off_, img_off_, img_len_;
    bool idx16_ = false, d8_ = false, d8_fused_ = false;
    std::vector<uint64_t> exp_len_;
    std::vector<uint8_t> d8_rec_;
    std::vector<uint32_t> row_nnz_;
    uint64_t image_bytes_ = 0;
    uint8_t* d_arena_ = nullptr;
    uint8_t* h_image_ = nullptr;
    uint64_t h_map_bytes_ = 0;     // > 0: h_image_ is an mmap'd staging image (else cudaHostAlloc)
    bool h_registered_ = false;    // ... page-locked with cudaHostRegister
    mutable int pull_ok_ = -1;     // pull_ok() cache
    uint64_t staged_bytes_ = 0;    // bytes of the staging image
    std::mutex mu_;
    void grow_slab(uint64_t slot_bytes);  // mu_ held
    std::vector<void*> slabs_;
    std::vector<cudaEvent_t> ev_free_, ev_all_;
    // per slot size, FIFO: reuse the slot released longest ago (its readers are done)
    std::map<uint64_t, std::deque<SlotRef>> free_;
    std::vector<OutBuffers> out_pool_;
    std::vector<std::pair<uint8_t*, uint64_t>> pinned_pool_;
};

// Read-ahead of a loader's fetch blocks for stream_file staging (the
// reference's BlockPrefetcher, loader.cpp:21-90, with the order known up front
// from the replay): I/O threads read blocks k+1 .. k+S-1 of this rank's fetch
// order into pinned buffers (4 KiB-aligned O_DIRECT reads with cache_bypass)
// while block k is staged; a buffer is refilled only after its H2D copy ended.
class BlockReader {
public:
    struct Block {
        uint64_t seq = ~0ull;       // position in the fetch order now held
        uint8_t* buf = nullptr;     // pinned, page aligned
        std::vector<uint64_t> pos;  // per record of the block: offset of its bytes in buf
        std::exception_ptr err;
    };
    BlockReader(std::shared_ptr<DStore> ds, std::vector<uint64_t> order, uint64_t f, uint32_t threads, uint32_t slots,
                bool direct);
    ~BlockReader();
    const Block& wait(uint64_t seq);              // the seq-th block of the order, once read
    void release(uint64_t seq, cudaStream_t st);  // its buffer is free after st's work so far

private:
    void worker();
    std::shared_ptr<DStore> ds_;
    std::vector<uint64_t> order_;
    uint64_t f_;
    bool direct_;
    bool validate_ = true;  // column checks of every fetched CSR record
    std::vector<Block> slots_;
    uint64_t buf_bytes_ = 0;
    std::vector<cudaEvent_t> ev_;
    std::vector<uint64_t> released_;  // per slot: last seq released (~0: none)
    std::mutex mu_;
    std::condition_variable cv_;
    uint64_t next_read_ = 0;
    bool stop_ = false;
    std::vector<std::thread> th_;
};

struct DeviceCfg {
    uint32_t output = 1;     // 0 csr, 1 dense
    OutDtype out_dtype = OutDtype::native;
    bool normalize = false;
    float target_sum = 1e4f;
    uint32_t out_slots = 2;
    cudaStream_t stream = nullptr;
    bool time_kernels = false;  // CUDA events around each batch's decode / assembly kernels
    // batches assembled per launch: next() replays, stages and assembles `group`
    // consecutive batches at once (one copy batch, one refs upload, one decode and one
    // assembly launch) into one output slot, then hands them out one per call
    uint32_t group = 1;
};

struct BatchOut {
    uint64_t epoch = 0, batch_index = 0, n_rows = 0, nnz = 0, n_var = 0;
    uint32_t layout = 0, dtype = 0, index_dtype = 0;
    void *d_gidx = nullptr, *d_indptr = nullptr, *d_indices = nullptr, *d_data = nullptr;
    const uint64_t* h_gidx = nullptr;
    cudaEvent_t ready = nullptr;
};

struct Counters {
    uint64_t blocks_fetched = 0, read_ops = 0, bytes_read = 0, chunks_decoded = 0, peak_buffer_rows = 0,
             h2d_bytes = 0, kernels_launched = 0;
    double decode_ms = 0, assembly_ms = 0;  // DeviceCfg::time_kernels, finished batches
};

class GpuLoader {
public:
    GpuLoader(std::shared_ptr<DStore> ds, const LoaderCfg& cfg, uint64_t epoch, const DeviceCfg& dev);
    ~GpuLoader();
    bool next(BatchOut& out);  // false at end of epoch (idempotent)
    // up to `max` further batches (fewer only at the end of the epoch); 0 at the end
    uint32_t next_many(BatchOut* out, uint32_t max);
    Counters counters() const;
    void sync();
    void harvest(OutBuffers& s) const;  // fold a finished batch's kernel times into the counters

private:
    using OutSlot = OutBuffers;
    struct Live {
        DStore::SlotRef slot;
        uint64_t live_rows = 0;
        uint64_t first_chunk = 0;
        uint64_t off0 = 0;     // device address of the block's first staged record
        bool single = false;   // the block is one chunk record (row refs skip chunk_off)
        std::vector<uint64_t> chunk_off;  // offset of each staged record inside the slot
    };
    // one replayed batch: its rows, the blocks pulled in while it was drawn, and the
    // replay's counters after it (the replay runs ahead on its own thread)
    struct Planned {
        std::vector<uint64_t> gidx, consumed;
        uint64_t batch_index = 0, blocks_fetched = 0, peak = 0;
    };
    void replay_worker();
    bool pop_planned(Planned& p);
    bool assemble_group();  // replay -> stage -> one launch for up to dev_.group batches
    void stage_block(uint64_t block_id);
    void count_fetch(uint64_t block_id);  // the reference's IoStats for one block fetch
    void ensure_capacity(OutSlot& s, uint64_t rows, uint64_t nnz);

    std::shared_ptr<DStore> ds_;
    LoaderCfg cfg_;
    uint64_t epoch_;
    DeviceCfg dev_;
    EpochReplay replay_;
    cudaStream_t compute_ = nullptr, copy_ = nullptr;
    bool own_compute_ = false;
    cudaEvent_t staged_ = nullptr;
    mutable std::vector<OutSlot> slots_;
    uint64_t next_slot_ = 0;
    std::vector<Planned> group_;             // the batches of the current output group
    std::vector<uint64_t> group_start_;      // first row of each batch of the group
    std::vector<BatchOut> ready_;            // assembled, not yet handed out
    size_t ready_pos_ = 0;
    uint64_t snap_blocks_ = 0, snap_peak_ = 0;  // replay counters after the last handed-out batch
    // replay-ahead
    std::thread replay_th_;
    std::mutex rq_mu_;
    std::condition_variable rq_cv_;
    std::deque<Planned> rq_;
    std::vector<Planned> rq_free_;  // recycled vectors
    bool rq_end_ = false, rq_stop_ = false;
    std::exception_ptr rq_err_;
    size_t rq_cap_ = 8;
    std::vector<uint8_t> footer_seen_;  // shards whose footer charge this loader already applied
    // dense output straight from the delta-staged records (K3d, no k_d8_decode)
    bool fused_ = false;
    // rows read in place from a device-resident image (resident, or resident_coded + fused_): no slots
    bool direct_ = false;
    std::vector<Live> live_;                 // indexed by block id (streaming)
    // the per-row reference loop's view of live_: the device address of a staged
    // single-record block (0: multi-record, look up chunk_off) and its rows still to
    // be handed out, as flat arrays (16 B per block instead of a Live per row)
    std::vector<uint64_t> blk_addr_;
    std::vector<uint32_t> blk_live_;
    FastDiv div_chunk_, div_f_;              // row -> chunk, row -> block
    // one release event per group, from a ring of kReleaseRing store-owned events: a
    // ring event is re-recorded only kReleaseRing groups later on the same stream, so a
    // slot still pointing at it waits on a later point of that stream (never earlier)
    static constexpr size_t kReleaseRing = 256;
    std::vector<cudaEvent_t> rel_ring_;
    size_t rel_pos_ = 0;
    std::vector<uint64_t> done_blocks_;      // blocks whose last rows this group took
    uint64_t block_bytes_ = 0;               // slot size: staged bytes of the largest block
    std::unique_ptr<BlockReader> reader_;        // stream_file read-ahead
    uint64_t read_seq_ = 0;
    std::vector<void*> batch_dst_, batch_src_;  // stream_pinned copies of one group (one pull kernel)
    std::vector<D8Job> d8_jobs_;                 // delta-staged records of this next() to expand
    std::vector<size_t> batch_size_;
    PullJobs pull_;                              // the pull kernel's job table (by value)
    mutable Counters ctr_;
    bool done_ = false;
    uint64_t batch_seq_ = 0;
    uint64_t id_ = 0;  // unique per loader (slot ownership; never reused like an address)
    // stream_pinned: the newest of this loader's own release events among the slots
    // acquired for the batch being staged -- one copy-stream wait per batch covers
    // them all (they were recorded in order on compute_)
    cudaEvent_t pend_ev_ = nullptr;
    uint64_t pend_seq_ = 0;
};

}  // namespace rfl
