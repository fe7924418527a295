// GPU pre-shuffle writer — run_shuffle (reference preshuffle.cpp:185-378).
//
// The output order is index-computable: round r's assembly is its blocks'
// rows in block order, permuted by Rng(seed).stream(1+r) (:336-338), and the
// output store is the concatenation of the rounds, re-chunked by the writer
// (store.cpp:170-213).  So the host only replays the plan on row ids; the
// device stages each input chunk record touched by the round once (as the
// reference decodes each chunk once per round), then one scan kernel + one
// record-pack kernel (K5) write the output chunk records directly in their
// on-disk encoding.  Rows of a chunk that straddles rounds are carried into a
// small device record so the round arena can be recycled.
//
// Output bytes are identical to the reference's (tests/test_gpu_preshuffle.py).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <future>
#include <thread>
#include <unordered_map>
#include <unordered_set>

#include "codec.hpp"
#include "engine.hpp"
#include "format.hpp"
#include "kernels.cuh"
#include "preshuffle.hpp"
#include "rng.hpp"
#include "schedule.hpp"

namespace rfl {

namespace {

constexpr uint64_t kAlign = 16;
constexpr uint64_t kHuge = 1ull << 63;           // chunk_rows of the "absolute" arena view
constexpr uint64_t kStageBytes = 256ull << 20;   // pinned staging window for round inputs (x2)
constexpr uint64_t kPieceBytes = 64ull << 20;    // pinned D2H piece of the output records (x2)
inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

struct DevBuf {
    uint8_t* p = nullptr;
    uint64_t cap = 0;
    void ensure(uint64_t n) {
        if (n <= cap) return;
        if (p) cuda_ok(cudaFree(p), "cudaFree");
        p = nullptr;
        cuda_ok(cudaMalloc(&p, n + 256), "cudaMalloc");
        cuda_ok(cudaMemset(p + n, 0, 256), "cudaMemset");
        cap = n;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};
struct PinBuf {
    uint8_t* p = nullptr;
    uint64_t cap = 0;
    void ensure(uint64_t n) {
        if (n <= cap) return;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cuda_ok(cudaHostAlloc(reinterpret_cast<void**>(&p), n, cudaHostAllocDefault), "cudaHostAlloc");
        cap = n;
    }
    ~PinBuf() {
        if (p) cudaFreeHost(p);
    }
};

struct Member {
    std::shared_ptr<HostStore> hs;
    uint64_t offset = 0;  // first global row
    // DatasetCollection column map (collection.cpp:55-63): unified column of
    // each member column, kMissing when an inner join dropped it
    std::vector<uint64_t> col_map;
    bool identity = true;
    bool remap = false;               // rows go through the reprojection kernels
    std::shared_ptr<DevBuf> d_map;    // CSR: u32 col_map; dense: u32 inverse map (unified -> member col)
    std::vector<uint64_t> dec_len;    // Codec::deflate: decoded length of every record (empty: codec none)
    uint64_t rec_bytes(uint64_t q) const { return dec_len.empty() ? hs->record_slot(q).len : dec_len[q]; }
};

constexpr uint64_t kMissing = ~0ull;  // kMissingColumn (collection.hpp:23)

std::string meta_json(uint64_t seed, uint64_t c, uint64_t m) {  // ProvenanceWriter::finish (:32-47)
    return std::string("{\n  \"rng\": \"") + Rng::kName + "\",\n  \"seed\": " + std::to_string(seed) +
           ",\n  \"block_rows\": " + std::to_string(c) + ",\n  \"buffer_rows\": " + std::to_string(m) + "\n}\n";
}

// DatasetCollection::rebuild_unified (collection.cpp:28-82): the unified axis
// (intersection in first-member order, or union in first-seen order), each
// member's column map and identity flag.
std::vector<std::string> unify(std::vector<Member>& ms, bool outer) {
    std::vector<std::string> uni;
    if (outer) {
        std::unordered_set<std::string> seen;
        for (const auto& m : ms)
            for (const auto& n : m.hs->manifest().var_names)
                if (seen.insert(n).second) uni.push_back(n);
    } else {
        for (const auto& n : ms.front().hs->manifest().var_names) {
            bool all = true;
            for (size_t i = 1; i < ms.size() && all; ++i) {
                const auto& v = ms[i].hs->manifest().var_names;
                all = std::find(v.begin(), v.end(), n) != v.end();
            }
            if (all) uni.push_back(n);
        }
    }
    std::unordered_map<std::string, uint64_t> index;
    index.reserve(uni.size());
    for (size_t i = 0; i < uni.size(); ++i) index.emplace(uni[i], i);
    for (auto& m : ms) {
        const auto& names = m.hs->manifest().var_names;
        m.col_map.assign(names.size(), kMissing);
        m.identity = names.size() == uni.size();
        for (size_t c = 0; c < names.size(); ++c) {
            const auto it = index.find(names[c]);
            if (it != index.end()) m.col_map[c] = it->second;
            if (m.col_map[c] != c) m.identity = false;
        }
    }
    return uni;
}

// RFL_TRACE=1: per-phase wall times of the single-GPU pass on stderr.
struct PhaseTrace {
    bool on = false;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    PhaseTrace() {
        const char* e = std::getenv("RFL_TRACE");
        on = e && e[0] == '1';
    }
    void mark(const char* what, uint64_t r) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "# shuffle r%llu %-10s %8.2f ms\n", static_cast<unsigned long long>(r), what,
                     std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

class GpuShuffler {
public:
    explicit GpuShuffler(const ShuffleArgs& a) : a_(a) {}
    ~GpuShuffler();
    void init();
    ShuffleResult run();  // single GPU, whole pass

    // ---- rank API (multi-GPU; the caller drives the control plane) ----
    uint64_t n_rounds() const { return plan_.rounds.size(); }
    void stage(uint64_t r, uint64_t* send_bytes);
    void recv_buffer(uint64_t bytes, void** ptr, void* ipc_handle, int* changed);
    void send(uint64_t r, void* const* dst);
    void emit_round(uint64_t r, const uint64_t* recv_bytes);
    ShuffleResult finish();

private:
    using Segs = std::vector<std::pair<uint32_t, std::pair<uint64_t, uint64_t>>>;
    void round_segments(uint64_t r, Segs& segs, std::vector<std::pair<uint32_t, uint64_t>>& prov,
                        std::vector<uint32_t>* src_rank);
    // nnz (CSR, may be null): per assembly row, the row's entry count read from the
    // staged records' indptrs on the host; cleared when a member is reprojected
    void stage_round(const Segs& segs, DevBuf& arena, std::vector<RowRef>& refs, uint64_t r,
                     std::vector<uint32_t>* nnz = nullptr);
    void reproject(uint32_t mi, std::vector<RowRef>& refs, const std::vector<uint64_t>& pos, DevBuf& out,
                   std::vector<uint64_t>& bad);
    void check_duplicates(uint64_t r, const std::vector<uint64_t>& bad_asm, uint64_t round_rows);
    void emit(const std::vector<RowRef>& refs, const std::vector<std::pair<uint32_t, uint64_t>>& prov, uint64_t n,
              const std::vector<uint64_t>* out_rows, const std::vector<uint32_t>* nnz = nullptr);
    void carry(std::vector<RowRef>& refs, uint64_t from, DevBuf& dst, const std::vector<uint32_t>* nnz = nullptr);
    // host-planned pack (no scan kernel, no host sync): refs + exclusive nnz prefix
    // staged through pinned buffer set `k`, then one K5 pack launch on st_
    uint64_t planned_upload(int k, const RowRef* refs, const uint32_t* nnz, uint64_t n);
    void harvest_timing();
    void upload_refs(const RowRef* refs, uint64_t n);

    ShuffleArgs a_;
    ShufflePlan plan_;
    uint64_t total_ = 0;
    std::vector<Member> ms_;
    Layout layout_ = Layout::csr;
    VDtype vdt_ = VDtype::f32;
    IDtype in_idt_ = IDtype::u32, out_idt_ = IDtype::u32;
    uint64_t n_var_ = 0, row_bytes_ = 0;
    std::unique_ptr<RecordWriter> out_, prov_;
    cudaStream_t st_ = nullptr;
    cudaEvent_t e0_ = nullptr, e1_ = nullptr, e2_ = nullptr, e3_ = nullptr;
    DevBuf d_refs_, d_prefix_, d_scratch_, d_out_[2];
    PinBuf h_stage_[2], h_refs_, h_prefix_, ring_[2];
    cudaEvent_t stage_ev_[2] = {nullptr, nullptr}, ring_ev_[2] = {nullptr, nullptr}, packed_[2] = {nullptr, nullptr};
    cudaStream_t wst_ = nullptr;                  // the writer's D2H stream
    // pack / D2H gate: the record pack never runs beside a D2H piece of an earlier
    // round (the pack waits for the pieces already issued; the writer issues no new
    // piece while a pack is launched but not finished).  A piece is 64 MB (~1.2 ms)
    // against a round of ~100+ ms of file writes, so the e2e does not move; the pack
    // gets the HBM to itself.  RFL_PACK_GATE=0 turns it off (A/B).
    bool gate_on_ = true;
    std::mutex gate_mu_;
    std::condition_variable gate_cv_;
    bool gate_busy_ = false;                      // a pack is being enqueued
    uint64_t gate_seq_ = 0, gate_seen_ = 0;       // packs enqueued / known complete
    cudaEvent_t gate_ev_ = nullptr, wgate_ = nullptr;
    void gate_begin() {
        if (!gate_on_) return;
        std::lock_guard<std::mutex> lk(gate_mu_);
        gate_busy_ = true;
        cuda_ok(cudaEventRecord(wgate_, wst_), "event");  // every piece issued so far
        cuda_ok(cudaStreamWaitEvent(st_, wgate_, 0), "wait D2H");
    }
    void gate_end() {
        if (!gate_on_) return;
        {
            std::lock_guard<std::mutex> lk(gate_mu_);
            cuda_ok(cudaEventRecord(gate_ev_, st_), "event");
            gate_busy_ = false;
            ++gate_seq_;
        }
        gate_cv_.notify_all();
    }
    // writer side: returns with the lock held once no pack is pending or running
    std::unique_lock<std::mutex> gate_wait() {
        std::unique_lock<std::mutex> lk(gate_mu_);
        if (!gate_on_) return lk;
        for (;;) {
            gate_cv_.wait(lk, [&] { return !gate_busy_; });
            if (gate_seen_ == gate_seq_) return lk;
            const uint64_t s = gate_seq_;
            lk.unlock();
            cuda_ok(cudaEventSynchronize(gate_ev_), "pack done");  // (the newest record: covers pack s)
            lk.lock();
            if (gate_seen_ < s) gate_seen_ = s;
        }
    }
    std::shared_future<void> wjob_[2], last_job_;  // writer job that drains d_out_[k]; the newest job
    uint64_t emits_ = 0;
    void drain_writes() {
        if (last_job_.valid()) last_job_.get();  // jobs are chained: the newest finishes last
        for (auto& f : wjob_)
            if (f.valid()) f.get();
    }
    ShuffleResult res_;
    std::vector<uint8_t> prov_rec_;
    // rank state
    DevBuf arena_[2], carry_[2], recv_, d_send_refs_, d_send_prefix_;
    std::vector<std::shared_ptr<DevBuf>> remap_[2];  // per round parity, per member: reprojected rows
    DevBuf d_counts_, d_flags_, d_dup_, d_vtab_;
    bool validate_ = true;                           // RFL_NO_VALIDATE=1 skips the staged-record checks
    std::vector<uint64_t> bad_asm_;                  // assembly rows of the staged round with duplicate columns
    std::vector<RowRef> pending_;
    std::vector<uint32_t> pend_nnz_;  // per pending row (single-GPU CSR pass, identity members)
    bool nnz_ok_ = false;
    std::vector<std::pair<uint32_t, uint64_t>> pend_prov_;
    // host-planned uploads: [0..1] emits (by parity), [2] carries
    PinBuf hp_[3];
    DevBuf dp_[3];
    cudaEvent_t hp_ev_[3] = {nullptr, nullptr, nullptr};
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> timing_;  // pack launches not yet added to gpu_ms
    std::vector<uint64_t> pend_out_;                 // global output row of each pending row (multi-rank)
    std::vector<uint64_t> send_start_, send_count_;  // per destination, into d_send_refs_
    std::vector<uint64_t> send_bytes_;               // per destination: message bytes of the staged round
    std::vector<uint64_t> round_first_out_;          // first global output row of each round
    std::vector<uint32_t> mine_src_;                 // per owned output row of the staged round: source rank
    std::vector<uint64_t> mine_out_;
    std::vector<std::pair<uint32_t, uint64_t>> mine_prov_;
    uint64_t staged_round_ = ~0ull;
    PhaseTrace tr_;
};

ArenaView absolute_view(Layout l, VDtype v, IDtype i, uint64_t n_var) {
    ArenaView av;
    av.base = nullptr;  // RowRef.rec_off holds absolute device addresses
    av.chunk_rows = kHuge;
    av.n_var = n_var;
    av.layout = l;
    av.vdt = v;
    av.idt = i;
    return av;
}

void GpuShuffler::upload_refs(const RowRef* refs, uint64_t n) {
    h_refs_.ensure(n * sizeof(RowRef));
    std::memcpy(h_refs_.p, refs, n * sizeof(RowRef));
    d_refs_.ensure(n * sizeof(RowRef));
    cuda_ok(cudaMemcpyAsync(d_refs_.p, h_refs_.p, n * sizeof(RowRef), cudaMemcpyHostToDevice, st_), "refs H2D");
    res_.h2d_bytes += n * sizeof(RowRef);
}

// Stage every input chunk record touched by the round's segments once into
// `arena`; fill refs[a] for every assembly row a (absolute record address, row
// within chunk).
void GpuShuffler::stage_round(const std::vector<std::pair<uint32_t, std::pair<uint64_t, uint64_t>>>& segs,
                              DevBuf& arena, std::vector<RowRef>& refs, uint64_t r, std::vector<uint32_t>* nnz) {
    // chunks per member, in (member, chunk) order
    std::vector<std::pair<uint32_t, uint64_t>> need;
    for (const auto& s : segs) {
        const Manifest& m = ms_[s.first].hs->manifest();
        for (uint64_t q = s.second.first / m.chunk_rows; q <= (s.second.second - 1) / m.chunk_rows; ++q)
            need.emplace_back(s.first, q);
    }
    std::sort(need.begin(), need.end());
    need.erase(std::unique(need.begin(), need.end()), need.end());
    std::vector<uint64_t> off(need.size()), len(need.size());
    uint64_t total = 0;
    for (size_t i = 0; i < need.size(); ++i) {
        len[i] = ms_[need[i].first].rec_bytes(need[i].second);
        off[i] = total;
        total = align_up(total + len[i], kAlign);
    }
    arena.ensure(std::max<uint64_t>(total, 16));
    std::vector<std::vector<uint32_t>> need_nnz(layout_ == Layout::csr && nnz ? need.size() : 0);
    auto row_counts = [&](size_t k, const uint8_t* rec) {  // per-row nnz from a staged record's indptr
        if (need_nnz.empty()) return;
        const Manifest& hm = ms_[need[k].first].hs->manifest();
        const uint64_t rows = hm.rows_in_chunk(need[k].second);
        const bool w4 = hm.index_dtype.value_or(IDtype::u32) == IDtype::u32;
        std::vector<uint32_t>& v = need_nnz[k];
        v.resize(rows);
        const uint8_t* ip = rec + kCsrHeaderBytes;
        for (uint64_t i = 0; i < rows; ++i)
            v[i] = static_cast<uint32_t>(w4 ? rd32(ip + 4 * (i + 1)) - rd32(ip + 4 * i) : rd64(ip + 8 * (i + 1)) - rd64(ip + 8 * i));
    };
    // coalesced reads of adjacent records of one shard (store.cpp:427-447)
    struct Run {
        size_t i, j;  // need[i..j)
        uint64_t shard, file_off, bytes;
    };
    std::vector<Run> runs;
    for (size_t i = 0; i < need.size();) {
        const HostStore& hs = *ms_[need[i].first].hs;
        const Manifest& m = hs.manifest();
        const uint64_t shard = need[i].second / m.chunks_per_shard;
        const Slot first = hs.record_slot(need[i].second);
        size_t j = i + 1;
        uint64_t run = first.len;
        while (j < need.size() && need[j].first == need[i].first && need[j].second == need[j - 1].second + 1 &&
               need[j].second / m.chunks_per_shard == shard) {
            const Slot s = hs.record_slot(need[j].second);
            if (s.off != first.off + run) break;
            run += s.len;
            ++j;
        }
        runs.push_back({i, j, shard, first.off, run});
        res_.input_bytes += run;
        i = j;
    }
    // windows of the arena image (<= kStageBytes, or one oversized run) read by a
    // thread pool into one of two pinned buffers — alignment gaps ride along —
    // then one async H2D, which overlaps the reads of the next window
    const unsigned T = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    for (size_t r = 0, wi = 0; r < runs.size(); ++wi) {
        const uint64_t w0 = off[runs[r].i];
        size_t r1 = r + 1;
        while (r1 < runs.size() && off[runs[r1].j - 1] + len[runs[r1].j - 1] - w0 <= kStageBytes) ++r1;
        const uint64_t w1 = off[runs[r1 - 1].j - 1] + len[runs[r1 - 1].j - 1];
        PinBuf& stage = h_stage_[wi & 1];
        cuda_ok(cudaEventSynchronize(stage_ev_[wi & 1]), "stage buffer reuse");  // its previous H2D is done
        stage.ensure(w1 - w0);
        std::vector<std::exception_ptr> errs(T);
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < T; ++t) {
            pool.emplace_back([&, t] {
                try {
                    for (size_t x = r + t; x < r1; x += T) {
                        const Run& ru = runs[x];
                        const HostStore& hs = *ms_[need[ru.i].first].hs;
                        const Manifest& hm = hs.manifest();
                        uint8_t* base = stage.p + (off[ru.i] - w0);
                        if (!ms_[need[ru.i].first].dec_len.empty()) {
                            // deflate member: inflate each record of the run to its aligned offset
                            // (decode_record, store.cpp:81-122), then the same checks
                            std::vector<uint8_t> enc(ru.bytes);
                            hs.read_shard_bytes(ru.shard, ru.file_off, enc.data(), ru.bytes, false);
                            for (size_t k = ru.i, rel = 0; k < ru.j; ++k) {
                                const uint64_t slen = hs.record_slot(need[k].second).len;
                                uint8_t* dst = base + (off[k] - off[ru.i]);
                                if (!inflate_fits(enc.data() + rel, slen, dst, len[k])) {
                                    decode_record_checked(hm, need[k].second, enc.data() + rel, slen);
                                    corrupt("chunk " + std::to_string(need[k].second) + " in shard " +
                                            std::to_string(ru.shard) + ": csr record invalid");
                                }
                                if (hm.layout == Layout::csr && !check_csr_record(hm, need[k].second, dst, len[k], nullptr))
                                    full_check_csr_record(hm, need[k].second, dst, len[k]);
                                if (hm.layout == Layout::csr) row_counts(k, dst);
                                rel += slen;
                            }
                            continue;
                        }
                        hs.read_shard_bytes(ru.shard, ru.file_off, base, ru.bytes, false);
                        // decode_record's checks (store.cpp:81-122) on each record of the run
                        for (size_t k = ru.i, rel = 0; k < ru.j; rel += len[k], ++k) {
                            if (hm.layout == Layout::dense) check_dense_record(hm, need[k].second, len[k]);
                            else if (!check_csr_record(hm, need[k].second, base + rel, len[k], nullptr))
                                full_check_csr_record(hm, need[k].second, base + rel, len[k]);
                        }
                        // spread to aligned offsets (targets move forward only: back to front)
                        std::vector<uint64_t> rel(ru.j - ru.i, 0);
                        for (size_t k = ru.i + 1; k < ru.j; ++k) rel[k - ru.i] = rel[k - ru.i - 1] + len[k - 1];
                        for (size_t k = ru.j - 1; k > ru.i; --k)
                            std::memmove(base + (off[k] - off[ru.i]), base + rel[k - ru.i], len[k]);
                        if (hm.layout == Layout::csr)
                            for (size_t k = ru.i; k < ru.j; ++k) row_counts(k, base + (off[k] - off[ru.i]));
                    }
                } catch (...) {
                    errs[t] = std::current_exception();
                }
            });
        }
        for (auto& th : pool) th.join();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
        tr_.mark(" read", wi);
        cuda_ok(cudaMemcpyAsync(arena.p + w0, stage.p, w1 - w0, cudaMemcpyHostToDevice, st_), "stage H2D");
        cuda_ok(cudaEventRecord(stage_ev_[wi & 1], st_), "event");
        res_.h2d_bytes += w1 - w0;
        r = r1;
    }
    cuda_ok(cudaStreamSynchronize(st_), "stage sync");
    tr_.mark(" h2d", r);
    // column checks of CsrBlock::validate for every staged record, on the GPU
    if (layout_ == Layout::csr && validate_) {
        std::vector<uint64_t> tab(2 * need.size());
        for (size_t i = 0; i < need.size();) {
            size_t j = i;
            while (j < need.size() && need[j].first == need[i].first) ++j;  // one member
            const Manifest& mm = ms_[need[i].first].hs->manifest();
            const uint64_t n = j - i;
            for (size_t k = 0; k < n; ++k) {
                tab[k] = off[i + k];
                tab[n + k] = need[i + k].second * mm.chunk_rows;
            }
            d_vtab_.ensure(16 * n);
            d_dup_.ensure(8);
            cuda_ok(cudaMemcpyAsync(d_vtab_.p, tab.data(), 16 * n, cudaMemcpyHostToDevice, st_), "H2D");
            cuda_ok(cudaMemsetAsync(d_dup_.p, 0xff, 8, st_), "memset");
            const uint64_t* t = reinterpret_cast<const uint64_t*>(d_vtab_.p);
            launch_validate_csr(arena.p, t, t + n, n, mm.n_var, mm.index_dtype.value_or(IDtype::u32),
                                reinterpret_cast<unsigned long long*>(d_dup_.p), st_);
            uint64_t bad = 0;
            cuda_ok(cudaMemcpyAsync(&bad, d_dup_.p, 8, cudaMemcpyDeviceToHost, st_), "D2H");
            cuda_ok(cudaStreamSynchronize(st_), "sync");
            if (bad != ~0ull) {
                const uint64_t q = bad / mm.chunk_rows;
                std::vector<uint8_t> rec(ms_[need[i].first].hs->record_slot(q).len);
                ms_[need[i].first].hs->read_record(q, rec.data(), rec.size());
                decode_record_checked(mm, q, rec.data(), rec.size());
                corrupt("chunk " + std::to_string(q) + " in shard " + std::to_string(q / mm.chunks_per_shard) +
                        ": csr record invalid");
            }
            i = j;
        }
    }
    tr_.mark(" validate", r);
    // refs per assembly row
    refs.clear();
    if (nnz) nnz->clear();
    bool any_remap = false;
    for (const auto& s : segs) any_remap = any_remap || ms_[s.first].remap;
    std::vector<std::vector<uint64_t>> remap_pos(ms_.size());
    for (const auto& s : segs) {
        const Manifest& m = ms_[s.first].hs->manifest();
        for (uint64_t row = s.second.first; row < s.second.second; ++row) {
            const uint64_t q = row / m.chunk_rows;
            const size_t k = std::lower_bound(need.begin(), need.end(), std::make_pair(s.first, q)) - need.begin();
            if (ms_[s.first].remap) remap_pos[s.first].push_back(refs.size());
            refs.push_back({reinterpret_cast<uint64_t>(arena.p) + off[k], row - q * m.chunk_rows});
            if (!need_nnz.empty() && !any_remap) nnz->push_back(need_nnz[k][row - q * m.chunk_rows]);
        }
    }
    // column reprojection of non-identity members (remap_csr_row / scatter_dense_row)
    bad_asm_.clear();
    auto& bufs = remap_[r % 2];
    if (bufs.size() < ms_.size()) bufs.resize(ms_.size());
    for (uint32_t mi = 0; mi < ms_.size(); ++mi) {
        if (remap_pos[mi].empty()) continue;
        if (!bufs[mi]) bufs[mi] = std::make_shared<DevBuf>();
        reproject(mi, refs, remap_pos[mi], *bufs[mi], bad_asm_);
    }
}

// Rows refs[pos[k]] of member mi -> one reprojected record (CSR) / block (dense)
// in `out`; the refs are re-pointed at it.  Rows with two columns mapping to one
// unified column are appended to `bad` (as positions into refs).
void GpuShuffler::reproject(uint32_t mi, std::vector<RowRef>& refs, const std::vector<uint64_t>& pos, DevBuf& out,
                            std::vector<uint64_t>& bad) {
    const Manifest& mm = ms_[mi].hs->manifest();
    const uint64_t n = pos.size();
    std::vector<RowRef> sub(n);
    for (uint64_t k = 0; k < n; ++k) sub[k] = refs[pos[k]];
    upload_refs(sub.data(), n);
    const RowRef* d_sub = reinterpret_cast<const RowRef*>(d_refs_.p);
    const ArenaView av = absolute_view(layout_, vdt_, mm.index_dtype.value_or(IDtype::u32), mm.n_var);
    const uint32_t* map = reinterpret_cast<const uint32_t*>(ms_[mi].d_map->p);
    if (layout_ == Layout::csr) {
        d_counts_.ensure(n * 8);
        d_prefix_.ensure((n + 1) * 8);
        d_scratch_.ensure(csr_gather_scratch_bytes(n));
        d_dup_.ensure(8);
        d_flags_.ensure(n);
        cuda_ok(cudaMemsetAsync(d_dup_.p, 0xff, 8, st_), "memset");
        cuda_ok(cudaMemsetAsync(d_flags_.p, 0, n, st_), "memset");
        launch_remap_count(av, d_sub, n, map, reinterpret_cast<uint64_t*>(d_counts_.p), st_);
        launch_count_scan(reinterpret_cast<uint64_t*>(d_counts_.p), n, reinterpret_cast<uint64_t*>(d_prefix_.p),
                          d_scratch_.p, st_);
        uint64_t nnz = 0;
        cuda_ok(cudaMemcpyAsync(&nnz, d_prefix_.p + n * 8, 8, cudaMemcpyDeviceToHost, st_), "D2H");
        cuda_ok(cudaStreamSynchronize(st_), "sync");
        const uint64_t os = index_size(in_idt_), vs = value_size(vdt_);
        out.ensure(kCsrHeaderBytes + os * (n + 1) + (os + vs) * nnz);
        launch_csr_remap(av, d_sub, n, map, n_var_, in_idt_, reinterpret_cast<uint64_t*>(d_prefix_.p), out.p,
                         reinterpret_cast<unsigned long long*>(d_dup_.p), d_flags_.p, st_);
        uint64_t dup = 0;
        cuda_ok(cudaMemcpyAsync(&dup, d_dup_.p, 8, cudaMemcpyDeviceToHost, st_), "D2H");
        cuda_ok(cudaStreamSynchronize(st_), "sync");
        if (dup != ~0ull) {
            std::vector<uint8_t> flags(n);
            cuda_ok(cudaMemcpy(flags.data(), d_flags_.p, n, cudaMemcpyDeviceToHost), "D2H");
            for (uint64_t k = 0; k < n; ++k)
                if (flags[k]) bad.push_back(pos[k]);
        }
    } else {
        out.ensure(std::max<uint64_t>(n * row_bytes_, 16));
        launch_dense_remap(av, d_sub, n, mm.n_var, map, n_var_, out.p, st_);
        cuda_ok(cudaStreamSynchronize(st_), "sync");
    }
    for (uint64_t k = 0; k < n; ++k) refs[pos[k]] = {reinterpret_cast<uint64_t>(out.p), k};
}

// StoreWriter::append -> CsrBlock::validate (store.cpp:261-275, block.cpp:127-129)
// rejects the first emitted c-row slice holding a row with a repeated column;
// report the same row (its position within that slice).
void GpuShuffler::check_duplicates(uint64_t r, const std::vector<uint64_t>& bad_asm, uint64_t round_rows) {
    if (bad_asm.empty()) return;
    const std::vector<uint64_t> perm = round_permutation(a_.seed, r, round_rows);
    std::vector<uint8_t> is_bad(round_rows, 0);
    for (uint64_t a : bad_asm) is_bad[a] = 1;
    for (uint64_t k = 0; k < round_rows; ++k)
        if (is_bad[perm[k]])
            invalid("csr block: column indices not strictly increasing in row " + std::to_string(k % a_.c));
}

// Write refs[0..n) as output chunk records (+ provenance records).
// out_rows (multi-rank) gives the global output row of each ref so records land
// in the owned chunk slots; single-GPU writes are consecutive.
uint64_t GpuShuffler::planned_upload(int k, const RowRef* refs, const uint32_t* nnz, uint64_t n) {
    const uint64_t rb = align_up(n * sizeof(RowRef), 16), bytes = rb + (n + 1) * 8;
    if (hp_ev_[k]) cuda_ok(cudaEventSynchronize(hp_ev_[k]), "pinned reuse");  // its last upload has been copied
    else cuda_ok(cudaEventCreateWithFlags(&hp_ev_[k], cudaEventDisableTiming), "event");
    hp_[k].ensure(bytes);
    dp_[k].ensure(bytes);
    std::memcpy(hp_[k].p, refs, n * sizeof(RowRef));
    uint64_t* P = reinterpret_cast<uint64_t*>(hp_[k].p + rb);
    uint64_t acc = 0;
    for (uint64_t i = 0; i < n; ++i) {
        P[i] = acc;
        acc += nnz[i];
    }
    P[n] = acc;
    cuda_ok(cudaMemcpyAsync(dp_[k].p, hp_[k].p, bytes, cudaMemcpyHostToDevice, st_), "refs+prefix H2D");
    cuda_ok(cudaEventRecord(hp_ev_[k], st_), "event");
    res_.h2d_bytes += bytes;
    return rb;
}

void GpuShuffler::harvest_timing() {
    for (auto& t : timing_) {
        float ms = 0.f;
        cuda_ok(cudaEventSynchronize(t.second), "sync");
        cuda_ok(cudaEventElapsedTime(&ms, t.first, t.second), "elapsed");
        res_.gpu_ms += ms;
        cudaEventDestroy(t.first);
        cudaEventDestroy(t.second);
    }
    timing_.clear();
}

void GpuShuffler::emit(const std::vector<RowRef>& refs, const std::vector<std::pair<uint32_t, uint64_t>>& prov,
                       uint64_t n, const std::vector<uint64_t>* out_rows, const std::vector<uint32_t>* nnz) {
    if (n == 0) return;
    const uint64_t cr = a_.out_chunk_rows;
    const uint64_t nq = (n + cr - 1) / cr;
    // d_out_[ob] is reused: the writer job that drained it two emits ago is done
    const int ob = static_cast<int>(emits_++ & 1u);
    if (wjob_[ob].valid()) wjob_[ob].get();
    std::vector<uint64_t> rec_len(nq), rec_rows(nq);
    uint64_t total = 0;
    DevBuf& dout = d_out_[ob];
    const bool planned = layout_ == Layout::csr && nnz != nullptr;
    if (!planned) upload_refs(refs.data(), n);
    if (planned) {
        // host-planned prefix: the rows' nnz were read from the staged records' indptrs, so
        // the record offsets are known here -- no scan kernel and no host<->device round trip
        const uint64_t rb = planned_upload(ob, refs.data(), nnz->data(), n);
        const uint64_t* P = reinterpret_cast<const uint64_t*>(hp_[ob].p + rb);
        const uint64_t os = index_size(out_idt_), vs = value_size(vdt_);
        for (uint64_t q = 0; q < nq; ++q) {
            const uint64_t r0 = q * cr, rows = std::min(cr, n - r0), cnt = P[r0 + rows] - P[r0];
            if (out_idt_ == IDtype::u32 && (cnt > 0xFFFFFFFFull || n_var_ > 0x100000000ull))
                invalid("csr record: value " + std::to_string(std::max<uint64_t>(cnt, n_var_ - 1)) +
                        " does not fit index_dtype u32");
            rec_rows[q] = rows;
            rec_len[q] = kCsrHeaderBytes + os * (rows + 1) + (os + vs) * cnt;
            total += rec_len[q];
        }
        dout.ensure(total + total / 8);
        cudaEvent_t ta = nullptr, tb = nullptr;
        cuda_ok(cudaEventCreate(&ta), "event");
        cuda_ok(cudaEventCreate(&tb), "event");
        static const bool isolate = [] {  // diagnostics: the pack kernel alone on the device
            const char* e = std::getenv("RFL_PACK_ISOLATE");
            return e && e[0] == '1';
        }();
        if (isolate) cuda_ok(cudaDeviceSynchronize(), "isolate");
        gate_begin();
        cuda_ok(cudaEventRecord(ta, st_), "event");
        launch_csr_pack(absolute_view(layout_, vdt_, in_idt_, n_var_), reinterpret_cast<const RowRef*>(dp_[ob].p), n,
                        cr, out_idt_, reinterpret_cast<const uint64_t*>(dp_[ob].p + rb), dout.p, st_);
        cuda_ok(cudaEventRecord(tb, st_), "event");
        gate_end();
        timing_.emplace_back(ta, tb);
    } else if (layout_ == Layout::csr) {
        const ArenaView av = absolute_view(layout_, vdt_, in_idt_, n_var_);
        d_prefix_.ensure((n + 1) * 8);
        d_scratch_.ensure(csr_gather_scratch_bytes(n));
        cuda_ok(cudaEventRecord(e0_, st_), "event");
        launch_csr_row_scan(av, reinterpret_cast<RowRef*>(d_refs_.p), n, reinterpret_cast<uint64_t*>(d_prefix_.p),
                            d_scratch_.p, st_);
        cuda_ok(cudaEventRecord(e2_, st_), "event");
        h_prefix_.ensure((n + 1) * 8);
        cuda_ok(cudaMemcpyAsync(h_prefix_.p, d_prefix_.p, (n + 1) * 8, cudaMemcpyDeviceToHost, st_), "prefix D2H");
        cuda_ok(cudaStreamSynchronize(st_), "sync");
        const uint64_t* P = reinterpret_cast<const uint64_t*>(h_prefix_.p);
        const uint64_t os = index_size(out_idt_), vs = value_size(vdt_);
        for (uint64_t q = 0; q < nq; ++q) {
            const uint64_t r0 = q * cr, rows = std::min(cr, n - r0), nnz = P[r0 + rows] - P[r0];
            if (out_idt_ == IDtype::u32 && (nnz > 0xFFFFFFFFull || n_var_ > 0x100000000ull))
                invalid("csr record: value " + std::to_string(std::max<uint64_t>(nnz, n_var_ - 1)) +
                        " does not fit index_dtype u32");
            rec_rows[q] = rows;
            rec_len[q] = kCsrHeaderBytes + os * (rows + 1) + (os + vs) * nnz;
            total += rec_len[q];
        }
        dout.ensure(total + total / 8);
        cuda_ok(cudaEventRecord(e3_, st_), "event");
        launch_csr_pack(av, reinterpret_cast<RowRef*>(d_refs_.p), n, cr, out_idt_,
                        reinterpret_cast<uint64_t*>(d_prefix_.p), dout.p, st_);
        cuda_ok(cudaEventRecord(e1_, st_), "event");
    } else {
        const ArenaView av = absolute_view(layout_, vdt_, in_idt_, n_var_);
        total = n * row_bytes_;
        for (uint64_t q = 0; q < nq; ++q) {
            rec_rows[q] = std::min(cr, n - q * cr);
            rec_len[q] = rec_rows[q] * row_bytes_;
        }
        dout.ensure(std::max<uint64_t>(total + total / 8, 16));
        cuda_ok(cudaEventRecord(e0_, st_), "event");
        launch_dense_gather(av, reinterpret_cast<RowRef*>(d_refs_.p), n, OutDtype::native, dout.p, nullptr, st_);
        cuda_ok(cudaEventRecord(e1_, st_), "event");
    }
    cuda_ok(cudaEventRecord(packed_[ob], st_), "event");
    tr_.mark(" kernels", emits_ - 1);
    res_.d2h_bytes += total;
    std::vector<uint64_t> chunk_id;
    if (out_rows)
        for (uint64_t q = 0; q < nq; ++q) chunk_id.push_back((*out_rows)[q * cr] / cr);
    // provenance: u32 dataset_id + u64 source_row, LE (preshuffle.cpp:27-91)
    std::vector<uint8_t> prov_bytes(n * 12);
    for (uint64_t k = 0; k < n; ++k) {
        wr32(prov_bytes.data() + 12 * k, prov[k].first);
        wr64(prov_bytes.data() + 12 * k + 4, prov[k].second);
    }
    // The records leave the device in 64 MB pieces through a two-buffer pinned
    // ring on the writer's own stream, each piece written (parallel pwrites at
    // its records' file offsets) while the next one is in flight.  Jobs run in
    // emit order (each waits for its predecessor), off the staging thread.
    std::shared_future<void> prev = last_job_;
    last_job_ = std::async(std::launch::async, [this, ob, total, prev, rec_len = std::move(rec_len),
                                                rec_rows = std::move(rec_rows), chunk_id = std::move(chunk_id),
                                                prov_bytes = std::move(prov_bytes)] {
                    if (prev.valid()) prev.get();
                    DeviceGuard g(a_.device);
                    cuda_ok(cudaEventSynchronize(packed_[ob]), "pack done");
                    const uint8_t* src = d_out_[ob].p;
                    const uint64_t S = kPieceBytes;
                    const uint64_t pieces = (total + S - 1) / S;
                    auto issue = [&](uint64_t i) {
                        const uint64_t off = i * S, len = std::min(S, total - off);
                        std::unique_lock<std::mutex> lk = gate_wait();  // held while the piece is enqueued
                        cuda_ok(cudaMemcpyAsync(ring_[i & 1].p, src + off, len, cudaMemcpyDeviceToHost, wst_), "D2H");
                        cuda_ok(cudaEventRecord(ring_ev_[i & 1], wst_), "event");
                    };
                    if (out_->codec() == Codec::deflate) {
                        // whole records to the host, deflated in parallel (codec_encode,
                        // store.cpp:200 / preshuffle.cpp:70), appended in order
                        std::vector<uint8_t> host(total);
                        if (pieces) issue(0);
                        for (uint64_t i = 0; i < pieces; ++i) {
                            if (i + 1 < pieces) issue(i + 1);
                            cuda_ok(cudaEventSynchronize(ring_ev_[i & 1]), "D2H done");
                            std::memcpy(host.data() + i * S, ring_[i & 1].p, std::min(S, total - i * S));
                        }
                        const size_t nq = rec_len.size();
                        std::vector<uint64_t> rs(nq + 1, 0), ps(nq + 1, 0);
                        for (size_t q = 0; q < nq; ++q) {
                            rs[q + 1] = rs[q] + rec_len[q];
                            ps[q + 1] = ps[q] + rec_rows[q] * 12;
                        }
                        std::vector<std::vector<uint8_t>> enc(nq), penc(nq);
                        std::atomic<size_t> next{0};
                        std::vector<std::exception_ptr> errs(16);
                        std::vector<std::thread> pool;
                        const unsigned T = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
                        for (unsigned t = 0; t < T; ++t)
                            pool.emplace_back([&, t] {
                                try {
                                    for (size_t q; (q = next.fetch_add(1)) < nq;) {
                                        enc[q] = deflate_encode(host.data() + rs[q], rec_len[q]);
                                        penc[q] = deflate_encode(prov_bytes.data() + ps[q], rec_rows[q] * 12);
                                    }
                                } catch (...) {
                                    errs[t] = std::current_exception();
                                }
                            });
                        for (auto& th : pool) th.join();
                        for (auto& e : errs)
                            if (e) std::rethrow_exception(e);
                        for (size_t q = 0; q < nq; ++q) {
                            const int64_t cid = chunk_id.empty() ? -1 : static_cast<int64_t>(chunk_id[q]);
                            out_->append_encoded(enc[q].data(), enc[q].size(), rec_rows[q], cid);
                            prov_->append_encoded(penc[q].data(), penc[q].size(), rec_rows[q], cid);
                        }
                        return;
                    }
                    if (pieces) issue(0);
                    size_t q = 0;
                    uint64_t rstart = 0, ppos = 0;
                    RecordWriter::Placement cur;
                    for (uint64_t i = 0; i < pieces; ++i) {
                        if (i + 1 < pieces) issue(i + 1);
                        cuda_ok(cudaEventSynchronize(ring_ev_[i & 1]), "D2H done");
                        const uint64_t p0 = i * S, p1 = std::min(total, p0 + S);
                        const uint8_t* buf = ring_[i & 1].p;
                        while (q < rec_len.size() && rstart < p1) {
                            if (rstart >= p0)  // the record starts in this piece
                                cur = out_->reserve_record(rec_len[q], rec_rows[q],
                                                           chunk_id.empty() ? -1 : static_cast<int64_t>(chunk_id[q]));
                            const uint64_t a = std::max(rstart, p0), b = std::min(rstart + rec_len[q], p1);
                            RecordWriter::write_part(cur, a - rstart, buf + (a - p0), b - a);
                            if (rstart + rec_len[q] > p1) break;  // continues in the next piece
                            const int64_t cid = chunk_id.empty() ? -1 : static_cast<int64_t>(chunk_id[q]);
                            RecordWriter::write_part(prov_->reserve_record(rec_rows[q] * 12, rec_rows[q], cid), 0,
                                                     prov_bytes.data() + ppos, rec_rows[q] * 12);
                            ppos += rec_rows[q] * 12;
                            rstart += rec_len[q];
                            ++q;
                        }
                    }
                    for (; q < rec_len.size(); ++q) {  // empty records (total == 0 tail)
                        const int64_t cid = chunk_id.empty() ? -1 : static_cast<int64_t>(chunk_id[q]);
                        out_->reserve_record(rec_len[q], rec_rows[q], cid);
                        RecordWriter::write_part(prov_->reserve_record(rec_rows[q] * 12, rec_rows[q], cid), 0,
                                                 prov_bytes.data() + ppos, rec_rows[q] * 12);
                        ppos += rec_rows[q] * 12;
                    }
                }).share();
    wjob_[ob] = last_job_;
    res_.rows_written += n;
    if (planned) return;  // kernel time harvested later (no host sync here)
    float ms = 0.f, ms2 = 0.f;
    cuda_ok(cudaEventSynchronize(e1_), "sync");
    if (layout_ == Layout::csr) {  // kernel time only: scan (e0..e2) + pack (e3..e1)
        cuda_ok(cudaEventElapsedTime(&ms, e0_, e2_), "elapsed");
        cuda_ok(cudaEventElapsedTime(&ms2, e3_, e1_), "elapsed");
    } else {
        cuda_ok(cudaEventElapsedTime(&ms, e0_, e1_), "elapsed");
    }
    res_.gpu_ms += ms + ms2;
}

// Materialise refs[from..) into one device record in `dst` (same encoding as
// the inputs) and point the refs at it, so round arenas can be recycled.
void GpuShuffler::carry(std::vector<RowRef>& refs, uint64_t from, DevBuf& dst, const std::vector<uint32_t>* nnz) {
    const uint64_t n = refs.size() - from;
    if (n == 0) return;
    const ArenaView av = absolute_view(layout_, vdt_, in_idt_, n_var_);
    if (layout_ == Layout::csr && nnz) {  // host-planned, no sync: one record of all carried rows
        const uint64_t rb = planned_upload(2, refs.data() + from, nnz->data() + from, n);
        const uint64_t cnt = reinterpret_cast<const uint64_t*>(hp_[2].p + rb)[n];
        const uint64_t is = index_size(in_idt_), vs = value_size(vdt_);
        dst.ensure(kCsrHeaderBytes + is * (n + 1) + (is + vs) * cnt);
        launch_csr_pack(av, reinterpret_cast<const RowRef*>(dp_[2].p), n, n, in_idt_,
                        reinterpret_cast<const uint64_t*>(dp_[2].p + rb), dst.p, st_);
        for (uint64_t k = 0; k < n; ++k) refs[from + k] = {reinterpret_cast<uint64_t>(dst.p), k};
        return;
    }
    upload_refs(refs.data() + from, n);
    if (layout_ == Layout::csr) {
        d_prefix_.ensure((n + 1) * 8);
        d_scratch_.ensure(csr_gather_scratch_bytes(n));
        launch_csr_row_scan(av, reinterpret_cast<RowRef*>(d_refs_.p), n, reinterpret_cast<uint64_t*>(d_prefix_.p),
                            d_scratch_.p, st_);
        uint64_t nnz = 0;
        cuda_ok(cudaMemcpyAsync(&nnz, d_prefix_.p + n * 8, 8, cudaMemcpyDeviceToHost, st_), "D2H");
        cuda_ok(cudaStreamSynchronize(st_), "sync");
        const uint64_t is = index_size(in_idt_), vs = value_size(vdt_);
        dst.ensure(kCsrHeaderBytes + is * (n + 1) + (is + vs) * nnz);
        launch_csr_pack(av, reinterpret_cast<RowRef*>(d_refs_.p), n, n, in_idt_,
                        reinterpret_cast<uint64_t*>(d_prefix_.p), dst.p, st_);
    } else {
        dst.ensure(std::max<uint64_t>(n * row_bytes_, 16));
        launch_dense_gather(av, reinterpret_cast<RowRef*>(d_refs_.p), n, OutDtype::native, dst.p, nullptr, st_);
    }
    cuda_ok(cudaStreamSynchronize(st_), "sync");
    for (uint64_t k = 0; k < n; ++k) refs[from + k] = {reinterpret_cast<uint64_t>(dst.p), k};
}

GpuShuffler::~GpuShuffler() {
    try {  // an abandoned pass (error) still joins its writer job
        if (last_job_.valid()) last_job_.wait();
    } catch (...) {
    }
    if (st_) cudaStreamSynchronize(st_);
    for (auto& t : timing_) {
        cudaEventDestroy(t.first);
        cudaEventDestroy(t.second);
    }
    for (auto& e : hp_ev_)
        if (e) cudaEventDestroy(e);
    if (wst_) {
        cudaStreamSynchronize(wst_);
        for (int k = 0; k < 2; ++k) {
            cudaEventDestroy(stage_ev_[k]);
            cudaEventDestroy(ring_ev_[k]);
            cudaEventDestroy(packed_[k]);
        }
        cudaEventDestroy(gate_ev_);
        cudaEventDestroy(wgate_);
        cudaStreamDestroy(wst_);
    }
    if (st_) {
        cudaStreamSynchronize(st_);
        cudaEventDestroy(e0_);
        cudaEventDestroy(e1_);
        cudaEventDestroy(e2_);
        cudaEventDestroy(e3_);
        cudaStreamDestroy(st_);
    }
}

void GpuShuffler::init() {
    if (a_.inputs.empty()) invalid("run_shuffle: empty collection");
    if (a_.world < 1 || a_.rank >= a_.world) invalid("run_shuffle: rank must satisfy 0 <= rank < world");
    total_ = 0;
    for (const auto& p : a_.inputs) {
        Member m;
        m.hs = std::make_shared<HostStore>(p);
        m.offset = total_;
        const Manifest& man = m.hs->manifest();
        if (!ms_.empty()) {  // DatasetCollection::add (collection.cpp:10-24)
            const Manifest& f = ms_.front().hs->manifest();
            if (man.layout != f.layout)
                invalid(std::string("collection: store layout ") + to_string(man.layout) +
                        " does not match collection layout " + to_string(f.layout));
            if (man.value_dtype != f.value_dtype)
                invalid(std::string("collection: store value_dtype ") + to_string(man.value_dtype) +
                        " does not match collection value_dtype " + to_string(f.value_dtype));
        }
        if (man.codec == Codec::deflate) deflate_record_lengths(*m.hs, m.dec_len, nullptr);
        total_ += man.n_obs;
        ms_.push_back(std::move(m));
    }
    plan_ = plan_shuffle(total_, a_.c, a_.m, a_.seed);
    // every rank creates its own shard files only; the directories may already exist
    if (a_.rank == 0 && dir_nonempty(a_.out_path))
        invalid("run_shuffle: output path '" + a_.out_path + "' is not fresh");
    const Manifest& f = ms_.front().hs->manifest();
    layout_ = f.layout;
    vdt_ = f.value_dtype;
    in_idt_ = f.index_dtype.value_or(IDtype::u32);
    out_idt_ = a_.out_idt < 0 ? in_idt_ : static_cast<IDtype>(a_.out_idt);
    if (a_.out_chunk_rows < 1 || a_.out_cps < 1) invalid("run_shuffle: output chunk geometry must be >= 1");
    Manifest om;
    om.layout = layout_;
    om.var_names = unify(ms_, a_.outer);
    om.n_var = om.var_names.size();
    if (om.n_var >= 0xFFFFFFFFull) invalid("run_shuffle: unified n_var too large for the GPU column maps");
    if (layout_ == Layout::csr && in_idt_ == IDtype::u32 && om.n_var > 0x100000000ull)
        invalid("run_shuffle: unified n_var does not fit index_dtype u32");
    for (auto& m : ms_) {
        const Manifest& mm = m.hs->manifest();
        m.remap = !m.identity || (layout_ == Layout::csr && mm.index_dtype.value_or(IDtype::u32) != in_idt_);
        if (!m.remap) continue;
        std::vector<uint32_t> map;
        if (layout_ == Layout::csr) {  // member column -> unified column
            map.resize(m.col_map.size());
            for (size_t c = 0; c < map.size(); ++c)
                map[c] = m.col_map[c] == kMissing ? ~0u : static_cast<uint32_t>(m.col_map[c]);
        } else {  // unified column -> last member column mapping to it (scatter_dense_row order)
            map.assign(om.n_var, ~0u);
            for (size_t c = 0; c < m.col_map.size(); ++c)
                if (m.col_map[c] != kMissing) map[m.col_map[c]] = static_cast<uint32_t>(c);
        }
        DeviceGuard g(a_.device);
        m.d_map = std::make_shared<DevBuf>();
        m.d_map->ensure(std::max<size_t>(map.size() * 4, 16));
        if (!map.empty()) cuda_ok(cudaMemcpy(m.d_map->p, map.data(), map.size() * 4, cudaMemcpyHostToDevice), "map H2D");
    }
    om.value_dtype = vdt_;
    if (layout_ == Layout::csr) om.index_dtype = out_idt_;
    om.chunk_rows = a_.out_chunk_rows;
    om.chunks_per_shard = a_.out_cps;
    om.codec = a_.out_codec ? Codec::deflate : Codec::none;
    om.has_provenance = true;
    n_var_ = om.n_var;
    row_bytes_ = n_var_ * value_size(vdt_);
    // defer_manifest (preshuffle.cpp:217): the manifest lands only when the pass completes (rank 0)
    out_ = std::make_unique<RecordWriter>(a_.out_path, om, /*defer_manifest=*/true, "shards", a_.rank == 0);
    Manifest pm;  // provenance sidecar: same chunk grid, 12-byte records
    pm.layout = Layout::dense;
    pm.chunk_rows = a_.out_chunk_rows;
    pm.chunks_per_shard = a_.out_cps;
    pm.codec = om.codec;  // ProvenanceWriter encodes with the store's codec (preshuffle.cpp:70,219)
    prov_ = std::make_unique<RecordWriter>(a_.out_path + "/provenance", pm, true, "shards", false);
    round_first_out_.assign(plan_.rounds.size() + 1, 0);
    for (size_t r = 0; r < plan_.rounds.size(); ++r) {
        uint64_t rows = 0;
        for (uint64_t id : plan_.rounds[r]) rows += plan_.block_end(id) - plan_.block_start(id);
        round_first_out_[r + 1] = round_first_out_[r] + rows;
    }
    if (const char* nv = std::getenv("RFL_NO_VALIDATE")) validate_ = nv[0] != '1';
    DeviceGuard g(a_.device);
    cuda_ok(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking), "stream");
    cuda_ok(cudaStreamCreateWithFlags(&wst_, cudaStreamNonBlocking), "stream");
    cuda_ok(cudaEventCreateWithFlags(&gate_ev_, cudaEventDisableTiming), "event");
    cuda_ok(cudaEventCreateWithFlags(&wgate_, cudaEventDisableTiming), "event");
    if (const char* ge = std::getenv("RFL_PACK_GATE")) gate_on_ = ge[0] != '0';
    for (int k = 0; k < 2; ++k) {  // pinned staging / output rings, allocated once (cudaHostAlloc is slow)
        h_stage_[k].ensure(kStageBytes);
        ring_[k].ensure(kPieceBytes);
        cuda_ok(cudaEventCreateWithFlags(&stage_ev_[k], cudaEventDisableTiming), "event");
        cuda_ok(cudaEventCreateWithFlags(&ring_ev_[k], cudaEventDisableTiming), "event");
        cuda_ok(cudaEventCreateWithFlags(&packed_[k], cudaEventDisableTiming), "event");
    }
    cuda_ok(cudaEventCreate(&e0_), "event");
    cuda_ok(cudaEventCreate(&e1_), "event");
    cuda_ok(cudaEventCreate(&e2_), "event");
    cuda_ok(cudaEventCreate(&e3_), "event");
}

// The round's blocks as per-member segments in block order (:234-251); with
// src_rank, the rank staging each assembly row (block index in round mod W).
void GpuShuffler::round_segments(uint64_t r, Segs& segs, std::vector<std::pair<uint32_t, uint64_t>>& prov,
                                 std::vector<uint32_t>* src_rank) {
    segs.clear();
    prov.clear();
    if (src_rank) src_rank->clear();
    for (size_t bi = 0; bi < plan_.rounds[r].size(); ++bi) {
        const uint64_t id = plan_.rounds[r][bi];
        const uint32_t owner = static_cast<uint32_t>(bi % a_.world);
        uint64_t row = plan_.block_start(id);
        const uint64_t end = plan_.block_end(id);
        while (row < end) {
            size_t mi = 0;
            while (mi + 1 < ms_.size() && ms_[mi + 1].offset <= row) ++mi;
            const uint64_t mend = ms_[mi].offset + ms_[mi].hs->manifest().n_obs;
            const uint64_t stop = std::min(end, mend);
            if (!src_rank || owner == a_.rank)
                segs.push_back({static_cast<uint32_t>(mi), {row - ms_[mi].offset, stop - ms_[mi].offset}});
            for (uint64_t x = row; x < stop; ++x) {
                prov.emplace_back(static_cast<uint32_t>(mi), x - ms_[mi].offset);
                if (src_rank) src_rank->push_back(owner);
            }
            row = stop;
        }
    }
}

ShuffleResult GpuShuffler::run() {
    PhaseTrace& tr = tr_;
    init();
    tr.mark("init", 0);
    DeviceGuard g(a_.device);
    std::vector<RowRef> round_refs;
    std::vector<uint32_t> round_nnz;
    Segs segs;
    std::vector<std::pair<uint32_t, uint64_t>> asm_prov;
    const uint64_t cr = a_.out_chunk_rows;
    for (size_t r = 0; r < plan_.rounds.size(); ++r) {
        round_segments(r, segs, asm_prov, nullptr);
        const uint64_t round_rows = asm_prov.size();
        res_.peak_resident_rows = std::max(res_.peak_resident_rows, round_rows + std::min(a_.c, round_rows));
        tr.mark("segments", r);
        stage_round(segs, arena_[r % 2], round_refs, r, &round_nnz);
        tr.mark("stage", r);
        check_duplicates(r, bad_asm_, round_rows);
        const std::vector<uint64_t> perm = round_permutation(a_.seed, r, round_rows);
        // host-planned packing while every row's nnz is known (identity members)
        const bool have = round_nnz.size() == round_rows && (r == 0 || nnz_ok_);
        if (!have) pend_nnz_.clear();
        nnz_ok_ = have;
        for (uint64_t k = 0; k < round_rows; ++k) {
            pending_.push_back(round_refs[perm[k]]);
            pend_prov_.push_back(asm_prov[perm[k]]);
            if (have) pend_nnz_.push_back(round_nnz[perm[k]]);
        }
        tr.mark("permute", r);
        const bool last = r + 1 == plan_.rounds.size();
        const uint64_t n_emit = last ? pending_.size() : pending_.size() / cr * cr;
        emit(pending_, pend_prov_, n_emit, nullptr, nnz_ok_ ? &pend_nnz_ : nullptr);
        tr.mark("emit", r);
        pending_.erase(pending_.begin(), pending_.begin() + n_emit);
        pend_prov_.erase(pend_prov_.begin(), pend_prov_.begin() + n_emit);
        if (nnz_ok_) pend_nnz_.erase(pend_nnz_.begin(), pend_nnz_.begin() + n_emit);
        if (!pending_.empty()) carry(pending_, 0, carry_[r % 2], nnz_ok_ ? &pend_nnz_ : nullptr);
        tr.mark("carry", r);
        res_.rounds++;
    }
    drain_writes();
    harvest_timing();
    tr.mark("drain", 0);
    out_->finish();
    prov_->finish();
    write_text_file(a_.out_path + "/provenance/meta.json", meta_json(a_.seed, a_.c, a_.m));
    return res_;
}

// ---- rank API ---------------------------------------------------------------
// Stage this rank's blocks of round r, group its rows by destination (owner of
// the output shard) in output order, scan them, and report the message size
// for every destination (one encoded record per destination).
void GpuShuffler::stage(uint64_t r, uint64_t* send_bytes) {
    if (r >= plan_.rounds.size()) invalid("run_shuffle: round out of range");
    DeviceGuard g(a_.device);
    Segs segs;
    std::vector<std::pair<uint32_t, uint64_t>> asm_prov;
    std::vector<uint32_t> asm_src;
    round_segments(r, segs, asm_prov, &asm_src);
    const uint64_t round_rows = asm_prov.size();
    res_.peak_resident_rows = std::max(res_.peak_resident_rows, round_rows + std::min(a_.c, round_rows));
    std::vector<RowRef> my_refs;
    stage_round(segs, arena_[r % 2], my_refs, r);  // refs of my assembly rows, in assembly order
    std::vector<int64_t> asm_to_mine(round_rows, -1);
    std::vector<uint64_t> mine_to_asm;
    for (uint64_t a = 0, k = 0; a < round_rows; ++a)
        if (asm_src[a] == a_.rank) {
            asm_to_mine[a] = static_cast<int64_t>(k++);
            mine_to_asm.push_back(a);
        }
    if (!bad_asm_.empty()) {
        std::vector<uint64_t> bad;
        for (uint64_t k : bad_asm_) bad.push_back(mine_to_asm[k]);
        check_duplicates(r, bad, round_rows);
    }
    const std::vector<uint64_t> perm = round_permutation(a_.seed, r, round_rows);
    const uint64_t shard_rows = a_.out_chunk_rows * a_.out_cps, first = round_first_out_[r];
    const uint32_t W = a_.world;
    std::vector<std::vector<RowRef>> by_dst(W);
    mine_src_.clear();
    mine_out_.clear();
    mine_prov_.clear();
    for (uint64_t k = 0; k < round_rows; ++k) {
        const uint64_t a = perm[k];
        const uint32_t dst = static_cast<uint32_t>(((first + k) / shard_rows) % W);
        if (asm_src[a] == a_.rank) by_dst[dst].push_back(my_refs[asm_to_mine[a]]);
        if (dst == a_.rank) {
            mine_src_.push_back(asm_src[a]);
            mine_out_.push_back(first + k);
            mine_prov_.push_back(asm_prov[a]);
        }
    }
    send_start_.assign(W, 0);
    send_count_.assign(W, 0);
    std::vector<RowRef> all;
    for (uint32_t d = 0; d < W; ++d) {
        send_start_[d] = all.size();
        send_count_[d] = by_dst[d].size();
        all.insert(all.end(), by_dst[d].begin(), by_dst[d].end());
    }
    const uint64_t n = all.size();
    d_send_refs_.ensure(std::max<uint64_t>(n, 1) * sizeof(RowRef));
    h_refs_.ensure(std::max<uint64_t>(n, 1) * sizeof(RowRef));
    std::memcpy(h_refs_.p, all.data(), n * sizeof(RowRef));
    if (n) cuda_ok(cudaMemcpyAsync(d_send_refs_.p, h_refs_.p, n * sizeof(RowRef), cudaMemcpyHostToDevice, st_), "H2D");
    res_.h2d_bytes += n * sizeof(RowRef);
    const uint64_t is = index_size(in_idt_), vs = value_size(vdt_);
    if (layout_ == Layout::csr) {
        d_send_prefix_.ensure((n + 1) * 8);
        d_scratch_.ensure(csr_gather_scratch_bytes(std::max<uint64_t>(n, 1)));
        launch_csr_row_scan(absolute_view(layout_, vdt_, in_idt_, n_var_), reinterpret_cast<RowRef*>(d_send_refs_.p),
                            n, reinterpret_cast<uint64_t*>(d_send_prefix_.p), d_scratch_.p, st_);
        h_prefix_.ensure((n + 1) * 8);
        cuda_ok(cudaMemcpyAsync(h_prefix_.p, d_send_prefix_.p, (n + 1) * 8, cudaMemcpyDeviceToHost, st_), "D2H");
        cuda_ok(cudaStreamSynchronize(st_), "sync");
        const uint64_t* P = reinterpret_cast<const uint64_t*>(h_prefix_.p);
        for (uint32_t d = 0; d < W; ++d) {
            const uint64_t c = send_count_[d];
            const uint64_t nnz = P[send_start_[d] + c] - P[send_start_[d]];
            send_bytes[d] = c ? kCsrHeaderBytes + is * (c + 1) + (is + vs) * nnz : 0;
        }
    } else {
        cuda_ok(cudaStreamSynchronize(st_), "sync");
        for (uint32_t d = 0; d < W; ++d) send_bytes[d] = send_count_[d] * row_bytes_;
    }
    send_bytes_.assign(send_bytes, send_bytes + W);
    staged_round_ = r;
}

void GpuShuffler::recv_buffer(uint64_t bytes, void** ptr, void* ipc_handle, int* changed) {
    DeviceGuard g(a_.device);
    const uint64_t before = recv_.cap;
    const uint8_t* old = recv_.p;
    if (bytes > recv_.cap) recv_.ensure(bytes + bytes / 4 + (1 << 20));
    *changed = (recv_.p != old || recv_.cap != before) ? 1 : 0;
    *ptr = recv_.p;
    if (ipc_handle) {
        cudaIpcMemHandle_t h;
        cuda_ok(cudaIpcGetMemHandle(&h, recv_.p), "cudaIpcGetMemHandle");
        std::memcpy(ipc_handle, &h, sizeof(h));
    }
}

// Pack my message for destination d straight into d's receive buffer (dst[d]
// = peer address over NVLink/IPC, or local): gather + exchange in one pass.
void GpuShuffler::send(uint64_t r, void* const* dst) {
    if (r != staged_round_) invalid("run_shuffle: send() without stage() of the same round");
    DeviceGuard g(a_.device);
    const ArenaView av = absolute_view(layout_, vdt_, in_idt_, n_var_);
    cuda_ok(cudaEventRecord(e0_, st_), "event");
    uint64_t sent = 0;
    for (uint32_t d = 0; d < a_.world; ++d) {
        const uint64_t c = send_count_[d];
        if (!c) continue;
        const RowRef* refs = reinterpret_cast<const RowRef*>(d_send_refs_.p) + send_start_[d];
        if (layout_ == Layout::csr)
            launch_csr_pack(av, refs, c, c, in_idt_, reinterpret_cast<uint64_t*>(d_send_prefix_.p) + send_start_[d],
                            static_cast<uint8_t*>(dst[d]), st_);
        else
            launch_dense_gather(av, refs, c, OutDtype::native, dst[d], nullptr, st_);
        sent += c;
    }
    cuda_ok(cudaEventRecord(e1_, st_), "event");
    cuda_ok(cudaStreamSynchronize(st_), "sync");  // peer writes complete before the caller's barrier
    float ms = 0.f;
    cuda_ok(cudaEventElapsedTime(&ms, e0_, e1_), "elapsed");
    res_.gpu_ms += ms;
    res_.send_ms += ms;
    for (uint32_t d = 0; d < a_.world; ++d)
        if (d != a_.rank) res_.peer_bytes += send_bytes_[d];
}

// Owner side: my rows of round r arrived as one record per source rank in my
// receive buffer (offsets = running 16-B aligned sums of recv_bytes).  Emit
// every owned chunk that is now complete; carry the rest.
void GpuShuffler::emit_round(uint64_t r, const uint64_t* recv_bytes) {
    if (r != staged_round_) invalid("run_shuffle: emit_round() without stage() of the same round");
    DeviceGuard g(a_.device);
    std::vector<uint64_t> off(a_.world, 0), cursor(a_.world, 0);
    for (uint32_t s = 1; s < a_.world; ++s) off[s] = align_up(off[s - 1] + recv_bytes[s - 1], kAlign);
    for (size_t i = 0; i < mine_src_.size(); ++i) {
        const uint32_t s = mine_src_[i];
        pending_.push_back({reinterpret_cast<uint64_t>(recv_.p) + off[s], cursor[s]++});
        pend_prov_.push_back(mine_prov_[i]);
        pend_out_.push_back(mine_out_[i]);
    }
    const bool last = r + 1 == plan_.rounds.size();
    const uint64_t cr = a_.out_chunk_rows;
    const uint64_t limit = last ? total_ : round_first_out_[r + 1] / cr * cr;  // rows of complete chunks
    const uint64_t n_emit = std::lower_bound(pend_out_.begin(), pend_out_.end(), limit) - pend_out_.begin();
    emit(pending_, pend_prov_, n_emit, &pend_out_);
    pending_.erase(pending_.begin(), pending_.begin() + n_emit);
    pend_prov_.erase(pend_prov_.begin(), pend_prov_.begin() + n_emit);
    pend_out_.erase(pend_out_.begin(), pend_out_.begin() + n_emit);
    if (!pending_.empty()) carry(pending_, 0, carry_[r % 2]);  // the receive buffer is reused next round
    res_.rounds++;
}

ShuffleResult GpuShuffler::finish() {
    drain_writes();
    harvest_timing();
    out_->finish(static_cast<int64_t>(total_));  // rank 0 writes the manifest (others: shards only)
    prov_->finish();
    if (a_.rank == 0) write_text_file(a_.out_path + "/provenance/meta.json", meta_json(a_.seed, a_.c, a_.m));
    return res_;
}

}  // namespace

ShuffleResult run_shuffle_gpu(const ShuffleArgs& a) {
    if (a.world != 1) invalid("run_shuffle: multi-GPU runs go through the rank API (rfl_pshuf_*)");
    return GpuShuffler(a).run();
}

// ---- rank API wrappers --------------------------------------------------------
struct RankShuffle {
    GpuShuffler s;
    explicit RankShuffle(const ShuffleArgs& a) : s(a) {}
};
RankShuffle* rank_shuffle_create(const ShuffleArgs& a, uint64_t* n_rounds) {
    auto* h = new RankShuffle(a);
    try {
        h->s.init();
    } catch (...) {
        delete h;
        throw;
    }
    *n_rounds = h->s.n_rounds();
    return h;
}
void rank_shuffle_stage(RankShuffle* h, uint64_t r, uint64_t* send_bytes) { h->s.stage(r, send_bytes); }
void rank_shuffle_recv(RankShuffle* h, uint64_t bytes, void** ptr, void* handle, int* changed) {
    h->s.recv_buffer(bytes, ptr, handle, changed);
}
void rank_shuffle_send(RankShuffle* h, uint64_t r, void* const* dst) { h->s.send(r, dst); }
void rank_shuffle_emit(RankShuffle* h, uint64_t r, const uint64_t* recv_bytes) { h->s.emit_round(r, recv_bytes); }
ShuffleResult rank_shuffle_finish(RankShuffle* h) { return h->s.finish(); }
void rank_shuffle_destroy(RankShuffle* h) { delete h; }

}  // namespace rfl
