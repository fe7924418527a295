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
#include <cstring>
#include <memory>
#include <numeric>
#include <unordered_map>
#include <unordered_set>

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
constexpr uint64_t kStageBytes = 128ull << 20;   // pinned bounce buffer per direction
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
};

std::string meta_json(uint64_t seed, uint64_t c, uint64_t m) {  // ProvenanceWriter::finish (:32-47)
    return std::string("{\n  \"rng\": \"") + Rng::kName + "\",\n  \"seed\": " + std::to_string(seed) +
           ",\n  \"block_rows\": " + std::to_string(c) + ",\n  \"buffer_rows\": " + std::to_string(m) + "\n}\n";
}

// DatasetCollection::rebuild_unified (collection.cpp:28-82): unified axis and
// per-member identity test.  Only identity members are supported on the GPU
// path (column reprojection is SURVEY §8f "next").
std::vector<std::string> unify(const std::vector<Member>& ms, bool outer) {
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
    for (size_t i = 0; i < ms.size(); ++i) {
        const auto& v = ms[i].hs->manifest().var_names;
        if (v.size() != uni.size() || !std::equal(v.begin(), v.end(), uni.begin()))
            invalid("run_shuffle: member " + std::to_string(i) +
                    " needs column reprojection, which the GPU path does not implement yet (identity columns only)");
    }
    return uni;
}

class GpuShuffler {
public:
    GpuShuffler(const ShuffleArgs& a) : a_(a) {}
    ShuffleResult run();

private:
    void stage_round(const std::vector<std::pair<uint32_t, std::pair<uint64_t, uint64_t>>>& segs, DevBuf& arena,
                     std::vector<RowRef>& refs);
    void emit(const std::vector<RowRef>& refs, const std::vector<std::pair<uint32_t, uint64_t>>& prov, uint64_t n);
    void carry(std::vector<RowRef>& refs, uint64_t from, DevBuf& dst);
    void upload_refs(const RowRef* refs, uint64_t n);

    ShuffleArgs a_;
    std::vector<Member> ms_;
    Layout layout_ = Layout::csr;
    VDtype vdt_ = VDtype::f32;
    IDtype in_idt_ = IDtype::u32, out_idt_ = IDtype::u32;
    uint64_t n_var_ = 0, row_bytes_ = 0;
    std::unique_ptr<RecordWriter> out_, prov_;
    cudaStream_t st_ = nullptr;
    cudaEvent_t e0_ = nullptr, e1_ = nullptr;
    DevBuf d_refs_, d_prefix_, d_scratch_, d_out_;
    PinBuf h_stage_, h_refs_, h_prefix_, h_out_;
    ShuffleResult res_;
    std::vector<uint8_t> prov_rec_;
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
                              DevBuf& arena, std::vector<RowRef>& refs) {
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
        len[i] = ms_[need[i].first].hs->record_slot(need[i].second).len;
        off[i] = total;
        total = align_up(total + len[i], kAlign);
    }
    arena.ensure(std::max<uint64_t>(total, 16));
    // coalesced reads of adjacent records of one shard (store.cpp:427-447) through a pinned bounce buffer
    h_stage_.ensure(kStageBytes);
    uint64_t fill = 0, fill_dst = 0;
    auto flush = [&] {
        if (!fill) return;
        cuda_ok(cudaMemcpyAsync(arena.p + fill_dst, h_stage_.p, fill, cudaMemcpyHostToDevice, st_), "stage H2D");
        cuda_ok(cudaStreamSynchronize(st_), "stage sync");
        res_.h2d_bytes += fill;
        fill = 0;
    };
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
        // bytes [off[i], off[j-1]+len) of the arena, laid out with alignment gaps
        const uint64_t span = off[j - 1] + len[j - 1] - off[i];
        if (span > kStageBytes) {  // a huge run: read record by record
            for (size_t k = i; k < j; ++k) {
                flush();
                h_stage_.ensure(len[k]);
                hs.read_record(need[k].second, h_stage_.p, len[k]);
                fill = len[k];
                fill_dst = off[k];
                flush();
                h_stage_.ensure(kStageBytes);
            }
        } else {
            // the bounce buffer mirrors arena bytes [fill_dst, fill_dst + fill); alignment gaps ride along
            if (fill && off[i] + span - fill_dst > kStageBytes) flush();
            if (!fill) fill_dst = off[i];
            uint8_t* base = h_stage_.p + (off[i] - fill_dst);
            hs.read_shard_bytes(shard, first.off, base, run, false);
            // spread to aligned offsets (targets move forward only: back to front)
            std::vector<uint64_t> rel(j - i, 0);
            for (size_t k = i + 1; k < j; ++k) rel[k - i] = rel[k - i - 1] + len[k - 1];
            for (size_t k = j - 1; k > i; --k) std::memmove(base + (off[k] - off[i]), base + rel[k - i], len[k]);
            fill = off[j - 1] + len[j - 1] - fill_dst;
        }
        res_.input_bytes += run;
        i = j;
    }
    flush();
    // refs per assembly row
    refs.clear();
    for (const auto& s : segs) {
        const Manifest& m = ms_[s.first].hs->manifest();
        for (uint64_t r = s.second.first; r < s.second.second; ++r) {
            const uint64_t q = r / m.chunk_rows;
            const size_t k = std::lower_bound(need.begin(), need.end(), std::make_pair(s.first, q)) - need.begin();
            refs.push_back({reinterpret_cast<uint64_t>(arena.p) + off[k], r - q * m.chunk_rows});
        }
    }
}

// Write refs[0..n) as output chunk records (+ provenance records).
void GpuShuffler::emit(const std::vector<RowRef>& refs, const std::vector<std::pair<uint32_t, uint64_t>>& prov,
                       uint64_t n) {
    if (n == 0) return;
    const uint64_t cr = a_.out_chunk_rows;
    const uint64_t nq = (n + cr - 1) / cr;
    upload_refs(refs.data(), n);
    std::vector<uint64_t> rec_len(nq), rec_rows(nq);
    uint64_t total = 0;
    if (layout_ == Layout::csr) {
        const ArenaView av = absolute_view(layout_, vdt_, in_idt_, n_var_);
        d_prefix_.ensure((n + 1) * 8);
        d_scratch_.ensure(csr_gather_scratch_bytes(n));
        cuda_ok(cudaEventRecord(e0_, st_), "event");
        launch_csr_row_scan(av, reinterpret_cast<RowRef*>(d_refs_.p), n, reinterpret_cast<uint64_t*>(d_prefix_.p),
                            d_scratch_.p, st_);
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
        d_out_.ensure(total);
        launch_csr_pack(av, reinterpret_cast<RowRef*>(d_refs_.p), n, cr, out_idt_,
                        reinterpret_cast<uint64_t*>(d_prefix_.p), d_out_.p, st_);
        cuda_ok(cudaEventRecord(e1_, st_), "event");
    } else {
        const ArenaView av = absolute_view(layout_, vdt_, in_idt_, n_var_);
        total = n * row_bytes_;
        for (uint64_t q = 0; q < nq; ++q) {
            rec_rows[q] = std::min(cr, n - q * cr);
            rec_len[q] = rec_rows[q] * row_bytes_;
        }
        d_out_.ensure(std::max<uint64_t>(total, 16));
        cuda_ok(cudaEventRecord(e0_, st_), "event");
        launch_dense_gather(av, reinterpret_cast<RowRef*>(d_refs_.p), n, OutDtype::native, d_out_.p, nullptr, st_);
        cuda_ok(cudaEventRecord(e1_, st_), "event");
    }
    h_out_.ensure(std::max<uint64_t>(total, 16));
    if (total) cuda_ok(cudaMemcpyAsync(h_out_.p, d_out_.p, total, cudaMemcpyDeviceToHost, st_), "records D2H");
    cuda_ok(cudaStreamSynchronize(st_), "sync");
    float ms = 0.f;
    cuda_ok(cudaEventElapsedTime(&ms, e0_, e1_), "elapsed");
    res_.gpu_ms += ms;
    res_.d2h_bytes += total;
    uint64_t pos = 0;
    for (uint64_t q = 0; q < nq; ++q) {
        out_->append_record(h_out_.p + pos, rec_len[q], rec_rows[q]);
        pos += rec_len[q];
        // provenance: u32 dataset_id + u64 source_row, LE (preshuffle.cpp:27-91)
        prov_rec_.resize(rec_rows[q] * 12);
        for (uint64_t k = 0; k < rec_rows[q]; ++k) {
            const auto& p = prov[q * cr + k];
            wr32(prov_rec_.data() + 12 * k, p.first);
            wr64(prov_rec_.data() + 12 * k + 4, p.second);
        }
        prov_->append_record(prov_rec_.data(), prov_rec_.size(), rec_rows[q]);
    }
    res_.rows_written += n;
}

// Materialise refs[from..) into one device record in `dst` (same encoding as
// the inputs) and point the refs at it, so round arenas can be recycled.
void GpuShuffler::carry(std::vector<RowRef>& refs, uint64_t from, DevBuf& dst) {
    const uint64_t n = refs.size() - from;
    if (n == 0) return;
    upload_refs(refs.data() + from, n);
    const ArenaView av = absolute_view(layout_, vdt_, in_idt_, n_var_);
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

ShuffleResult GpuShuffler::run() {
    if (a_.inputs.empty()) invalid("run_shuffle: empty collection");
    if (a_.world != 1) invalid("run_shuffle: multi-GPU runs go through the rank API (world must be 1 here)");
    uint64_t total = 0;
    for (const auto& p : a_.inputs) {
        Member m;
        m.hs = std::make_shared<HostStore>(p);
        m.offset = total;
        const Manifest& man = m.hs->manifest();
        if (!ms_.empty()) {  // DatasetCollection::add (collection.cpp:10-24)
            const Manifest& f = ms_.front().hs->manifest();
            if (man.layout != f.layout)
                invalid(std::string("collection: store layout ") + to_string(man.layout) +
                        " does not match collection layout " + to_string(f.layout));
            if (man.value_dtype != f.value_dtype)
                invalid(std::string("collection: store value_dtype ") + to_string(man.value_dtype) +
                        " does not match collection value_dtype " + to_string(f.value_dtype));
            if (man.index_dtype != f.index_dtype)
                invalid("run_shuffle: members with different index dtypes are not supported on the GPU path");
        }
        if (man.codec != Codec::none) invalid("GPU path requires codec none (deflate decode is out of scope)");
        total += man.n_obs;
        ms_.push_back(std::move(m));
    }
    const ShufflePlan plan = plan_shuffle(total, a_.c, a_.m, a_.seed);
    if (dir_nonempty(a_.out_path)) invalid("run_shuffle: output path '" + a_.out_path + "' is not fresh");
    const Manifest& f = ms_.front().hs->manifest();
    layout_ = f.layout;
    vdt_ = f.value_dtype;
    in_idt_ = f.index_dtype.value_or(IDtype::u32);
    out_idt_ = a_.out_idt < 0 ? in_idt_ : static_cast<IDtype>(a_.out_idt);
    Manifest om;
    om.layout = layout_;
    om.var_names = unify(ms_, a_.outer);
    om.n_var = om.var_names.size();
    om.value_dtype = vdt_;
    if (layout_ == Layout::csr) om.index_dtype = out_idt_;
    om.chunk_rows = a_.out_chunk_rows;
    om.chunks_per_shard = a_.out_cps;
    om.codec = Codec::none;
    om.has_provenance = true;
    n_var_ = om.n_var;
    row_bytes_ = n_var_ * value_size(vdt_);
    if (a_.out_chunk_rows < 1 || a_.out_cps < 1) invalid("run_shuffle: output chunk geometry must be >= 1");
    out_ = std::make_unique<RecordWriter>(a_.out_path, om, /*defer_manifest=*/true);
    Manifest pm;  // provenance sidecar: same chunk grid, 12-byte records
    pm.layout = Layout::dense;
    pm.chunk_rows = a_.out_chunk_rows;
    pm.chunks_per_shard = a_.out_cps;
    prov_ = std::make_unique<RecordWriter>(a_.out_path + "/provenance", pm, true, "shards", false);

    DeviceGuard g(a_.device);
    cuda_ok(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking), "stream");
    cuda_ok(cudaEventCreate(&e0_), "event");
    cuda_ok(cudaEventCreate(&e1_), "event");
    DevBuf arena[2], carry_buf[2];
    std::vector<RowRef> pending, round_refs;
    std::vector<std::pair<uint32_t, uint64_t>> pend_prov;
    const uint64_t cr = a_.out_chunk_rows;
    try {
        for (size_t r = 0; r < plan.rounds.size(); ++r) {
            // split the round's blocks into per-member segments, in block order (:234-251)
            std::vector<std::pair<uint32_t, std::pair<uint64_t, uint64_t>>> segs;
            std::vector<std::pair<uint32_t, uint64_t>> asm_prov;
            for (const uint64_t id : plan.rounds[r]) {
                uint64_t row = plan.block_start(id);
                const uint64_t end = plan.block_end(id);
                while (row < end) {
                    size_t mi = 0;
                    while (mi + 1 < ms_.size() && ms_[mi + 1].offset <= row) ++mi;
                    const uint64_t mend = ms_[mi].offset + ms_[mi].hs->manifest().n_obs;
                    const uint64_t stop = std::min(end, mend);
                    segs.push_back({static_cast<uint32_t>(mi), {row - ms_[mi].offset, stop - ms_[mi].offset}});
                    for (uint64_t x = row; x < stop; ++x) asm_prov.emplace_back(static_cast<uint32_t>(mi), x - ms_[mi].offset);
                    row = stop;
                }
            }
            const uint64_t round_rows = asm_prov.size();
            res_.peak_resident_rows = std::max(res_.peak_resident_rows, round_rows + std::min(a_.c, round_rows));
            stage_round(segs, arena[r % 2], round_refs);
            const std::vector<uint64_t> perm = round_permutation(a_.seed, r, round_rows);
            for (uint64_t k = 0; k < round_rows; ++k) {
                pending.push_back(round_refs[perm[k]]);
                pend_prov.push_back(asm_prov[perm[k]]);
            }
            const bool last = r + 1 == plan.rounds.size();
            const uint64_t n_emit = last ? pending.size() : pending.size() / cr * cr;
            emit(pending, pend_prov, n_emit);
            pending.erase(pending.begin(), pending.begin() + n_emit);
            pend_prov.erase(pend_prov.begin(), pend_prov.begin() + n_emit);
            if (!pending.empty()) carry(pending, 0, carry_buf[r % 2]);
            res_.rounds++;
        }
        out_->finish();
        prov_->finish();
        write_text_file(a_.out_path + "/provenance/meta.json", meta_json(a_.seed, a_.c, a_.m));
    } catch (...) {
        cudaStreamSynchronize(st_);
        cudaEventDestroy(e0_);
        cudaEventDestroy(e1_);
        cudaStreamDestroy(st_);
        throw;
    }
    cudaEventDestroy(e0_);
    cudaEventDestroy(e1_);
    cudaStreamDestroy(st_);
    return res_;
}

}  // namespace

ShuffleResult run_shuffle_gpu(const ShuffleArgs& a) { return GpuShuffler(a).run(); }

}  // namespace rfl
