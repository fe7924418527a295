// Device store images + GPU BatchIterator (see engine.hpp).
#include <sys/mman.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>

#include "codec.hpp"
#include "engine.hpp"

namespace rfl {

void cuda_ok(cudaError_t e, const char* what) {
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();  // not sticky: clear it so the context stays usable
        throw Error(kNoMem, std::string(what) + ": " + cudaGetErrorString(e));
    }
    if (e != cudaSuccess) throw Error(kCuda, std::string(what) + ": " + cudaGetErrorString(e));
}

DeviceGuard::DeviceGuard(int dev) {
    cuda_ok(cudaGetDevice(&prev), "cudaGetDevice");
    if (dev != prev) cuda_ok(cudaSetDevice(dev), "cudaSetDevice");
}
DeviceGuard::~DeviceGuard() { cudaSetDevice(prev); }

namespace {
constexpr uint64_t kAlign = kRecAlign;
constexpr uint64_t kPad = kRecPad;
constexpr uint64_t kUploadRun = 64ull << 20;    // pinned bounce buffer for uploads
}  // namespace

// ====================================================== record checks ===
namespace {
std::string chunk_where(const Manifest& m, uint64_t q) {  // process_shard's wrapping (store.cpp:455-457)
    return "chunk " + std::to_string(q) + " in shard " + std::to_string(q / m.chunks_per_shard) + ": ";
}
uint64_t rd_index(const Manifest& m, const uint8_t* p) { return *m.index_dtype == IDtype::u32 ? rd32(p) : rd64(p); }
}  // namespace

void full_check_csr_record(const Manifest& m, uint64_t q, const uint8_t* rec, uint64_t len) {
    const std::string at = chunk_where(m, q);
    if (len < kCsrHeaderBytes) corrupt(at + "csr record shorter than header");
    const uint64_t rows = m.rows_in_chunk(q);
    const uint32_t hdr_rows = rd32(rec);
    const uint64_t nnz = rd64(rec + 4);
    if (hdr_rows != rows)
        corrupt(at + "csr record header declares " + std::to_string(hdr_rows) + " rows, chunk has " +
                std::to_string(rows));
    const uint64_t is = index_size(*m.index_dtype), vs = value_size(m.value_dtype);
    const uint64_t expected = kCsrHeaderBytes + (rows + 1) * is + nnz * (is + vs);
    if (len != expected)
        corrupt(at + "csr record length " + std::to_string(len) + ", expected " + std::to_string(expected));
    // CsrBlock::validate (block.cpp:110-133), in its order
    const std::string inv = at + "csr record invalid: csr block: ";
    const uint8_t* ip = rec + kCsrHeaderBytes;
    const uint8_t* idx = ip + (rows + 1) * is;
    if (rd_index(m, ip) != 0) corrupt(inv + "indptr[0] != 0");
    for (uint64_t r = 0; r < rows; ++r) {
        const uint64_t lo = rd_index(m, ip + r * is), hi = rd_index(m, ip + (r + 1) * is);
        if (hi < lo) corrupt(inv + "indptr decreasing at row " + std::to_string(r));
        for (uint64_t k = lo; k < hi && k < nnz; ++k) {
            const uint64_t c = rd_index(m, idx + k * is);
            if (c >= m.n_var)
                corrupt(inv + "column index " + std::to_string(c) + " >= n_var " + std::to_string(m.n_var) +
                        " in row " + std::to_string(r));
            if (k > lo && c <= rd_index(m, idx + (k - 1) * is))
                corrupt(inv + "column indices not strictly increasing in row " + std::to_string(r));
        }
        if (hi > nnz) corrupt(inv + "indices length does not match indptr");
    }
    if (rd_index(m, ip + rows * is) != nnz) corrupt(inv + "indices length does not match indptr");
}

void check_dense_record(const Manifest& m, uint64_t q, uint64_t len) {  // codec_decode none (codec.cpp:40-44)
    const uint64_t expected = m.rows_in_chunk(q) * m.n_var * value_size(m.value_dtype);
    if (len != expected)
        corrupt(chunk_where(m, q) + "chunk record: expected " + std::to_string(expected) + " bytes, found " +
                std::to_string(len));
}

bool check_csr_record(const Manifest& m, uint64_t q, const uint8_t* rec, uint64_t len, uint32_t* row_nnz) {
    if (len < kCsrHeaderBytes) return false;
    const uint64_t rows = m.rows_in_chunk(q);
    const uint64_t nnz = rd64(rec + 4);
    const uint64_t is = index_size(*m.index_dtype), vs = value_size(m.value_dtype);
    if (rd32(rec) != rows || len != kCsrHeaderBytes + (rows + 1) * is + nnz * (is + vs)) return false;
    const uint8_t* ip = rec + kCsrHeaderBytes;
    uint64_t prev = rd_index(m, ip);
    if (prev != 0) return false;
    for (uint64_t r = 1; r <= rows; ++r) {
        const uint64_t v = rd_index(m, ip + r * is);
        if (v < prev) return false;
        if (row_nnz) row_nnz[r - 1] = static_cast<uint32_t>(v - prev);
        prev = v;
    }
    return prev == nnz;
}

uint64_t csr_record_bytes(const Manifest& m, uint64_t rows, uint64_t nnz) {
    const uint64_t is = index_size(*m.index_dtype), vs = value_size(m.value_dtype);
    return kCsrHeaderBytes + (rows + 1) * is + nnz * (is + vs);
}

std::vector<uint8_t> decode_record_checked(const Manifest& m, uint64_t q, const uint8_t* enc, uint64_t n) {
    std::vector<uint8_t> raw;
    if (m.codec == Codec::none) {
        raw.assign(enc, enc + n);
    } else {
        try {
            if (m.layout == Layout::dense) {  // codec_decode to the known size (store.cpp:84-87)
                raw.resize(m.rows_in_chunk(q) * m.n_var * value_size(m.value_dtype));
                inflate_exact(enc, n, raw.data(), raw.size());
            } else {  // codec_decode_any with the reference's size hint (store.cpp:92-93)
                raw = inflate_any(enc, n, n * 3 + kCsrHeaderBytes);
            }
        } catch (const Error& e) {
            if (e.code == kCorrupt) corrupt(chunk_where(m, q) + e.what());
            throw;
        }
    }
    if (m.layout == Layout::dense) check_dense_record(m, q, raw.size());
    else full_check_csr_record(m, q, raw.data(), raw.size());
    return raw;
}

// ================================================================= DStore ===
DStore::DStore(std::shared_ptr<HostStore> hs, int device, uint32_t staging)
    : hs_(std::move(hs)), device_(device), staging_(staging) {
    const Manifest& m = hs_->manifest();
    if (staging > kResidentCoded) invalid("unknown staging mode");
    const uint64_t nch = m.chunk_count();
    rec_off_.resize(nch);
    slot_len_.resize(nch);
    slot_off_.resize(nch);
    for (uint64_t q = 0; q < nch; ++q) {
        const Slot sl = hs_->record_slot(q);
        slot_off_[q] = sl.off;
        slot_len_[q] = sl.len;
    }
    if (m.layout == Layout::csr) row_nnz_.resize(m.n_obs);
    // the image holds DECODED records: deflate stores are inflated on the host
    // (open / read-ahead threads), so every kernel reads plain records
    if (m.codec == Codec::deflate) deflate_layout();
    else rec_len_ = slot_len_;
    uint64_t off = 0;
    for (uint64_t q = 0; q < nch; ++q) {
        rec_off_[q] = off;
        off = align_up(off + rec_len_[q], kAlign);
    }
    image_bytes_ = off;
    DeviceGuard g(device_);
    try {
        open_image();
        if (d8_ && (m.value_dtype == VDtype::f32 || m.value_dtype == VDtype::i32)) {
            d8_fused_ = true;
            for (uint8_t k : d8_rec_)
                d8_fused_ = d8_fused_ && ((k & ~kD8Packed) == kD8Raw || (k & ~kD8Packed) == kD8Coded ||
                                          (k & ~kD8Packed) == kD8Coded16 || (k & ~kD8Packed) == kD8Int8 ||
                                          (k & ~kD8Packed) == kD8IntP);
            for (uint32_t n : row_nnz_) d8_fused_ = d8_fused_ && n <= kD8FusedMaxNnz;
        }
    } catch (...) {  // the destructor does not run for a throwing constructor
        if (d_arena_) cudaFree(d_arena_);
        d_arena_ = nullptr;
        free_host_image();
        throw;
    }
}

bool DStore::pull_ok() const {
    if (pull_ok_ < 0) {
        bool ok = h_image_ != nullptr;
        const uint64_t bytes = h_map_bytes_ ? h_map_bytes_ : image_bytes_ + kPad;
        for (uint64_t o = 0; ok && o < bytes; o += kPinPiece) {
            void* dp = nullptr;
            ok = cudaHostGetDevicePointer(&dp, h_image_ + o, 0) == cudaSuccess && dp == h_image_ + o;
        }
        cudaGetLastError();
        pull_ok_ = ok ? 1 : 0;
    }
    return pull_ok_ == 1;
}

void DStore::free_host_image() {
    if (!h_image_) return;
    if (h_map_bytes_) {
        if (h_registered_)
            for (uint64_t o = 0; o < h_map_bytes_; o += kPinPiece) cudaHostUnregister(h_image_ + o);
        munmap(h_image_, h_map_bytes_);
    } else {
        cudaFreeHost(h_image_);
    }
    h_image_ = nullptr;
    h_map_bytes_ = 0;
    h_registered_ = false;
}

// load (resident / stream_pinned), validate and re-encode the image; per-row nnz
void DStore::open_image() {
    const Manifest& m = hs_->manifest();
    const uint64_t nch = m.chunk_count();
    img_off_ = rec_off_;
    img_len_ = rec_len_;
    // stream_pinned / resident_coded: the re-encoded staging image, built streaming
    // from the store (records checked on the host as they are encoded)
    if (staging_ == kStreamPinned || staging_ == kResidentCoded) {
        const uint32_t mode = stage_mode();
        if (mode != kStageVerbatim && build_staged_image(mode)) {
            if (staging_ == kResidentCoded) {  // the image goes to HBM; the host copy is dropped
                cuda_ok(cudaMalloc(&d_arena_, staged_bytes_ + kPad), "cudaMalloc staging image");
                for (uint64_t o = 0; o < staged_bytes_ + kPad; o += kUploadRun)
                    cuda_ok(cudaMemcpy(d_arena_ + o, h_image_ + o, std::min(kUploadRun, staged_bytes_ + kPad - o),
                                       cudaMemcpyHostToDevice),
                            "upload staging image");
                free_host_image();
            }
            return;
        }
        if (staging_ == kResidentCoded) invalid("resident_coded staging needs a re-encodable store (csr u32 ids "
                                                "with n_var <= 65536, or one-hot dense u8 rows)");
    }
    if (m.codec == Codec::deflate) {
        if (staging_ != kStreamFile) load_records_deflate(staging_ == kResident);
    } else if (staging_ == kResident) {
        load_records(true);
    } else if (staging_ == kStreamPinned) {
        load_records(false);
    }
    // CsrBlock::validate of every record, once, on the GPU (the reference
    // re-validates on each decode, store.cpp:116-120); the pinned image is read
    // in place over PCIe (mapped pinned memory)
    if (m.layout == Layout::csr && staging_ != kStreamFile) {
        const char* nv = std::getenv("RFL_NO_VALIDATE");
        if (!(nv && nv[0] == '1')) validate_records(staging_ == kResident ? d_arena_ : h_image_);
    }
    if (m.layout == Layout::csr && staging_ == kStreamFile && m.codec == Codec::none) {
        // file streaming: only headers + indptrs now (deflate: read by deflate_layout)
        std::vector<uint8_t> buf;
        for (uint64_t q = 0; q < nch; ++q) {
            const uint64_t want = std::min<uint64_t>(
                rec_len_[q], kCsrHeaderBytes + (m.rows_in_chunk(q) + 1) * index_size(*m.index_dtype));
            buf.resize(want);
            const Slot s = hs_->record_slot(q);
            hs_->read_shard_bytes(q / m.chunks_per_shard, s.off, buf.data(), want, false);
            if (want < kCsrHeaderBytes || !check_csr_record(m, q, buf.data(), rec_len_[q],
                                                             row_nnz_.data() + q * m.chunk_rows)) {
                buf.resize(rec_len_[q]);
                hs_->read_record(q, buf.data(), buf.size());
                full_check_csr_record(m, q, buf.data(), buf.size());
            }
        }
    }
}

void DStore::load_records(bool to_device) {
    const Manifest& m = hs_->manifest();
    const uint64_t nch = m.chunk_count();
    if (to_device) {
        cuda_ok(cudaMalloc(&d_arena_, image_bytes_ + kPad), "cudaMalloc arena");
        cuda_ok(cudaMemset(d_arena_ + image_bytes_, 0, kPad), "cudaMemset pad");
    } else {
        cuda_ok(cudaHostAlloc(reinterpret_cast<void**>(&h_image_), image_bytes_ + kPad, cudaHostAllocPortable | cudaHostAllocMapped),
                "cudaHostAlloc image");
    }
    uint64_t max_rec = 0;
    for (auto l : rec_len_) max_rec = std::max(max_rec, l);
    const uint64_t run_cap = std::max(kUploadRun, max_rec);
    uint8_t* bounce[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    cudaStream_t st = nullptr;
    if (to_device) {
        cuda_ok(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
        for (int i = 0; i < 2; ++i) {
            cuda_ok(cudaHostAlloc(reinterpret_cast<void**>(&bounce[i]), run_cap, cudaHostAllocDefault), "bounce");
            cuda_ok(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming), "event");
        }
    }
    int which = 0;
    uint64_t q = 0;
    while (q < nch) {  // a run of consecutive records of one shard, read with one pread
        const uint64_t shard = q / m.chunks_per_shard;
        const Slot first = hs_->record_slot(q);
        uint64_t end = q + 1, run_len = first.len;
        while (end < nch && end / m.chunks_per_shard == shard) {
            const Slot s = hs_->record_slot(end);
            if (s.off != first.off + run_len || run_len + s.len > run_cap) break;
            run_len += s.len;
            ++end;
        }
        uint8_t* buf;
        if (to_device) {
            cuda_ok(cudaEventSynchronize(ev[which]), "event sync");
            buf = bounce[which];
            hs_->read_shard_bytes(shard, first.off, buf, run_len, false);
        } else {
            buf = h_image_ + rec_off_[q];  // records land contiguously, then get spread to their slots
            if (end - q > 1) {
                buf = static_cast<uint8_t*>(std::malloc(run_len));
                if (!buf) invalid("out of host memory");
            }
            hs_->read_shard_bytes(shard, first.off, buf, run_len, false);
        }
        uint64_t rel = 0;
        for (uint64_t k = q; k < end; ++k) {
            const uint8_t* rec = buf + rel;
            if (m.layout == Layout::csr) {
                if (!check_csr_record(m, k, rec, rec_len_[k], row_nnz_.data() + k * m.chunk_rows))
                    full_check_csr_record(m, k, rec, rec_len_[k]);
            } else {
                check_dense_record(m, k, rec_len_[k]);
            }
            if (to_device)
                cuda_ok(cudaMemcpyAsync(d_arena_ + rec_off_[k], rec, rec_len_[k], cudaMemcpyHostToDevice, st),
                        "upload");
            else if (end - q > 1)
                std::memcpy(h_image_ + rec_off_[k], rec, rec_len_[k]);
            rel += rec_len_[k];
        }
        if (to_device) {
            cuda_ok(cudaEventRecord(ev[which], st), "event record");
            which ^= 1;
        } else if (end - q > 1) {
            std::free(buf);
        }
        q = end;
    }
    if (to_device) {
        cuda_ok(cudaStreamSynchronize(st), "upload sync");
        for (int i = 0; i < 2; ++i) {
            cudaFreeHost(bounce[i]);
            cudaEventDestroy(ev[i]);
        }
        cudaStreamDestroy(st);
    }
}

namespace {
template <class F>
void parallel_chunks(uint64_t n, F&& fn) {  // fn(q) over [0, n) on up to 16 threads, first error rethrown
    const unsigned T = static_cast<unsigned>(
        std::max<uint64_t>(1, std::min<uint64_t>({16u, std::max(1u, std::thread::hardware_concurrency()), n})));
    std::vector<std::exception_ptr> errs(T);
    std::atomic<uint64_t> next{0};
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < T; ++t)
        pool.emplace_back([&, t] {
            try {
                for (uint64_t q; (q = next.fetch_add(1)) < n;) fn(q);
            } catch (...) {
                errs[t] = std::current_exception();
                next = n;
            }
        });
    for (auto& th : pool) th.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
}
}  // namespace

// Codec::deflate: decoded record lengths (dense: rows x row bytes; CSR: from
// the header, by inflating only the record's head) and, for CSR, per-row nnz
// from the inflated indptr -- the same header / indptr checks as
// check_csr_record; a record failing them is decoded the reference's way for
// the exact error.
void deflate_record_lengths(const HostStore& hs, std::vector<uint64_t>& rec_len, uint32_t* row_nnz) {
    const Manifest& m = hs.manifest();
    const uint64_t nch = m.chunk_count();
    rec_len.assign(nch, 0);
    if (m.layout == Layout::dense) {
        for (uint64_t q = 0; q < nch; ++q) rec_len[q] = m.rows_in_chunk(q) * m.n_var * value_size(m.value_dtype);
        return;
    }
    const uint64_t is = index_size(*m.index_dtype);
    parallel_chunks(nch, [&](uint64_t q) {
        const Slot sl = hs.record_slot(q);
        const uint64_t rows = m.rows_in_chunk(q);
        const uint64_t want = kCsrHeaderBytes + (rows + 1) * is;
        std::vector<uint8_t> enc, head(want);
        uint64_t got = 0;
        for (uint64_t take = std::min<uint64_t>(sl.len, 16384);; take = sl.len) {  // head first, whole record if short
            enc.resize(take);
            hs.read_shard_bytes(q / m.chunks_per_shard, sl.off, enc.data(), take, false);
            got = inflate_prefix(enc.data(), take, head.data(), want);
            if (got == want || take == sl.len) break;
        }
        bool ok = got == want && rd32(head.data()) == rows;
        if (ok) {
            const uint64_t nnz = rd64(head.data() + 4);
            rec_len[q] = csr_record_bytes(m, rows, nnz);
            // check_csr_record's indptr pass on the inflated head (the length is right by construction)
            uint64_t prev = is == 4 ? rd32(head.data() + kCsrHeaderBytes) : rd64(head.data() + kCsrHeaderBytes);
            ok = prev == 0;
            for (uint64_t r = 1; ok && r <= rows; ++r) {
                const uint8_t* p = head.data() + kCsrHeaderBytes + r * is;
                const uint64_t v = is == 4 ? rd32(p) : rd64(p);
                ok = v >= prev;
                if (row_nnz) row_nnz[q * m.chunk_rows + r - 1] = static_cast<uint32_t>(v - prev);
                prev = v;
            }
            ok = ok && prev == nnz;
        }
        if (!ok) {  // the reference's decode for its message (throws); anything it accepts is still corrupt here
            if (enc.size() != sl.len) {
                enc.resize(sl.len);
                hs.read_shard_bytes(q / m.chunks_per_shard, sl.off, enc.data(), sl.len, false);
            }
            decode_record_checked(m, q, enc.data(), enc.size());
            corrupt(chunk_where(m, q) + "csr record invalid");
        }
    });
}

void DStore::deflate_layout() { deflate_record_lengths(*hs_, rec_len_, row_nnz_.empty() ? nullptr : row_nnz_.data()); }

// Codec::deflate, resident / stream_pinned: every record inflated (in parallel)
// straight into a pinned image at its aligned offset; resident then uploads the
// image to HBM and drops it.
void DStore::load_records_deflate(bool to_device) {
    const Manifest& m = hs_->manifest();
    const uint64_t nch = m.chunk_count();
    cuda_ok(cudaHostAlloc(reinterpret_cast<void**>(&h_image_), image_bytes_ + kPad, cudaHostAllocPortable | cudaHostAllocMapped),
            "cudaHostAlloc image");
    std::memset(h_image_ + image_bytes_, 0, kPad);
    parallel_chunks(nch, [&](uint64_t q) {
        const Slot sl = hs_->record_slot(q);
        std::vector<uint8_t> enc(sl.len);
        hs_->read_shard_bytes(q / m.chunks_per_shard, sl.off, enc.data(), sl.len, false);
        if (!inflate_fits(enc.data(), enc.size(), h_image_ + rec_off_[q], rec_len_[q])) {
            decode_record_checked(m, q, enc.data(), enc.size());  // throws the reference's error
            corrupt(chunk_where(m, q) + "csr record invalid");
        }
    });
    if (!to_device) return;
    cuda_ok(cudaMalloc(&d_arena_, image_bytes_ + kPad), "cudaMalloc arena");
    cuda_ok(cudaMemcpy(d_arena_, h_image_, image_bytes_ + kPad, cudaMemcpyHostToDevice), "upload");
    cudaFreeHost(h_image_);
    h_image_ = nullptr;
}

void DStore::validate_records(const uint8_t* base) {
    const Manifest& m = hs_->manifest();
    const uint64_t nch = m.chunk_count();
    if (nch == 0) return;
    std::vector<uint64_t> first(nch);
    for (uint64_t q = 0; q < nch; ++q) first[q] = q * m.chunk_rows;
    uint64_t* d_tab = nullptr;
    unsigned long long* d_bad = nullptr;
    cuda_ok(cudaMalloc(&d_tab, 2 * nch * sizeof(uint64_t)), "cudaMalloc");
    cuda_ok(cudaMalloc(&d_bad, sizeof(unsigned long long)), "cudaMalloc");
    cuda_ok(cudaMemcpy(d_tab, rec_off_.data(), nch * 8, cudaMemcpyHostToDevice), "H2D");
    cuda_ok(cudaMemcpy(d_tab + nch, first.data(), nch * 8, cudaMemcpyHostToDevice), "H2D");
    cuda_ok(cudaMemset(d_bad, 0xff, sizeof(unsigned long long)), "memset");
    launch_validate_csr(base, d_tab, d_tab + nch, nch, m.n_var, *m.index_dtype, d_bad, nullptr);
    unsigned long long bad = 0;
    cuda_ok(cudaMemcpy(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost), "D2H");
    cudaFree(d_tab);
    cudaFree(d_bad);
    if (bad == ~0ull) return;
    // reproduce the reference's message (first error of the record, in validate's order)
    const uint64_t q = bad / m.chunk_rows;
    std::vector<uint8_t> rec(slot_len_[q]);
    hs_->read_record(q, rec.data(), rec.size());
    decode_record_checked(m, q, rec.data(), rec.size());
    corrupt(chunk_where(m, q) + "csr record invalid");
}

DStore::~DStore() {
    DeviceGuard g(device_);
    for (auto& b : out_pool_) b.free_all();
    for (auto& pb : pinned_pool_) cudaFreeHost(pb.first);
    for (cudaEvent_t e : ev_all_) cudaEventDestroy(e);
    for (void* p : slabs_) cudaFree(p);
    if (d_arena_) cudaFree(d_arena_);
    free_host_image();
}

uint64_t DStore::max_block_bytes(uint64_t f, bool expanded) const {
    const Manifest& m = manifest();
    uint64_t best = 0;
    for (uint64_t s = 0; s < m.n_obs; s += f) {
        const uint64_t e = std::min(m.n_obs, s + f);
        uint64_t bytes = 0;
        for (uint64_t q = s / m.chunk_rows; q <= (e - 1) / m.chunk_rows; ++q) {
            bytes = align_up(bytes + img_len_[q], kAlign);
            if (d8_ && expanded) bytes = align_up(bytes + exp_len_[q], kAlign);  // expanded records + staged deltas
        }
        best = std::max(best, bytes);
    }
    return best;
}

ArenaView DStore::view(const uint8_t* base) const {
    const Manifest& m = manifest();
    ArenaView a;
    a.base = base;
    a.chunk_rows = m.chunk_rows;
    a.n_var = m.n_var;
    a.layout = m.layout;
    a.vdt = m.value_dtype;
    a.idt = m.index_dtype.value_or(IDtype::u32);
    a.idx16 = idx16_ && (staging_ == kStreamPinned || staging_ == kResidentCoded);
    return a;
}

void DStore::reserve_slots(uint64_t bytes, uint64_t n) {
    const uint64_t key = align_up(std::max<uint64_t>(bytes, 1), 256);
    std::lock_guard<std::mutex> lk(mu_);
    std::deque<SlotRef>& pool = free_[key];
    while (pool.size() < n) grow_slab(key);
}

void DStore::grow_slab(uint64_t slot_bytes) {
    const uint64_t n = 32;
    void* slab = nullptr;
    cuda_ok(cudaMalloc(&slab, n * slot_bytes + kPad), "cudaMalloc slab");
    slabs_.push_back(slab);
    std::deque<SlotRef>& pool = free_[slot_bytes];
    for (uint64_t i = 0; i < n; ++i) {
        SlotRef s;
        s.ptr = static_cast<uint8_t*>(slab) + i * slot_bytes;
        s.bytes = slot_bytes;
        pool.push_back(s);
    }
}

DStore::SlotRef DStore::acquire_slot(uint64_t bytes) {
    // one FIFO pool per slot size: iterators with different fetch_block_rows over one
    // store each recycle their own geometry's slabs (nothing is orphaned)
    const uint64_t key = align_up(std::max<uint64_t>(bytes, 1), 256);
    std::lock_guard<std::mutex> lk(mu_);
    std::deque<SlotRef>& pool = free_[key];
    if (pool.empty()) grow_slab(key);
    // oldest first: a LIFO pop would hand the next batch's copy the slot the
    // previous batch's kernel just released, serialising copy(i+1) behind kernel(i)
    SlotRef s = pool.front();
    pool.pop_front();
    return s;
}

void OutBuffers::free_all() {
    cudaFree(gidx);
    cudaFree(indptr);
    cudaFree(indices);
    cudaFree(data);
    cudaFree(scratch);
    cudaFree(d_refs);
    cudaFreeHost(h_refs);
    cudaFreeHost(h_gidx);
    cudaFreeHost(h_prefix);
    if (done) cudaEventDestroy(done);
    for (auto& e : tk)
        if (e) cudaEventDestroy(e);
    *this = OutBuffers{};
}

uint8_t* DStore::take_pinned(uint64_t bytes) {
    {
        std::lock_guard<std::mutex> lk(mu_);
        for (size_t i = 0; i < pinned_pool_.size(); ++i)
            if (pinned_pool_[i].second == bytes) {
                uint8_t* p = pinned_pool_[i].first;
                pinned_pool_.erase(pinned_pool_.begin() + static_cast<std::ptrdiff_t>(i));
                return p;
            }
    }
    uint8_t* p = nullptr;
    cuda_ok(cudaHostAlloc(reinterpret_cast<void**>(&p), bytes, cudaHostAllocDefault), "pinned");
    return p;
}

void DStore::give_pinned(uint8_t* p, uint64_t bytes) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(mu_);
    if (pinned_pool_.size() < 64) pinned_pool_.emplace_back(p, bytes);
    else cudaFreeHost(p);
}

OutBuffers DStore::take_out(uint32_t key) {
    std::lock_guard<std::mutex> lk(mu_);
    for (size_t i = 0; i < out_pool_.size(); ++i)
        if (out_pool_[i].key == key) {
            OutBuffers b = out_pool_[i];
            out_pool_.erase(out_pool_.begin() + static_cast<std::ptrdiff_t>(i));
            b.used = false;
            return b;
        }
    OutBuffers b;
    b.key = key;
    return b;
}

void DStore::give_out(OutBuffers&& b) {
    std::lock_guard<std::mutex> lk(mu_);
    if (out_pool_.size() < 16) {
        b.used = false;
        out_pool_.push_back(b);
    } else {
        b.free_all();
    }
    b = OutBuffers{};
}

void DStore::release_slot(const SlotRef& s) {
    std::lock_guard<std::mutex> lk(mu_);
    free_[s.bytes].push_back(s);
}

std::vector<cudaEvent_t> DStore::take_events(size_t n) {
    std::lock_guard<std::mutex> lk(mu_);
    std::vector<cudaEvent_t> out;
    while (out.size() < n && !ev_free_.empty()) {
        out.push_back(ev_free_.back());
        ev_free_.pop_back();
    }
    while (out.size() < n) {
        cudaEvent_t e = nullptr;
        cuda_ok(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        ev_all_.push_back(e);
        out.push_back(e);
    }
    return out;
}

// (the giving loader has drained its stream: every record of these events is complete,
// so slots still pointing at them wait on nothing, or on a later point of a later user)
void DStore::give_events(std::vector<cudaEvent_t>&& ev) {
    std::lock_guard<std::mutex> lk(mu_);
    ev_free_.insert(ev_free_.end(), ev.begin(), ev.end());
    ev.clear();
}

// ============================================================ BlockReader ===
// CsrBlock::validate's column checks (block.cpp:110-133) on a record whose header
// and indptr were already checked: every id < n_var, strictly increasing per row
bool columns_ok(const Manifest& m, uint64_t q, const uint8_t* rec) {
    const uint64_t rows = rd32(rec);
    const uint8_t* ip = rec + kCsrHeaderBytes;
    if (m.index_dtype == IDtype::u32) {
        const uint8_t* ix = ip + 4 * (rows + 1);
        const uint32_t nv = m.n_var > 0xFFFFFFFFull ? 0xFFFFFFFFu : static_cast<uint32_t>(m.n_var);
        for (uint64_t r = 0; r < rows; ++r) {
            const uint64_t lo = rd32(ip + 4 * r), hi = rd32(ip + 4 * (r + 1));
            if (lo == hi) continue;
            // branch-free, vectorisable: any id >= n_var, any id <= its predecessor
            uint32_t bad = rd32(ix + 4 * lo) >= nv;
            for (uint64_t k = lo + 1; k < hi; ++k) {
                const uint32_t c = rd32(ix + 4 * k), p = rd32(ix + 4 * (k - 1));
                bad |= static_cast<uint32_t>(c >= nv) | static_cast<uint32_t>(c <= p);
            }
            if (bad) return false;
        }
        return true;
    }
    (void)q;
    return false;  // u64 ids: the full check (rare layout)
}

BlockReader::BlockReader(std::shared_ptr<DStore> ds, std::vector<uint64_t> order, uint64_t f, uint32_t threads,
                         uint32_t slots, bool direct)
    : ds_(std::move(ds)), order_(std::move(order)), f_(f), direct_(direct) {
    const char* nv = std::getenv("RFL_NO_VALIDATE");
    validate_ = ds_->manifest().layout == Layout::csr && !(nv && nv[0] == '1');
    const Manifest& m = ds_->manifest();
    // a block's records, each run read as its 4 KiB-aligned superset into a page-aligned position
    const uint64_t bytes = ds_->max_block_bytes(f) + (f / m.chunk_rows + 2) * 3 * 4096;
    buf_bytes_ = bytes;
    slots_.resize(slots);
    ev_.resize(slots);
    released_.assign(slots, ~0ull);
    DeviceGuard g(ds_->device());
    for (uint32_t i = 0; i < slots; ++i) {
        slots_[i].buf = ds_->take_pinned(bytes);
        cuda_ok(cudaEventCreateWithFlags(&ev_[i], cudaEventDisableTiming), "event");
    }
    for (uint32_t t = 0; t < threads; ++t) th_.emplace_back([this] { worker(); });
}

BlockReader::~BlockReader() {
    {
        std::lock_guard<std::mutex> lk(mu_);
        stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
    for (size_t i = 0; i < slots_.size(); ++i) {
        cudaEventSynchronize(ev_[i]);
        cudaEventDestroy(ev_[i]);
        ds_->give_pinned(slots_[i].buf, buf_bytes_);
    }
}

void BlockReader::worker() {
    cudaSetDevice(ds_->device());
    const Manifest& m = ds_->manifest();
    const HostStore& hs = ds_->host();
    const uint64_t S = slots_.size();
    uint8_t* scratch = nullptr;  // deflate stores: the encoded run (4 KiB aligned for O_DIRECT)
    uint64_t scratch_cap = 0;
    struct Free {
        uint8_t*& p;
        ~Free() { std::free(p); }
    } free_scratch{scratch};
    for (;;) {
        uint64_t k = 0;
        {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] {
                return stop_ || (next_read_ < order_.size() &&
                                 (next_read_ < S || released_[next_read_ % S] == next_read_ - S));
            });
            if (stop_) return;
            k = next_read_++;
        }
        Block& b = slots_[k % S];
        std::exception_ptr err;
        try {
            if (k >= S) cuda_ok(cudaEventSynchronize(ev_[k % S]), "pinned reuse");  // H2D of block k-S done
            const uint64_t id = order_[k];
            const uint64_t s = id * f_, e = std::min(m.n_obs, s + f_);
            const uint64_t q0 = s / m.chunk_rows, q1 = (e - 1) / m.chunk_rows;
            b.pos.assign(q1 - q0 + 1, 0);
            uint64_t cursor = 0, q = q0;
            while (q <= q1) {  // coalesced runs of adjacent records of one shard (store.cpp:427-447)
                const uint64_t shard = q / m.chunks_per_shard;
                const Slot first = hs.record_slot(q);
                uint64_t end = q + 1, run = first.len;
                while (end <= q1 && end / m.chunks_per_shard == shard) {
                    const Slot sl = hs.record_slot(end);
                    if (sl.off != first.off + run) break;
                    run += sl.len;
                    ++end;
                }
                if (ds_->deflate()) {  // inflate the run's records into the pinned buffer (codec.cpp:38-107)
                    const uint64_t span = HostStore::aligned_span(first.off, run);
                    if (scratch_cap < span) {
                        std::free(scratch);
                        scratch = nullptr;
                        if (posix_memalign(reinterpret_cast<void**>(&scratch), 4096, span) != 0) {
                            scratch = nullptr;
                            scratch_cap = 0;
                            throw Error(kIo, "out of host memory");
                        }
                        scratch_cap = span;
                    }
                    const uint64_t lead = hs.read_shard_span(shard, first.off, scratch, run, direct_);
                    for (uint64_t x = q, rel = 0; x < end; ++x) {
                        uint8_t* dst = b.buf + cursor;
                        const uint8_t* enc = scratch + lead + rel;
                        if (!inflate_fits(enc, ds_->slot_len()[x], dst, ds_->rec_len()[x])) {
                            decode_record_checked(m, x, enc, ds_->slot_len()[x]);
                            corrupt("chunk " + std::to_string(x) + " in shard " + std::to_string(shard) +
                                    ": csr record invalid");
                        }
                        b.pos[x - q0] = cursor;
                        if (validate_ && !columns_ok(m, x, dst)) full_check_csr_record(m, x, dst, ds_->rec_len()[x]);
                        cursor = align_up(cursor + ds_->rec_len()[x], 16);
                        rel += ds_->slot_len()[x];
                    }
                    q = end;
                    continue;
                }
                const uint64_t lead = hs.read_shard_span(shard, first.off, b.buf + cursor, run, direct_);
                for (uint64_t x = q, rel = 0; x < end; ++x) {
                    b.pos[x - q0] = cursor + lead + rel;
                    // decode_record validates every fetched record (store.cpp:116-120); headers and
                    // indptrs were checked at open, the columns are checked here, per fetch
                    if (validate_ && !columns_ok(m, x, b.buf + b.pos[x - q0]))
                        full_check_csr_record(m, x, b.buf + b.pos[x - q0], ds_->rec_len()[x]);
                    rel += ds_->rec_len()[x];
                }
                cursor += (HostStore::aligned_span(first.off, run) + 4095) & ~4095ull;
                q = end;
            }
        } catch (...) {
            err = std::current_exception();
        }
        {
            std::lock_guard<std::mutex> lk(mu_);
            b.err = err;
            b.seq = k;
        }
        cv_.notify_all();
    }
}

const BlockReader::Block& BlockReader::wait(uint64_t seq) {
    if (seq >= order_.size()) invalid("block reader: read past the fetch order");
    Block& b = slots_[seq % slots_.size()];
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return b.seq == seq; });
    if (b.err) {  // BlockPrefetcher rethrows naming the block (loader.cpp:70-73)
        try {
            std::rethrow_exception(b.err);
        } catch (const std::exception& e) {
            const uint64_t s = order_[seq] * f_;
            throw Error(kIo, "fetch block [" + std::to_string(s) + ", " +
                                 std::to_string(std::min(ds_->manifest().n_obs, s + f_)) + "): " + e.what());
        }
    }
    return b;
}

void BlockReader::release(uint64_t seq, cudaStream_t st) {
    const uint64_t slot = seq % slots_.size();
    cuda_ok(cudaEventRecord(ev_[slot], st), "event");
    {
        std::lock_guard<std::mutex> lk(mu_);
        released_[slot] = seq;
    }
    cv_.notify_all();
}

// ============================================================== GpuLoader ===
GpuLoader::GpuLoader(std::shared_ptr<DStore> ds, const LoaderCfg& cfg, uint64_t epoch, const DeviceCfg& dev)
    : ds_(std::move(ds)), cfg_(cfg), epoch_(epoch), dev_(dev), replay_(ds_->manifest().n_obs, cfg, epoch) {
    static std::atomic<uint64_t> next_id{1};
    id_ = next_id++;
    const Manifest& m = ds_->manifest();
    if (m.layout == Layout::dense && dev_.output == 0) invalid("csr output requested from a dense store");
    if (dev_.normalize && (m.layout != Layout::csr || dev_.output != 1))
        invalid("normalize_log1p applies to csr -> dense output");
    if (dev_.out_slots == 0) dev_.out_slots = 2;
    DeviceGuard g(ds_->device());
    if (dev_.stream) {
        compute_ = dev_.stream;
    } else {
        cuda_ok(cudaStreamCreateWithFlags(&compute_, cudaStreamNonBlocking), "stream");
        own_compute_ = true;
    }
    cuda_ok(cudaStreamCreateWithFlags(&copy_, cudaStreamNonBlocking), "stream");
    cuda_ok(cudaEventCreateWithFlags(&staged_, cudaEventDisableTiming), "event");
    const uint32_t key = dev_.output | (static_cast<uint32_t>(dev_.out_dtype) << 4) | (dev_.normalize ? 1u << 8 : 0u);
    slots_.resize(dev_.out_slots);
    for (auto& s : slots_) {
        s = ds_->take_out(key);
        if (!s.done) cuda_ok(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming), "event");
        if (dev_.time_kernels)
            for (auto& e : s.tk)
                if (!e) cuda_ok(cudaEventCreate(&e), "event");
        s.timed = false;
    }
    {
        const char* e = std::getenv("RFL_FUSED");  // RFL_FUSED=0: k_d8_decode + idx16 densify (A/B)
        const bool coded = ds_->staging() == kStreamPinned || ds_->staging() == kResidentCoded;
        // CSR -> dense from delta records (K3d), or dense rows from one-hot records (K4o)
        fused_ = !(e && e[0] == '0') && coded &&
                 ((dev_.output == 1 && m.layout == Layout::csr && ds_->d8_fused()) ||
                  (m.layout == Layout::dense && ds_->d8()));
    }
    direct_ = ds_->staging() == kResident || (ds_->staging() == kResidentCoded && fused_);
    if (!direct_) {
        live_.resize((m.n_obs + cfg_.f - 1) / cfg_.f);
        blk_addr_.assign(live_.size(), 0);
        blk_live_.assign(live_.size(), 0);
        block_bytes_ = ds_->max_block_bytes(cfg_.f, !fused_);
        // live blocks peak at ~5x B/f (cfg1 318 for B/f = 64, cfg4 230 for 32).
        // On top, (out_slots + 2) batches' worth of free slots: the host runs out_slots
        // batches ahead, and the FIFO pool must hand batch j a slot whose releasing
        // kernel already ran, or copy(j) queues behind kernel(j-1) and the copy
        // engine idles for every kernel (profiles/r1_pcie.md)
        const uint64_t nb = (m.n_obs + cfg_.f - 1) / cfg_.f;
        const uint64_t per_batch = (cfg_.b + cfg_.f - 1) / cfg_.f + 1;
        const uint64_t want = std::min<uint64_t>(
            nb, 6 * ((cfg_.B + cfg_.f - 1) / cfg_.f) + 32 + (dev_.out_slots + 2) * per_batch * std::max<uint32_t>(1, dev_.group));
        ds_->reserve_slots(block_bytes_, std::min<uint64_t>(want, (8ull << 30) / std::max<uint64_t>(block_bytes_, 1)));
        if (ds_->staging() == kStreamFile) {
            const uint32_t threads = std::min<uint32_t>(16, std::max<uint32_t>(1, cfg_.prefetch_depth));
            reader_ = std::make_unique<BlockReader>(ds_, replay_.plan(), cfg_.f, threads, 2 * threads + 2,
                                                    cfg_.cache_bypass);
        }
    }
    footer_seen_.assign(m.shard_count(), 0);
    if (!direct_) rel_ring_ = ds_->take_events(kReleaseRing);
    div_chunk_ = FastDiv(m.chunk_rows);
    div_f_ = FastDiv(cfg_.f);
    // every output slot sized for a full group up front (first-use cudaMalloc /
    // cudaHostAlloc would stall the first groups' steps)
    for (auto& s : slots_) ensure_capacity(s, static_cast<uint64_t>(std::max<uint32_t>(1, dev_.group)) * cfg_.b, 0);
    rq_cap_ = std::max<size_t>(8, 2 * static_cast<size_t>(std::max<uint32_t>(1, dev_.group)) + 2);
    replay_th_ = std::thread([this] { replay_worker(); });
}

GpuLoader::~GpuLoader() {
    {
        std::lock_guard<std::mutex> lk(rq_mu_);
        rq_stop_ = true;
    }
    rq_cv_.notify_all();
    if (replay_th_.joinable()) replay_th_.join();
    DeviceGuard g(ds_->device());
    if (compute_) cudaStreamSynchronize(compute_);
    if (copy_) cudaStreamSynchronize(copy_);
    cudaEvent_t last = rel_ring_.empty() ? nullptr : rel_ring_[rel_pos_ % rel_ring_.size()];
    if (last) cudaEventRecord(last, compute_);
    for (auto& l : live_)
        if (l.slot.ptr) {
            l.slot.released = last;
            ds_->release_slot(l.slot);
        }
    if (!rel_ring_.empty()) ds_->give_events(std::move(rel_ring_));
    for (auto& s : slots_) ds_->give_out(std::move(s));  // the compute stream is drained: reusable as is
    reader_.reset();
    cudaEventDestroy(staged_);
    cudaStreamDestroy(copy_);
    if (own_compute_) cudaStreamDestroy(compute_);
}

void GpuLoader::stage_block(uint64_t id) {
    const Manifest& m = ds_->manifest();
    const uint64_t s = id * cfg_.f, e = std::min(m.n_obs, s + cfg_.f);
    const uint64_t q0 = s / m.chunk_rows, q1 = (e - 1) / m.chunk_rows;
    Live& lv = live_[id];
    lv.first_chunk = q0;
    lv.chunk_off.clear();
    const bool coded = ds_->staging() == kResidentCoded;  // staging image in HBM: decode device-to-device
    const bool d8 = (ds_->staging() == kStreamPinned || coded) && ds_->d8() && !fused_;  // fused: no expansion
    uint64_t bytes = 0;
    for (uint64_t q = q0; q <= q1; ++q) {
        lv.chunk_off.push_back(bytes);
        bytes = align_up(bytes + (d8 ? ds_->exp_len()[q] : ds_->img_len()[q]), kAlign);
    }
    lv.slot = ds_->acquire_slot(block_bytes_);
    lv.live_rows = e - s;
    // the slot's previous kernel readers are done (skip the stream wait if already complete)
    if (ds_->staging() == kStreamPinned && lv.slot.owner == id_ && lv.slot.released) {
        if (!pend_ev_ || lv.slot.seq >= pend_seq_) {  // coalesced into one wait in next()
            pend_ev_ = lv.slot.released;
            pend_seq_ = lv.slot.seq;
        }
    } else if (!lv.slot.released) {
        // never used: nothing to wait for
    } else if (coded) {  // the decode writes the slot on compute_, where this loader's releases were recorded
        if (lv.slot.owner != id_ && cudaEventQuery(lv.slot.released) != cudaSuccess)
            cuda_ok(cudaStreamWaitEvent(compute_, lv.slot.released, 0), "wait slot");
    } else if (cudaEventQuery(lv.slot.released) != cudaSuccess) {
        cuda_ok(cudaStreamWaitEvent(copy_, lv.slot.released, 0), "wait slot");
    }
    if (coded) {
        for (uint64_t q = q0; q <= q1; ++q)
            d8_jobs_.push_back({ds_->d_arena() + ds_->img_off()[q], lv.slot.ptr + lv.chunk_off[q - q0],
                                ds_->exp_len()[q], ds_->d8_kind(q), 0});
    } else if (ds_->staging() == kStreamPinned) {
        // records of one block are contiguous in the pinned image except for alignment padding;
        // the copies of all blocks fetched for this group are issued together (assemble_group)
        const uint64_t img0 = ds_->img_off()[q0];
        const uint64_t img1 = ds_->img_off()[q1] + ds_->img_len()[q1];
        uint8_t* land = d8 ? lv.slot.ptr + bytes : lv.slot.ptr;  // delta records land after the expanded area
        for (uint64_t a = img0; a < img1;) {  // one copy per pinned piece the range touches
            const uint64_t b = std::min(img1, (a / kPinPiece + 1) * kPinPiece);
            batch_dst_.push_back(land + (a - img0));
            batch_src_.push_back(const_cast<uint8_t*>(ds_->h_image() + a));
            batch_size_.push_back(b - a);
            a = b;
        }
        if (d8) {
            for (uint64_t q = q0; q <= q1; ++q)
                d8_jobs_.push_back({land + (ds_->img_off()[q] - img0), lv.slot.ptr + lv.chunk_off[q - q0],
                                    ds_->exp_len()[q], ds_->d8_kind(q), 0});
        } else {
            for (uint64_t q = q0; q <= q1; ++q) lv.chunk_off[q - q0] = ds_->img_off()[q] - img0;
        }
        ctr_.h2d_bytes += img1 - img0;
    } else {
        // read ahead by the BlockReader; one copy per record into its aligned slot offset
        // (copied and released right away: one next() may consume more blocks than there are buffers)
        const uint64_t seq = read_seq_++;
        const BlockReader::Block& bk = reader_->wait(seq);
        for (uint64_t q = q0; q <= q1; ++q) {
            cuda_ok(cudaMemcpyAsync(lv.slot.ptr + lv.chunk_off[q - q0], bk.buf + bk.pos[q - q0], ds_->rec_len()[q],
                                    cudaMemcpyHostToDevice, copy_),
                    "stage H2D");
            ctr_.h2d_bytes += ds_->rec_len()[q];
        }
        reader_->release(seq, copy_);
    }
    lv.off0 = reinterpret_cast<uint64_t>(lv.slot.ptr) + lv.chunk_off[0];
    lv.single = q0 == q1;
    blk_addr_[id] = lv.single ? lv.off0 : 0;
    blk_live_[id] = static_cast<uint32_t>(lv.live_rows);
    count_fetch(id);
}

// IoStats of BlockPrefetcher's read_rows({block}) (store.cpp:371-470): per shard
// the footer on first use, one read op per run of adjacent records, bytes_read =
// the run length (cache_bypass: the 4 KiB-aligned superset actually read,
// store.cpp:374-392), one decode per chunk.  Whatever the staging mode, the
// counters equal the reference's for the same fetch order.
void GpuLoader::count_fetch(uint64_t id) {
    const Manifest& m = ds_->manifest();
    const HostStore& hs = ds_->host();
    const uint64_t s = id * cfg_.f, e = std::min(m.n_obs, s + cfg_.f);
    const uint64_t q0 = s / m.chunk_rows, q1 = (e - 1) / m.chunk_rows;
    uint64_t q = q0;
    const std::vector<uint64_t>& so = ds_->slot_off();
    while (q <= q1) {
        const uint64_t shard = q / m.chunks_per_shard;
        if (!footer_seen_[shard]) {  // (the store's own charge is shared by its readers)
            footer_seen_[shard] = 1;
            ctr_.bytes_read += hs.charge_footer(shard);
        }
        const uint64_t first_off = so[q];
        uint64_t end = q + 1, run = ds_->slot_len()[q];
        while (end <= q1 && end / m.chunks_per_shard == shard && so[end] == first_off + run)
            run += ds_->slot_len()[end++];
        ctr_.read_ops += 1;
        if (cfg_.cache_bypass && hs.direct_ok(shard)) {
            const uint64_t a0 = first_off & ~4095ull;
            const uint64_t span = HostStore::aligned_span(first_off, run);
            ctr_.bytes_read += std::min(span, hs.shard_bytes(shard) - a0);
        } else {
            ctr_.bytes_read += run;
        }
        ctr_.chunks_decoded += end - q;
        q = end;
    }
}

void GpuLoader::ensure_capacity(OutSlot& s, uint64_t rows, uint64_t nnz) {
    const Manifest& m = ds_->manifest();
    const ArenaView av = ds_->view(nullptr);
    if (rows > s.cap_rows) {
        cudaFree(s.gidx);
        cudaFree(s.indptr);
        cudaFree(s.scratch);
        cudaFree(s.d_refs);
        cudaFreeHost(s.h_refs);
        cudaFreeHost(s.h_gidx);
        cudaFreeHost(s.h_prefix);
        // CSR indptrs of a group: the group prefix (rows+1) + each later batch's own (<= rows + group)
        const uint64_t ip = 2 * (rows + 1) + std::max<uint32_t>(1, dev_.group);
        cuda_ok(cudaHostAlloc(reinterpret_cast<void**>(&s.h_prefix), ip * 8, cudaHostAllocDefault), "pinned");
        cuda_ok(cudaMalloc(&s.gidx, rows * 8), "malloc");
        cuda_ok(cudaMalloc(&s.indptr, ip * 8), "malloc");
        cuda_ok(cudaMalloc(&s.scratch, csr_gather_scratch_bytes(rows)), "malloc");
        cuda_ok(cudaMalloc(reinterpret_cast<void**>(&s.d_refs), rows * sizeof(RowRef)), "malloc");
        cuda_ok(cudaHostAlloc(reinterpret_cast<void**>(&s.h_refs), rows * sizeof(RowRef), cudaHostAllocDefault),
                "pinned");
        cuda_ok(cudaHostAlloc(reinterpret_cast<void**>(&s.h_gidx), rows * 8, cudaHostAllocDefault), "pinned");
        s.cap_rows = rows;
        if (dev_.output == 1) {
            cudaFree(s.data);
            s.data_bytes = rows * m.n_var * dense_out_elem_size(av, dev_.out_dtype);
            cuda_ok(cudaMalloc(&s.data, s.data_bytes + 16), "malloc");
        }
    }
    if (dev_.output == 0 && nnz > s.cap_nnz) {
        cudaFree(s.indices);
        cudaFree(s.data);
        const uint64_t cap = nnz + nnz / 8 + 1024;
        cuda_ok(cudaMalloc(&s.indices, cap * index_size(av.idt) + 16), "malloc");
        cuda_ok(cudaMalloc(&s.data, cap * value_size(av.vdt) + 16), "malloc");
        s.cap_nnz = cap;
    }
}

namespace {
// RFL_TRACE_LOADER=1: per next() host phase times on stderr (replay, staging, slot wait, launch)
struct NextTrace {
    bool on = [] {
        const char* e = std::getenv("RFL_TRACE_LOADER");
        return e && e[0] == '1';
    }();
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    double lap() {
        const auto n = std::chrono::steady_clock::now();
        const double us = std::chrono::duration<double, std::micro>(n - t).count();
        t = n;
        return us;
    }
};
}  // namespace

// ---- replay-ahead: the occupancy-driven schedule runs on its own thread, a few
// batches ahead of the consumer (the host replay is the one sequential step)
void GpuLoader::replay_worker() {
    try {
        for (;;) {
            Planned p;
            {
                std::unique_lock<std::mutex> lk(rq_mu_);
                rq_cv_.wait(lk, [&] { return rq_stop_ || rq_.size() < rq_cap_; });
                if (rq_stop_) return;
                if (!rq_free_.empty()) {
                    p = std::move(rq_free_.back());
                    rq_free_.pop_back();
                }
            }
            const bool more = replay_.next(p.gidx, p.consumed);
            p.batch_index = replay_.batch_index() - 1;
            p.blocks_fetched = replay_.blocks_fetched();
            p.peak = replay_.peak_buffer_rows();
            {
                std::lock_guard<std::mutex> lk(rq_mu_);
                if (more) rq_.push_back(std::move(p));
                else rq_end_ = true;
            }
            rq_cv_.notify_all();
            if (!more) return;
        }
    } catch (...) {
        {
            std::lock_guard<std::mutex> lk(rq_mu_);
            rq_err_ = std::current_exception();
            rq_end_ = true;
        }
        rq_cv_.notify_all();
    }
}

bool GpuLoader::pop_planned(Planned& p) {
    std::unique_lock<std::mutex> lk(rq_mu_);
    rq_cv_.wait(lk, [&] { return !rq_.empty() || rq_end_; });
    if (rq_.empty()) {
        if (rq_err_) std::rethrow_exception(rq_err_);
        return false;
    }
    p = std::move(rq_.front());
    rq_.pop_front();
    lk.unlock();
    rq_cv_.notify_all();
    return true;
}

bool GpuLoader::next(BatchOut& out) {
    if (ready_pos_ >= ready_.size()) {
        if (done_) return false;
        if (!assemble_group()) {
            done_ = true;
            return false;
        }
    }
    out = ready_[ready_pos_];
    snap_blocks_ = group_[ready_pos_].blocks_fetched;
    snap_peak_ = group_[ready_pos_].peak;
    ++ready_pos_;
    return true;
}

uint32_t GpuLoader::next_many(BatchOut* out, uint32_t max) {
    uint32_t n = 0;
    while (n < max && next(out[n])) ++n;
    return n;
}

bool GpuLoader::assemble_group() {
    DeviceGuard g(ds_->device());
    const Manifest& m = ds_->manifest();
    NextTrace tr;
    double t_replay = 0, t_stage = 0, t_slot = 0;
    {
        std::lock_guard<std::mutex> lk(rq_mu_);  // recycle the last group's vectors
        for (auto& p : group_) rq_free_.push_back(std::move(p));
    }
    group_.clear();
    ready_.clear();
    ready_pos_ = 0;
    static const bool device_scan = [] {
        const char* e = std::getenv("RFL_GATHER");
        return e && std::string(e) == "scan";
    }();
    const bool planned = m.layout == Layout::csr && dev_.output == 0 && (!device_scan || ds_->view(nullptr).idx16);
    // the device-scan CSR path writes one batch's indptr itself: one batch per launch
    const uint32_t k = m.layout == Layout::csr && dev_.output == 0 && !planned ? 1u : std::max<uint32_t>(1, dev_.group);
    while (group_.size() < k) {
        Planned p;
        if (!pop_planned(p)) break;
        group_.push_back(std::move(p));
    }
    if (group_.empty()) return false;
    if (tr.on) t_replay = tr.lap();
    const bool resident = direct_;
    if (!resident) {
        batch_dst_.clear();
        batch_src_.clear();
        batch_size_.clear();
        pend_ev_ = nullptr;
        d8_jobs_.clear();
        for (const Planned& p : group_)
            for (uint64_t id : p.consumed) stage_block(id);  // (counts each fetch)
        if (pend_ev_ && cudaEventQuery(pend_ev_) != cudaSuccess)
            cuda_ok(cudaStreamWaitEvent(copy_, pend_ev_, 0), "wait slots");
        if (!batch_dst_.empty()) {
            // the group's block copies: ONE TMA pull kernel on the copy stream (default), or
            // one copy-engine transfer per block (RFL_STAGE=ce; ~4.7 us setup each)
            static const bool ce = [] {
                const char* e = std::getenv("RFL_STAGE");
                return e && std::string(e) == "ce";
            }();
            if (ce || !ds_->pull_ok()) {
                for (size_t i = 0; i < batch_dst_.size(); ++i)
                    cuda_ok(cudaMemcpyAsync(batch_dst_[i], batch_src_[i], batch_size_[i], cudaMemcpyHostToDevice,
                                            copy_),
                            "stage H2D");
            } else {
                const uint64_t P = stage_pull_piece_bytes();
                for (size_t i0 = 0; i0 < batch_dst_.size(); i0 += kMaxPullJobs) {
                    pull_.n = static_cast<uint32_t>(std::min<size_t>(kMaxPullJobs, batch_dst_.size() - i0));
                    pull_.first_piece[0] = 0;
                    for (uint32_t k = 0; k < pull_.n; ++k) {
                        // 16-B multiples: records sit at 16-B aligned image offsets with zeroed gaps,
                        // and slots hold the aligned sizes
                        const uint64_t bytes = align_up(batch_size_[i0 + k], kAlign);
                        pull_.job[k] = {static_cast<const uint8_t*>(batch_src_[i0 + k]),
                                        static_cast<uint8_t*>(batch_dst_[i0 + k]), bytes};
                        pull_.first_piece[k + 1] = pull_.first_piece[k] + static_cast<uint32_t>((bytes + P - 1) / P);
                    }
                    launch_stage_pull(pull_, copy_);
                    ctr_.kernels_launched += 1;
                }
            }
        }
    } else {
        for (const Planned& p : group_)
            for (uint64_t id : p.consumed) count_fetch(id);
    }
    if (tr.on) t_stage = tr.lap();
    OutSlot& s = slots_[next_slot_++ % slots_.size()];
    if (s.used) {
        cuda_ok(cudaEventSynchronize(s.done), "slot reuse");  // the callers' views of it expire here
        harvest(s);
    }
    if (tr.on) t_slot = tr.lap();
    s.used = true;
    const size_t nb = group_.size();
    group_start_.assign(nb + 1, 0);
    for (size_t i = 0; i < nb; ++i) group_start_[i + 1] = group_start_[i] + group_[i].gidx.size();
    const uint64_t n = group_start_[nb];
    std::vector<uint64_t> bnnz(nb, 0);
    uint64_t nnz = 0;
    if (m.layout == Layout::csr)
        for (size_t i = 0; i < nb; ++i) {
            for (uint64_t gr : group_[i].gidx) bnnz[i] += ds_->row_nnz(gr);
            nnz += bnnz[i];
        }
    ensure_capacity(s, std::max<uint64_t>(n, static_cast<uint64_t>(k) * cfg_.b), nnz);

    // row references of every row of the group
    const uint8_t* base = resident ? ds_->d_arena() : nullptr;
    const bool kinds = fused_ && m.layout == Layout::csr;
    const uint64_t* offs = resident ? (fused_ ? ds_->img_off().data() : ds_->rec_off().data()) : nullptr;
    uint64_t* const baddr = blk_addr_.data();
    uint32_t* const blive = blk_live_.data();
    for (size_t i = 0; i < nb; ++i) {
        RowRef* hr = s.h_refs + group_start_[i];
        uint64_t* hg = s.h_gidx + group_start_[i];
        const std::vector<uint64_t>& gv = group_[i].gidx;
        const size_t ng = gv.size();
        const uint64_t* g = gv.data();
        if (resident) {
            for (size_t j = 0; j < ng; ++j) {
                const uint64_t gr = g[j], q = div_chunk_.div(gr);
                hr[j] = {offs[q], gr};
                if (kinds) hr[j].rec_off |= static_cast<uint64_t>(ds_->d8_kind(q)) << kRowKindShift;
            }
        } else {
            // streamed: base == nullptr, row refs hold device addresses
            for (size_t j = 0; j < ng; ++j) {
                const uint64_t gr = g[j], blk = div_f_.div(gr);
                uint64_t a = baddr[blk];
                if (!a || kinds) {  // a block of several records (or a kind tag): its chunk's record
                    const uint64_t q = div_chunk_.div(gr);
                    const Live& lv = live_[blk];
                    if (!a) a = reinterpret_cast<uint64_t>(lv.slot.ptr) + lv.chunk_off[q - lv.first_chunk];
                    if (kinds) a |= static_cast<uint64_t>(ds_->d8_kind(q)) << kRowKindShift;
                }
                hr[j] = {a, gr};
                if (--blive[blk] == 0) done_blocks_.push_back(blk);  // released after this group's kernel
            }
        }
        std::memcpy(hg, g, ng * sizeof(uint64_t));
    }
    double t_refs = 0;
    if (tr.on) t_refs = tr.lap();
    cuda_ok(cudaMemcpyAsync(s.d_refs, s.h_refs, n * sizeof(RowRef), cudaMemcpyHostToDevice, copy_), "refs H2D");
    ctr_.h2d_bytes += n * sizeof(RowRef);
    // CSR output: the batch indptrs are prefixes of the schedule's per-row nnz
    // (CsrBlock::append_rows rebase, block.cpp:92-108) -- planned here, so the
    // device runs one balanced copy kernel and no scan.  [P: the group's prefix,
    // n+1 entries = batch 0's indptr][batch 1's indptr][batch 2's] ...
    std::vector<uint64_t> ip_off(nb, 0);
    if (planned) {
        uint64_t acc = 0, w = n + 1, row = 0;
        for (size_t i = 0; i < nb; ++i)
            for (uint64_t gr : group_[i].gidx) {
                s.h_prefix[row++] = acc;
                acc += ds_->row_nnz(gr);
            }
        s.h_prefix[n] = acc;
        for (size_t i = 1; i < nb; ++i) {
            ip_off[i] = w;
            const uint64_t r0 = group_start_[i], rn = group_start_[i + 1] - r0, p0 = s.h_prefix[r0];
            for (uint64_t j = 0; j <= rn; ++j) s.h_prefix[w + j] = s.h_prefix[r0 + j] - p0;
            w += rn + 1;
        }
        cuda_ok(cudaMemcpyAsync(s.indptr, s.h_prefix, w * 8, cudaMemcpyHostToDevice, copy_), "indptr H2D");
        ctr_.h2d_bytes += w * 8;
    }
    cuda_ok(cudaEventRecord(staged_, copy_), "event");
    cuda_ok(cudaStreamWaitEvent(compute_, staged_, 0), "wait staged");
    const bool timing = dev_.time_kernels && s.tk[0];
    if (timing) cuda_ok(cudaEventRecord(s.tk[0], compute_), "event");
    // delta-staged records expand into idx16 records on the compute stream, so the
    // copy stream goes straight on to the next group's blocks
    if (!d8_jobs_.empty()) {
        launch_d8_decode(d8_jobs_.data(), d8_jobs_.size(), static_cast<uint32_t>(value_size(m.value_dtype)),
                         m.chunk_rows, compute_, m.n_var, m.value_dtype != VDtype::i32);
        ctr_.kernels_launched += (d8_jobs_.size() + kMaxD8Jobs - 1) / kMaxD8Jobs;
    }

    if (timing) cuda_ok(cudaEventRecord(s.tk[1], compute_), "event");
    const ArenaView av = ds_->view(base);
    if (m.layout == Layout::dense && fused_) {
        launch_onehot_gather(av, s.d_refs, n, dev_.out_dtype, s.data, static_cast<uint64_t*>(s.gidx), compute_);
    } else if (m.layout == Layout::dense) {
        launch_dense_gather(av, s.d_refs, n, dev_.out_dtype, s.data, static_cast<uint64_t*>(s.gidx), compute_);
    } else if (dev_.output == 1 && fused_) {
        launch_csr_densify_d8(av, s.d_refs, n, dev_.out_dtype, dev_.normalize, dev_.target_sum, s.data,
                              static_cast<uint64_t*>(s.gidx), compute_);
    } else if (dev_.output == 1) {
        launch_csr_densify(av, s.d_refs, n, dev_.out_dtype, dev_.normalize, dev_.target_sum, s.data,
                           static_cast<uint64_t*>(s.gidx), compute_, n ? (nnz + n - 1) / n : 0);
    } else if (planned) {
        launch_csr_gather_prefixed(av, s.d_refs, n, static_cast<const uint64_t*>(s.indptr), s.indices, s.data,
                                   static_cast<uint64_t*>(s.gidx), compute_);
    } else {
        launch_csr_gather(av, s.d_refs, n, static_cast<uint64_t*>(s.indptr), s.indices, s.data,
                          static_cast<uint64_t*>(s.gidx), s.scratch, compute_);
    }
    ctr_.kernels_launched += 1;
    if (timing) {
        cuda_ok(cudaEventRecord(s.tk[2], compute_), "event");
        s.timed = true;
    }
    cuda_ok(cudaEventRecord(s.done, compute_), "event");
    ++batch_seq_;

    // blocks whose rows are all taken go back to the pool once this group's kernel is done
    if (!done_blocks_.empty()) {
        cudaEvent_t e = rel_ring_[rel_pos_++ % rel_ring_.size()];
        cuda_ok(cudaEventRecord(e, compute_), "event");
        for (uint64_t blk : done_blocks_) {
            Live& lv = live_[blk];
            lv.slot.released = e;
            lv.slot.owner = id_;
            lv.slot.seq = batch_seq_;
            ds_->release_slot(lv.slot);
            lv.slot = DStore::SlotRef{};
        }
        done_blocks_.clear();
    }

    size_t n_blocks = 0;
    for (const Planned& p : group_) n_blocks += p.consumed.size();
    if (tr.on)
        std::fprintf(stderr,
                     "# next %llu (+%zu): replay %.1f us, stage %.1f us (%zu blocks), slot wait %.1f us, "
                     "row refs %.1f us, rest %.1f us\n",
                     static_cast<unsigned long long>(group_[0].batch_index), nb - 1, t_replay, t_stage, n_blocks,
                     t_slot, t_refs, tr.lap());
    const uint32_t layout = (m.layout == Layout::csr && dev_.output == 0) ? 1u : 0u;
    const uint32_t native = static_cast<uint32_t>(m.value_dtype);
    const uint32_t dtype =
        layout == 1 ? native : (dev_.out_dtype == OutDtype::bf16 ? 4u : dev_.out_dtype == OutDtype::f32 ? 0u : native);
    const uint64_t out_row = layout == 1 ? 0 : m.n_var * dense_out_elem_size(av, dev_.out_dtype);
    const uint64_t is = index_size(av.idt), vs = value_size(m.value_dtype);
    ready_.resize(nb);
    for (size_t i = 0; i < nb; ++i) {
        BatchOut& out = ready_[i];
        const uint64_t r0 = group_start_[i];
        out.epoch = epoch_;
        out.batch_index = group_[i].batch_index;
        out.n_rows = group_start_[i + 1] - r0;
        out.nnz = bnnz[i];
        out.n_var = m.n_var;
        out.layout = layout;
        out.dtype = dtype;
        out.index_dtype = static_cast<uint32_t>(av.idt);
        out.d_gidx = static_cast<uint64_t*>(s.gidx) + r0;
        out.h_gidx = s.h_gidx + r0;
        if (layout == 1) {
            const uint64_t p0 = planned ? s.h_prefix[r0] : 0;
            out.d_indptr = static_cast<uint64_t*>(s.indptr) + ip_off[i];
            out.d_indices = static_cast<uint8_t*>(s.indices) + p0 * is;
            out.d_data = static_cast<uint8_t*>(s.data) + p0 * vs;
        } else {
            out.d_indptr = nullptr;
            out.d_indices = nullptr;
            out.d_data = static_cast<uint8_t*>(s.data) + r0 * out_row;
        }
        out.ready = s.done;
    }
    return true;
}

void GpuLoader::harvest(OutBuffers& s) const {
    if (!s.timed) return;
    float a = 0.f, b = 0.f;
    if (cudaEventElapsedTime(&a, s.tk[0], s.tk[1]) == cudaSuccess &&
        cudaEventElapsedTime(&b, s.tk[1], s.tk[2]) == cudaSuccess) {
        ctr_.decode_ms += a;
        ctr_.assembly_ms += b;
        s.timed = false;
    }
}

Counters GpuLoader::counters() const {
    for (auto& s : slots_)
        if (s.timed && cudaEventQuery(s.tk[2]) == cudaSuccess) harvest(s);
    Counters c = ctr_;
    c.blocks_fetched = snap_blocks_;  // as of the last batch handed out (the replay runs ahead)
    c.peak_buffer_rows = snap_peak_;
    return c;
}

void GpuLoader::sync() {
    DeviceGuard g(ds_->device());
    cuda_ok(cudaStreamSynchronize(compute_), "sync");
}

}  // namespace rfl
