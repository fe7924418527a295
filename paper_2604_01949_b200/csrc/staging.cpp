// Re-encoding of a stream_pinned store's pinned image for PCIe (DESIGN.md,
// "Re-encoded staging image"): u16 column ids, u8 column deltas (+ top-byte
// coded values), one-hot channel codes.  Host-side, once per store at open;
// the GPU expands the staged records (k_d8_decode) before the batch kernels.
#include <algorithm>
#include <array>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>

#include "engine.hpp"

namespace rfl {

namespace {
constexpr uint64_t kAlign = kRecAlign;
constexpr uint64_t kPad = kRecPad;
}  // namespace

// The pinned staging image with u16 column indices (lossless: n_var <= 65536):
// 2 of every 8 bytes per stored entry never cross PCIe.  The records were
// validated in their store encoding first; kernels read this layout through
// ArenaView::idx16 (csr_row<uint16_t>).
namespace {
template <typename F>
void parallel_records(uint64_t n, F&& f) {
    const unsigned T = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < T; ++t)
        pool.emplace_back([&, t] {
            for (uint64_t q = t; q < n; q += T) f(q);
        });
    for (auto& th : pool) th.join();
}
}  // namespace

// Delta staging image (kernels.cuh d8_* / d8v_*): records whose in-row column
// gaps are all <= 255 stage as u8 deltas (1 B per stored column id instead of
// 4), with 4-byte values also top-byte coded when that is smaller
// (RFL_NARROW_VALUES=0 keeps them raw); the rest stage as idx16 records.  A
// kernel expands every kind into idx16 records in the slot.  Analysed read-only
// and encoded in parallel into a separate buffer, then copied over the
// verbatim image (false: the encoding would not fit; narrow_image() runs).
bool DStore::delta_image() {
    const Manifest& m = hs_->manifest();
    const uint64_t nch = m.chunk_count();
    const uint64_t vs = value_size(m.value_dtype);
    // per record: delta-eligible (every in-row gap <= 255)?  With 4-byte values, also
    // the top-byte dictionary (3 most frequent) and its escape count, kept when smaller
    std::vector<uint8_t> kind(nch, kD8Raw);
    std::vector<std::array<uint8_t, 4>> dict(nch);
    std::vector<uint64_t> n_esc(nch, 0);
    const char* ve = std::getenv("RFL_NARROW_VALUES");
    const bool code_values = vs == 4 && !(ve && ve[0] == '0');
    {
        const unsigned T = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < T; ++t)
            pool.emplace_back([&, t] {
                for (uint64_t q = t; q < nch; q += T) {
                    const uint8_t* rec = h_image_ + rec_off_[q];
                    const uint64_t rows = rd32(rec), nnz = rd64(rec + 4);
                    const uint8_t* ip = rec + kCsrHeaderBytes;
                    const uint8_t* ix = ip + 4 * (rows + 1);
                    bool ok = true;
                    for (uint64_t r = 0; r < rows && ok; ++r) {
                        const uint64_t lo = rd32(ip + 4 * r), hi = rd32(ip + 4 * (r + 1));
                        for (uint64_t k = lo + 1; k < hi; ++k)
                            if (rd32(ix + 4 * k) - rd32(ix + 4 * (k - 1)) > 255) {
                                ok = false;
                                break;
                            }
                    }
                    if (!ok) {
                        kind[q] = kIdx16Copy;
                        continue;
                    }
                    if (!code_values) continue;
                    uint64_t hist[256] = {0};
                    const uint8_t* val = ix + 4 * nnz;
                    for (uint64_t k = 0; k < nnz; ++k) ++hist[val[4 * k + 3]];
                    std::array<uint8_t, 4> d{0, 0, 0, 0};
                    uint64_t covered = 0;
                    for (int c = 0; c < 3; ++c) {
                        int best = 0;
                        for (int b = 1; b < 256; ++b)
                            if (hist[b] > hist[best]) best = b;
                        d[c] = static_cast<uint8_t>(best);
                        covered += hist[best];
                        hist[best] = 0;
                    }
                    const uint64_t esc = nnz - covered;
                    bool low16_zero = true;
                    for (uint64_t k = 0; k < nnz && low16_zero; ++k) low16_zero = val[4 * k] == 0 && val[4 * k + 1] == 0;
                    const uint64_t lb = low16_zero ? 1 : 3;
                    if (d8v_layout(rows, nnz, esc, lb).bytes < d8_record_bytes(rows, nnz, vs)) {
                        kind[q] = low16_zero ? kD8Coded16 : kD8Coded;
                        dict[q] = d;
                        n_esc[q] = esc;
                    }
                }
            });
        for (auto& th : pool) th.join();
    }
    std::vector<uint64_t> off(nch), len(nch), elen(nch);
    uint64_t total = 0;
    for (uint64_t q = 0; q < nch; ++q) {
        const uint8_t* rec = h_image_ + rec_off_[q];
        const uint64_t rows = rd32(rec), nnz = rd64(rec + 4);
        elen[q] = idx16_record_bytes(rows, nnz, vs);
        len[q] = kind[q] == kIdx16Copy  ? elen[q]
                 : kind[q] == kD8Coded   ? d8v_layout(rows, nnz, n_esc[q]).bytes
                 : kind[q] == kD8Coded16 ? d8v_layout(rows, nnz, n_esc[q], 1).bytes
                                         : d8_record_bytes(rows, nnz, vs);
        off[q] = total;
        total = align_up(total + len[q], kAlign);
    }
    if (total > image_bytes_) return false;
    // encode in parallel into a separate buffer (the verbatim image stays read-only), then copy back
    std::vector<uint8_t> img(total, 0);
    parallel_records(nch, [&](uint64_t q) {
        const uint8_t* src = h_image_ + rec_off_[q];
        uint8_t* dst = img.data() + off[q];
        const uint64_t rows = rd32(src), nnz = rd64(src + 4);
        const uint64_t head = kCsrHeaderBytes + 4 * (rows + 1);
        std::memcpy(dst, src, head);
        const uint8_t* ip = src + kCsrHeaderBytes;
        const uint8_t* ix = src + head;
        const uint8_t* val = ix + 4 * nnz;
        if (kind[q] == kIdx16Copy) {
            for (uint64_t k = 0; k < nnz; ++k) {
                const uint16_t w = static_cast<uint16_t>(rd32(ix + 4 * k));
                std::memcpy(dst + head + 2 * k, &w, 2);
            }
            std::memcpy(dst + head + ((2 * nnz + 7) & ~7ull), val, vs * nnz);
            return;
        }
        uint8_t* first = dst + head;
        uint8_t* delta = first + ((2 * rows + 3) & ~3ull);
        for (uint64_t r = 0; r < rows; ++r) {
            const uint64_t lo = rd32(ip + 4 * r), hi = rd32(ip + 4 * (r + 1));
            const uint16_t f = lo < hi ? static_cast<uint16_t>(rd32(ix + 4 * lo)) : 0;
            std::memcpy(first + 2 * r, &f, 2);
            for (uint64_t k = lo; k < hi; ++k)
                delta[k] = k == lo ? 0 : static_cast<uint8_t>(rd32(ix + 4 * k) - rd32(ix + 4 * (k - 1)));
        }
        if (kind[q] == kD8Raw) {
            std::memcpy(dst + d8_values_offset(rows, nnz), val, vs * nnz);
            return;
        }
        const bool c16 = kind[q] == kD8Coded16;
        const D8vLayout L = d8v_layout(rows, nnz, n_esc[q], c16 ? 1 : 3);
        const std::array<uint8_t, 4>& d = dict[q];
        std::memcpy(dst + L.dict, d.data(), 4);
        const uint32_t ne = static_cast<uint32_t>(n_esc[q]);
        std::memcpy(dst + L.n_esc, &ne, 4);
        uint32_t e = 0;
        for (uint64_t r = 0; r < rows; ++r) {
            std::memcpy(dst + L.esc_base + 4 * r, &e, 4);
            const uint64_t lo = rd32(ip + 4 * r), hi = rd32(ip + 4 * (r + 1));
            for (uint64_t k = lo; k < hi; ++k) {
                const uint8_t top = val[4 * k + 3];
                const uint32_t code = top == d[0] ? 0u : top == d[1] ? 1u : top == d[2] ? 2u : 3u;
                dst[L.codes + (k >> 2)] |= static_cast<uint8_t>(code << (2 * (k & 3)));
                if (code == 3) dst[L.esc + e++] = top;
                if (c16) dst[L.low3 + k] = val[4 * k + 2];
                else std::memcpy(dst + L.low3 + 3 * k, val + 4 * k, 3);
            }
        }
    });
    std::memcpy(h_image_, img.data(), total);
    std::memset(h_image_ + total, 0, std::min<uint64_t>(kPad, image_bytes_ + kPad - total));
    img_off_ = std::move(off);
    img_len_ = std::move(len);
    exp_len_ = std::move(elen);
    d8_rec_ = std::move(kind);
    idx16_ = d8_ = true;
    return true;
}

// One-hot staging image (kernels.cuh kOneHot4): when every row of a dense u8
// store is one-hot over 4 channel planes ([4][n_var/4], exactly one 1 per
// position -- the WGS-window encoding of BASELINE config 4), each row stages
// as n_var/16 bytes of 2-bit channel codes; the decode kernel rebuilds the
// verbatim rows in the slot.  Checked read-only first; false = not one-hot.
bool DStore::one_hot_image() {
    const Manifest& m = hs_->manifest();
    const uint64_t nch = m.chunk_count();
    const uint64_t L = m.n_var / 4;
    std::atomic<bool> ok{true};
    {
        const unsigned T = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < T; ++t)
            pool.emplace_back([&, t] {
                for (uint64_t q = t; q < nch && ok.load(std::memory_order_relaxed); q += T) {
                    const uint8_t* rec = h_image_ + rec_off_[q];
                    const uint64_t rows = m.rows_in_chunk(q);
                    for (uint64_t i = 0; i < rows; ++i) {
                        const uint8_t* row = rec + i * m.n_var;
                        for (uint64_t p = 0; p < L; ++p) {
                            const uint32_t a = row[p], b = row[L + p], c = row[2 * L + p], d = row[3 * L + p];
                            if ((a | b | c | d) > 1 || a + b + c + d != 1) {
                                ok = false;
                                return;
                            }
                        }
                    }
                }
            });
        for (auto& th : pool) th.join();
    }
    if (!ok) return false;
    std::vector<uint64_t> off(nch), len(nch);
    uint64_t total = 0;
    for (uint64_t q = 0; q < nch; ++q) {
        len[q] = m.rows_in_chunk(q) * (L / 4);
        off[q] = total;
        total = align_up(total + len[q], kAlign);
    }
    std::vector<uint8_t> img(total, 0);  // encoded in parallel, then copied over the verbatim image
    parallel_records(nch, [&](uint64_t q) {
        uint8_t* dst = img.data() + off[q];
        const uint64_t rows = m.rows_in_chunk(q);
        for (uint64_t i = 0; i < rows; ++i) {
            const uint8_t* row = h_image_ + rec_off_[q] + i * m.n_var;
            uint8_t* codes = dst + i * (L / 4);
            for (uint64_t p = 0; p < L; ++p) {
                const uint32_t ch = row[L + p] ? 1u : row[2 * L + p] ? 2u : row[3 * L + p] ? 3u : 0u;
                codes[p >> 2] |= static_cast<uint8_t>(ch << (2 * (p & 3)));
            }
        }
    });
    std::memcpy(h_image_, img.data(), total);
    std::memset(h_image_ + total, 0, std::min<uint64_t>(kPad, image_bytes_ + kPad - total));
    img_off_ = std::move(off);
    img_len_ = std::move(len);
    exp_len_ = rec_len_;
    d8_rec_.assign(nch, kOneHot4);
    d8_ = true;
    return true;
}

void DStore::narrow_image() {
    const Manifest& m = hs_->manifest();
    const uint64_t nch = m.chunk_count();
    const uint64_t vs = value_size(m.value_dtype);
    std::vector<uint64_t> off(nch), len(nch);
    uint64_t total = 0;
    for (uint64_t q = 0; q < nch; ++q) {
        const uint8_t* rec = h_image_ + rec_off_[q];
        len[q] = idx16_record_bytes(rd32(rec), rd64(rec + 4), vs);
        off[q] = total;
        total = align_up(total + len[q], kAlign);
    }
    // In place, front to back (no second pinned image): safe when every narrowed
    // record ends before the next record's old start (it starts at or below its
    // old offset, and within a record each destination byte lies below every
    // source byte still to be read).  Only records with < 4 entries can grow
    // (index padding); if that ever breaks the rule, keep the verbatim image.
    for (uint64_t q = 0; q < nch; ++q) {
        const uint64_t next_old = q + 1 < nch ? rec_off_[q + 1] : image_bytes_;
        if (off[q] > rec_off_[q] || off[q] + len[q] > next_old) return;
    }
    for (uint64_t q = 0; q < nch; ++q) {
        const uint8_t* src = h_image_ + rec_off_[q];
        uint8_t* dst = h_image_ + off[q];
        const uint64_t rows = rd32(src), nnz = rd64(src + 4);
        const uint64_t head = kCsrHeaderBytes + 4 * (rows + 1);
        std::memmove(dst, src, head);  // header + u32 indptr unchanged
        const uint8_t* si = src + head;
        uint8_t* di = dst + head;
        for (uint64_t k = 0; k < nnz; ++k) {
            uint32_t v;
            std::memcpy(&v, si + 4 * k, 4);
            const uint16_t w = static_cast<uint16_t>(v);
            std::memcpy(di + 2 * k, &w, 2);
        }
        const uint64_t ib = (2 * nnz + 7) & ~7ull;
        std::memmove(dst + head + ib, src + head + 4 * nnz, vs * nnz);  // before the pad may overwrite it
        std::memset(dst + head + 2 * nnz, 0, ib - 2 * nnz);
    }
    std::memset(h_image_ + total, 0, std::min<uint64_t>(kPad, image_bytes_ + kPad - total));
    img_off_ = std::move(off);
    img_len_ = std::move(len);
    idx16_ = true;
}

}  // namespace rfl
