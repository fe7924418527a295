// The re-encoded staging image of a store ("Re-encoded staging
// image"): u16 column ids, u8 column deltas (+ top-byte coded values), one-hot
// channel codes.  Built on the host once per store at open, streaming: records
// are read (and inflated) a window at a time by a thread pool, checked as
// decode_record checks them, encoded, and written straight into the image, so
// the verbatim store never has to fit in host memory.  The image lives in a
// virtual reservation that is page-locked (cudaHostRegister) once filled --
// pinned host memory for stream_pinned, or uploaded to HBM for resident_coded.
// The GPU expands the staged records (k_d8_decode) before the batch kernels.
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cstdio>
#include <array>
#include <atomic>
#include <cstdlib>
#include <cctype>
#include <cstring>
#include <fstream>
#include <string>
#include <thread>

#include "codec.hpp"
#include "engine.hpp"

namespace rfl {

namespace {
constexpr uint64_t kAlign = kRecAlign;
constexpr uint64_t kPad = kRecPad;
constexpr uint64_t kWindowBytes = 512ull << 20;  // verbatim records held per window

// NUMA node of the GPU's PCIe attachment (sysfs), -1 when unknown
int gpu_numa_node(int dev) {
    char bus[64] = {0};
    if (cudaDeviceGetPCIBusId(bus, sizeof bus, dev) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    std::string b(bus);
    for (char& c : b) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    const size_t colon = b.find(':');
    if (colon != std::string::npos && colon > 4) b = b.substr(colon - 4);  // 8-digit PCI domain -> 4
    std::ifstream f("/sys/bus/pci/devices/" + b + "/numa_node");
    int node = -1;
    if (!(f >> node)) return -1;
    return node;
}

// Prefer the GPU's NUMA node for the pages of [p, p + bytes) (first touched later):
// on a multi-socket node the staging pull then reads socket-local memory instead
// of crossing the socket interconnect for half the image.  Best effort, no-op on
// one-node hosts.
void prefer_gpu_node(void* p, uint64_t bytes, int dev) {
    const int node = gpu_numa_node(dev);
    if (node < 0 || node >= 256) return;
    unsigned long mask[4] = {0, 0, 0, 0};
    mask[node / 64] |= 1ul << (node % 64);
    constexpr int kMpolPreferred = 1;
    syscall(SYS_mbind, p, bytes, kMpolPreferred, mask, 256ul, 0u);
}

template <typename F>
void parallel_for(uint64_t n, F&& f) {  // f(i) over [0, n) on up to 16 threads; first error rethrown
    const unsigned T = static_cast<unsigned>(
        std::max<uint64_t>(1, std::min<uint64_t>({16u, std::max(1u, std::thread::hardware_concurrency()), n})));
    std::atomic<uint64_t> next{0};
    std::vector<std::exception_ptr> errs(T);
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < T; ++t)
        pool.emplace_back([&, t] {
            try {
                for (uint64_t i; (i = next.fetch_add(1)) < n;) f(i);
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

// ---------------------------------------------------------- per-record codecs --
namespace {
// column delta of record entry k (0 at a row's first entry)
struct Deltas {
    const uint8_t* ip;
    const uint8_t* ix;
    uint64_t rows, nnz;
    std::vector<uint8_t> d;
    Deltas(const uint8_t* rec) : ip(rec + kCsrHeaderBytes) {
        rows = rd32(rec);
        nnz = rd64(rec + 4);
        ix = ip + 4 * (rows + 1);
        d.assign(nnz, 0);
        for (uint64_t r = 0; r < rows; ++r) {
            const uint64_t lo = rd32(ip + 4 * r), hi = rd32(ip + 4 * (r + 1));
            for (uint64_t k = lo + 1; k < hi; ++k) d[k] = static_cast<uint8_t>(rd32(ix + 4 * k) - rd32(ix + 4 * (k - 1)));
        }
    }
};
uint32_t bit_width(uint32_t v) {
    uint32_t w = 0;
    while (v >> w) ++w;
    return w;
}
// write v[0..n) as the packed groups of d8_packed_at(at, n, pb) into rec (zeroed)
void write_packed(uint8_t* rec, uint64_t at, const std::vector<uint8_t>& v, uint64_t pb) {
    const uint64_t n = v.size();
    const D8Packed L = d8_packed_at(at, n, pb);
    const uint32_t pb32 = static_cast<uint32_t>(pb);
    std::memcpy(rec + L.pbytes_at, &pb32, 4);
    uint64_t bit = 0;
    for (uint64_t g = 0; g * 16 < n; ++g) {
        if (g % 32 == 0) {
            const uint32_t b32 = static_cast<uint32_t>(bit);
            std::memcpy(rec + L.skip + 4 * (g / 32), &b32, 4);
        }
        uint32_t mx = 0;
        const uint64_t k1 = std::min<uint64_t>(n, g * 16 + 16);
        for (uint64_t k = g * 16; k < k1; ++k) mx = std::max<uint32_t>(mx, v[k]);
        uint32_t w = 0;
        while (mx >> w) ++w;
        rec[L.widths + g / 2] |= static_cast<uint8_t>(w << (4 * (g & 1)));
        for (uint64_t k = g * 16; k < g * 16 + 16; ++k, bit += w) {
            const uint32_t x = k < k1 ? v[k] : 0u;
            for (uint32_t b = 0; b < w; ++b)
                if ((x >> b) & 1u) rec[L.bits + ((bit + b) >> 3)] |= static_cast<uint8_t>(1u << ((bit + b) & 7));
        }
    }
}
// the value byte of each entry of an integer-valued record (kD8Int8 eligibility holds)
std::vector<uint8_t> int8_values(const uint8_t* val, uint64_t nnz) {
    std::vector<uint8_t> v(nnz);
    for (uint64_t k = 0; k < nnz; ++k) {
        uint32_t b;
        std::memcpy(&b, val + 4 * k, 4);
        if (b > 255u) {  // f32 bits of an integer value
            float f;
            std::memcpy(&f, &b, 4);
            b = static_cast<uint32_t>(f);
        }
        v[k] = static_cast<uint8_t>(b);
    }
    return v;
}
// bytes of the bit-packed delta stream (sum over groups of 16 x width)
uint64_t packed_bits_bytes(const std::vector<uint8_t>& d) {
    uint64_t bits = 0;
    for (uint64_t g = 0; g * 16 < d.size(); ++g) {
        uint32_t mx = 0;
        for (uint64_t k = g * 16; k < std::min<uint64_t>(d.size(), g * 16 + 16); ++k) mx = std::max<uint32_t>(mx, d[k]);
        bits += 16ull * bit_width(mx);
    }
    return (bits + 7) / 8;
}
}  // namespace

StagePlan plan_csr_stage_u8(const uint8_t* rec, uint64_t vs, bool allow_delta, bool code_values, bool vfloat);

StagePlan plan_csr_stage(const uint8_t* rec, uint64_t vs, bool allow_delta, bool code_values, bool vfloat,
                         bool pack_deltas) {
    StagePlan p = plan_csr_stage_u8(rec, vs, allow_delta, code_values, vfloat);
    if (!pack_deltas || (p.kind != kD8Raw && p.kind != kD8Coded && p.kind != kD8Coded16 && p.kind != kD8Int8)) return p;
    const uint64_t rows = rd32(rec), nnz = rd64(rec + 4);
    const Deltas dl(rec);
    const uint64_t pb = packed_bits_bytes(dl.d);
    const uint64_t dsec = d8_packed_section(rows, nnz, pb);
    if (dsec >= nnz) return p;  // (tiny records: the u8 deltas are smaller)
    const uint64_t ovs = p.kind == kD8Int8 ? 1 : vs;
    p.pbytes = pb;
    if (p.kind == kD8Raw || p.kind == kD8Int8) p.bytes = d8_record_bytes(rows, nnz, ovs, dsec);
    else p.bytes = d8v_layout(rows, nnz, p.n_esc, p.kind == kD8Coded16 ? 1 : 3, dsec).bytes;
    if (p.kind == kD8Int8) {  // the value bytes bit-packed too (kD8IntP) when smaller
        const uint8_t* val = rec + kCsrHeaderBytes + 4 * (rows + 1) + 4 * nnz;
        const uint64_t pbv = packed_bits_bytes(int8_values(val, nnz));
        const uint64_t vo = d8_values_offset(rows, nnz, dsec);
        const D8Packed V = d8_packed_at(vo, nnz, pbv);
        if (V.end - vo < nnz) {
            p.kind = kD8IntP;
            p.pbytes_v = pbv;
            p.bytes = V.end;
        }
    }
    p.kind |= kD8Packed;
    return p;
}

StagePlan plan_csr_stage_u8(const uint8_t* rec, uint64_t vs, bool allow_delta, bool code_values, bool vfloat) {
    const uint64_t rows = rd32(rec), nnz = rd64(rec + 4);
    const uint8_t* ip = rec + kCsrHeaderBytes;
    const uint8_t* ix = ip + 4 * (rows + 1);
    StagePlan p;
    p.exp = idx16_record_bytes(rows, nnz, vs);
    p.kind = kIdx16Copy;
    p.bytes = p.exp;
    if (!allow_delta) return p;
    for (uint64_t r = 0; r < rows; ++r) {  // every in-row column gap <= 255?
        const uint64_t lo = rd32(ip + 4 * r), hi = rd32(ip + 4 * (r + 1));
        uint32_t big = 0;
        for (uint64_t k = lo + 1; k < hi; ++k) big |= static_cast<uint32_t>(rd32(ix + 4 * k) - rd32(ix + 4 * (k - 1)) > 255);
        if (big) return p;
    }
    p.kind = kD8Raw;
    p.bytes = d8_record_bytes(rows, nnz, vs);
    if (!code_values || vs != 4) return p;
    {  // every value an integer in [0, 255]: one byte per value, nothing else (kD8Int8)
        const uint8_t* v = ix + 4 * nnz;
        bool small = true;
        for (uint64_t k = 0; k < nnz && small; ++k) {
            uint32_t b;
            std::memcpy(&b, v + 4 * k, 4);
            if (vfloat) {
                float f;
                std::memcpy(&f, &b, 4);
                uint32_t back;
                const float r = static_cast<float>(static_cast<uint32_t>(f >= 0.f && f <= 255.f ? f : 0.f));
                std::memcpy(&back, &r, 4);
                small = f >= 0.f && f <= 255.f && back == b;  // exact (and not -0.0)
            } else {
                small = b <= 255u;
            }
        }
        if (small) {
            p.kind = kD8Int8;
            p.bytes = d8_record_bytes(rows, nnz, 1);
            return p;
        }
    }
    // top-byte dictionary (3 most frequent) + escapes, kept when smaller
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
    const uint64_t bytes = d8v_layout(rows, nnz, esc, low16_zero ? 1 : 3).bytes;
    if (bytes < p.bytes) {
        p.kind = low16_zero ? kD8Coded16 : kD8Coded;
        p.dict = d;
        p.n_esc = esc;
        p.bytes = bytes;
    }
    return p;
}

void encode_csr_stage(const uint8_t* src, uint64_t vs, const StagePlan& p, uint8_t* dst) {
    std::memset(dst, 0, p.bytes);
    const uint64_t rows = rd32(src), nnz = rd64(src + 4);
    const uint64_t head = kCsrHeaderBytes + 4 * (rows + 1);
    std::memcpy(dst, src, head);  // header + u32 indptr unchanged
    const uint8_t* ip = src + kCsrHeaderBytes;
    const uint8_t* ix = src + head;
    const uint8_t* val = ix + 4 * nnz;
    if (p.kind == kIdx16Copy) {
        for (uint64_t k = 0; k < nnz; ++k) {
            const uint16_t w = static_cast<uint16_t>(rd32(ix + 4 * k));
            std::memcpy(dst + head + 2 * k, &w, 2);
        }
        std::memcpy(dst + head + ((2 * nnz + 7) & ~7ull), val, vs * nnz);
        return;
    }
    uint8_t* first = dst + head;
    uint8_t* delta = first + ((2 * rows + 3) & ~3ull);
    const bool packed = (p.kind & kD8Packed) != 0;
    const uint32_t kind = p.kind & ~kD8Packed;
    for (uint64_t r = 0; r < rows; ++r) {
        const uint64_t lo = rd32(ip + 4 * r), hi = rd32(ip + 4 * (r + 1));
        const uint16_t f = lo < hi ? static_cast<uint16_t>(rd32(ix + 4 * lo)) : 0;
        std::memcpy(first + 2 * r, &f, 2);
        if (!packed)
            for (uint64_t k = lo; k < hi; ++k)
                delta[k] = k == lo ? 0 : static_cast<uint8_t>(rd32(ix + 4 * k) - rd32(ix + 4 * (k - 1)));
    }
    uint64_t dsec = ~0ull;
    if (packed) {
        const Deltas dl(src);
        const D8Packed L = d8_packed_layout(rows, nnz, p.pbytes);
        dsec = L.end - L.pbytes_at;
        write_packed(dst, L.pbytes_at, dl.d, p.pbytes);
    }
    if (kind == kD8IntP) {
        write_packed(dst, d8_values_offset(rows, nnz, dsec), int8_values(val, nnz), p.pbytes_v);
        return;
    }
    if (kind == kD8Raw) {
        std::memcpy(dst + d8_values_offset(rows, nnz, dsec), val, vs * nnz);
        return;
    }
    if (kind == kD8Int8) {
        uint8_t* v8 = dst + d8_values_offset(rows, nnz, dsec);
        for (uint64_t k = 0; k < nnz; ++k) {
            uint32_t b;
            std::memcpy(&b, val + 4 * k, 4);
            if (vs == 4 && b > 255u) {  // f32 bits of an integer value
                float f;
                std::memcpy(&f, &b, 4);
                b = static_cast<uint32_t>(f);
            }
            v8[k] = static_cast<uint8_t>(b);
        }
        return;
    }
    const bool c16 = kind == kD8Coded16;
    const D8vLayout L = d8v_layout(rows, nnz, p.n_esc, c16 ? 1 : 3, dsec);
    std::memcpy(dst + L.dict, p.dict.data(), 4);
    const uint32_t ne = static_cast<uint32_t>(p.n_esc);
    std::memcpy(dst + L.n_esc, &ne, 4);
    uint32_t e = 0;
    for (uint64_t r = 0; r < rows; ++r) {
        std::memcpy(dst + L.esc_base + 4 * r, &e, 4);
        const uint64_t lo = rd32(ip + 4 * r), hi = rd32(ip + 4 * (r + 1));
        for (uint64_t k = lo; k < hi; ++k) {
            const uint8_t top = val[4 * k + 3];
            const uint32_t code = top == p.dict[0] ? 0u : top == p.dict[1] ? 1u : top == p.dict[2] ? 2u : 3u;
            dst[L.codes + (k >> 2)] |= static_cast<uint8_t>(code << (2 * (k & 3)));
            if (code == 3) dst[L.esc + e++] = top;
            if (c16) dst[L.low3 + k] = val[4 * k + 2];
            else std::memcpy(dst + L.low3 + 3 * k, val + 4 * k, 3);
        }
    }
}

bool one_hot_record(const uint8_t* rec, uint64_t rows, uint64_t n_var) {
    const uint64_t L = n_var / 4;
    for (uint64_t i = 0; i < rows; ++i) {
        const uint8_t* row = rec + i * n_var;
        uint32_t bad = 0;
        for (uint64_t p = 0; p < L; ++p) {
            const uint32_t a = row[p], b = row[L + p], c = row[2 * L + p], d = row[3 * L + p];
            bad |= static_cast<uint32_t>((a | b | c | d) > 1) | static_cast<uint32_t>(a + b + c + d != 1);
        }
        if (bad) return false;
    }
    return true;
}

void encode_one_hot(const uint8_t* rec, uint64_t rows, uint64_t n_var, uint8_t* dst) {
    const uint64_t L = n_var / 4;
    std::memset(dst, 0, rows * (L / 4));
    for (uint64_t i = 0; i < rows; ++i) {
        const uint8_t* row = rec + i * n_var;
        uint8_t* codes = dst + i * (L / 4);
        for (uint64_t p = 0; p < L; ++p) {
            const uint32_t ch = row[L + p] ? 1u : row[2 * L + p] ? 2u : row[3 * L + p] ? 3u : 0u;
            codes[p >> 2] |= static_cast<uint8_t>(ch << (2 * (p & 3)));
        }
    }
}

// ------------------------------------------------------------ image builder --
// Which encoding the staging image of this store can use (kStageVerbatim: none).
// RFL_NARROW=0 keeps the verbatim image, =16 u16 ids only; default: deltas where
// every in-row gap <= 255 (+ coded values unless RFL_NARROW_VALUES=0), u16 ids
// elsewhere; dense u8 rows one-hot over 4 planes (n_var % 64 == 0) as 2-bit codes.
uint32_t DStore::stage_mode() const {
    const Manifest& m = manifest();
    const char* e = std::getenv("RFL_NARROW");
    if (e && e[0] == '0') return kStageVerbatim;
    if (m.layout == Layout::csr && m.index_dtype == IDtype::u32 && m.n_var <= 65536)
        return e && std::string(e) == "16" ? kStageIdx16 : kStageDelta;
    if (m.layout == Layout::dense && m.value_dtype == VDtype::u8 && m.n_var % 64 == 0) return kStageOneHot;
    return kStageVerbatim;
}

// Verbatim (decoded) record q into dst[0, rec_len_[q]), checked like
// decode_record (store.cpp:81-122) incl. CsrBlock::validate's column checks;
// per-row nnz of CSR records into row_nnz_.
void DStore::read_checked(uint64_t q, uint8_t* dst, std::vector<uint8_t>& scratch, bool validate) const {
    const Manifest& m = manifest();
    const Slot sl = hs_->record_slot(q);
    if (m.codec == Codec::deflate) {
        scratch.resize(sl.len);
        hs_->read_shard_bytes(q / m.chunks_per_shard, sl.off, scratch.data(), sl.len, false);
        if (!inflate_fits(scratch.data(), sl.len, dst, rec_len_[q])) {
            decode_record_checked(m, q, scratch.data(), sl.len);
            corrupt("chunk " + std::to_string(q) + " in shard " + std::to_string(q / m.chunks_per_shard) +
                    ": csr record invalid");
        }
    } else {
        hs_->read_shard_bytes(q / m.chunks_per_shard, sl.off, dst, sl.len, false);
    }
    if (m.layout == Layout::dense) {
        check_dense_record(m, q, rec_len_[q]);
        return;
    }
    uint32_t* rn = const_cast<uint32_t*>(row_nnz_.data()) + q * m.chunk_rows;
    if (!check_csr_record(m, q, dst, rec_len_[q], rn)) full_check_csr_record(m, q, dst, rec_len_[q]);
    if (validate && !columns_ok(m, q, dst)) full_check_csr_record(m, q, dst, rec_len_[q]);
}

bool DStore::build_staged_image(uint32_t mode) {
    const Manifest& m = manifest();
    const uint64_t nch = m.chunk_count();
    const uint64_t vs = value_size(m.value_dtype);
    const char* nv = std::getenv("RFL_NO_VALIDATE");
    const bool validate = m.layout == Layout::csr && !(nv && nv[0] == '1');
    const char* ve = std::getenv("RFL_NARROW_VALUES");
    const char* te = std::getenv("RFL_TRACE");
    const bool trace = te && te[0] == '1';
    const bool code_values = !(ve && ve[0] == '0');
    // bit-packed column deltas for the PCIe-bound pinned image (RFL_PACK_DELTAS=0: u8 deltas);
    // the HBM-resident coded image keeps u8 deltas (K3d there is bound by its dense writes)
    const char* pe = std::getenv("RFL_PACK_DELTAS");
    const bool pack = staging_ == kStreamPinned && !(pe && pe[0] == '0');
    // virtual reservation bounding every encoding (each kind is at most the
    // verbatim record + 2 B per row + padding), committed page by page as filled
    uint64_t bound = kPad + 4096;
    for (uint64_t q = 0; q < nch; ++q) bound += align_up(rec_len_[q] + 4 * m.rows_in_chunk(q) + 64, kAlign);
    void* map = mmap(nullptr, bound, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
    if (map == MAP_FAILED) throw Error(kIo, "staging image: mmap of " + std::to_string(bound) + " bytes failed");
    if (staging_ == kStreamPinned) prefer_gpu_node(map, bound, device_);
    uint8_t* img = static_cast<uint8_t*>(map);
    std::vector<uint64_t> off(nch), len(nch), elen(nch);
    std::vector<uint8_t> kind(nch);
    std::vector<uint8_t> win;
    std::vector<uint64_t> wpos;
    std::vector<StagePlan> plans;
    uint64_t cursor = 0;
    try {
        for (uint64_t q0 = 0; q0 < nch;) {
            uint64_t q1 = q0, wb = 0;
            wpos.clear();
            while (q1 < nch && (q1 == q0 || wb + rec_len_[q1] <= kWindowBytes)) {
                wpos.push_back(wb);
                wb = align_up(wb + rec_len_[q1], kAlign);
                ++q1;
            }
            if (win.size() < wb + kPad) win.resize(wb + kPad);
            plans.assign(q1 - q0, StagePlan{});
            std::atomic<bool> one_hot_ok{true};
            parallel_for(q1 - q0, [&](uint64_t k) {
                thread_local std::vector<uint8_t> scratch;
                const uint64_t q = q0 + k;
                uint8_t* rec = win.data() + wpos[k];
                read_checked(q, rec, scratch, validate);
                if (mode == kStageOneHot) {
                    if (!one_hot_record(rec, m.rows_in_chunk(q), m.n_var)) one_hot_ok = false;
                    plans[k].kind = kOneHot4;
                    plans[k].bytes = m.rows_in_chunk(q) * (m.n_var / 16);
                    plans[k].exp = rec_len_[q];
                } else {
                    plans[k] = plan_csr_stage(rec, vs, mode == kStageDelta, code_values, m.value_dtype != VDtype::i32, pack);
                }
            });
            if (!one_hot_ok) {  // not a one-hot store: the verbatim image
                munmap(map, bound);
                return false;
            }
            for (uint64_t k = 0; k < q1 - q0; ++k) {
                const uint64_t q = q0 + k;
                off[q] = cursor;
                len[q] = plans[k].bytes;
                elen[q] = plans[k].exp;
                kind[q] = plans[k].kind;
                cursor = align_up(cursor + len[q], kAlign);
            }
            if (cursor + kPad > bound) throw Error(kIo, "staging image: encoding exceeds its reservation");
            parallel_for(q1 - q0, [&](uint64_t k) {
                const uint64_t q = q0 + k;
                const uint8_t* rec = win.data() + wpos[k];
                if (mode == kStageOneHot) encode_one_hot(rec, m.rows_in_chunk(q), m.n_var, img + off[q]);
                else encode_csr_stage(rec, vs, plans[k], img + off[q]);
                const uint64_t gap = (q + 1 < nch ? align_up(off[q] + len[q], kAlign) : off[q] + len[q] + kPad) -
                                     (off[q] + len[q]);
                std::memset(img + off[q] + len[q], 0, gap);
            });
            q0 = q1;
            if (trace && (q0 == nch || q0 / 1024 != (q0 - (q1 - wpos.size())) / 1024))
                std::fprintf(stderr, "# staging image: %llu / %llu records, %.2f GB staged\n",
                             static_cast<unsigned long long>(q0), static_cast<unsigned long long>(nch), cursor / 1e9);
        }
    } catch (...) {
        munmap(map, bound);
        throw;
    }
    std::vector<uint8_t>().swap(win);
    // release the unused tail of the reservation, then page-lock the image
    const uint64_t used = (cursor + kPad + 4095) & ~4095ull;
    if (used < bound) munmap(img + used, bound - used);
    h_map_bytes_ = used;
    h_image_ = img;
    if (staging_ == kStreamPinned) {
        // page-locked in kPinPiece pieces: one cudaHostRegister of the whole
        // multi-GB range fails on the B200 boxes ("OS call failed") while every
        // 1 GiB piece of it registers; copies never cross a piece boundary
        // (stage_block splits them), so the pieces behave as one pinned image
        for (uint64_t o = 0; o < used; o += kPinPiece) {
            const cudaError_t rc = cudaHostRegister(img + o, std::min(kPinPiece, used - o), cudaHostRegisterPortable | cudaHostRegisterMapped);
            if (rc != cudaSuccess) {
                for (uint64_t u = 0; u < o; u += kPinPiece) cudaHostUnregister(img + u);
                munmap(img, used);
                h_image_ = nullptr;
                h_map_bytes_ = 0;
                cuda_ok(rc, ("cudaHostRegister of the staging image at byte " + std::to_string(o)).c_str());
            }
        }
        h_registered_ = true;
    }
    img_off_ = std::move(off);
    img_len_ = std::move(len);
    exp_len_ = std::move(elen);
    d8_rec_ = std::move(kind);
    staged_bytes_ = cursor;
    if (mode == kStageIdx16 && staging_ == kStreamPinned) {
        // u16 ids only: the kernels read the staged records in place (no decode)
        idx16_ = true;
        d8_ = false;
        exp_len_.clear();
        d8_rec_.clear();
    } else {
        idx16_ = mode != kStageOneHot;
        d8_ = true;
    }
    return true;
}

}  // namespace rfl
