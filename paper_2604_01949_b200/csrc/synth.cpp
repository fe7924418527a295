// Seeded synthetic stores, byte-identical to the reference synth_store
// (reference src/synth.cpp:15-144) so parity inputs can be produced on the GPU
// box without the reference: one Rng stream per 4096-row block, column-0
// identity channel, CSR columns by geometric skipping with std::log1p/floor.
// Blocks are generated in parallel (each owns its stream) and streamed into
// chunk records in order (StoreWriter::append -> emit_chunk, store.cpp:170-213).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <thread>

#include "format.hpp"
#include "rng.hpp"
#include "synth.hpp"

namespace rfl {

namespace {

constexpr uint64_t kSynthBlockRows = 4096;  // synth.cpp:15

double identity_value(VDtype dt, uint64_t row) {  // synth.cpp:39-48
    switch (dt) {
        case VDtype::f32: return static_cast<double>(static_cast<float>(row));
        case VDtype::f64: return static_cast<double>(row);
        case VDtype::i32: return static_cast<double>(static_cast<int32_t>(row % 0x80000000ull));
        case VDtype::u8: return static_cast<double>(row % 256);
    }
    return 0.0;
}
double random_value(Rng& r, VDtype dt) {  // synth.cpp:17-25
    switch (dt) {
        case VDtype::f32:
        case VDtype::f64: return r.next_double();
        case VDtype::i32: return static_cast<double>(r.bounded(1000));
        case VDtype::u8: return static_cast<double>(r.bounded(256));
    }
    return 0.0;
}
double random_nonzero_value(Rng& r, VDtype dt) {  // synth.cpp:27-35
    switch (dt) {
        case VDtype::f32:
        case VDtype::f64: return 1.0 - r.next_double();
        case VDtype::i32: return 1.0 + static_cast<double>(r.bounded(999));
        case VDtype::u8: return 1.0 + static_cast<double>(r.bounded(255));
    }
    return 1.0;
}
void put_value(uint8_t* dst, VDtype dt, double v) {  // scalar_set, block.cpp:36-55
    switch (dt) {
        case VDtype::f32: { const float f = static_cast<float>(v); std::memcpy(dst, &f, 4); return; }
        case VDtype::f64: std::memcpy(dst, &v, 8); return;
        case VDtype::i32: { const int32_t n = static_cast<int32_t>(v); std::memcpy(dst, &n, 4); return; }
        case VDtype::u8: *dst = static_cast<uint8_t>(v); return;
    }
}

struct CsrRows {  // one synth block: chunk-independent CSR
    std::vector<uint64_t> indptr{0};
    std::vector<uint64_t> indices;
    std::vector<uint8_t> data;
};

void gen_csr_block(const SynthCfg& c, uint64_t start, uint64_t rows, uint64_t block_index, double resid,
                   CsrRows& out) {
    Rng rng = Rng(c.seed).stream(block_index);
    const size_t vs = value_size(c.value_dtype);
    const double log1mp = resid > 0.0 && resid < 1.0 ? std::log1p(-resid) : 0.0;
    const size_t expect = static_cast<size_t>(static_cast<double>(rows) * (1.0 + resid * c.n_var) * 1.05) + 16;
    out.indices.reserve(expect);
    out.data.reserve(expect * vs);
    out.indptr.reserve(rows + 1);
    auto push = [&](uint64_t col, double v) {
        out.indices.push_back(col);
        const size_t o = out.data.size();
        out.data.resize(o + vs);
        put_value(out.data.data() + o, c.value_dtype, v);
    };
    for (uint64_t i = 0; i < rows; ++i) {
        push(0, identity_value(c.value_dtype, start + i));
        if (resid >= 1.0) {
            for (uint64_t col = 1; col < c.n_var; ++col) push(col, random_nonzero_value(rng, c.value_dtype));
        } else if (resid > 0.0) {
            uint64_t col = 0;
            for (;;) {
                const double u = rng.next_double();
                const double skip = std::floor(std::log1p(-u) / log1mp);
                if (skip >= static_cast<double>(c.n_var)) break;
                col += 1 + static_cast<uint64_t>(skip);
                if (col >= c.n_var) break;
                push(col, random_nonzero_value(rng, c.value_dtype));
            }
        }
        out.indptr.push_back(out.indices.size());
    }
}

void gen_dense_block(const SynthCfg& c, uint64_t start, uint64_t rows, uint64_t block_index,
                     std::vector<uint8_t>& out) {
    Rng rng = Rng(c.seed).stream(block_index);
    const size_t vs = value_size(c.value_dtype);
    const size_t rb = c.n_var * vs;
    out.assign(rows * rb, 0);
    for (uint64_t i = 0; i < rows; ++i) {
        uint8_t* row = out.data() + i * rb;
        put_value(row, c.value_dtype, identity_value(c.value_dtype, start + i));
        for (uint64_t col = 1; col < c.n_var; ++col) put_value(row + col * vs, c.value_dtype, random_value(rng, c.value_dtype));
    }
}

void put_index(std::vector<uint8_t>& rec, size_t& pos, IDtype idt, uint64_t v) {
    if (idt == IDtype::u64) {
        wr64(rec.data() + pos, v);
        pos += 8;
    } else {
        if (v > 0xFFFFFFFFull) invalid("csr record: value " + std::to_string(v) + " does not fit index_dtype u32");
        wr32(rec.data() + pos, static_cast<uint32_t>(v));
        pos += 4;
    }
}

}  // namespace

// encode_csr_record (store.cpp:52-64) for rows [r0, r1) of `src` (indptr rebased).
void encode_csr_rows(const uint64_t* indptr, const uint64_t* indices, const uint8_t* data, size_t vs,
                     IDtype idt, uint64_t r0, uint64_t r1, std::vector<uint8_t>& rec) {
    const uint64_t rows = r1 - r0, base = indptr[r0], nnz = indptr[r1] - base;
    const size_t is = index_size(idt);
    rec.resize(kCsrHeaderBytes + (rows + 1) * is + nnz * is + nnz * vs);
    wr32(rec.data(), static_cast<uint32_t>(rows));
    wr64(rec.data() + 4, nnz);
    size_t pos = kCsrHeaderBytes;
    for (uint64_t r = r0; r <= r1; ++r) put_index(rec, pos, idt, indptr[r] - base);
    for (uint64_t k = base; k < base + nnz; ++k) put_index(rec, pos, idt, indices[k]);
    std::memcpy(rec.data() + pos, data + base * vs, nnz * vs);
}

namespace {
Manifest synth_one_hot(const std::string& path, const SynthCfg& c) {
    if (c.layout != Layout::dense || c.value_dtype != VDtype::u8 || c.n_var % c.one_hot != 0)
        invalid("synth: one_hot needs a dense u8 store with n_var a multiple of the channel count");
    Manifest man;
    man.layout = Layout::dense;
    man.n_var = c.n_var;
    man.value_dtype = VDtype::u8;
    man.chunk_rows = c.chunk_rows;
    man.chunks_per_shard = c.chunks_per_shard;
    man.codec = c.codec;
    man.var_names.reserve(c.n_var);
    for (uint64_t i = 0; i < c.n_var; ++i) man.var_names.push_back("v" + std::to_string(i));
    RecordWriter w(path, man, /*defer_manifest=*/false);
    const uint64_t L = c.n_var / c.one_hot;
    const unsigned T = c.threads ? c.threads : std::max(1u, std::thread::hardware_concurrency());
    std::vector<uint8_t> rec;
    for (uint64_t r0 = 0; r0 < c.n_obs; r0 += c.chunk_rows) {
        const uint64_t rows = std::min<uint64_t>(c.chunk_rows, c.n_obs - r0);
        rec.assign(rows * c.n_var, 0);
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < T; ++t)
            pool.emplace_back([&, t] {
                for (uint64_t i = t; i < rows; i += T) {
                    const uint64_t hr = mix64(c.seed ^ mix64(r0 + i));
                    uint8_t* row = rec.data() + i * c.n_var;
                    for (uint64_t p = 0; p < L; ++p) row[(mix64(hr ^ p) % c.one_hot) * L + p] = 1;
                }
            });
        for (auto& th : pool) th.join();
        w.append_record(rec.data(), rec.size(), rows);
    }
    return w.finish();
}
}  // namespace

namespace {
Manifest counts_manifest(const SynthCfg& c) {
    if (c.layout != Layout::csr || (c.value_dtype != VDtype::f32 && c.value_dtype != VDtype::i32))
        invalid("synth: counts needs a csr store with f32 or i32 values");
    Manifest man;
    man.layout = Layout::csr;
    man.n_var = c.n_var;
    man.value_dtype = c.value_dtype;
    man.index_dtype = c.index_dtype;
    man.chunk_rows = c.chunk_rows;
    man.chunks_per_shard = c.chunks_per_shard;
    man.codec = c.codec;
    man.var_names.reserve(c.n_var);
    for (uint64_t i = 0; i < c.n_var; ++i) man.var_names.push_back("v" + std::to_string(i));
    man.validate();
    return man;
}
uint64_t counts_row_nnz(const SynthCfg& c, uint64_t row) {
    return std::min<uint64_t>(c.n_var, 2000 + mix64(c.seed ^ mix64(row)) % 2001);
}
}  // namespace

// The counts record of rows [r0, r0 + rows) (encode_csr_record layout), rows
// generated on `threads` threads (each row owns its hash stream).
void counts_record(const SynthCfg& c, uint64_t r0, uint64_t rows, std::vector<uint8_t>& rec, unsigned threads) {
    const size_t vs = value_size(c.value_dtype);
    std::vector<uint64_t> indptr(rows + 1, 0);
    for (uint64_t i = 0; i < rows; ++i) indptr[i + 1] = indptr[i] + counts_row_nnz(c, r0 + i);
    std::vector<uint64_t> indices(indptr[rows]);
    std::vector<uint8_t> data(indptr[rows] * vs);
    auto gen = [&](unsigned t, unsigned T) {
        for (uint64_t i = t; i < rows; i += T) {
            const uint64_t h = mix64(c.seed ^ mix64(r0 + i)), n = indptr[i + 1] - indptr[i];
            for (uint64_t k = 0; k < n; ++k) {
                const uint64_t lo = k * c.n_var / n, hi = (k + 1) * c.n_var / n;  // stratum
                indices[indptr[i] + k] = lo + mix64(h ^ k) % (hi - lo);
                const uint32_t cnt = 1 + static_cast<uint32_t>(mix64(h ^ (k + (1ull << 32))) % 64);
                if (c.value_dtype == VDtype::f32) {
                    const float f = static_cast<float>(cnt);
                    std::memcpy(data.data() + (indptr[i] + k) * 4, &f, 4);
                } else {
                    std::memcpy(data.data() + (indptr[i] + k) * 4, &cnt, 4);
                }
            }
        }
    };
    if (threads <= 1) {
        gen(0, 1);
    } else {
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < threads; ++t) pool.emplace_back(gen, t, threads);
        for (auto& th : pool) th.join();
    }
    encode_csr_rows(indptr.data(), indices.data(), data.data(), vs, c.index_dtype, 0, rows, rec);
}

Manifest synth_counts(const std::string& path, const SynthCfg& c) {
    const Manifest man = counts_manifest(c);
    RecordWriter w(path, man, /*defer_manifest=*/false);
    const unsigned T = c.threads ? c.threads : std::max(1u, std::thread::hardware_concurrency());
    std::vector<uint8_t> rec;
    for (uint64_t r0 = 0; r0 < c.n_obs; r0 += c.chunk_rows) {
        const uint64_t rows = std::min<uint64_t>(c.chunk_rows, c.n_obs - r0);
        counts_record(c, r0, rows, rec, T);
        w.append_record(rec.data(), rec.size(), rows);
    }
    return w.finish();
}

// ---- procedural record source ---------------------------------------------------
namespace {
class CountsSource : public RecordSource {
public:
    explicit CountsSource(SynthCfg c) : c_(std::move(c)) {}
    uint64_t record_bytes(uint64_t q) const override {
        const uint64_t r0 = q * c_.chunk_rows, rows = std::min<uint64_t>(c_.chunk_rows, c_.n_obs - r0);
        uint64_t nnz = 0;
        for (uint64_t i = 0; i < rows; ++i) nnz += counts_row_nnz(c_, r0 + i);
        return kCsrHeaderBytes + (rows + 1) * index_size(c_.index_dtype) +
               nnz * (index_size(c_.index_dtype) + value_size(c_.value_dtype));
    }
    void record(uint64_t q, std::vector<uint8_t>& out) const override {
        const uint64_t r0 = q * c_.chunk_rows, rows = std::min<uint64_t>(c_.chunk_rows, c_.n_obs - r0);
        counts_record(c_, r0, rows, out, 1);
    }

private:
    SynthCfg c_;
};

uint64_t spec_u64(const std::string& v, const std::string& key) {
    if (v.empty() || v.find_first_not_of("0123456789") != std::string::npos)
        invalid("procedural store: bad value for " + key + ": '" + v + "'");
    return std::stoull(v);
}
}  // namespace

std::shared_ptr<const RecordSource> make_record_source(const std::string& spec, Manifest& man) {
    // procedural:counts?n_obs=N&n_var=V&seed=S&chunk_rows=C&chunks_per_shard=P[&value_dtype=f32|i32]
    const std::string pre = "procedural:counts";
    if (spec.compare(0, pre.size(), pre) != 0)
        invalid("procedural store: unknown generator in '" + spec + "' (known: procedural:counts?...)");
    SynthCfg c;
    c.layout = Layout::csr;
    c.value_dtype = VDtype::f32;
    c.index_dtype = IDtype::u32;
    c.counts = true;
    const size_t qm = spec.find('?');
    std::string rest = qm == std::string::npos ? "" : spec.substr(qm + 1);
    while (!rest.empty()) {
        const size_t amp = rest.find('&');
        const std::string kv = rest.substr(0, amp);
        rest = amp == std::string::npos ? "" : rest.substr(amp + 1);
        const size_t eq = kv.find('=');
        const std::string k = kv.substr(0, eq), v = eq == std::string::npos ? "" : kv.substr(eq + 1);
        if (k == "n_obs") c.n_obs = spec_u64(v, k);
        else if (k == "n_var") c.n_var = spec_u64(v, k);
        else if (k == "seed") c.seed = spec_u64(v, k);
        else if (k == "chunk_rows") c.chunk_rows = spec_u64(v, k);
        else if (k == "chunks_per_shard") c.chunks_per_shard = spec_u64(v, k);
        else if (k == "value_dtype" && (v == "f32" || v == "i32")) c.value_dtype = v == "f32" ? VDtype::f32 : VDtype::i32;
        else invalid("procedural store: unknown parameter '" + kv + "'");
    }
    if (c.n_obs == 0 || c.n_var == 0) invalid("procedural store: n_obs and n_var must be >= 1");
    man = counts_manifest(c);
    man.n_obs = c.n_obs;
    return std::make_shared<CountsSource>(c);
}

Manifest synth_store(const std::string& path, const SynthCfg& c) {
    if (c.n_obs == 0 || c.n_var == 0) invalid("synth: n_obs and n_var must be >= 1");
    if (c.one_hot) return synth_one_hot(path, c);
    if (c.counts) return synth_counts(path, c);
    if (c.layout == Layout::csr && (c.density <= 0.0 || c.density > 1.0))
        invalid("synth: density must lie in (0, 1] for csr stores");
    Manifest man;
    man.layout = c.layout;
    man.n_var = c.n_var;
    man.value_dtype = c.value_dtype;
    if (c.layout == Layout::csr) man.index_dtype = c.index_dtype;
    man.chunk_rows = c.chunk_rows;
    man.chunks_per_shard = c.chunks_per_shard;
    man.codec = c.codec;
    man.var_names.reserve(c.n_var);
    for (uint64_t i = 0; i < c.n_var; ++i) man.var_names.push_back("v" + std::to_string(i));
    RecordWriter w(path, man, /*defer_manifest=*/false);

    const double resid = c.n_var > 1 ? std::clamp((static_cast<double>(c.n_var) * c.density - 1.0) /
                                                      static_cast<double>(c.n_var - 1),
                                                  0.0, 1.0)
                                     : 0.0;
    const uint64_t n_blocks = (c.n_obs + kSynthBlockRows - 1) / kSynthBlockRows;
    unsigned T = c.threads ? c.threads : std::max(1u, std::thread::hardware_concurrency());
    T = static_cast<unsigned>(std::min<uint64_t>(T, n_blocks));
    const size_t vs = value_size(c.value_dtype);

    // pending rows not yet emitted as a chunk
    CsrRows pend;
    std::vector<uint8_t> pend_dense;
    uint64_t pend_rows = 0;
    std::vector<uint8_t> rec;
    const size_t rb = c.n_var * vs;

    uint64_t head = 0;  // first pending row not yet emitted (compacted once per generation batch)
    auto emit = [&](uint64_t rows) {
        if (c.layout == Layout::csr) {
            encode_csr_rows(pend.indptr.data(), pend.indices.data(), pend.data.data(), vs, c.index_dtype, head,
                            head + rows, rec);
            w.append_record(rec.data(), rec.size(), rows);
        } else {
            w.append_record(pend_dense.data() + head * rb, rows * rb, rows);
        }
        head += rows;
        pend_rows -= rows;
    };
    auto compact = [&] {
        if (head == 0) return;
        if (c.layout == Layout::csr) {
            const uint64_t cut = pend.indptr[head];
            pend.indices.erase(pend.indices.begin(), pend.indices.begin() + cut);
            pend.data.erase(pend.data.begin(), pend.data.begin() + cut * vs);
            pend.indptr.erase(pend.indptr.begin(), pend.indptr.begin() + head);
            for (auto& v : pend.indptr) v -= cut;
        } else {
            pend_dense.erase(pend_dense.begin(), pend_dense.begin() + head * rb);
        }
        head = 0;
    };

    for (uint64_t b0 = 0; b0 < n_blocks; b0 += T) {
        const uint64_t nb = std::min<uint64_t>(T, n_blocks - b0);
        std::vector<CsrRows> cs(c.layout == Layout::csr ? nb : 0);
        std::vector<std::vector<uint8_t>> ds(c.layout == Layout::dense ? nb : 0);
        std::vector<std::thread> th;
        for (uint64_t k = 0; k < nb; ++k) {
            th.emplace_back([&, k] {
                const uint64_t bi = b0 + k, start = bi * kSynthBlockRows;
                const uint64_t rows = std::min(kSynthBlockRows, c.n_obs - start);
                if (c.layout == Layout::csr) gen_csr_block(c, start, rows, bi, resid, cs[k]);
                else gen_dense_block(c, start, rows, bi, ds[k]);
            });
        }
        for (auto& t : th) t.join();
        for (uint64_t k = 0; k < nb; ++k) {  // StoreWriter::append (store.cpp:245-277)
            if (c.layout == Layout::csr) {
                const uint64_t base = pend.indptr.back();
                for (size_t r = 1; r < cs[k].indptr.size(); ++r) pend.indptr.push_back(base + cs[k].indptr[r]);
                pend.indices.insert(pend.indices.end(), cs[k].indices.begin(), cs[k].indices.end());
                pend.data.insert(pend.data.end(), cs[k].data.begin(), cs[k].data.end());
                pend_rows += cs[k].indptr.size() - 1;
                cs[k] = CsrRows{};
            } else {
                pend_dense.insert(pend_dense.end(), ds[k].begin(), ds[k].end());
                pend_rows += rb ? ds[k].size() / rb : 0;
                std::vector<uint8_t>().swap(ds[k]);
            }
            while (pend_rows >= c.chunk_rows) emit(c.chunk_rows);
        }
        compact();
    }
    if (pend_rows > 0) emit(pend_rows);
    return w.finish();
}

}  // namespace rfl
