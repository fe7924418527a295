// Drop-in parity of the C++ host API (include/riffle_b200.hpp) against the
// reference library itself (/root/reference/proj/core, compiled unmodified into
// oracle/_ref/libriffle_ref.so): the same program drives `riffle::` (the CPU
// reference) and `riffle_b200::` (the B200 path) on identical stores and
// configs and requires identical results — the loader's MiniBatch stream,
// plans, validation errors, and the pre-shuffled output store byte for byte.
// Written in the style of the reference's doctest suite (tests/test_store.cpp).
//
// TEST INFRASTRUCTURE: links the reference as the checker.  Built by
// oracle/Makefile (`make -C oracle dropin`) into oracle/_ref/test_dropin.
//   test_dropin            host-only cases (no GPU needed)
//   test_dropin --gpu      + the device cases (BatchIterator, run_shuffle)
#include <riffle/block.hpp>
#include <riffle/collection.hpp>
#include <riffle/error.hpp>
#include <riffle/loader.hpp>
#include <riffle/preshuffle.hpp>
#include <riffle/store.hpp>
#include <riffle/synth.hpp>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <functional>
#include <iterator>
#include <string>
#include <vector>

#include "riffle_b200.hpp"

namespace fs = std::filesystem;
namespace B = riffle_b200;

// ------------------------------------------------------------ mini harness --
static int g_checks = 0, g_failures = 0;
static std::vector<std::pair<std::string, std::function<void()>>>& registry(bool gpu) {
    static std::vector<std::pair<std::string, std::function<void()>>> host, dev;
    return gpu ? dev : host;
}
struct Reg {
    Reg(const char* name, bool gpu, std::function<void()> fn) { registry(gpu).emplace_back(name, std::move(fn)); }
};
#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define TEST_CASE_IMPL(name, gpu, fn)             \
    static void fn();                             \
    static Reg CAT(reg_, fn)(name, gpu, fn);      \
    static void fn()
#define TEST_CASE(name) TEST_CASE_IMPL(name, false, CAT(tc_, __LINE__))
#define GPU_CASE(name) TEST_CASE_IMPL(name, true, CAT(tc_, __LINE__))
#define CHECK(cond)                                                                       \
    do {                                                                                  \
        ++g_checks;                                                                       \
        if (!(cond)) {                                                                    \
            ++g_failures;                                                                 \
            std::fprintf(stderr, "  %s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #cond); \
        }                                                                                 \
    } while (0)

struct TempDir {  // test_support.hpp:15-37
    fs::path path;
    TempDir() {
        char tmpl[] = "/tmp/riffle_dropin_XXXXXX";
        path = ::mkdtemp(tmpl);
    }
    ~TempDir() {
        std::error_code ec;
        fs::remove_all(path, ec);
    }
};

// error type + message of a throwing call, for both libraries
template <typename F>
static std::pair<std::string, std::string> error_of(F&& f) {
    try {
        f();
    } catch (const riffle::InvalidArgument& e) {
        return {"InvalidArgument", e.what()};
    } catch (const riffle::CorruptStore& e) {
        return {"CorruptStore", e.what()};
    } catch (const riffle::IoError& e) {
        return {"IoError", e.what()};
    } catch (const B::InvalidArgument& e) {
        return {"InvalidArgument", e.what()};
    } catch (const B::CorruptStore& e) {
        return {"CorruptStore", e.what()};
    } catch (const B::IoError& e) {
        return {"IoError", e.what()};
    } catch (const std::exception& e) {
        return {"other", e.what()};
    }
    return {"none", ""};
}

static riffle::SynthConfig synth_cfg(std::uint64_t n, std::uint64_t nv, riffle::Layout l, riffle::ValueDtype vd,
                                     riffle::IndexDtype id, double dens, std::uint64_t seed, std::uint64_t cr,
                                     std::uint64_t cps) {
    riffle::SynthConfig c;
    c.n_obs = n;
    c.n_var = nv;
    c.layout = l;
    c.value_dtype = vd;
    c.index_dtype = id;
    c.density = dens;
    c.seed = seed;
    c.chunk_rows = cr;
    c.chunks_per_shard = cps;
    return c;
}

static riffle::LoaderConfig ref_cfg(const B::LoaderConfig& c) {
    riffle::LoaderConfig r;
    r.fetch_block_rows = c.fetch_block_rows;
    r.buffer_capacity_rows = c.buffer_capacity_rows;
    r.batch_rows = c.batch_rows;
    r.seed = c.seed;
    r.prefetch_depth = c.prefetch_depth;
    r.drop_last = c.drop_last;
    r.cache_bypass = c.cache_bypass;
    return r;
}

// ------------------------------------------------------------- host cases --
TEST_CASE("plan_epoch matches the reference block permutation") {
    for (std::uint64_t n : {1ull, 10ull, 999ull, 100000ull})
        for (std::uint64_t f : {1ull, 4ull, 64ull, 1000ull})
            for (std::uint64_t e : {0ull, 1ull, 7ull}) {
                B::LoaderConfig c;
                c.fetch_block_rows = f;
                c.buffer_capacity_rows = std::max<std::uint64_t>(f, 16);
                c.batch_rows = 16;
                c.seed = 42 + e;
                const auto ours = B::plan_epoch(n, c, e);
                const auto ref = riffle::plan_epoch(n, ref_cfg(c), e);
                CHECK(ours.blocks.size() == ref.blocks.size());
                bool same = ours.epoch_index == ref.epoch_index;
                for (std::size_t i = 0; same && i < ref.blocks.size(); ++i)
                    same = ours.blocks[i].start == ref.blocks[i].start && ours.blocks[i].end == ref.blocks[i].end;
                CHECK(same);
            }
}

TEST_CASE("LoaderConfig::validate and plan_epoch errors match the reference") {
    std::vector<B::LoaderConfig> bad(5);
    bad[0].fetch_block_rows = 0;
    bad[1].buffer_capacity_rows = 10, bad[1].fetch_block_rows = 20;
    bad[2].batch_rows = 0;
    bad[3].batch_rows = 20000;
    bad[4].buffer_capacity_rows = 0;
    for (const auto& c : bad) {
        const auto ours = error_of([&] { c.validate(); });
        const auto ref = error_of([&] { ref_cfg(c).validate(); });
        CHECK(ours == ref);
        CHECK(ours.first == "InvalidArgument");
    }
    const auto ours = error_of([&] { (void)B::plan_epoch(0, bad[0], 0); });
    const auto ref = error_of([&] { (void)riffle::plan_epoch(0, ref_cfg(bad[0]), 0); });
    CHECK(ours == ref);
}

TEST_CASE("plan_shuffle matches the reference (rounds, ids, errors)") {
    for (auto [n, c, m, s] : std::vector<std::array<std::uint64_t, 4>>{
             {100, 10, 30, 0}, {1, 1, 1, 5}, {12345, 64, 1024, 7}, {1000, 7, 50, 3}, {50, 10, 1000, 1}}) {
        const auto ours = B::plan_shuffle(n, c, m, s);
        const auto ref = riffle::plan_shuffle(n, c, m, s);
        CHECK(ours.rounds == ref.rounds);
        CHECK(ours.block_count() == ref.block_count());
    }
    for (auto [n, c, m] : std::vector<std::array<std::uint64_t, 3>>{{100, 0, 10}, {100, 20, 10}}) {
        const auto ours = error_of([&] { (void)B::plan_shuffle(n, c, m, 0); });
        const auto ref = error_of([&] { (void)riffle::plan_shuffle(n, c, m, 0); });
        CHECK(ours == ref);
    }
}

TEST_CASE("StoreReader manifest and raw records match; missing store errors alike") {
    TempDir t;
    riffle::synth_store(t.path / "s", synth_cfg(500, 40, riffle::Layout::csr, riffle::ValueDtype::f32,
                                                riffle::IndexDtype::u64, 0.2, 3, 64, 4));
    const B::StoreReader ours(t.path / "s");
    const riffle::StoreReader ref(t.path / "s");
    CHECK(ours.manifest().n_obs == ref.manifest().n_obs);
    CHECK(ours.manifest().n_var == ref.manifest().n_var);
    CHECK(ours.manifest().chunk_rows == ref.manifest().chunk_rows);
    CHECK(static_cast<int>(ours.manifest().layout) == static_cast<int>(ref.manifest().layout));
    CHECK(static_cast<int>(*ours.manifest().index_dtype) == static_cast<int>(*ref.manifest().index_dtype));
    // a raw record decodes to the reference's rows: header rows == chunk rows
    const auto rec = ours.read_record(1);
    std::uint32_t rows = 0;
    std::memcpy(&rows, rec.data(), 4);
    CHECK(rows == 64);
    const auto e1 = error_of([&] { B::StoreReader x(t.path / "nope"); });
    const auto e2 = error_of([&] { riffle::StoreReader x(t.path / "nope"); });
    CHECK(e1.first == e2.first);
}

// ----------------------------------------------------------- device cases --
static bool same_batch(const B::MiniBatch& o, const riffle::MiniBatch& r) {
    if (o.global_indices != r.global_indices || o.epoch_index != r.epoch_index || o.batch_index != r.batch_index)
        return false;
    if (std::holds_alternative<riffle::CsrBlock>(r.block)) {
        const auto& rb = std::get<riffle::CsrBlock>(r.block);
        if (!std::holds_alternative<B::CsrBlock>(o.block)) return false;
        const auto& ob = std::get<B::CsrBlock>(o.block);
        return ob.n_rows == rb.n_rows && ob.n_var == rb.n_var && ob.indptr == rb.indptr && ob.indices == rb.indices &&
               ob.data == rb.data;
    }
    const auto& rb = std::get<riffle::DenseBlock>(r.block);
    if (!std::holds_alternative<B::DenseBlock>(o.block)) return false;
    const auto& ob = std::get<B::DenseBlock>(o.block);
    return ob.n_rows == rb.n_rows && ob.n_var == rb.n_var && ob.values == rb.values;
}

GPU_CASE("BatchIterator: the MiniBatch stream equals the reference's (csr + dense stores, all stagings)") {
    TempDir t;
    riffle::synth_store(t.path / "csr", synth_cfg(3000, 300, riffle::Layout::csr, riffle::ValueDtype::f32,
                                                  riffle::IndexDtype::u32, 0.05, 1, 64, 8));
    riffle::synth_store(t.path / "dense", synth_cfg(2000, 96, riffle::Layout::dense, riffle::ValueDtype::u8,
                                                    riffle::IndexDtype::u32, 0.0, 2, 100, 4));
    struct Case {
        const char* store;
        std::uint64_t f, B_, b, seed, epoch;
        bool drop_last;
    };
    const Case cases[] = {{"csr", 64, 4096, 4096, 0, 0, false}, {"csr", 50, 700, 256, 3, 1, false},
                          {"csr", 1, 32, 32, 9, 2, true},       {"dense", 100, 1000, 300, 1, 0, false},
                          {"dense", 37, 400, 128, 5, 3, true}};
    for (const Case& k : cases) {
        auto ref_store = std::make_shared<const riffle::StoreReader>(t.path / k.store);
        auto our_store = std::make_shared<const B::StoreReader>(t.path / k.store);
        for (B::Staging st : {B::Staging::resident, B::Staging::stream_pinned, B::Staging::stream_file}) {
            B::LoaderConfig c;
            c.fetch_block_rows = k.f;
            c.buffer_capacity_rows = k.B_;
            c.batch_rows = k.b;
            c.seed = k.seed;
            c.drop_last = k.drop_last;
            c.prefetch_depth = st == B::Staging::stream_file ? 4 : 0;
            B::DeviceOptions opt;
            opt.staging = st;
            B::BatchIterator ours = B::open_epoch(our_store, c, k.epoch, opt);
            riffle::BatchIterator ref = riffle::open_epoch(ref_store, ref_cfg(c), k.epoch);
            std::size_t n = 0;
            bool same = true;
            for (;;) {
                auto a = ours.next();
                auto r = ref.next();
                if (!a || !r) {
                    same = same && !a && !r;
                    break;
                }
                same = same && same_batch(*a, *r);
                ++n;
            }
            CHECK(same);
            CHECK(n > 0);
            CHECK(!ours.next());  // idempotent end of epoch (loader.cpp:259)
            CHECK(ours.counters().blocks_fetched == ref.counters().blocks_fetched);
            CHECK(ours.peak_buffer_rows() == ref.peak_buffer_rows());
            // the reference's IoStats in every staging mode (both store handles are shared
            // across the stagings, so footer loads are charged to the first iterator in both)
            CHECK(ours.counters().io.read_ops == ref.counters().io.read_ops);
            CHECK(ours.counters().io.chunks_decoded == ref.counters().io.chunks_decoded);
            CHECK(ours.counters().io.bytes_read == ref.counters().io.bytes_read);
        }
    }
}

GPU_CASE("densified batches equal riffle::to_dense of the reference's batches") {
    TempDir t;
    riffle::synth_store(t.path / "s", synth_cfg(2500, 500, riffle::Layout::csr, riffle::ValueDtype::f32,
                                                riffle::IndexDtype::u64, 0.1, 4, 128, 4));
    B::LoaderConfig c;
    c.fetch_block_rows = 128;
    c.buffer_capacity_rows = 1024;
    c.batch_rows = 512;
    c.seed = 11;
    B::DeviceOptions opt;
    opt.output = B::Output::dense;
    B::BatchIterator ours(std::make_shared<const B::StoreReader>(t.path / "s"), c, 0, opt);
    riffle::BatchIterator ref(std::make_shared<const riffle::StoreReader>(t.path / "s"), ref_cfg(c), 0);
    bool same = true;
    std::size_t n = 0;
    while (auto r = ref.next()) {
        auto a = ours.next();
        if (!a) {
            same = false;
            break;
        }
        const riffle::DenseBlock d = riffle::to_dense(std::get<riffle::CsrBlock>(r->block));
        const auto& ob = std::get<B::DenseBlock>(a->block);
        same = same && a->global_indices == r->global_indices && ob.values == d.values && ob.n_var == d.n_var;
        ++n;
    }
    CHECK(same);
    CHECK(n == 5);
    CHECK(!ours.next());
}

static std::vector<std::pair<std::string, std::string>> tree(const fs::path& root) {
    std::vector<std::pair<std::string, std::string>> out;
    for (const auto& e : fs::recursive_directory_iterator(root)) {
        if (!e.is_regular_file()) continue;
        std::ifstream in(e.path(), std::ios::binary);
        out.emplace_back(fs::relative(e.path(), root).string(),
                         std::string(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>()));
    }
    std::sort(out.begin(), out.end());
    return out;
}

GPU_CASE("run_shuffle writes the reference's output store byte for byte (inner/outer joins)") {
    TempDir t;
    riffle::synth_store(t.path / "a", synth_cfg(900, 60, riffle::Layout::csr, riffle::ValueDtype::f32,
                                                riffle::IndexDtype::u32, 0.1, 1, 32, 4));
    riffle::synth_store(t.path / "b", synth_cfg(400, 60, riffle::Layout::csr, riffle::ValueDtype::f32,
                                                riffle::IndexDtype::u32, 0.2, 2, 50, 2));
    for (bool outer : {true, false}) {
        const std::string tag = outer ? "outer" : "inner";
        riffle::DatasetCollection rc(outer ? riffle::JoinMode::outer : riffle::JoinMode::inner);
        rc.add(std::make_shared<const riffle::StoreReader>(t.path / "a"));
        rc.add(std::make_shared<const riffle::StoreReader>(t.path / "b"));
        B::DatasetCollection oc(outer ? B::JoinMode::outer : B::JoinMode::inner);
        oc.add(std::make_shared<const B::StoreReader>(t.path / "a"));
        oc.add(std::make_shared<const B::StoreReader>(t.path / "b"));
        riffle::ShuffleOutputConfig roc;
        roc.chunk_rows = 100;
        roc.chunks_per_shard = 3;
        B::ShuffleOutputConfig ooc;
        ooc.chunk_rows = 100;
        ooc.chunks_per_shard = 3;
        riffle::ShuffleRunStats rs;
        B::ShuffleRunStats os;
        riffle::run_shuffle(rc, riffle::plan_shuffle(1300, 24, 256, 9), t.path / ("ref_" + tag), roc, &rs);
        const auto man = B::run_shuffle(oc, B::plan_shuffle(1300, 24, 256, 9), t.path / ("gpu_" + tag), ooc, &os);
        CHECK(tree(t.path / ("ref_" + tag)) == tree(t.path / ("gpu_" + tag)));
        CHECK(man.n_obs == 1300);
        CHECK(os.rows_written == rs.rows_written && os.rounds_executed == rs.rounds_executed);
        CHECK(os.peak_resident_rows == rs.peak_resident_rows);
    }
    const auto e1 = error_of([&] {
        B::DatasetCollection oc(B::JoinMode::outer);
        (void)B::run_shuffle(oc, B::plan_shuffle(10, 1, 1, 0), t.path / "x", {});
    });
    const auto e2 = error_of([&] {
        riffle::DatasetCollection rc(riffle::JoinMode::outer);
        (void)riffle::run_shuffle(rc, riffle::plan_shuffle(10, 1, 1, 0), t.path / "y", {});
    });
    CHECK(e1 == e2);
}

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && std::strcmp(argv[1], "--gpu") == 0;
    int cases = 0;
    for (bool dev : {false, true}) {
        if (dev && !gpu) break;
        for (auto& [name, fn] : registry(dev)) {
            const int before = g_failures;
            try {
                fn();
            } catch (const std::exception& e) {
                ++g_failures;
                std::fprintf(stderr, "  unexpected exception: %s\n", e.what());
            }
            std::printf("[%s] %s\n", g_failures == before ? "pass" : "FAIL", name.c_str());
            ++cases;
        }
    }
    std::printf("%d test cases, %d checks, %d failures\n", cases, g_checks, g_failures);
    return g_failures == 0 ? 0 : 1;
}
