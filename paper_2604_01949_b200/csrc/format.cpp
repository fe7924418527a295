// riffle store format, host side (see format.hpp for the reference map).
#include "format.hpp"
#include "codec.hpp"

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cctype>
#include <cerrno>
#include <cinttypes>
#include <cstdio>
#include <exception>
#include <filesystem>
#include <thread>

namespace rfl {

const char* to_string(Layout l) { return l == Layout::dense ? "dense" : "csr"; }
const char* to_string(VDtype d) {
    switch (d) {
        case VDtype::f32: return "f32";
        case VDtype::f64: return "f64";
        case VDtype::i32: return "i32";
        case VDtype::u8: return "u8";
    }
    return "";
}
const char* to_string(IDtype d) { return d == IDtype::u32 ? "u32" : "u64"; }
const char* to_string(Codec c) { return c == Codec::none ? "none" : "deflate"; }

// ------------------------------------------------------------------ JSON ------
// A small recursive-descent reader for the manifest / provenance meta objects
// and an emitter reproducing nlohmann::ordered_json::dump(2) byte for byte.
namespace {

struct JVal {
    enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
    bool b = false;
    bool is_uint = false;
    uint64_t u = 0;
    std::string s;
    std::vector<JVal> arr;
    std::vector<std::pair<std::string, JVal>> obj;
    const JVal* get(const char* k) const {
        for (auto& kv : obj)
            if (kv.first == k) return &kv.second;
        return nullptr;
    }
};

struct JParser {
    const std::string& t;
    size_t i = 0;
    explicit JParser(const std::string& text) : t(text) {}
    [[noreturn]] void fail(const char* what) {
        corrupt(std::string("manifest: invalid JSON: ") + what + " at offset " + std::to_string(i));
    }
    void ws() {
        while (i < t.size() && (t[i] == ' ' || t[i] == '\n' || t[i] == '\r' || t[i] == '\t')) ++i;
    }
    bool lit(const char* w) {
        const size_t n = std::strlen(w);
        if (t.compare(i, n, w) == 0) {
            i += n;
            return true;
        }
        return false;
    }
    static void put_utf8(std::string& o, uint32_t cp) {
        if (cp < 0x80) {
            o += char(cp);
        } else if (cp < 0x800) {
            o += char(0xC0 | (cp >> 6));
            o += char(0x80 | (cp & 0x3F));
        } else if (cp < 0x10000) {
            o += char(0xE0 | (cp >> 12));
            o += char(0x80 | ((cp >> 6) & 0x3F));
            o += char(0x80 | (cp & 0x3F));
        } else {
            o += char(0xF0 | (cp >> 18));
            o += char(0x80 | ((cp >> 12) & 0x3F));
            o += char(0x80 | ((cp >> 6) & 0x3F));
            o += char(0x80 | (cp & 0x3F));
        }
    }
    uint32_t hex4() {
        if (i + 4 > t.size()) fail("short \\u escape");
        uint32_t v = 0;
        for (int k = 0; k < 4; ++k) {
            const char c = t[i++];
            v <<= 4;
            if (c >= '0' && c <= '9') v |= c - '0';
            else if (c >= 'a' && c <= 'f') v |= c - 'a' + 10;
            else if (c >= 'A' && c <= 'F') v |= c - 'A' + 10;
            else fail("bad \\u escape");
        }
        return v;
    }
    std::string str() {
        if (t[i] != '"') fail("expected string");
        ++i;
        std::string o;
        while (i < t.size() && t[i] != '"') {
            char c = t[i++];
            if (c != '\\') {
                o += c;
                continue;
            }
            if (i >= t.size()) fail("bad escape");
            c = t[i++];
            switch (c) {
                case '"': o += '"'; break;
                case '\\': o += '\\'; break;
                case '/': o += '/'; break;
                case 'b': o += '\b'; break;
                case 'f': o += '\f'; break;
                case 'n': o += '\n'; break;
                case 'r': o += '\r'; break;
                case 't': o += '\t'; break;
                case 'u': {
                    uint32_t cp = hex4();
                    if (cp >= 0xD800 && cp < 0xDC00 && i + 1 < t.size() && t[i] == '\\' && t[i + 1] == 'u') {
                        i += 2;
                        const uint32_t lo = hex4();
                        cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                    }
                    put_utf8(o, cp);
                    break;
                }
                default: fail("bad escape");
            }
        }
        if (i >= t.size()) fail("unterminated string");
        ++i;
        return o;
    }
    JVal value() {
        ws();
        if (i >= t.size()) fail("unexpected end");
        JVal v;
        const char c = t[i];
        if (c == '{') {
            v.kind = JVal::Obj;
            ++i;
            ws();
            if (t[i] == '}') {
                ++i;
                return v;
            }
            for (;;) {
                ws();
                std::string k = str();
                ws();
                if (t[i] != ':') fail("expected ':'");
                ++i;
                JVal x = value();
                v.obj.emplace_back(std::move(k), std::move(x));
                ws();
                if (t[i] == ',') {
                    ++i;
                    continue;
                }
                if (t[i] == '}') {
                    ++i;
                    break;
                }
                fail("expected ',' or '}'");
            }
        } else if (c == '[') {
            v.kind = JVal::Arr;
            ++i;
            ws();
            if (t[i] == ']') {
                ++i;
                return v;
            }
            for (;;) {
                v.arr.push_back(value());
                ws();
                if (t[i] == ',') {
                    ++i;
                    continue;
                }
                if (t[i] == ']') {
                    ++i;
                    break;
                }
                fail("expected ',' or ']'");
            }
        } else if (c == '"') {
            v.kind = JVal::Str;
            v.s = str();
        } else if (lit("true")) {
            v.kind = JVal::Bool;
            v.b = true;
        } else if (lit("false")) {
            v.kind = JVal::Bool;
        } else if (lit("null")) {
        } else if (c == '-' || (c >= '0' && c <= '9')) {
            v.kind = JVal::Num;
            const size_t s = i;
            if (t[i] == '-') ++i;
            while (i < t.size() && (std::isdigit(static_cast<unsigned char>(t[i])) || t[i] == '.' ||
                                    t[i] == 'e' || t[i] == 'E' || t[i] == '+' || t[i] == '-'))
                ++i;
            const std::string num = t.substr(s, i - s);
            v.is_uint = num.find_first_of("-.eE") == std::string::npos;
            if (v.is_uint) v.u = std::stoull(num);
        } else {
            fail("unexpected character");
        }
        return v;
    }
};

uint64_t uint_field(const JVal& j, const char* k) {
    const JVal* v = j.get(k);
    if (!v || v->kind != JVal::Num || !v->is_uint)
        invalid(std::string("manifest: missing or non-integer field '") + k + "'");
    return v->u;
}
std::string str_field(const JVal& j, const char* k) {
    const JVal* v = j.get(k);
    if (!v || v->kind != JVal::Str) invalid(std::string("manifest: missing or non-string field '") + k + "'");
    return v->s;
}
[[noreturn]] void bad_enum(const std::string& s, const char* k) {
    invalid("manifest: bad value '" + s + "' for '" + k + "'");
}

}  // namespace

std::string json_escape(const std::string& s) {
    std::string o;
    o.reserve(s.size() + 2);
    for (const unsigned char c : s) {
        switch (c) {
            case '"': o += "\\\""; break;
            case '\\': o += "\\\\"; break;
            case '\b': o += "\\b"; break;
            case '\f': o += "\\f"; break;
            case '\n': o += "\\n"; break;
            case '\r': o += "\\r"; break;
            case '\t': o += "\\t"; break;
            default:
                if (c < 0x20) {
                    char buf[8];
                    std::snprintf(buf, sizeof buf, "\\u%04x", c);
                    o += buf;
                } else {
                    o += static_cast<char>(c);
                }
        }
    }
    return o;
}

void Manifest::validate() const {
    if (format_version != 1) invalid("manifest: unsupported format_version " + std::to_string(format_version));
    if (chunk_rows < 1) invalid("manifest: chunk_rows must be >= 1");
    if (chunks_per_shard < 1) invalid("manifest: chunks_per_shard must be >= 1");
    if (var_names.size() != n_var)
        invalid("manifest: var_names length " + std::to_string(var_names.size()) + " != n_var " +
                std::to_string(n_var));
    if ((layout == Layout::csr) != index_dtype.has_value())
        invalid(layout == Layout::csr ? "manifest: csr layout requires index_dtype"
                                      : "manifest: index_dtype is only valid for csr layout");
}

std::string Manifest::serialize() const {
    std::string o = "{\n";
    auto kv = [&](const char* k, const std::string& v, bool last = false) {
        o += "  \"";
        o += k;
        o += "\": ";
        o += v;
        o += last ? "\n" : ",\n";
    };
    auto q = [](const char* s) { return std::string("\"") + s + "\""; };
    kv("format_version", std::to_string(format_version));
    kv("layout", q(to_string(layout)));
    kv("n_obs", std::to_string(n_obs));
    kv("n_var", std::to_string(n_var));
    kv("value_dtype", q(to_string(value_dtype)));
    if (index_dtype) kv("index_dtype", q(to_string(*index_dtype)));
    kv("chunk_rows", std::to_string(chunk_rows));
    kv("chunks_per_shard", std::to_string(chunks_per_shard));
    kv("codec", q(to_string(codec)));
    std::string names;
    if (var_names.empty()) {
        names = "[]";
    } else {
        names = "[\n";
        for (size_t i = 0; i < var_names.size(); ++i) {
            names += "    \"" + json_escape(var_names[i]) + "\"";
            names += i + 1 < var_names.size() ? ",\n" : "\n";
        }
        names += "  ]";
    }
    kv("var_names", names);
    kv("has_provenance", has_provenance ? "true" : "false", true);
    o += "}\n";
    return o;
}

Manifest Manifest::parse(const std::string& text) {
    JParser p(text);
    const JVal j = p.value();
    if (j.kind != JVal::Obj) corrupt("manifest: root is not an object");
    Manifest m;
    m.format_version = static_cast<uint32_t>(uint_field(j, "format_version"));
    const std::string lay = str_field(j, "layout");
    if (lay == "dense") m.layout = Layout::dense;
    else if (lay == "csr") m.layout = Layout::csr;
    else bad_enum(lay, "layout");
    m.n_obs = uint_field(j, "n_obs");
    m.n_var = uint_field(j, "n_var");
    const std::string vd = str_field(j, "value_dtype");
    if (vd == "f32") m.value_dtype = VDtype::f32;
    else if (vd == "f64") m.value_dtype = VDtype::f64;
    else if (vd == "i32") m.value_dtype = VDtype::i32;
    else if (vd == "u8") m.value_dtype = VDtype::u8;
    else bad_enum(vd, "value_dtype");
    if (j.get("index_dtype")) {
        const std::string id = str_field(j, "index_dtype");
        if (id == "u32") m.index_dtype = IDtype::u32;
        else if (id == "u64") m.index_dtype = IDtype::u64;
        else bad_enum(id, "index_dtype");
    }
    m.chunk_rows = uint_field(j, "chunk_rows");
    m.chunks_per_shard = uint_field(j, "chunks_per_shard");
    const std::string cd = str_field(j, "codec");
    if (cd == "none") m.codec = Codec::none;
    else if (cd == "deflate") m.codec = Codec::deflate;
    else bad_enum(cd, "codec");
    const JVal* vn = j.get("var_names");
    if (!vn || vn->kind != JVal::Arr) invalid("manifest: missing or non-array field 'var_names'");
    m.var_names.reserve(vn->arr.size());
    for (const auto& v : vn->arr) {
        if (v.kind != JVal::Str) invalid("manifest: var_names entries must be strings");
        m.var_names.push_back(v.s);
    }
    const JVal* hp = j.get("has_provenance");
    if (!hp || hp->kind != JVal::Bool) invalid("manifest: missing or non-boolean field 'has_provenance'");
    m.has_provenance = hp->b;
    m.validate();
    return m;
}

std::string shard_file_name(uint64_t shard_index) {
    char buf[32];
    std::snprintf(buf, sizeof buf, "s%08" PRIu64 ".bin", shard_index);
    return buf;
}

// ------------------------------------------------------------------ files -----
File& File::operator=(File&& o) noexcept {
    if (this != &o) {
        if (fd_ >= 0) ::close(fd_);
        fd_ = o.fd_;
        o.fd_ = -1;
    }
    return *this;
}
File::~File() {
    if (fd_ >= 0) ::close(fd_);
}
File File::open_read(const std::string& p) {
    File f;
    f.fd_ = ::open(p.c_str(), O_RDONLY | O_CLOEXEC);
    if (f.fd_ < 0) ioerr("open '" + p + "': " + std::strerror(errno));
    return f;
}
File File::try_open_direct(const std::string& p) {
    File f;
#ifdef O_DIRECT
    f.fd_ = ::open(p.c_str(), O_RDONLY | O_CLOEXEC | O_DIRECT);
#endif
    return f;
}
File File::create_write(const std::string& p) {
    File f;
    f.fd_ = ::open(p.c_str(), O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
    if (f.fd_ < 0) ioerr("create '" + p + "': " + std::strerror(errno));
    return f;
}
uint64_t File::size() const {
    struct stat st {};
    if (::fstat(fd_, &st) != 0) ioerr(std::string("fstat: ") + std::strerror(errno));
    return static_cast<uint64_t>(st.st_size);
}
void File::pread_exact(uint64_t off, void* dst, uint64_t n) const {
    uint64_t done = 0;
    auto* d = static_cast<uint8_t*>(dst);
    while (done < n) {
        const ssize_t r = ::pread(fd_, d + done, n - done, static_cast<off_t>(off + done));
        if (r < 0) {
            if (errno == EINTR) continue;
            ioerr(std::string("pread: ") + std::strerror(errno));
        }
        if (r == 0) ioerr("pread: unexpected end of file at offset " + std::to_string(off + done));
        done += static_cast<uint64_t>(r);
    }
}
void File::pread_upto(uint64_t off, void* dst, uint64_t n, uint64_t need) const {
    uint64_t done = 0;
    auto* d = static_cast<uint8_t*>(dst);
    while (done < n) {
        const ssize_t r = ::pread(fd_, d + done, n - done, static_cast<off_t>(off + done));
        if (r < 0) {
            if (errno == EINTR) continue;
            ioerr(std::string("pread: ") + std::strerror(errno));
        }
        if (r == 0) {
            if (done >= need) return;
            ioerr("pread: unexpected end of file at offset " + std::to_string(off + done));
        }
        done += static_cast<uint64_t>(r);
    }
}
void File::pwrite_all(uint64_t off, const void* src, uint64_t n) const {
    uint64_t done = 0;
    const auto* s = static_cast<const uint8_t*>(src);
    while (done < n) {
        const ssize_t r = ::pwrite(fd_, s + done, n - done, static_cast<off_t>(off + done));
        if (r < 0) {
            if (errno == EINTR) continue;
            ioerr(std::string("pwrite: ") + std::strerror(errno));
        }
        done += static_cast<uint64_t>(r);
    }
}
void File::write_all(const void* src, uint64_t n) {
    uint64_t done = 0;
    const auto* s = static_cast<const uint8_t*>(src);
    while (done < n) {
        const ssize_t r = ::write(fd_, s + done, n - done);
        if (r < 0) {
            if (errno == EINTR) continue;
            ioerr(std::string("write: ") + std::strerror(errno));
        }
        done += static_cast<uint64_t>(r);
    }
}

std::string read_text_file(const std::string& p) {
    File f = File::open_read(p);
    std::string s(f.size(), '\0');
    if (!s.empty()) f.pread_exact(0, s.data(), s.size());
    return s;
}
void write_text_file(const std::string& p, const std::string& text) {
    File f = File::create_write(p);
    f.write_all(text.data(), text.size());
}
void make_dirs(const std::string& p) {
    std::error_code ec;
    std::filesystem::create_directories(p, ec);
    if (ec) ioerr("cannot create directories at '" + p + "': " + ec.message());
}
bool path_exists(const std::string& p) { return std::filesystem::exists(p); }
bool dir_nonempty(const std::string& p) {
    return std::filesystem::exists(p) && !std::filesystem::is_empty(p);
}

// ------------------------------------------------------------------ shards ----
static const char kMagic[8] = {'S', 'H', 'R', 'D', 'I', 'D', 'X', '1'};

std::vector<Slot> read_footer(const File& f, const std::string& path, uint64_t slots) {
    const uint64_t size = f.size();
    const uint64_t tail = slots * 16 + 8;
    if (size < tail)
        corrupt("shard '" + path + "': truncated (size " + std::to_string(size) + " < footer " +
                std::to_string(tail) + ")");
    std::vector<uint8_t> buf(tail);
    f.pread_exact(size - tail, buf.data(), tail);
    if (std::memcmp(buf.data() + slots * 16, kMagic, 8) != 0) corrupt("shard '" + path + "': bad footer magic");
    const uint64_t payload = size - tail;
    std::vector<Slot> out(slots);
    bool seen_empty = false;
    for (uint64_t i = 0; i < slots; ++i) {
        out[i].off = rd64(buf.data() + i * 16);
        out[i].len = rd64(buf.data() + i * 16 + 8);
        if (out[i].empty()) {
            seen_empty = true;
            continue;
        }
        if (seen_empty)
            corrupt("shard '" + path + "': chunk slot " + std::to_string(i) + " follows an empty slot");
        if (out[i].off > payload || out[i].len > payload || out[i].off + out[i].len > payload)
            corrupt("shard '" + path + "': chunk slot " + std::to_string(i) + " extends past the payload area");
    }
    return out;
}

HostStore::HostStore(std::string root) : root_(std::move(root)) {
    if (root_.compare(0, 11, "procedural:") == 0) {
        src_ = make_record_source(root_, man_);
        const uint64_t nch = man_.chunk_count();
        src_slots_.resize(nch);
        std::vector<uint64_t> len(nch);
        const unsigned T = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < T; ++t)
            pool.emplace_back([&, t] {
                for (uint64_t q = t; q < nch; q += T) len[q] = src_->record_bytes(q);
            });
        for (auto& th : pool) th.join();
        uint64_t off = 0;
        for (uint64_t q = 0; q < nch; ++q) {  // records back to back per shard, as the writer lays them out
            if (q % man_.chunks_per_shard == 0) off = 0;
            src_slots_[q] = {off, len[q]};
            off += len[q];
        }
        return;
    }
    const std::string mp = root_ + "/manifest.json";
    if (!path_exists(mp)) ioerr("store '" + root_ + "': no manifest found (absent or unfinished store)");
    man_ = Manifest::parse(read_text_file(mp));
}

const File& HostStore::fd(uint64_t shard, bool direct) const {
    std::lock_guard<std::mutex> lk(mu_);
    auto& m = direct ? dfds_ : fds_;
    auto it = m.find(shard);
    if (it == m.end()) {
        const std::string p = root_ + "/shards/" + shard_file_name(shard);
        it = m.emplace(shard, direct ? File::try_open_direct(p) : File::open_read(p)).first;
    }
    return it->second;
}

uint64_t HostStore::shard_bytes(uint64_t shard) const {
    if (src_) {
        const uint64_t last = std::min(man_.chunk_count(), (shard + 1) * man_.chunks_per_shard) - 1;
        return src_slots_[last].off + src_slots_[last].len + man_.chunks_per_shard * 16 + 8;
    }
    return fd(shard, false).size();
}
bool HostStore::direct_ok(uint64_t shard) const { return !src_ && fd(shard, true).valid(); }

// procedural store: bytes [off, off + n) of a shard's record area, generated
void HostStore::gen_range(uint64_t shard, uint64_t off, uint8_t* dst, uint64_t n) const {
    const uint64_t q_begin = shard * man_.chunks_per_shard;
    const uint64_t q_end = std::min(man_.chunk_count(), q_begin + man_.chunks_per_shard);
    std::vector<uint8_t> rec;
    for (uint64_t q = q_begin; q < q_end && n; ++q) {
        const Slot s = src_slots_[q];
        if (s.off + s.len <= off) continue;
        if (s.off >= off + n) break;
        src_->record(q, rec);
        const uint64_t a = std::max(off, s.off), b = std::min(off + n, s.off + s.len);
        std::memcpy(dst + (a - off), rec.data() + (a - s.off), b - a);
    }
}

uint64_t HostStore::charge_footer(uint64_t shard) const {
    std::lock_guard<std::mutex> lk(mu_);
    if (footer_charged_.empty()) footer_charged_.assign(man_.shard_count(), 0);
    if (footer_charged_[shard]) return 0;
    footer_charged_[shard] = 1;
    return man_.chunks_per_shard * 16 + 8;  // ShardFooter::footer_bytes + magic
}

Slot HostStore::record_slot(uint64_t chunk) const {
    if (src_) {
        if (chunk >= src_slots_.size()) invalid("chunk " + std::to_string(chunk) + " out of range");
        return src_slots_[chunk];
    }
    const uint64_t shard = chunk / man_.chunks_per_shard;
    const File& f = fd(shard, false);
    std::vector<Slot>* foot;
    {
        std::lock_guard<std::mutex> lk(mu_);
        auto it = footers_.find(shard);
        if (it == footers_.end())
            it = footers_
                     .emplace(shard, read_footer(f, root_ + "/shards/" + shard_file_name(shard),
                                                 man_.chunks_per_shard))
                     .first;
        foot = &it->second;
    }
    const uint64_t slot = chunk % man_.chunks_per_shard;
    const Slot s = (*foot)[slot];
    if (s.empty())
        corrupt("chunk " + std::to_string(chunk) + ": slot " + std::to_string(slot) + " of shard " +
                std::to_string(shard) + " is empty");
    return s;
}

void HostStore::read_record(uint64_t chunk, void* dst, uint64_t cap) const {
    const Slot s = record_slot(chunk);
    if (s.len > cap) invalid("read_record: buffer too small");
    if (src_) {
        std::vector<uint8_t> rec;
        src_->record(chunk, rec);
        std::memcpy(dst, rec.data(), s.len);
        return;
    }
    fd(chunk / man_.chunks_per_shard, false).pread_exact(s.off, dst, s.len);
}

void HostStore::read_shard_bytes(uint64_t shard, uint64_t off, void* dst, uint64_t n, bool direct) const {
    if (src_) return gen_range(shard, off, static_cast<uint8_t*>(dst), n);
    if (direct) {
        const File& d = fd(shard, true);
        // O_DIRECT needs 4 KiB-aligned offset/length/buffer; only used when the
        // caller hands an aligned request (pinned staging is page-aligned).
        if (d.valid() && (off % 4096 == 0) && (n % 4096 == 0) &&
            (reinterpret_cast<uintptr_t>(dst) % 4096 == 0)) {
            d.pread_exact(off, dst, n);
            return;
        }
    }
    fd(shard, false).pread_exact(off, dst, n);
}

uint64_t HostStore::read_shard_span(uint64_t shard, uint64_t off, void* dst, uint64_t n, bool direct) const {
    if (src_) {
        gen_range(shard, off, static_cast<uint8_t*>(dst), n);
        return 0;
    }
    if (direct) {
        const File& d = fd(shard, true);
        if (d.valid()) {
            const uint64_t a0 = off & ~4095ull;
            d.pread_upto(a0, dst, aligned_span(off, n), off + n - a0);
            return off - a0;
        }
    }
    fd(shard, false).pread_exact(off, dst, n);
    return 0;
}

// ------------------------------------------------------------------ writer ----
RecordWriter::RecordWriter(std::string root, Manifest man, bool defer_manifest, const char* shard_dir,
                           bool write_manifest_file)
    : root_(std::move(root)), shard_dir_(shard_dir), man_(std::move(man)),
      write_manifest_file_(write_manifest_file) {
    man_.n_obs = 0;
    man_.validate();
    if (write_manifest_file_ && path_exists(root_ + "/manifest.json"))
        invalid("store '" + root_ + "' already contains a manifest; refusing to clobber");
    make_dirs(root_ + "/" + shard_dir_);
    if (write_manifest_file_ && !defer_manifest) write_text_file(root_ + "/manifest.json", man_.serialize());
}

void RecordWriter::open_shard() {
    const uint64_t idx = chunks_emitted_ / man_.chunks_per_shard;
    shard_.emplace(File::create_write(root_ + "/" + shard_dir_ + "/" + shard_file_name(idx)));
    slots_.assign(man_.chunks_per_shard, Slot{});
    shard_bytes_ = 0;
    chunk_in_shard_ = 0;
}

void RecordWriter::close_shard() {
    std::vector<uint8_t> tail(slots_.size() * 16 + 8);
    for (size_t i = 0; i < slots_.size(); ++i) {
        wr64(tail.data() + i * 16, slots_[i].off);
        wr64(tail.data() + i * 16 + 8, slots_[i].len);
    }
    std::memcpy(tail.data() + slots_.size() * 16, kMagic, 8);
    shard_->pwrite_all(shard_bytes_, tail.data(), tail.size());
    shard_.reset();
}

// Large records (the pre-shuffle's output chunks are tens of MB) go out as
// parallel pwrites of disjoint slices: one writer thread is page-cache-copy bound.
static void write_parallel(const File& f, uint64_t off, const uint8_t* src, uint64_t n) {
    constexpr uint64_t kSlice = 8ull << 20;
    const unsigned T = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
    if (n < 2 * kSlice || T == 1) {
        f.pwrite_all(off, src, n);
        return;
    }
    const uint64_t slices = (n + kSlice - 1) / kSlice;
    std::vector<std::exception_ptr> errs(T);
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < T; ++t)
        pool.emplace_back([&, t] {
            try {
                for (uint64_t k = t; k < slices; k += T) {
                    const uint64_t a = k * kSlice, b = std::min(n, a + kSlice);
                    f.pwrite_all(off + a, src + a, b - a);
                }
            } catch (...) {
                errs[t] = std::current_exception();
            }
        });
    for (auto& th : pool) th.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
}

RecordWriter::Placement RecordWriter::reserve_record(uint64_t nbytes, uint64_t rows, int64_t chunk) {
    if (finished_) invalid("store writer: append after finish");
    if (chunk >= 0) {
        const uint64_t c = static_cast<uint64_t>(chunk);
        const uint64_t shard = c / man_.chunks_per_shard;
        if (shard_ && shard != (chunks_emitted_ - 1) / man_.chunks_per_shard) close_shard();
        if (!shard_) {
            if (c % man_.chunks_per_shard != 0) invalid("store writer: owned shard must be filled from slot 0");
            chunks_emitted_ = c;
            open_shard();
        } else if (c != chunks_emitted_) {
            invalid("store writer: non-consecutive chunk " + std::to_string(c));
        }
    }
    // a full shard is closed lazily, once the records written into it are complete
    if (shard_ && chunk_in_shard_ >= man_.chunks_per_shard) close_shard();
    if (!shard_) open_shard();
    const Placement p{&*shard_, shard_bytes_};
    slots_[chunk_in_shard_] = {shard_bytes_, nbytes};
    shard_bytes_ += nbytes;
    ++chunk_in_shard_;
    ++chunks_emitted_;
    man_.n_obs += rows;
    return p;
}

void RecordWriter::write_part(const Placement& p, uint64_t rel, const void* src, uint64_t n) {
    write_parallel(*p.file, p.off + rel, static_cast<const uint8_t*>(src), n);
}

void RecordWriter::append_record(const void* rec, uint64_t nbytes, uint64_t rows) {
    if (man_.codec != Codec::none) {  // emit_chunk: codec_encode, then the shard append (store.cpp:200-203)
        const std::vector<uint8_t> enc = deflate_encode(static_cast<const uint8_t*>(rec), nbytes);
        write_part(reserve_record(enc.size(), rows), 0, enc.data(), enc.size());
        return;
    }
    write_part(reserve_record(nbytes, rows), 0, rec, nbytes);
}

void RecordWriter::append_record_at(uint64_t chunk, const void* rec, uint64_t nbytes, uint64_t rows) {
    if (man_.codec != Codec::none) {
        const std::vector<uint8_t> enc = deflate_encode(static_cast<const uint8_t*>(rec), nbytes);
        write_part(reserve_record(enc.size(), rows, static_cast<int64_t>(chunk)), 0, enc.data(), enc.size());
        return;
    }
    write_part(reserve_record(nbytes, rows, static_cast<int64_t>(chunk)), 0, rec, nbytes);
}

void RecordWriter::append_encoded(const void* enc, uint64_t nbytes, uint64_t rows, int64_t chunk) {
    write_part(reserve_record(nbytes, rows, chunk), 0, enc, nbytes);
}

Manifest RecordWriter::finish(int64_t n_obs_override) {
    if (finished_) invalid("store writer: finish called twice");
    if (shard_) close_shard();
    if (n_obs_override >= 0) man_.n_obs = static_cast<uint64_t>(n_obs_override);
    if (write_manifest_file_) write_text_file(root_ + "/manifest.json", man_.serialize());
    finished_ = true;
    return man_;
}

}  // namespace rfl
