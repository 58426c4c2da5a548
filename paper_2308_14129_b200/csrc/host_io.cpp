// On-disk formats of the hot path's inputs:
//
//  * edge CSV "src,dst,ts" with the reference's exact acceptance rules and
//    error texts (graph_io.hpp load_edges / write_edges, graph_io.cpp:19-154);
//  * a binary event file: a 32-byte header and the spd_edge records verbatim
//    (the TemporalEdge layout, types.hpp:15-20), read with large fread calls
//    straight into the caller's array — the practical format at GDELT scale
//    (191M edges: 3.06 GB binary vs ~4.5 GB of CSV parsed row by row);
//  * the partition assignment JSON that the reference CLI writes and reads
//    between `partition` and the trainer (speedpart_main.cpp:110-119 writer,
//    :129-166 reader): {"config", "edge_part", "node_parts", "shared",
//    "discards"}, compact (nlohmann dump() without indent), node_parts keyed
//    by decimal node id.
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <memory>
#include <string>
#include <string_view>
#include <vector>

#include "capi_types.hpp"
#include "host.hpp"

using namespace spd;

namespace {

// ------------------------------------------------------------------- CSV
constexpr std::string_view kWs = " \t\r";

std::string_view trim(std::string_view v) {
    const auto b = v.find_first_not_of(kWs);
    if (b == std::string_view::npos) return {};
    return v.substr(b, v.find_last_not_of(kWs) - b + 1);
}

// the first `want` comma-separated fields of a row (later columns ignored);
// returns how many fields the row has, capped at want
int fields(std::string_view row, std::string_view* out, int want) {
    int n = 0;
    std::size_t pos = 0;
    while (n < want) {
        const std::size_t c = row.find(',', pos);
        out[n++] = row.substr(pos, c == std::string_view::npos ? std::string_view::npos : c - pos);
        if (c == std::string_view::npos) break;
        pos = c + 1;
    }
    return n;
}

std::string row_tag(std::uint64_t row) { return "row " + std::to_string(row) + ": "; }

// Node id: decimal digits only, below the NodeId sentinel (graph_io.cpp parse_node).
NodeId node_field(std::string_view raw, std::uint64_t row) {
    const std::string_view t = trim(raw);
    const auto bad = [&] {
        data_error("ParseError", row_tag(row) + "bad node id '" + std::string(raw) + "'");
    };
    if (t.empty()) bad();
    unsigned long long v = 0;
    for (char ch : t) {
        if (ch < '0' || ch > '9') bad();
        const unsigned d = static_cast<unsigned>(ch - '0');
        if (v > (std::numeric_limits<unsigned long long>::max() - d) / 10) bad();  // stoull range
        v = v * 10 + d;
    }
    if (v > std::numeric_limits<NodeId>::max() - 1)
        data_error("ParseError", row_tag(row) + "node id out of range");
    return static_cast<NodeId>(v);
}

// Timestamp: the whole trimmed field must convert (std::stod, so the accepted
// spellings are libstdc++'s), finite and non-negative.
double ts_field(std::string_view raw, std::uint64_t row) {
    const std::string t(trim(raw));
    std::size_t used = 0;
    double v = 0.0;
    bool ok = true;
    try {
        v = std::stod(t, &used);
    } catch (const std::exception&) {
        ok = false;
    }
    if (!ok || used != t.size() || !std::isfinite(v) || v < 0.0)
        data_error("ParseError", row_tag(row) + "bad timestamp '" + std::string(raw) + "'");
    return v;
}

struct Loaded {
    std::vector<spd_edge> e;
    NodeId node_count = 0;
    double t_max = 0.0;
};

void finish(Loaded& L, bool assume_sorted) {
    if (!assume_sorted)
        std::stable_sort(L.e.begin(), L.e.end(),
                         [](const spd_edge& a, const spd_edge& b) { return a.ts < b.ts; });
    NodeId hi = 0;
    double tm = 0.0;
    for (const spd_edge& x : L.e) {
        hi = std::max(hi, std::max(x.src, x.dst));
        tm = std::max(tm, x.ts);
    }
    L.node_count = L.e.empty() ? 0 : hi + 1;
    L.t_max = L.e.empty() ? 0.0 : tm;
}

Loaded load_csv(const char* path, bool assume_sorted) {
    std::ifstream in(path);
    if (!in) data_error("FileNotFound", std::string("cannot open '") + path + "'");
    Loaded L;
    std::string line;
    if (!std::getline(in, line)) data_error("ParseError", "empty input: expected header src,dst,ts");
    std::string_view h[3];
    if (fields(line, h, 3) < 3 || trim(h[0]) != "src" || trim(h[1]) != "dst" || trim(h[2]) != "ts")
        data_error("ParseError", "expected header src,dst,ts");
    std::uint64_t row = 0;
    while (std::getline(in, line)) {
        if (trim(line).empty()) continue;  // blank rows are not counted
        ++row;
        std::string_view f[3];
        if (fields(line, f, 3) < 3) data_error("ParseError", row_tag(row) + "expected 3 fields");
        spd_edge x;
        x.src = node_field(f[0], row);
        x.dst = node_field(f[1], row);
        x.ts = ts_field(f[2], row);
        L.e.push_back(x);
    }
    finish(L, assume_sorted);
    return L;
}

// ---------------------------------------------------------------- binary
constexpr char kMagic[8] = {'S', 'P', 'D', 'E', 'D', 'G', 'E', '1'};
struct BinHeader {
    char magic[8];
    std::uint64_t n;
    std::uint32_t node_count;
    std::uint32_t flags;  // 0
    double t_max;
};
static_assert(sizeof(BinHeader) == 32 && sizeof(spd_edge) == 16, "on-disk layout");

struct File {
    std::FILE* f = nullptr;
    ~File() {
        if (f) std::fclose(f);
    }
};

// ------------------------------------------------------------------ JSON
// Minimal reader for the assignment document: objects, arrays, numbers,
// strings, literals. Values the caller does not need are skipped; the config
// object is returned as its raw text.
struct Json {
    std::string_view s;
    std::size_t i = 0;

    [[noreturn]] void fail(const std::string& what) const {
        data_error("ParseError", "assignment: " + what + " at byte " + std::to_string(i));
    }
    void ws() {
        while (i < s.size() && (s[i] == ' ' || s[i] == '\t' || s[i] == '\n' || s[i] == '\r')) ++i;
    }
    char peek() {
        ws();
        if (i >= s.size()) fail("unexpected end of input");
        return s[i];
    }
    void expect(char c) {
        if (peek() != c) fail(std::string("expected '") + c + "'");
        ++i;
    }
    std::string str() {
        expect('"');
        std::string out;
        while (true) {
            if (i >= s.size()) fail("unterminated string");
            const char c = s[i++];
            if (c == '"') return out;
            if (c == '\\') {
                if (i >= s.size()) fail("bad escape");
                const char e = s[i++];
                switch (e) {
                    case 'n': out += '\n'; break;
                    case 't': out += '\t'; break;
                    case 'r': out += '\r'; break;
                    case 'b': out += '\b'; break;
                    case 'f': out += '\f'; break;
                    case 'u':
                        if (i + 4 > s.size()) fail("bad escape");
                        out += '?';  // keys/values we read are ASCII; keep position
                        i += 4;
                        break;
                    default: out += e;
                }
            } else {
                out += c;
            }
        }
    }
    double num() {
        ws();
        const std::size_t b = i;
        while (i < s.size() && std::strchr("+-0123456789.eE", s[i])) ++i;
        if (b == i) fail("expected a number");
        const std::string t(s.substr(b, i - b));
        char* end = nullptr;
        const double v = std::strtod(t.c_str(), &end);
        if (end != t.c_str() + t.size()) fail("bad number");
        return v;
    }
    std::int64_t integer() {
        const double v = num();
        if (v != std::floor(v) || std::fabs(v) > 9.007199254740992e15) fail("expected an integer");
        return static_cast<std::int64_t>(v);
    }
    void skip() {
        const char c = peek();
        if (c == '{') {
            ++i;
            if (peek() == '}') { ++i; return; }
            while (true) {
                str();
                expect(':');
                skip();
                if (peek() == ',') { ++i; continue; }
                expect('}');
                return;
            }
        } else if (c == '[') {
            ++i;
            if (peek() == ']') { ++i; return; }
            while (true) {
                skip();
                if (peek() == ',') { ++i; continue; }
                expect(']');
                return;
            }
        } else if (c == '"') {
            str();
        } else if (s.compare(i, 4, "true") == 0 || s.compare(i, 4, "null") == 0) {
            i += 4;
        } else if (s.compare(i, 5, "false") == 0) {
            i += 5;
        } else {
            num();
        }
    }
    template <class T>
    std::vector<T> int_array() {
        std::vector<T> out;
        expect('[');
        if (peek() == ']') { ++i; return out; }
        while (true) {
            out.push_back(static_cast<T>(integer()));
            if (peek() == ',') { ++i; continue; }
            expect(']');
            return out;
        }
    }
    // visit each member of an object: f(key) must consume the value
    template <class F>
    void object(F&& f) {
        expect('{');
        if (peek() == '}') { ++i; return; }
        while (true) {
            const std::string k = str();
            expect(':');
            f(k);
            if (peek() == ',') { ++i; continue; }
            expect('}');
            return;
        }
    }
};

std::string read_file(const char* path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) data_error("FileNotFound", std::string("cannot open assignment ") + path);
    return std::string(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
}

template <class T>
void put_ints(std::string& o, const T* v, std::size_t n) {
    o += '[';
    char buf[24];
    for (std::size_t k = 0; k < n; ++k) {
        if (k) o += ',';
        const int len = std::snprintf(buf, sizeof buf, "%lld", static_cast<long long>(v[k]));
        o.append(buf, len);
    }
    o += ']';
}

spd_edge* export_edges(const std::vector<spd_edge>& e) {
    auto* p = static_cast<spd_edge*>(std::malloc(sizeof(spd_edge) * (e.empty() ? 1 : e.size())));
    if (!p) throw std::bad_alloc();
    if (!e.empty()) std::memcpy(p, e.data(), sizeof(spd_edge) * e.size());
    return p;
}

}  // namespace

extern "C" {

void spd_free(void* p) { std::free(p); }

spd_status spd_load_edges_csv(const char* path, int32_t assume_sorted, spd_edge** out, uint64_t* n,
                              uint32_t* node_count, double* t_max) {
    GUARD({
        if (!path || !out || !n) usage_error("null argument");
        Loaded L = load_csv(path, assume_sorted != 0);
        *out = export_edges(L.e);
        *n = L.e.size();
        if (node_count) *node_count = L.node_count;
        if (t_max) *t_max = L.t_max;
    });
}

spd_status spd_write_edges_csv(const char* path, const spd_edge* e, uint64_t n) {
    GUARD({
        if (!path || (n && !e)) usage_error("null argument");
        File f{std::fopen(path, "wb")};
        if (!f.f) data_error("FileNotFound", std::string("cannot open '") + path + "' for writing");
        std::string buf = "src,dst,ts\n";
        char row[96];
        for (std::uint64_t k = 0; k < n; ++k) {
            // %.17g: every double round-trips through the reader
            const int len = std::snprintf(row, sizeof row, "%u,%u,%.17g\n", e[k].src, e[k].dst, e[k].ts);
            buf.append(row, len);
            if (buf.size() > (1u << 22)) {
                if (std::fwrite(buf.data(), 1, buf.size(), f.f) != buf.size())
                    data_error("FileNotFound", "short write");
                buf.clear();
            }
        }
        if (std::fwrite(buf.data(), 1, buf.size(), f.f) != buf.size())
            data_error("FileNotFound", "short write");
    });
}

spd_status spd_write_edges_bin(const char* path, const spd_edge* e, uint64_t n, uint32_t node_count,
                               double t_max) {
    GUARD({
        if (!path || (n && !e)) usage_error("null argument");
        // the reader's acceptance rules, checked before anything is written, so
        // every file this writes reads back (ids < node_count, finite ts >= 0,
        // time-ordered)
        double prev = 0.0;
        for (std::uint64_t q = 0; q < n; ++q) {
            if (e[q].src >= node_count || e[q].dst >= node_count)
                data_error("InvalidParams", "edge " + std::to_string(q) + ": node id out of range");
            if (!std::isfinite(e[q].ts) || e[q].ts < 0.0)
                data_error("ParseError", "edge " + std::to_string(q) + ": timestamp is negative or not finite");
            if (e[q].ts < prev)
                data_error("UnsortedStream", "edge " + std::to_string(q) + ": timestamp decreases");
            prev = e[q].ts;
        }
        File f{std::fopen(path, "wb")};
        if (!f.f) data_error("FileNotFound", std::string("cannot open '") + path + "' for writing");
        BinHeader h{};
        std::memcpy(h.magic, kMagic, 8);
        h.n = n;
        h.node_count = node_count;
        h.t_max = t_max;
        if (std::fwrite(&h, sizeof h, 1, f.f) != 1 ||
            (n && std::fwrite(e, sizeof(spd_edge), n, f.f) != n))
            data_error("FileNotFound", "short write");
    });
}

spd_status spd_edges_bin_info(const char* path, uint64_t* n, uint32_t* node_count, double* t_max) {
    GUARD({
        if (!path || !n) usage_error("null argument");
        File f{std::fopen(path, "rb")};
        if (!f.f) data_error("FileNotFound", std::string("cannot open '") + path + "'");
        BinHeader h{};
        if (std::fread(&h, sizeof h, 1, f.f) != 1 || std::memcmp(h.magic, kMagic, 8) != 0)
            data_error("ParseError", "not a binary edge file (bad header)");
        *n = h.n;
        if (node_count) *node_count = h.node_count;
        if (t_max) *t_max = h.t_max;
    });
}

// Reads into caller memory of spd_edges_bin_info's n records (zero-copy into
// e.g. pinned host buffers); validates ids against node_count and time order.
spd_status spd_load_edges_bin(const char* path, spd_edge* out, uint64_t cap) {
    GUARD({
        if (!path) usage_error("null argument");
        File f{std::fopen(path, "rb")};
        if (!f.f) data_error("FileNotFound", std::string("cannot open '") + path + "'");
        BinHeader h{};
        if (std::fread(&h, sizeof h, 1, f.f) != 1 || std::memcmp(h.magic, kMagic, 8) != 0)
            data_error("ParseError", "not a binary edge file (bad header)");
        if (h.n > cap) usage_error("output buffer smaller than the file's edge count");
        if (h.n && !out) usage_error("null argument");
        constexpr std::uint64_t kChunk = 1u << 20;
        double prev = -std::numeric_limits<double>::infinity();
        for (std::uint64_t k = 0; k < h.n; k += kChunk) {
            const std::uint64_t m = std::min(kChunk, h.n - k);
            if (std::fread(out + k, sizeof(spd_edge), m, f.f) != m)
                data_error("ParseError", "binary edge file truncated");
            for (std::uint64_t q = k; q < k + m; ++q) {
                if (out[q].src >= h.node_count || out[q].dst >= h.node_count)
                    data_error("ParseError", "edge " + std::to_string(q) + ": node id out of range");
                if (!std::isfinite(out[q].ts) || out[q].ts < 0.0)  // parse_ts's rule (graph_io.cpp)
                    data_error("ParseError", "edge " + std::to_string(q) + ": timestamp is negative or not finite");
                if (!(out[q].ts >= prev))
                    data_error("UnsortedStream", "edge " + std::to_string(q) + ": timestamp decreases");
                prev = out[q].ts;
            }
        }
        if (std::fgetc(f.f) != EOF) data_error("ParseError", "trailing bytes after the edge records");
    });
}

spd_status spd_assignment_write_json(const spd_assignment* a, const char* config_json,
                                     const char* path) {
    GUARD({
        if (!a || !path) usage_error("null argument");
        const Assignment& x = a->a;
        std::string o;
        o.reserve(x.edge_part.size() * 3 + x.np_parts.size() * 8 + 256);
        o += "{\"config\":";
        o += config_json && *config_json ? config_json : "{}";
        o += ",\"edge_part\":";
        put_ints(o, x.edge_part.data(), x.edge_part.size());
        o += ",\"node_parts\":{";
        for (NodeId i = 0; i < x.node_count; ++i) {
            if (i) o += ',';
            o += '"';
            o += std::to_string(i);
            o += "\":";
            put_ints(o, x.np_parts.data() + x.np_off[i], x.np_off[i + 1] - x.np_off[i]);
        }
        o += "},\"shared\":";
        put_ints(o, x.shared.data(), x.shared.size());
        o += ",\"discards\":";
        o += std::to_string(x.discards);
        o += "}\n";
        File f{std::fopen(path, "wb")};
        if (!f.f) data_error("FileNotFound", std::string("cannot open '") + path + "' for writing");
        if (std::fwrite(o.data(), 1, o.size(), f.f) != o.size()) data_error("FileNotFound", "short write");
    });
}

// Reader of the same document (speedpart_main.cpp:129-166 load_assignment):
// missing keys are ParseError "assignment is missing '<key>'"; num_parts and
// k_eff come from config.parts / config.topk. config_out (optional) receives
// the raw config object text, malloc'ed (spd_free).
spd_status spd_assignment_read_json(const char* path, spd_assignment** out, char** config_out) {
    GUARD({
        if (!path || !out) usage_error("null argument");
        const std::string text = read_file(path);
        Json j{text};
        auto res = std::make_unique<spd_assignment>();
        Assignment& x = res->a;
        bool has_cfg = false, has_ep = false, has_np = false, has_sh = false, has_dc = false;
        bool has_parts = false, has_topk = false;
        std::string cfg_text;
        std::vector<std::vector<PartId>> np;
        j.object([&](const std::string& key) {
            if (key == "config") {
                has_cfg = true;
                const std::size_t b = (j.ws(), j.i);
                if (j.peek() != '{') j.fail("config is not an object");
                j.object([&](const std::string& ck) {
                    if (ck == "parts") {
                        x.num_parts = static_cast<int>(j.integer());
                        has_parts = true;
                    } else if (ck == "topk") {
                        x.k_eff = j.num();
                        has_topk = true;
                    } else {
                        j.skip();
                    }
                });
                cfg_text.assign(text, b, j.i - b);
            } else if (key == "edge_part") {
                has_ep = true;
                x.edge_part = j.int_array<PartId>();
            } else if (key == "node_parts") {
                has_np = true;
                j.object([&](const std::string& nk) {
                    char* end = nullptr;
                    errno = 0;
                    const unsigned long id = std::strtoul(nk.c_str(), &end, 10);
                    if (nk.empty() || *end || errno || id >= std::numeric_limits<NodeId>::max())
                        data_error("ParseError", "node_parts key '" + nk + "' is not a node id");
                    if (id >= np.size()) np.resize(id + 1);
                    np[id] = j.int_array<PartId>();
                });
            } else if (key == "shared") {
                has_sh = true;
                x.shared = j.int_array<NodeId>();
            } else if (key == "discards") {
                has_dc = true;
                x.discards = static_cast<std::uint64_t>(j.integer());
            } else {
                j.skip();
            }
        });
        j.ws();
        if (j.i != text.size()) j.fail("trailing content");
        const auto need = [](bool have, const char* what, const char* k) {
            if (!have) data_error("ParseError", std::string(what) + " is missing '" + k + "'");
        };
        need(has_cfg, "assignment", "config");
        need(has_np, "assignment", "node_parts");
        need(has_ep, "assignment", "edge_part");
        need(has_sh, "assignment", "shared");
        need(has_dc, "assignment", "discards");
        need(has_parts, "assignment config", "parts");
        need(has_topk, "assignment config", "topk");
        if (x.num_parts < 1) data_error("InvalidParams", "assignment config parts < 1");
        x.node_count = static_cast<NodeId>(np.size());
        x.np_off.assign(1, 0);
        for (const auto& v : np) {
            for (PartId p : v)
                if (p < 0 || p >= x.num_parts)
                    data_error("InvalidPartition", "node_parts entry outside [0, parts)");
            x.np_parts.insert(x.np_parts.end(), v.begin(), v.end());
            x.np_off.push_back(x.np_parts.size());
        }
        for (PartId p : x.edge_part)
            if (p < kDiscarded || p >= x.num_parts)
                data_error("InvalidPartition", "edge_part entry outside [-1, parts)");
        if (config_out) {
            char* c = static_cast<char*>(std::malloc(cfg_text.size() + 1));
            if (!c) throw std::bad_alloc();
            std::memcpy(c, cfg_text.c_str(), cfg_text.size() + 1);
            *config_out = c;
        }
        *out = res.release();
    });
}

}  // extern "C"
