// loader.cu -- text ingestion at scale.
//
// load_edge_list / load_node_types / load_edge_types (graph.cpp:70-177) with
// the reference's exact acceptance rules and messages, parsed by all host
// cores: the file is split at newlines into one range per thread, each range
// is scanned independently and the first error in file order wins (its line
// number is recovered by counting newlines before it). The CSR is then built
// on the device with build_csr semantics (graph.cu graph_from_edges).
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "internal.h"
#include "loader.h"

namespace mhw {

namespace {

struct Text {
    std::vector<char> data;
};

Text read_file(const std::string& path, const char* what) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw Error(MHW_ERR_IO, std::string("cannot open ") + what + ": " + path);
    Text t;
    std::fseek(f, 0, SEEK_END);
    const long sz = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    t.data.resize(sz > 0 ? (size_t)sz : 0);
    if (sz > 0 && std::fread(t.data.data(), 1, (size_t)sz, f) != (size_t)sz) {
        std::fclose(f);
        throw Error(MHW_ERR_IO, std::string("cannot read ") + what + ": " + path);
    }
    std::fclose(f);
    return t;
}

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

// blank_or_comment (graph.cpp:27-33): a '#' before any non-space char, or
// only whitespace.
inline bool blank_or_comment(const char* b, const char* e) {
    for (const char* p = b; p < e; ++p) {
        if (*p == '#') return true;
        if (!is_space(*p)) return false;
    }
    return true;
}

// istream >> long long: skip whitespace, optional sign, digits (overflow fails).
inline bool read_ll(const char*& p, const char* e, long long& out) {
    while (p < e && is_space(*p)) ++p;
    bool neg = false;
    if (p < e && (*p == '+' || *p == '-')) {
        neg = *p == '-';
        ++p;
    }
    if (p >= e || *p < '0' || *p > '9') return false;
    unsigned long long v = 0;
    while (p < e && *p >= '0' && *p <= '9') {
        const unsigned d = (unsigned)(*p - '0');
        if (v > (9223372036854775807ull - d) / 10 + (neg ? 1 : 0)) return false;
        v = v * 10 + d;
        ++p;
    }
    out = neg ? -(long long)v : (long long)v;
    return true;
}

// istream >> double: the characters num_get accumulates for a float
// ([+-] digits [. digits] [(e|E) [+-] digits]) converted with strtod.
inline bool read_double(const char*& p, const char* e, double& out) {
    while (p < e && is_space(*p)) ++p;
    char buf[128];
    size_t k = 0;
    const char* q = p;
    auto put = [&](char c) {
        if (k + 1 < sizeof buf) buf[k++] = c;
    };
    if (q < e && (*q == '+' || *q == '-')) put(*q++);
    bool digits = false;
    while (q < e && *q >= '0' && *q <= '9') {
        put(*q++);
        digits = true;
    }
    if (q < e && *q == '.') {
        put(*q++);
        while (q < e && *q >= '0' && *q <= '9') {
            put(*q++);
            digits = true;
        }
    }
    if (!digits) return false;
    if (q < e && (*q == 'e' || *q == 'E')) {
        const char* r = q + 1;
        if (r < e && (*r == '+' || *r == '-')) ++r;
        if (r < e && *r >= '0' && *r <= '9') {
            put(*q++);
            if (*q == '+' || *q == '-') put(*q++);
            while (q < e && *q >= '0' && *q <= '9') put(*q++);
        } else {
            return false;  // num_get consumed 'e' and failed
        }
    }
    buf[k] = 0;
    errno = 0;
    out = std::strtod(buf, nullptr);
    if (errno == ERANGE && std::isinf(out)) return false;
    p = q;
    return true;
}

struct LineError {
    size_t pos = SIZE_MAX;  // byte offset of the failing line's start
    mhw_status code = MHW_OK;
    std::string what;       // message after "path:line: "
};

template <class Rec, class ParseLine>
std::vector<Rec> parse_lines(const Text& t, const std::string& path, ParseLine&& parse_line) {
    const char* base = t.data.data();
    const size_t n = t.data.size();
    unsigned threads = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    if (n < (1u << 20)) threads = 1;
    std::vector<size_t> cut(threads + 1, n);
    cut[0] = 0;
    for (unsigned i = 1; i < threads; ++i) {
        size_t c = n * i / threads;
        while (c < n && base[c - 1] != '\n') ++c;
        cut[i] = std::max(c, cut[i - 1]);
    }
    std::vector<std::vector<Rec>> parts(threads);
    std::vector<LineError> errs(threads);
    auto work = [&](unsigned i) {
        const char* p = base + cut[i];
        const char* end = base + cut[i + 1];
        while (p < end) {
            const char* nl = static_cast<const char*>(std::memchr(p, '\n', (size_t)(end - p)));
            const char* le = nl ? nl : end;
            if (!blank_or_comment(p, le)) {
                Rec r;
                LineError e;
                if (!parse_line(p, le, r, e)) {
                    e.pos = (size_t)(p - base);
                    errs[i] = e;
                    return;
                }
                parts[i].push_back(r);
            }
            p = nl ? nl + 1 : end;
        }
    };
    if (threads == 1) {
        work(0);
    } else {
        std::vector<std::thread> pool;
        for (unsigned i = 0; i < threads; ++i) pool.emplace_back(work, i);
        for (auto& th : pool) th.join();
    }
    for (unsigned i = 0; i < threads; ++i) {
        if (errs[i].pos != SIZE_MAX) {
            const size_t line = 1 + (size_t)std::count(base, base + errs[i].pos, '\n');
            throw Error(errs[i].code, path + ":" + std::to_string(line) + ": " + errs[i].what);
        }
    }
    size_t total = 0;
    for (auto& v : parts) total += v.size();
    std::vector<Rec> all;
    all.reserve(total);
    for (auto& v : parts) all.insert(all.end(), v.begin(), v.end());
    return all;
}

struct EdgeRec {
    uint32_t s, d;
    double w;
    bool rev;  // symmetrize && src != dst on the untruncated values (graph.cpp:95)
};

}  // namespace

void parse_edge_list(const std::string& path, bool weighted, bool symmetrize, std::vector<uint32_t>& src,
                     std::vector<uint32_t>& dst, std::vector<double>& w) {
    const Text t = read_file(path, "edge list");
    auto recs = parse_lines<EdgeRec>(t, path, [&](const char* p, const char* e, EdgeRec& r, LineError& err) {
        long long a, b;
        if (!read_ll(p, e, a) || !read_ll(p, e, b) || a < 0 || b < 0) {
            err.code = MHW_ERR_INVALID;
            err.what = "expected \"src dst [weight]\"";
            return false;
        }
        double x = 1.0;
        if (weighted) {
            if (!read_double(p, e, x)) {
                err.code = MHW_ERR_INVALID;
                err.what = "missing edge weight";
                return false;
            }
            if (x < 0) {
                err.code = MHW_ERR_INVALID;
                err.what = "negative edge weight";
                return false;
            }
        }
        r.s = (uint32_t)a;  // static_cast<NodeId>, graph.cpp:94
        r.d = (uint32_t)b;
        r.w = x;
        r.rev = symmetrize && a != b;
        return true;
    });
    // the reference's edge vector: each edge, then its reverse (graph.cpp:94-97)
    size_t k = 0;
    for (const auto& r : recs) k += r.rev ? 2 : 1;
    src.resize(k);
    dst.resize(k);
    w.resize(k);
    k = 0;
    for (const auto& r : recs) {
        src[k] = r.s;
        dst[k] = r.d;
        w[k++] = r.w;
        if (r.rev) {
            src[k] = r.d;
            dst[k] = r.s;
            w[k++] = r.w;
        }
    }
}

void load_node_types(Graph& g, const std::string& path) {
    const Text t = read_file(path, "node-type file");
    struct R {
        uint32_t v;
        uint16_t t;
    };
    const uint32_t n = g.n;
    auto recs = parse_lines<R>(t, path, [&](const char* p, const char* e, R& r, LineError& err) {
        long long node, type;
        if (!read_ll(p, e, node) || !read_ll(p, e, type) || node < 0 || type < 0) {
            err.code = MHW_ERR_INVALID;
            err.what = "expected \"node_id type_id\"";
            return false;
        }
        if (node >= n) {
            err.code = MHW_ERR_INVALID;
            err.what = "unknown node id " + std::to_string(node);
            return false;
        }
        r.v = (uint32_t)node;
        r.t = (uint16_t)type;
        return true;
    });
    std::vector<uint16_t> types(n, 0);
    std::vector<uint8_t> covered(n, 0);
    uint16_t mx = 0;
    for (const auto& r : recs) {  // file order: a later line overrides (graph.cpp:124)
        types[r.v] = r.t;
        covered[r.v] = 1;
        mx = std::max(mx, r.t);
    }
    for (uint32_t v = 0; v < n; ++v)
        if (!covered[v]) invalid(path + ": node " + std::to_string(v) + " has no type assignment");
    graph_set_node_types(g, types.data(), (uint16_t)(mx + 1));
}

void load_edge_types(Graph& g, const std::string& path) {
    const Text t = read_file(path, "edge-type file");
    struct R {
        uint32_t s, d;
        uint16_t t;
        uint64_t line_pos;
    };
    const uint32_t n = g.n;
    const char* base = t.data.data();
    auto recs = parse_lines<R>(t, path, [&](const char* p, const char* e, R& r, LineError& err) {
        const char* line = p;
        long long a, b, c;
        if (!read_ll(p, e, a) || !read_ll(p, e, b) || !read_ll(p, e, c) || a < 0 || b < 0 || c < 0) {
            err.code = MHW_ERR_INVALID;
            err.what = "expected \"src dst type_id\"";
            return false;
        }
        if (a >= n || b >= n) {
            err.code = MHW_ERR_INVALID;
            err.what = "edge not present in graph";
            return false;
        }
        r.s = (uint32_t)a;
        r.d = (uint32_t)b;
        r.t = (uint16_t)c;
        r.line_pos = (uint64_t)(line - base);
        return true;
    });
    // arc lookup on the host copy of the CSR (same lower_bound as graph.cpp:13-18)
    std::vector<int64_t> off(n + 1);
    std::vector<int32_t> ids(g.m);
    graph_download(g, off.data(), ids.data(), nullptr, nullptr, nullptr);
    auto index_of = [&](uint32_t v, uint32_t u) -> int64_t {
        const int32_t* b = ids.data() + off[v];
        const int32_t* e = ids.data() + off[v + 1];
        const int32_t* it = std::lower_bound(b, e, (int32_t)u, [](int32_t x, int32_t y) {
            return (uint32_t)x < (uint32_t)y;
        });
        if (it == e || (uint32_t)*it != u) return -1;
        return off[v] + (it - b);
    };
    std::vector<uint16_t> types(g.m, 0);
    std::vector<uint8_t> covered(g.m, 0);
    uint16_t mx = 0;
    for (const auto& r : recs) {
        const int64_t a = index_of(r.s, r.d);
        if (a < 0) {
            const size_t line = 1 + (size_t)std::count(base, base + r.line_pos, '\n');
            invalid(path + ":" + std::to_string(line) + ": edge not present in graph");
        }
        types[a] = r.t;
        covered[a] = 1;
        if (g.symmetric) {  // both directions (graph.cpp:165-167)
            const int64_t bk = index_of(r.d, r.s);
            if (bk >= 0) {
                types[bk] = r.t;
                covered[bk] = 1;
            }
        }
        mx = std::max(mx, r.t);
    }
    for (uint64_t i = 0; i < g.m; ++i)
        if (!covered[i]) invalid(path + ": arc " + std::to_string(i) + " has no type assignment");
    graph_set_edge_types(g, types.data(), (uint16_t)(mx + 1));
}

void load_edge_list(Graph& g, const std::string& path, bool weighted, bool symmetrize) {
    std::vector<uint32_t> src, dst;
    std::vector<double> w;
    parse_edge_list(path, weighted, symmetrize, src, dst, w);
    build_parsed(g, src, dst, w, weighted, symmetrize);
}

void build_parsed(Graph& g, const std::vector<uint32_t>& src, const std::vector<uint32_t>& dst,
                  const std::vector<double>& w, bool weighted, bool symmetrize) {
    std::vector<float> wf;
    if (weighted) {
        wf.resize(w.size());
        for (size_t i = 0; i < w.size(); ++i) wf[i] = (float)w[i];
    }
    // reverse arcs are already in the list: build without symmetrising again
    graph_from_edges(g, src.size(), src.data(), dst.data(), weighted ? wf.data() : nullptr, false, 0);
    g.symmetric = symmetrize;
}

}  // namespace mhw
