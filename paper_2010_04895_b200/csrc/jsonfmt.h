// jsonfmt.h -- the reference's JSON sidecars byte for byte, without a JSON
// library: the `.stats.jsonl` line of write_corpus (engine.cpp:248-259,
// nlohmann::json::dump()) and the `.manifest.json` of cmd_walk
// (tools/mhwalk.cpp:142-169, dump(2)).
//
// What the bytes depend on (nlohmann 3.11 semantics, restated):
//  * objects are std::map-ordered: keys sorted by byte value;
//  * dump() has no whitespace; dump(2) puts one member per line, indented
//    by two spaces per level, ": " after keys, "{}" for empty objects;
//  * integers print in decimal; doubles print as Grisu2's digits (a decimal
//    that reads back to the same double, nearly always the shortest), laid
//    out as nlohmann's format_buffer
//    does (decimal exponent window (-4, 15]: "2959152.659515442", "0.0",
//    "1234500.0", "0.000123"; otherwise "1.5e+16", "1e-05", "2.5e-07"),
//    non-finite values as null;
//  * strings are quoted with '"', '\\', and control characters escaped
//    (\b \f \n \r \t, else \u00XX).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

namespace mhw {
namespace json {

// Decimal digits of a finite, non-zero |x| by Grisu2 (F. Loitsch, "Printing
// floating-point numbers quickly and accurately with integers", PLDI 2010),
// the variant nlohmann's dtoa_impl runs: boundaries m- / m+ of x, a cached
// power c = 10^-k with the scaled exponent in [-60, -32], digit generation
// from M+ = w+ - 1 ulp against delta = M+ - M-, then round-weeding toward w.
// It returns the shortest digits in almost all cases but not always (e.g.
// 6.6340809261215234e+181), which is why it is restated rather than
// replaced by a true shortest search. x = d1...dk * 10^dec_exp.
namespace grisu {
struct Fp {
    uint64_t f;
    int e;
};
inline Fp mul(Fp x, Fp y) {  // upper 64 bits of the 128-bit product, rounded (ties up)
    const uint64_t a = x.f >> 32, b = x.f & 0xFFFFFFFFu, c = y.f >> 32, d = y.f & 0xFFFFFFFFu;
    const uint64_t ac = a * c, bc = b * c, ad = a * d, bd = b * d;
    uint64_t mid = (bd >> 32) + (ad & 0xFFFFFFFFu) + (bc & 0xFFFFFFFFu);
    mid += uint64_t(1) << 31;
    return {ac + (ad >> 32) + (bc >> 32) + (mid >> 32), x.e + y.e + 64};
}
inline Fp normalize(Fp x) {
    while (!(x.f >> 63)) {
        x.f <<= 1;
        --x.e;
    }
    return x;
}

// 10^k ~ f * 2^e, f in [2^63, 2^64) rounded to nearest, for k = -300 + 8 i
// (i < 79): computed once with a small bignum (exact powers of ten, and
// floor(2^(s+1) / 10^n) by repeated exact division for negative k).
struct CachedPower {
    uint64_t f;
    int e;
    int k;
};
struct Big {
    std::vector<uint32_t> w;  // little-endian limbs
    void mul10() {
        uint64_t c = 0;
        for (auto& x : w) {
            const uint64_t t = (uint64_t)x * 10 + c;
            x = (uint32_t)t;
            c = t >> 32;
        }
        if (c) w.push_back((uint32_t)c);
    }
    void div10() {
        uint64_t r = 0;
        for (size_t i = w.size(); i-- > 0;) {
            const uint64_t t = (r << 32) | w[i];
            w[i] = (uint32_t)(t / 10);
            r = t % 10;
        }
        while (!w.empty() && !w.back()) w.pop_back();
    }
    int bits() const {
        if (w.empty()) return 0;
        int b = 32 * (int)(w.size() - 1);
        for (uint32_t x = w.back(); x; x >>= 1) ++b;
        return b;
    }
    uint64_t top(int from, int count) const {  // bits [from, from + count) as an integer
        uint64_t r = 0;
        for (int i = count - 1; i >= 0; --i) {
            const int b = from + i;
            const uint32_t bit = (b >= 0 && b / 32 < (int)w.size()) ? (w[b / 32] >> (b % 32)) & 1u : 0u;
            r = (r << 1) | bit;
        }
        return r;
    }
};
inline CachedPower power_of_ten(int k) {
    Big t;
    t.w = {1};
    const int n = k < 0 ? -k : k;
    for (int i = 0; i < n; ++i) t.mul10();  // 10^n
    const int L = t.bits();                 // 2^(L-1) <= 10^n < 2^L
    if (k >= 0) {
        // f = round(10^k / 2^(L-64))
        const int e = L - 64;
        uint64_t f;
        if (e <= 0) {
            f = t.top(0, 64) << (-e);
        } else {
            const uint64_t hi = t.top(e, 64), half = t.top(e - 1, 1);
            f = hi + half;
            if (f == 0) return {uint64_t(1) << 63, e + 1, k};  // carried out of 64 bits
        }
        return {f, e, k};
    }
    // f = round(2^s / 10^n), s = 63 + L: q = floor(2^(s+1) / 10^n) has 65 bits
    const int s = 63 + L;
    Big q;
    q.w.assign((size_t)((s + 1) / 32 + 1), 0u);
    q.w[(size_t)((s + 1) / 32)] = 1u << ((s + 1) % 32);
    for (int i = 0; i < n; ++i) q.div10();
    const uint64_t f = (q.top(1, 64)) + q.top(0, 1);
    if (f == 0) return {uint64_t(1) << 63, -s + 1, k};
    return {f, -s, k};
}
inline const CachedPower& cached_power_for(int e) {
    // the power whose product with 2^e lands in [2^-60, 2^-32] (alpha, gamma)
    static const std::vector<CachedPower> table = [] {
        std::vector<CachedPower> t;
        for (int i = 0; i < 79; ++i) t.push_back(power_of_ten(-300 + 8 * i));
        return t;
    }();
    const int f = -60 - e - 1;
    const int k = (f * 78913) / (1 << 18) + (f > 0 ? 1 : 0);
    const int index = (300 + k + 7) / 8;
    return table[(size_t)index];
}
inline void round_weed(std::string& buf, uint64_t dist, uint64_t delta, uint64_t rest, uint64_t ten_k) {
    while (rest < dist && delta - rest >= ten_k && (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
        --buf.back();
        rest += ten_k;
    }
}
inline void digits(double x, std::string& buf, int& dec_exp) {
    uint64_t bits;
    std::memcpy(&bits, &x, 8);
    const uint64_t E = (bits >> 52) & 0x7FF, F = bits & ((uint64_t(1) << 52) - 1);
    const Fp v = E == 0 ? Fp{F, 1 - 1075} : Fp{F + (uint64_t(1) << 52), (int)E - 1075};
    const bool lower_closer = F == 0 && E > 1;
    const Fp mp = normalize(Fp{2 * v.f + 1, v.e - 1});
    Fp mm = lower_closer ? Fp{4 * v.f - 1, v.e - 2} : Fp{2 * v.f - 1, v.e - 1};
    mm = Fp{mm.f << (mm.e - mp.e), mp.e};
    const Fp w0 = normalize(v);
    const CachedPower& cp = cached_power_for(mp.e);
    const Fp c{cp.f, cp.e};
    const Fp w = mul(w0, c), wm = mul(mm, c), wp = mul(mp, c);
    const Fp Mm{wm.f + 1, wm.e}, Mp{wp.f - 1, wp.e};
    dec_exp = -cp.k;
    uint64_t delta = Mp.f - Mm.f, dist = Mp.f - w.f;
    const int sh = -Mp.e;
    const uint64_t one = uint64_t(1) << sh;
    uint32_t p1 = (uint32_t)(Mp.f >> sh);
    uint64_t p2 = Mp.f & (one - 1);
    uint32_t pow10 = 1;
    int n = 1;
    while (pow10 <= p1 / 10) {
        pow10 *= 10;
        ++n;
    }
    buf.clear();
    while (n > 0) {
        buf.push_back((char)('0' + p1 / pow10));
        p1 %= pow10;
        --n;
        const uint64_t rest = ((uint64_t)p1 << sh) + p2;
        if (rest <= delta) {
            dec_exp += n;
            round_weed(buf, dist, delta, rest, (uint64_t)pow10 << sh);
            return;
        }
        pow10 /= 10;
    }
    int m = 0;
    for (;;) {
        p2 *= 10;
        buf.push_back((char)('0' + (p2 >> sh)));
        p2 &= one - 1;
        ++m;
        delta *= 10;
        dist *= 10;
        if (p2 <= delta) break;
    }
    dec_exp -= m;
    round_weed(buf, dist, delta, p2, one);
}
}  // namespace grisu

inline std::string number(double x) {
    if (!std::isfinite(x)) return "null";
    std::string out;
    if (std::signbit(x)) {
        out.push_back('-');
        x = -x;
    }
    if (x == 0.0) return out + "0.0";
    std::string d;
    int dec_exp = 0;
    grisu::digits(x, d, dec_exp);
    const int k = (int)d.size();
    const int n = k + dec_exp;  // decimal point position: value = 0.d * 10^n
    constexpr int kMinExp = -4, kMaxExp = 15;
    if (k <= n && n <= kMaxExp) {  // integral: digits, zeros, ".0"
        out += d;
        out.append((size_t)(n - k), '0');
        out += ".0";
    } else if (0 < n && n <= kMaxExp) {  // 123.45
        out += d.substr(0, (size_t)n);
        out.push_back('.');
        out += d.substr((size_t)n);
    } else if (kMinExp < n && n <= 0) {  // 0.00123
        out += "0.";
        out.append((size_t)(-n), '0');
        out += d;
    } else {  // d.ddde+XX
        out.push_back(d[0]);
        if (k > 1) {
            out.push_back('.');
            out += d.substr(1);
        }
        int e = n - 1;
        out.push_back('e');
        out.push_back(e < 0 ? '-' : '+');
        e = e < 0 ? -e : e;
        char eb[8];
        std::snprintf(eb, sizeof eb, e < 10 ? "0%d" : "%d", e);
        out += eb;
    }
    return out;
}

inline std::string number(uint64_t x) { return std::to_string(x); }
inline std::string number(int64_t x) { return std::to_string(x); }

inline std::string quote(const std::string& s) {
    std::string o = "\"";
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
                    char b[8];
                    std::snprintf(b, sizeof b, "\\u%04x", c);
                    o += b;
                } else {
                    o.push_back((char)c);
                }
        }
    }
    return o + "\"";
}

// A JSON value: a scalar already rendered, or an object (sorted keys).
struct Value {
    std::string scalar;
    std::map<std::string, Value> obj;
    bool is_obj = false;
    Value() : is_obj(true) {}
    Value(const char* s) : scalar(quote(s)) {}
    Value(const std::string& s) : scalar(quote(s)) {}
    Value(bool b) : scalar(b ? "true" : "false") {}
    Value(double x) : scalar(number(x)) {}
    Value(uint64_t x) : scalar(number(x)) {}
    Value(uint32_t x) : scalar(number((uint64_t)x)) {}
    Value(int64_t x) : scalar(number(x)) {}
    Value(int x) : scalar(number((int64_t)x)) {}
    Value& operator[](const std::string& k) { return obj[k]; }

    // dump(-1) compact, dump(indent) pretty (nlohmann serializer layout)
    void dump(std::string& o, int indent, int level) const {
        if (!is_obj) {
            o += scalar;
            return;
        }
        if (obj.empty()) {
            o += "{}";
            return;
        }
        o.push_back('{');
        bool first = true;
        for (const auto& kv : obj) {
            if (!first) o.push_back(',');
            first = false;
            if (indent >= 0) {
                o.push_back('\n');
                o.append((size_t)(indent * (level + 1)), ' ');
            }
            o += quote(kv.first);
            o += indent >= 0 ? ": " : ":";
            kv.second.dump(o, indent, level + 1);
        }
        if (indent >= 0) {
            o.push_back('\n');
            o.append((size_t)(indent * level), ' ');
        }
        o.push_back('}');
    }
    std::string dump(int indent = -1) const {
        std::string o;
        dump(o, indent, 0);
        return o;
    }
};

}  // namespace json

// write_corpus's sidecar line (engine.cpp:248-259): dump() of the stats
// object (sorted keys) plus '\n'.
template <class Stats>
inline std::string stats_line(const Stats& st) {
    json::Value v;
    v["walks"] = (uint64_t)st.walks;
    v["early_terminations"] = (uint64_t)st.early_terminations;
    v["skipped_starts"] = (uint64_t)st.skipped_starts;
    v["steps"] = (uint64_t)st.steps;
    v["steps_per_sec"] = (double)st.steps_per_sec;
    v["init_seconds"] = (double)st.init_seconds;
    v["walk_seconds"] = (double)st.walk_seconds;
    return v.dump() + "\n";
}

}  // namespace mhw
