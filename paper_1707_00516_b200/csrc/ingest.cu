// Bulk panel ingest: the reference's text panel format
// (io.load_panel, pkg/src/fastid/io.py:45-127) parsed in native code with
// the same validation, error precedence and messages, multi-threaded over
// profile lines.  Host code only; the words it produces go to the device
// through fastid_load_words.
//
// Format: UTF-8 lines (universal newlines), a required `#bits=<L>` header,
// `#` comments, blank lines, and one `<id><TAB><hex>` profile per line; the
// hex is a bit string, most significant nibble of word 0 first, zero-extended
// or truncated (surplus digits must be 0) to ceil(L/W) words, padding past
// bit L must be zero.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "common.cuh"

struct fastid_parsed_panel {
    int64_t n = 0, bit_length = 0, n_words = 0;
    int word_width = 64;
    std::vector<uint8_t> words;   // n x n_words words of word_width bits (native endian)
    std::vector<char> ids;        // concatenated id bytes
    std::vector<int64_t> offsets; // n + 1
};

namespace fastid {
namespace {

struct Line {
    int64_t start, len, lineno;
};

// Error ranks within one line, in the reference's check order (io.py:79-125);
// the duplicate-id check sits between the id checks and the hex checks.
enum Rank { kRankFields = 0, kRankDup = 1, kRankHex = 2 };

struct Err {
    int64_t lineno = INT64_MAX;
    int rank = 0;
    int status = FASTID_OK;
    std::string msg;
    bool before(const Err& o) const { return lineno < o.lineno || (lineno == o.lineno && rank < o.rank); }
};

struct HexTable {
    uint8_t v[256];
    HexTable() {
        for (int c = 0; c < 256; ++c) v[c] = 0xFF;
        for (int c = '0'; c <= '9'; ++c) v[c] = (uint8_t)(c - '0');
        for (int c = 'a'; c <= 'f'; ++c) v[c] = (uint8_t)(c - 'a' + 10);
        for (int c = 'A'; c <= 'F'; ++c) v[c] = (uint8_t)(c - 'A' + 10);
    }
};
const HexTable kHex;
inline int8_t hexval(unsigned char c) { return (int8_t)kHex.v[c]; }

// 8 validated hex digits (most significant first) -> 32-bit value, SWAR.
inline uint32_t hex8(const unsigned char* p) {
    uint64_t x;
    memcpy(&x, p, 8);
    x = (x & 0x0F0F0F0F0F0F0F0Full) + 9 * ((x >> 6) & 0x0101010101010101ull);  // byte i = digit i
    x = ((x << 4) | (x >> 8)) & 0x00FF00FF00FF00FFull;                           // (d0 d1) (d2 d3) ...
    x = (x | (x >> 8)) & 0x0000FFFF0000FFFFull;
    x = (x | (x >> 16)) & 0x00000000FFFFFFFFull;                                  // bytes b0 b1 b2 b3
    return __builtin_bswap32((uint32_t)x);
}

std::string pyrepr(std::string_view s) {  // enough of Python's str repr for ids
    const bool sq = s.find('\'') != std::string_view::npos && s.find('"') == std::string_view::npos;
    const char q = sq ? '"' : '\'';
    std::string r(1, q);
    for (char c : s) {
        if (c == '\\' || c == q) r += '\\';
        if (c == '\t') {
            r += "\\t";
            continue;
        }
        r += c;
    }
    r += q;
    return r;
}

std::string fmt(const char* f, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, f);
    vsnprintf(buf, sizeof buf, f, ap);
    va_end(ap);
    return buf;
}

bool is_space(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\f' || c == '\v'; }

// Python int() of an ASCII decimal literal: whitespace, optional sign, digits
// with single underscores between them.
bool py_int(std::string_view s, int64_t* v) {
    size_t a = 0, b = s.size();
    while (a < b && is_space(s[a])) ++a;
    while (b > a && is_space(s[b - 1])) --b;
    if (a == b) return false;
    bool neg = false;
    if (s[a] == '+' || s[a] == '-') neg = s[a++] == '-';
    if (a == b || s[a] == '_' || s[b - 1] == '_') return false;
    int64_t x = 0;
    for (size_t i = a; i < b; ++i) {
        if (s[i] == '_') {
            if (s[i - 1] == '_') return false;
            continue;
        }
        if (s[i] < '0' || s[i] > '9') return false;
        if (x > (INT64_MAX - 9) / 10) return false;
        x = x * 10 + (s[i] - '0');
    }
    *v = neg ? -x : x;
    return true;
}

// One profile line -> words (or the first error of that line, ignoring the duplicate check).
bool parse_line(const char* text, const Line& ln, int64_t bit_length, int word_width, int64_t n_words,
                int64_t first_hex_len, bool first, uint8_t* dst, Err* err, std::string_view* id_out) {
    const char* p = text + ln.start;
    const char* tab = (const char*)memchr(p, '\t', (size_t)ln.len);
    const bool one_tab = tab && !memchr(tab + 1, '\t', (size_t)(p + ln.len - tab - 1));
    auto fail = [&](int rank, int status, std::string m) {
        err->lineno = ln.lineno;
        err->rank = rank;
        err->status = status;
        err->msg = fmt("line %lld: ", (long long)ln.lineno) + m;
        return false;
    };
    if (!one_tab) return fail(kRankFields, FASTID_E_FORMAT, "expected '<id><TAB><hex>'");
    const std::string_view id(p, (size_t)(tab - p));
    const std::string_view hex(tab + 1, (size_t)(p + ln.len - tab - 1));
    if (id.empty()) return fail(kRankFields, FASTID_E_FORMAT, "empty profile id");
    if (id.find(',') != std::string_view::npos)
        return fail(kRankFields, FASTID_E_FORMAT, "id " + pyrepr(id) + " contains a CSV separator");
    *id_out = id;
    uint8_t acc = 0;  // 0xFF bits appear only for a non-hex byte
    for (unsigned char c : hex) acc |= kHex.v[c] & 0xF0;
    if (acc) {
        bool bad[256] = {};
        for (unsigned char c : hex)
            if (hexval(c) < 0) bad[c] = true;
        std::string list = "[";
        for (int c = 0; c < 256; ++c)
            if (bad[c]) {
                if (list.size() > 1) list += ", ";
                list += pyrepr(std::string_view((const char*)&c, 1));
            }
        return fail(kRankHex, FASTID_E_FORMAT, "invalid hex characters " + list + "] in " + pyrepr(id));
    }
    const int64_t h = (int64_t)hex.size();
    if (first) {
        if (4 * h < bit_length)
            return fail(kRankHex, FASTID_E_FORMAT,
                        fmt("%lld bits of hex cannot hold %lld panel bits", (long long)(4 * h), (long long)bit_length));
    } else if (h != first_hex_len) {
        return fail(kRankHex, FASTID_E_FORMAT,
                    fmt("hex length %lld differs from %lld on earlier lines", (long long)h, (long long)first_hex_len));
    }
    const int dpw = word_width / 4;
    const int64_t target = n_words * dpw;
    if (h > target)
        for (int64_t i = target; i < h; ++i)
            if (hex[(size_t)i] != '0')
                return fail(kRankHex, FASTID_E_CORRUPT,
                            fmt("nonzero padding past bit %lld in ", (long long)bit_length) + pyrepr(id));
    uint64_t last = 0;
    const unsigned char* hx = (const unsigned char*)hex.data();
    for (int64_t w = 0; w < n_words; ++w) {
        uint64_t v = 0;
        if ((w + 1) * dpw <= h) {
            v = dpw == 16 ? ((uint64_t)hex8(hx + w * 16) << 32) | hex8(hx + w * 16 + 8) : hex8(hx + w * 8);
        } else {
            for (int d = 0; d < dpw; ++d) {
                const int64_t i = w * dpw + d;
                v = (v << 4) | (uint64_t)(i < h ? kHex.v[hx[i]] : 0);
            }
        }
        if (word_width == 64)
            reinterpret_cast<uint64_t*>(dst)[w] = v;
        else
            reinterpret_cast<uint32_t*>(dst)[w] = (uint32_t)v;
        last = v;
    }
    const int tail = (int)(bit_length % word_width);
    if (tail && (last & ((uint64_t(1) << (word_width - tail)) - 1)))
        return fail(kRankHex, FASTID_E_CORRUPT,
                    fmt("nonzero padding past bit %lld in ", (long long)bit_length) + pyrepr(id));
    return true;
}

}  // namespace
}  // namespace fastid

using namespace fastid;

extern "C" int fastid_parse_panel(const char* text, int64_t len, int word_width, int n_threads,
                                  fastid_parsed_panel** out) {
    if (!out) FASTID_FAIL(FASTID_E_INVALID, "out is NULL");
    *out = nullptr;
    if (word_width != 32 && word_width != 64) FASTID_FAIL(FASTID_E_INVALID, "word width must be 32 or 64");
    if (len < 0 || (len && !text)) FASTID_FAIL(FASTID_E_INVALID, "bad text buffer");
    const bool prof = getenv("FASTID_INGEST_PROFILE") != nullptr;
    auto tick = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (!prof) return;
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[ingest] %-10s %.3f s\n", what, std::chrono::duration<double>(now - tick).count());
        tick = now;
    };
    // ---- pass 1 (sequential): lines, header, comments ----
    std::vector<Line> lines;
    Err err;
    int64_t bit_length = -1, lineno = 0;
    for (int64_t i = 0; i < len && err.lineno == INT64_MAX;) {
        // next line end: memchr for '\n', then any '\r' before it (universal newlines)
        const char* nl = (const char*)memchr(text + i, '\n', (size_t)(len - i));
        int64_t j = nl ? (int64_t)(nl - text) : len;
        const char* cr = (const char*)memchr(text + i, '\r', (size_t)(j - i));
        if (cr) j = (int64_t)(cr - text);
        ++lineno;
        const int64_t n = j - i;
        if (n > 0) {
            const char* p = text + i;
            if (p[0] == '#') {
                std::string_view body(p + 1, (size_t)(n - 1));
                size_t a = 0, b = body.size();
                while (a < b && is_space(body[a])) ++a;
                while (b > a && is_space(body[b - 1])) --b;
                body = body.substr(a, b - a);
                if (body.substr(0, 5) == "bits=") {
                    int64_t v = 0;
                    if (bit_length >= 0) {
                        err = {lineno, 0, FASTID_E_FORMAT, fmt("line %lld: duplicate #bits header", (long long)lineno)};
                    } else if (!py_int(body.substr(5), &v)) {
                        err = {lineno, 0, FASTID_E_FORMAT,
                               fmt("line %lld: bad header ", (long long)lineno) + pyrepr(std::string_view(p, (size_t)n))};
                    } else if (v <= 0) {
                        err = {lineno, 0, FASTID_E_FORMAT, fmt("line %lld: bit length must be positive", (long long)lineno)};
                    } else {
                        bit_length = v;
                    }
                }
            } else if (bit_length < 0) {
                err = {lineno, 0, FASTID_E_FORMAT,
                       fmt("line %lld: profile before the #bits=<L> header", (long long)lineno)};
            } else {
                lines.push_back({i, n, lineno});
            }
        }
        // universal newlines: \r\n, \r and \n each end one line
        if (j < len && text[j] == '\r' && j + 1 < len && text[j + 1] == '\n') ++j;
        i = j + 1;
    }
    if (err.lineno == INT64_MAX && bit_length < 0) FASTID_FAIL(FASTID_E_FORMAT, "missing #bits=<L> header");
    mark("lines");
    const int64_t n_words = bit_length > 0 ? (bit_length + word_width - 1) / word_width : 0;
    const int64_t n = (int64_t)lines.size();
    // ---- pass 2 (parallel): per-line checks and words ----
    auto* P = new fastid_parsed_panel();
    P->bit_length = bit_length;
    P->n_words = n_words;
    P->word_width = word_width;
    P->words.resize((size_t)(n * n_words * (word_width / 8)));
    std::vector<std::string_view> ids((size_t)n);
    int64_t first_hex_len = 0;
    if (n) {
        const char* p = text + lines[0].start;
        const char* tab = (const char*)memchr(p, '\t', (size_t)lines[0].len);
        first_hex_len = tab ? (int64_t)(p + lines[0].len - tab - 1) : 0;
    }
    int nt = n_threads > 0 ? n_threads : (int)std::max(1u, std::thread::hardware_concurrency());
    nt = (int)std::max<int64_t>(1, std::min<int64_t>(nt, n / 4096 + 1));
    std::vector<Err> terr((size_t)nt);
    mark("setup");
    auto work = [&](int t) {
        const int64_t lo = n * t / nt, hi = n * (t + 1) / nt;
        const size_t row = (size_t)n_words * (word_width / 8);
        for (int64_t k = lo; k < hi && lines[(size_t)k].lineno < err.lineno; ++k)
            if (!parse_line(text, lines[(size_t)k], bit_length, word_width, n_words, first_hex_len, k == 0,
                            P->words.data() + (size_t)k * row, &terr[(size_t)t], &ids[(size_t)k]))
                break;
    };
    {
        std::vector<std::thread> pool;
        for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
        work(0);
        for (auto& th : pool) th.join();
    }
    mark("parse");
    for (auto& e : terr)
        if (e.before(err)) err = e;
    // ---- pass 3 (sequential, line order): duplicate ids before the first error ----
    {
        // open-addressing set of line indices keyed by the id bytes (hashes precomputed in parallel)
        int64_t limit = 0;
        while (limit < n && (lines[(size_t)limit].lineno < err.lineno ||
                             (lines[(size_t)limit].lineno == err.lineno && err.rank > kRankDup)))
            ++limit;
        std::vector<uint64_t> hs((size_t)limit);
        {
            std::vector<std::thread> pool;
            auto hw = [&](int t) {
                for (int64_t k = limit * t / nt; k < limit * (t + 1) / nt; ++k)
                    hs[(size_t)k] = std::hash<std::string_view>{}(ids[(size_t)k]);
            };
            for (int t = 1; t < nt; ++t) pool.emplace_back(hw, t);
            hw(0);
            for (auto& th : pool) th.join();
        }
        size_t cap = 16;
        while (cap < (size_t)limit * 2) cap <<= 1;
        std::vector<int64_t> slot(cap, -1);
        for (int64_t k = 0; k < limit; ++k) {
            size_t h = (size_t)hs[(size_t)k] & (cap - 1);
            bool dup = false;
            while (slot[h] >= 0) {
                const int64_t o = slot[h];
                if (hs[(size_t)o] == hs[(size_t)k] && ids[(size_t)o] == ids[(size_t)k]) {
                    dup = true;
                    break;
                }
                h = (h + 1) & (cap - 1);
            }
            if (dup) {
                const Line& ln = lines[(size_t)k];
                err = {ln.lineno, kRankDup, FASTID_E_FORMAT,
                       fmt("line %lld: duplicate id ", (long long)ln.lineno) + pyrepr(ids[(size_t)k])};
                break;
            }
            slot[h] = k;
        }
    }
    mark("dups");
    if (err.lineno != INT64_MAX) {
        delete P;
        FASTID_FAIL(err.status, "%s", err.msg.c_str());
    }
    // ids joined by '\n' (an id holds neither a tab nor a line break), offsets
    // of each id's first byte (+ total) for callers that slice
    P->n = n;
    P->offsets.resize((size_t)n + 1);
    size_t total = 0;
    for (int64_t k = 0; k < n; ++k) {
        P->offsets[(size_t)k] = (int64_t)total;
        total += ids[(size_t)k].size() + (k + 1 < n ? 1 : 0);
    }
    P->offsets[(size_t)n] = (int64_t)total;
    P->ids.resize(total);
    for (int64_t k = 0; k < n; ++k) {
        char* d = P->ids.data() + P->offsets[(size_t)k];
        memcpy(d, ids[(size_t)k].data(), ids[(size_t)k].size());
        if (k + 1 < n) d[ids[(size_t)k].size()] = '\n';
    }
    mark("ids");
    *out = P;
    return FASTID_OK;
}

extern "C" int fastid_parsed_panel_shape(const fastid_parsed_panel* p, int64_t* n_profiles, int64_t* bit_length,
                                         int64_t* n_words, int64_t* id_bytes) {
    if (!p) FASTID_FAIL(FASTID_E_INVALID, "panel is NULL");
    if (n_profiles) *n_profiles = p->n;
    if (bit_length) *bit_length = p->bit_length;
    if (n_words) *n_words = p->n_words;
    if (id_bytes) *id_bytes = (int64_t)p->ids.size();
    return FASTID_OK;
}

extern "C" int fastid_parsed_panel_copy(const fastid_parsed_panel* p, void* words, char* ids, int64_t* id_offsets) {
    if (!p) FASTID_FAIL(FASTID_E_INVALID, "panel is NULL");
    if (words && !p->words.empty()) memcpy(words, p->words.data(), p->words.size());
    if (ids && !p->ids.empty()) memcpy(ids, p->ids.data(), p->ids.size());
    if (id_offsets) memcpy(id_offsets, p->offsets.data(), p->offsets.size() * sizeof(int64_t));
    return FASTID_OK;
}

extern "C" void fastid_parsed_panel_free(fastid_parsed_panel* p) { delete p; }
