// gd_textio.cpp -- native parsers for the reference's text formats
// (graph/io.py:11-39 edge lines, graph/updates.py:77-104 update lines).
//
// The Python parsers handle ~1M lines/s; C2 is 67M edge lines and C5 ~20 GB
// of text.  These read the file with one fread, split it into chunks at line
// boundaries and parse the chunks on all host threads, with the reference's
// validation and the line number of the FIRST bad line (the same line the
// sequential Python loop would report).  Fields are whitespace separated;
// `#` starts a comment; blank lines are skipped; \n, \r\n and \r end lines.
#include <omp.h>

#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

namespace {

struct Parsed {
    std::vector<int64_t> a, b, c;  // src, dst, weight
    std::vector<uint8_t> k;        // update kind ('a' / 'd')
    int64_t max_id = -1;
    int weighted = -1;  // edges: -1 = no line yet
};

inline bool is_ws(char ch) { return ch == ' ' || ch == '\t' || ch == '\v' || ch == '\f'; }
inline bool is_eol(char ch) { return ch == '\n' || ch == '\r'; }

// parse an optionally signed decimal integer spanning exactly [p, e)
inline bool parse_int(const char* p, const char* e, int64_t& out) {
    bool neg = false;
    if (p < e && (*p == '+' || *p == '-')) neg = *p++ == '-';
    if (p == e) return false;
    uint64_t v = 0;
    for (; p < e; ++p) {
        if (*p < '0' || *p > '9') return false;
        uint64_t nv = v * 10 + (uint64_t)(*p - '0');
        if (nv / 10 != v) return false;  // overflow
        v = nv;
    }
    if (v > (uint64_t)INT64_MAX + (neg ? 1 : 0)) return false;
    out = neg ? (int64_t)(0 - v) : (int64_t)v;
    return true;
}

struct Error {
    int64_t line = -1;  // 1-based within the chunk until rebased
    std::string msg;
};

// split [p, e) into whitespace fields, up to 5
inline int fields(const char* p, const char* e, const char* fs[5], const char* fe[5]) {
    int n = 0;
    while (p < e) {
        while (p < e && is_ws(*p)) ++p;
        if (p >= e) break;
        const char* s = p;
        while (p < e && !is_ws(*p)) ++p;
        if (n < 5) {
            fs[n] = s;
            fe[n] = p;
        }
        ++n;
    }
    return n;
}

// mode 0: edge lines "src dst [w]"; mode 1: update lines "a s d [w]" / "d s d"
void parse_chunk(const char* p, const char* e, int mode, Parsed& out, Error& err, int64_t& lines) {
    lines = 0;
    while (p < e) {
        const char* ls = p;
        while (p < e && !is_eol(*p)) ++p;
        const char* le = p;
        if (p < e && *p == '\r' && p + 1 < e && p[1] == '\n') ++p;
        if (p < e) ++p;
        ++lines;
        if (err.line >= 0) continue;  // keep counting lines only
        const char* hash = (const char*)memchr(ls, '#', (size_t)(le - ls));
        if (hash) le = hash;
        const char* fs[5];
        const char* fe[5];
        int nf = fields(ls, le, fs, fe);
        if (nf == 0) continue;
        if (mode == 0) {
            if (nf != 2 && nf != 3) {
                err = {lines, "expected 'src dst [weight]'"};
                continue;
            }
            int64_t s, d, w = 1;
            if (!parse_int(fs[0], fe[0], s) || !parse_int(fs[1], fe[1], d) ||
                (nf == 3 && !parse_int(fs[2], fe[2], w))) {
                err = {lines, "non-integer field"};
                continue;
            }
            if (s < 0 || d < 0) {
                err = {lines, "negative node id"};
                continue;
            }
            int has_w = nf == 3;
            if (out.weighted < 0) out.weighted = has_w;
            else if (out.weighted != has_w) {
                err = {lines, "mixed weighted/unweighted edge lines"};
                continue;
            }
            if (has_w && w < 0) {
                err = {lines, "negative edge weight"};
                continue;
            }
            out.a.push_back(s);
            out.b.push_back(d);
            out.c.push_back(w);
            if (s > out.max_id) out.max_id = s;
            if (d > out.max_id) out.max_id = d;
        } else {
            char kind = (fe[0] - fs[0] == 1) ? fs[0][0] : '?';
            if (kind != 'a' && kind != 'd') {
                err = {lines, "unknown update kind '" + std::string(fs[0], fe[0]) + "'"};
                continue;
            }
            if (kind == 'a' ? (nf != 3 && nf != 4) : nf != 3) {
                err = {lines, kind == 'a' ? "expected 'a <src> <dst> [weight]'" : "expected 'd <src> <dst>'"};
                continue;
            }
            // ids and weights are range-checked by the store (ExecError /
            // ContractViolation), as the reference leaves them to it
            int64_t s, d, w = 1;
            if (!parse_int(fs[1], fe[1], s) || !parse_int(fs[2], fe[2], d) ||
                (nf == 4 && !parse_int(fs[3], fe[3], w))) {
                err = {lines, "non-integer field"};
                continue;
            }
            out.k.push_back((uint8_t)kind);
            out.a.push_back(s);
            out.b.push_back(d);
            out.c.push_back(w);
        }
    }
}

struct Result {
    Parsed all;
    int64_t err_line = -1;
    std::string err_msg;
};

Result* parse_file(const char* path, int mode) {
    auto* r = new Result;
    FILE* f = fopen(path, "rb");
    if (!f) {
        r->err_line = 0;
        r->err_msg = std::string("cannot open file: ") + strerror(errno);
        return r;
    }
    fseek(f, 0, SEEK_END);
    long sz = ftell(f);
    fseek(f, 0, SEEK_SET);
    std::vector<char> buf((size_t)(sz > 0 ? sz : 0));
    if (sz > 0 && fread(buf.data(), 1, (size_t)sz, f) != (size_t)sz) {
        fclose(f);
        r->err_line = 0;
        r->err_msg = "short read";
        return r;
    }
    fclose(f);
    const char* base = buf.data();
    const size_t n = buf.size();
    int nt = omp_get_max_threads();
    int nchunk = n < (1u << 20) ? 1 : nt * 4;
    // chunk boundaries just after a line end
    std::vector<size_t> cut(nchunk + 1, n);
    cut[0] = 0;
    for (int i = 1; i < nchunk; ++i) {
        size_t c = n * (size_t)i / (size_t)nchunk;
        if (c < cut[i - 1]) c = cut[i - 1];
        while (c < n && !is_eol(base[c])) ++c;
        if (c < n && base[c] == '\r' && c + 1 < n && base[c + 1] == '\n') ++c;
        if (c < n) ++c;
        cut[i] = c;
    }
    std::vector<Parsed> parts(nchunk);
    std::vector<Error> errs(nchunk);
    std::vector<int64_t> lines(nchunk, 0);
#pragma omp parallel for schedule(dynamic, 1)
    for (int i = 0; i < nchunk; ++i)
        parse_chunk(base + cut[i], base + cut[i + 1], mode, parts[i], errs[i], lines[i]);
    // first error in file order; a weighted/unweighted mix across chunks is
    // reported at the first line of the first chunk that disagrees
    int64_t before = 0;
    int w = -1;
    for (int i = 0; i < nchunk; ++i) {
        int64_t bad = errs[i].line >= 0 ? errs[i].line : INT64_MAX;
        std::string msg = errs[i].msg;
        if (mode == 0 && parts[i].weighted >= 0) {
            if (w < 0) {
                w = parts[i].weighted;
            } else if (w != parts[i].weighted) {
                // the chunk is self-consistent, so its first edge line is the
                // first line that disagrees with the chunks before it
                Parsed tmp;
                Error e2;
                int64_t l2 = 0, ln = 0;
                const char* p = base + cut[i];
                const char* e = base + cut[i + 1];
                while (p < e && tmp.a.empty()) {
                    const char* ls = p;
                    while (p < e && !is_eol(*p)) ++p;
                    const char* le = p;
                    if (p < e && *p == '\r' && p + 1 < e && p[1] == '\n') ++p;
                    if (p < e) ++p;
                    ++ln;
                    parse_chunk(ls, le, 0, tmp, e2, l2);
                }
                if (ln < bad) {
                    bad = ln;
                    msg = "mixed weighted/unweighted edge lines";
                }
            }
        }
        if (bad != INT64_MAX) {
            r->err_line = before + bad;
            r->err_msg = msg;
            return r;
        }
        before += lines[i];
    }
    size_t tot = 0;
    for (auto& p : parts) tot += p.a.size();
    Parsed& o = r->all;
    o.a.resize(tot);
    o.b.resize(tot);
    o.c.resize(tot);
    if (mode == 1) o.k.resize(tot);
    size_t off = 0;
    for (auto& p : parts) {
        std::copy(p.a.begin(), p.a.end(), o.a.begin() + off);
        std::copy(p.b.begin(), p.b.end(), o.b.begin() + off);
        std::copy(p.c.begin(), p.c.end(), o.c.begin() + off);
        if (mode == 1) std::copy(p.k.begin(), p.k.end(), o.k.begin() + off);
        off += p.a.size();
        if (p.max_id > o.max_id) o.max_id = p.max_id;
    }
    o.weighted = w < 0 ? 0 : w;
    return r;
}

}  // namespace

extern "C" {

// Parse a graph (mode 0) or update (mode 1) text file.  Returns a handle;
// *count = records, *weighted (edges), *max_id (edges), *err_line = -1 or
// the 1-based line of the first malformed line (0 = I/O error) with the
// message in err (NUL-terminated, truncated to err_cap).
__attribute__((visibility("default"))) void* gdgen_parse_file(const char* path, int mode, int64_t* count,
                                                              int* weighted, int64_t* max_id, int64_t* err_line,
                                                              char* err, int err_cap) {
    Result* r = parse_file(path, mode);
    *count = (int64_t)r->all.a.size();
    *weighted = r->all.weighted;
    *max_id = r->all.max_id;
    *err_line = r->err_line;
    if (err_cap > 0) {
        strncpy(err, r->err_msg.c_str(), (size_t)err_cap - 1);
        err[err_cap - 1] = 0;
    }
    return r;
}

__attribute__((visibility("default"))) void gdgen_parsed_copy(void* h, uint8_t* kind, int64_t* src, int64_t* dst,
                                                              int64_t* w) {
    auto* r = (Result*)h;
    size_t n = r->all.a.size();
    if (n == 0) return;
    memcpy(src, r->all.a.data(), n * 8);
    memcpy(dst, r->all.b.data(), n * 8);
    if (w) memcpy(w, r->all.c.data(), n * 8);
    if (kind && !r->all.k.empty()) memcpy(kind, r->all.k.data(), n);
}

__attribute__((visibility("default"))) void gdgen_parsed_free(void* h) { delete (Result*)h; }

}  // extern "C"
