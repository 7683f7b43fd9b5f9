// Native CONEPROB reader/writer (host code): the reference's text format
// (conefree/fileio.py:1-25) parsed and written by all host cores.
//
// The reference parser (fileio.py:98-190) is a per-line Python loop with a set
// of (i, j) tuples — minutes and 10+ GB at 1e8 nonzeros. This one
// memory-maps the file, finds line starts in parallel, parses entries, b and c
// in parallel into caller-owned arrays, and finds duplicates with a parallel
// bucketed sort. It reproduces the reference's errors exactly: the FIRST
// failing line in file order wins, with the same message text (Python repr()
// quoting included). Inputs outside the handled subset (non-ASCII bytes,
// integers beyond int64) return CF_IO_FALLBACK and the Python restatement in
// binio.py handles them.
//
// Line semantics follow str.splitlines() / str.strip() / str.split() for ASCII:
// breaks are \n, \r, \r\n, \v, \f, \x1c, \x1d, \x1e; whitespace additionally
// includes ' ', \t and \x1f.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <charconv>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/cfb200.h"

namespace {

inline bool is_break(unsigned char c) { return c == '\n' || c == '\r' || c == '\v' || c == '\f' || (c >= 0x1c && c <= 0x1e); }
inline bool is_space(unsigned char c) { return c == ' ' || c == '\t' || is_break(c) || c == 0x1f; }

// Python repr() of an ASCII str
std::string py_repr(const char* s, size_t n) {
    bool has_sq = false, has_dq = false;
    for (size_t i = 0; i < n; ++i) {
        has_sq |= s[i] == '\'';
        has_dq |= s[i] == '"';
    }
    const char q = (has_sq && !has_dq) ? '"' : '\'';
    std::string out(1, q);
    for (size_t i = 0; i < n; ++i) {
        const unsigned char c = (unsigned char)s[i];
        if (c == (unsigned char)q || c == '\\') {
            out += '\\';
            out += (char)c;
        } else if (c == '\t') {
            out += "\\t";
        } else if (c == '\n') {
            out += "\\n";
        } else if (c == '\r') {
            out += "\\r";
        } else if (c < 0x20 || c == 0x7f) {
            char buf[8];
            snprintf(buf, sizeof buf, "\\x%02x", c);
            out += buf;
        } else {
            out += (char)c;
        }
    }
    out += q;
    return out;
}

struct Tok {
    const char* p;
    size_t n;
    std::string str() const { return std::string(p, n); }
    bool eq(const char* s) const { return strlen(s) == n && memcmp(p, s, n) == 0; }
};

// str.split() of one stripped line (at most `cap` tokens are recorded; count returned)
size_t split(const char* b, const char* e, Tok* out, size_t cap) {
    size_t k = 0;
    const char* p = b;
    while (p < e) {
        while (p < e && is_space((unsigned char)*p)) ++p;
        if (p >= e) break;
        const char* q = p;
        while (q < e && !is_space((unsigned char)*q)) ++q;
        if (k < cap) out[k] = Tok{p, (size_t)(q - p)};
        ++k;
        p = q;
    }
    return k;
}

enum { PARSE_OK = 0, PARSE_BAD = 1, PARSE_BIG = 2 };

// int(tok) for base-10 ASCII: [sign] digit (['_'] digit)*
int parse_int(const Tok& t, int64_t* out) {
    size_t i = 0;
    bool neg = false;
    if (i < t.n && (t.p[i] == '+' || t.p[i] == '-')) neg = t.p[i++] == '-';
    if (i >= t.n || t.p[i] < '0' || t.p[i] > '9') return PARSE_BAD;
    unsigned long long v = 0;
    bool big = false, prev_digit = false;
    for (; i < t.n; ++i) {
        const char c = t.p[i];
        if (c >= '0' && c <= '9') {
            if (v > (ULLONG_MAX - 9) / 10) big = true;
            v = v * 10 + (unsigned)(c - '0');
            prev_digit = true;
        } else if (c == '_' && prev_digit && i + 1 < t.n && t.p[i + 1] >= '0' && t.p[i + 1] <= '9') {
            prev_digit = false;
        } else {
            return PARSE_BAD;
        }
    }
    if (big || v > (unsigned long long)INT64_MAX) return PARSE_BIG;
    *out = neg ? -(int64_t)v : (int64_t)v;
    return PARSE_OK;
}

// float(tok) for ASCII (decimal, inf/infinity/nan, underscores between digits)
int parse_float(const Tok& t, double* out) {
    size_t i = 0;
    bool neg = false;
    if (i < t.n && (t.p[i] == '+' || t.p[i] == '-')) neg = t.p[i++] == '-';
    const size_t rest = t.n - i;
    auto ieq = [&](const char* w) {
        const size_t L = strlen(w);
        if (rest != L) return false;
        for (size_t k = 0; k < L; ++k)
            if ((char)tolower((unsigned char)t.p[i + k]) != w[k]) return false;
        return true;
    };
    if (ieq("inf") || ieq("infinity")) {
        *out = neg ? -INFINITY : INFINITY;
        return PARSE_OK;
    }
    if (ieq("nan")) {
        *out = neg ? -NAN : NAN;
        return PARSE_OK;
    }
    // validate the decimal grammar, copying digits without underscores
    char stackbuf[128];
    std::string heap;
    char* buf = stackbuf;
    if (t.n + 2 > sizeof stackbuf) {
        heap.resize(t.n + 2);
        buf = &heap[0];
    }
    size_t w = 0;
    if (neg) buf[w++] = '-';
    auto digits = [&](size_t& k) -> bool {   // digitpart: digit (['_'] digit)*
        if (k >= t.n || t.p[k] < '0' || t.p[k] > '9') return false;
        while (k < t.n) {
            const char c = t.p[k];
            if (c >= '0' && c <= '9') {
                buf[w++] = c;
                ++k;
            } else if (c == '_' && k + 1 < t.n && t.p[k + 1] >= '0' && t.p[k + 1] <= '9') {
                ++k;
            } else {
                break;
            }
        }
        return true;
    };
    size_t k = i;
    bool int_part = false, frac_part = false;
    if (k < t.n && t.p[k] >= '0' && t.p[k] <= '9') int_part = digits(k);
    if (k < t.n && t.p[k] == '.') {
        buf[w++] = '.';
        ++k;
        if (k < t.n && t.p[k] >= '0' && t.p[k] <= '9') frac_part = digits(k);
    }
    if (!int_part && !frac_part) return PARSE_BAD;
    if (k < t.n && (t.p[k] == 'e' || t.p[k] == 'E')) {
        buf[w++] = 'e';
        ++k;
        if (k < t.n && (t.p[k] == '+' || t.p[k] == '-')) buf[w++] = t.p[k++];
        if (!digits(k)) return PARSE_BAD;
    }
    if (k != t.n) return PARSE_BAD;
    buf[w] = 0;
    errno = 0;
    *out = strtod(buf, nullptr);   // glibc strtod: correctly rounded, like float()
    return PARSE_OK;
}

struct Error {
    int64_t line = INT64_MAX;   // 0 = "file ended" class (reported after every line error)
    std::string msg;
    bool set = false;
};

}  // namespace

struct cf_text {
    const char* data = nullptr;
    int64_t len = 0;
    bool mapped = false;
    std::string owned;
    // header results
    int64_t m = 0, n = 0, nnz = 0;
    std::vector<int64_t> sizes;
    int64_t body_off = 0;      // byte offset of the first line after the CONES line
    int64_t body_line = 0;     // its 1-based line number
};

namespace {

// next line [b, e) starting at *pos; advances *pos past the break; false at `len`
inline bool next_line(const char* data, int64_t len, int64_t* pos, const char** b, const char** e) {
    if (*pos >= len) return false;
    const char* s = data + *pos;
    const char* end = data + len;
    const char* q = s;
    while (q < end && !is_break((unsigned char)*q)) ++q;
    *b = s;
    *e = q;
    if (q < end) {
        if (*q == '\r' && q + 1 < end && q[1] == '\n')
            q += 2;
        else
            q += 1;
    }
    *pos = q - data;
    return true;
}

// strip; returns false for blank or '#' lines
inline bool content(const char*& b, const char*& e) {
    while (b < e && is_space((unsigned char)*b)) ++b;
    while (e > b && is_space((unsigned char)e[-1])) --e;
    return b < e && *b != '#';
}

void set_msg(char* msg, int64_t cap, const std::string& s) {
    if (!msg || cap <= 0) return;
    const size_t n = std::min<size_t>(s.size(), (size_t)cap - 1);
    memcpy(msg, s.data(), n);
    msg[n] = 0;
}

int fail(int64_t* err_line, char* msg, int64_t cap, int64_t line, const std::string& s) {
    if (err_line) *err_line = line;
    set_msg(msg, cap, s);
    return CF_IO_PARSE;
}

int n_threads(int req) {
    if (req > 0) return std::min(req, 256);
    const unsigned hw = std::thread::hardware_concurrency();
    return (int)std::max(1u, std::min(hw ? hw : 4u, 64u));
}

}  // namespace

extern "C" {

int cf_coneprob_open(const char* path, const char* text, int64_t len, cf_text** out) {
    if (!out) return CF_EINVAL;
    *out = nullptr;
    cf_text* t = new cf_text();
    if (path) {
        const int fd = open(path, O_RDONLY);
        if (fd < 0) {
            delete t;
            return CF_EINVAL;
        }
        struct stat st;
        if (fstat(fd, &st) != 0) {
            close(fd);
            delete t;
            return CF_EINVAL;
        }
        t->len = (int64_t)st.st_size;
        if (t->len > 0) {
            void* p = mmap(nullptr, (size_t)t->len, PROT_READ, MAP_PRIVATE, fd, 0);
            if (p == MAP_FAILED) {
                close(fd);
                delete t;
                return CF_EINVAL;
            }
            madvise(p, (size_t)t->len, MADV_SEQUENTIAL);
            t->data = static_cast<const char*>(p);
            t->mapped = true;
        } else {
            t->data = "";
        }
        close(fd);
    } else {
        t->owned.assign(text ? text : "", text ? (size_t)len : 0);
        t->data = t->owned.data();
        t->len = (int64_t)t->owned.size();
    }
    *out = t;
    return CF_OK;
}

void cf_coneprob_close(cf_text* t) {
    if (!t) return;
    if (t->mapped && t->len > 0) munmap(const_cast<char*>(t->data), (size_t)t->len);
    delete t;
}

// header, dimensions and CONES line (fileio.py:98-138)
int cf_coneprob_header(cf_text* t, int64_t dims[4], int64_t* err_line, char* msg, int64_t cap) {
    if (!t || !dims) return CF_EINVAL;
    // the handled subset is ASCII (str.splitlines/strip/split have more
    // separators for non-ASCII text); the header bytes are checked here, the
    // body bytes by cf_coneprob_body
    int64_t pos = 0, line = 0;
    const char *b, *e;
    auto take = [&](const char* what, int64_t* num, const char** lb, const char** le) -> int {
        while (next_line(t->data, t->len, &pos, &b, &e)) {
            for (const char* q = b; q < e; ++q)
                if ((unsigned char)*q >= 0x80) return CF_IO_FALLBACK;
            ++line;
            if (content(b, e)) {
                *num = line;
                *lb = b;
                *le = e;
                return CF_OK;
            }
        }
        return fail(err_line, msg, cap, 0, std::string("file ended before ") + what);
    };
    int64_t num;
    const char *lb, *le;
    int rc = take("header", &num, &lb, &le);
    if (rc) return rc;
    if (!(le - lb == 10 && memcmp(lb, "CONEPROB 1", 10) == 0))
        return fail(err_line, msg, cap, num,
                    "expected 'CONEPROB 1' header, got " + py_repr(lb, (size_t)(le - lb)));
    rc = take("dimensions", &num, &lb, &le);
    if (rc) return rc;
    Tok tk[4];
    size_t nt = split(lb, le, tk, 4);
    if (nt != 3) return fail(err_line, msg, cap, num, "expected 'm n nnz', got " + py_repr(lb, (size_t)(le - lb)));
    int64_t v[3];
    const char* what[3] = {"m", "n", "nnz"};
    for (int k = 0; k < 3; ++k) {
        const int r = parse_int(tk[k], &v[k]);
        if (r == PARSE_BIG) return CF_IO_FALLBACK;
        if (r != PARSE_OK)
            return fail(err_line, msg, cap, num,
                        std::string("expected integer ") + what[k] + ", got " + py_repr(tk[k].p, tk[k].n));
    }
    if (v[0] < 1 || v[1] < 1 || v[2] < 0)
        return fail(err_line, msg, cap, num,
                    "bad dimensions m=" + std::to_string(v[0]) + " n=" + std::to_string(v[1]) +
                        " nnz=" + std::to_string(v[2]));
    if (v[0] > INT32_MAX || v[1] > INT32_MAX || v[2] > ((int64_t)1 << 40)) return CF_IO_FALLBACK;
    rc = take("CONES line", &num, &lb, &le);
    if (rc) return rc;
    // tokens of the CONES line (may hold n block sizes)
    std::vector<Tok> ct;
    {
        const char* p = lb;
        while (p < le) {
            while (p < le && is_space((unsigned char)*p)) ++p;
            if (p >= le) break;
            const char* q = p;
            while (q < le && !is_space((unsigned char)*q)) ++q;
            ct.push_back(Tok{p, (size_t)(q - p)});
            p = q;
        }
    }
    if (ct.empty() || !ct[0].eq("CONES"))
        return fail(err_line, msg, cap, num, "expected 'CONES ...', got " + py_repr(lb, (size_t)(le - lb)));
    if (ct.size() < 2) return fail(err_line, msg, cap, num, "CONES line missing block count");
    int64_t count;
    {
        const int r = parse_int(ct[1], &count);
        if (r == PARSE_BIG) return CF_IO_FALLBACK;
        if (r != PARSE_OK)
            return fail(err_line, msg, cap, num, "expected integer cone block count, got " + py_repr(ct[1].p, ct[1].n));
    }
    if ((int64_t)ct.size() != 2 + count)
        return fail(err_line, msg, cap, num,
                    "CONES declares " + std::to_string(count) + " blocks but lists " + std::to_string(ct.size() - 2));
    t->sizes.resize((size_t)count);
    for (int64_t q = 0; q < count; ++q) {
        const int r = parse_int(ct[2 + q], &t->sizes[q]);
        if (r == PARSE_BIG) return CF_IO_FALLBACK;
        if (r != PARSE_OK)
            return fail(err_line, msg, cap, num, "expected integer cone size, got " + py_repr(ct[2 + q].p, ct[2 + q].n));
    }
    __int128 total = 0;
    for (int64_t s : t->sizes) {
        if (s < 1) return fail(err_line, msg, cap, num, "cone size " + std::to_string(s) + " < 1");
        total += s;
    }
    if (total != v[1]) {
        if (total > INT64_MAX) return CF_IO_FALLBACK;
        return fail(err_line, msg, cap, num,
                    "cone sizes sum " + std::to_string((int64_t)total) + " != n=" + std::to_string(v[1]));
    }
    t->m = v[0];
    t->n = v[1];
    t->nnz = v[2];
    t->body_off = pos;
    t->body_line = line + 1;
    dims[0] = t->m;
    dims[1] = t->n;
    dims[2] = t->nnz;
    dims[3] = count;
    return CF_OK;
}

int cf_coneprob_sizes(const cf_text* t, int64_t* sizes) {
    if (!t || (!sizes && !t->sizes.empty())) return CF_EINVAL;
    std::copy(t->sizes.begin(), t->sizes.end(), sizes);
    return CF_OK;
}

// entries, b, c and trailing content (fileio.py:140-190), in parallel
int cf_coneprob_body(cf_text* t, int64_t* rows, int64_t* cols, double* vals, double* b, double* c, int threads,
                     int64_t* err_line, char* msg, int64_t cap) {
    if (!t) return CF_EINVAL;
    const int64_t m = t->m, n = t->n, nnz = t->nnz;
    const int64_t need = nnz + m + n;   // content lines after the CONES line
    const int T = n_threads(threads);
    const int64_t L = t->len - t->body_off;
    // ---- chunk boundaries at line starts
    const int C = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)T * 4, L / (1 << 16) + 1));
    std::vector<int64_t> cut(C + 1);
    cut[0] = t->body_off;
    cut[C] = t->len;
    for (int k = 1; k < C; ++k) {
        int64_t p = t->body_off + L * k / C;
        p = std::max(p, cut[k - 1]);
        while (p < t->len && !is_break((unsigned char)t->data[p])) ++p;
        if (p < t->len) p += (t->data[p] == '\r' && p + 1 < t->len && t->data[p + 1] == '\n') ? 2 : 1;
        cut[k] = p;
    }
    // ---- pass 1: lines and content lines per chunk (and the ASCII check)
    std::vector<int64_t> nlines(C, 0), ncontent(C, 0);
    std::atomic<int> non_ascii{0};
    auto run = [&](auto&& fn) {
        std::atomic<int> next{0};
        std::vector<std::thread> th;
        for (int w = 0; w < std::min(T, C); ++w)
            th.emplace_back([&]() {
                for (int k = next++; k < C; k = next++) fn(k);
            });
        for (auto& x : th) x.join();
    };
    run([&](int k) {
        for (int64_t q = cut[k]; q < cut[k + 1]; ++q)
            if ((unsigned char)t->data[q] >= 0x80) {
                non_ascii = 1;
                return;
            }
        int64_t pos = cut[k];
        const char *lb, *le;
        int64_t nl = 0, nc = 0;
        while (next_line(t->data, cut[k + 1], &pos, &lb, &le)) {
            ++nl;
            nc += content(lb, le);
        }
        nlines[k] = nl;
        ncontent[k] = nc;
    });
    if (non_ascii) return CF_IO_FALLBACK;
    std::vector<int64_t> line0(C), cidx0(C);
    int64_t ln = t->body_line, ci = 0;
    for (int k = 0; k < C; ++k) {
        line0[k] = ln;
        cidx0[k] = ci;
        ln += nlines[k];
        ci += ncontent[k];
    }
    const int64_t total_content = ci;
    // ---- pass 2: parse; each chunk keeps its first error
    std::vector<Error> errs(C);
    std::vector<int64_t> valid_entries(C, 0);   // entries parsed before the chunk's first error
    std::atomic<int> fallback{0};
    run([&](int k) {
        int64_t pos = cut[k];
        const char *lb, *le;
        int64_t line = line0[k] - 1, cidx = cidx0[k];
        Error& er = errs[k];
        auto err = [&](const std::string& s) {
            er.line = line;
            er.msg = s;
            er.set = true;
        };
        Tok tk[4];
        while (next_line(t->data, cut[k + 1], &pos, &lb, &le)) {
            ++line;
            if (!content(lb, le)) continue;
            const int64_t idx = cidx++;
            if (idx < nnz) {
                const size_t nt = split(lb, le, tk, 4);
                if (nt != 3) {
                    err("expected 'i j value', got " + py_repr(lb, (size_t)(le - lb)));
                    return;
                }
                int64_t i, j;
                double v;
                int r = parse_int(tk[0], &i);
                if (r == PARSE_BIG) {
                    fallback = 1;
                    return;
                }
                if (r != PARSE_OK) {
                    err("expected integer row index, got " + py_repr(tk[0].p, tk[0].n));
                    return;
                }
                r = parse_int(tk[1], &j);
                if (r == PARSE_BIG) {
                    fallback = 1;
                    return;
                }
                if (r != PARSE_OK) {
                    err("expected integer column index, got " + py_repr(tk[1].p, tk[1].n));
                    return;
                }
                if (parse_float(tk[2], &v) != PARSE_OK) {
                    err("expected number value, got " + py_repr(tk[2].p, tk[2].n));
                    return;
                }
                if (!(0 <= i && i < m)) {
                    err("row index " + std::to_string(i) + " outside [0, " + std::to_string(m) + ")");
                    return;
                }
                if (!(0 <= j && j < n)) {
                    err("column index " + std::to_string(j) + " outside [0, " + std::to_string(n) + ")");
                    return;
                }
                if (!std::isfinite(v)) {
                    err("value " + tk[2].str() + " is not finite");
                    return;
                }
                if (v == 0.0) {
                    err("zero value at (" + std::to_string(i) + ", " + std::to_string(j) + ")");
                    return;
                }
                rows[idx] = i;
                cols[idx] = j;
                vals[idx] = v;
                ++valid_entries[k];
            } else if (idx < need) {
                const bool isb = idx < nnz + m;
                const int64_t q = isb ? idx - nnz : idx - nnz - m;
                const std::string name = std::string(isb ? "b" : "c") + "[" + std::to_string(q) + "]";
                double v;
                const Tok whole{lb, (size_t)(le - lb)};
                if (parse_float(whole, &v) != PARSE_OK) {
                    err("expected number " + name + ", got " + py_repr(lb, (size_t)(le - lb)));
                    return;
                }
                if (!std::isfinite(v)) {
                    err(name + " = " + whole.str() + " is not finite");
                    return;
                }
                if (isb)
                    b[q] = v;
                else
                    c[q] = v;
            } else {
                err("unexpected trailing content " + py_repr(lb, (size_t)(le - lb)));
                return;
            }
        }
    });
    if (fallback) return CF_IO_FALLBACK;
    // first line error in file order
    Error first;
    for (int k = 0; k < C; ++k)
        if (errs[k].set) {
            first = errs[k];
            break;
        }
    // entries known good: those before the first error (all, if none)
    int64_t good = 0;
    for (int k = 0; k < C; ++k) {
        good += valid_entries[k];
        if (errs[k].set) break;
    }
    good = std::min(good, nnz);
    // ---- duplicates among the good entries: bucketed parallel sort of (key, k)
    int64_t dup_k = -1;
    if (good > 1) {
        const int B = std::max(1, T * 4);
        const unsigned __int128 cells = (unsigned __int128)m * (unsigned __int128)n;
        std::vector<std::vector<std::pair<int64_t, int64_t>>> bucket(B);
        {
            // per-thread scatter into per-thread buckets, then concatenate
            const int W = std::min<int64_t>(T, good);
            std::vector<std::vector<std::vector<std::pair<int64_t, int64_t>>>> part(
                W, std::vector<std::vector<std::pair<int64_t, int64_t>>>(B));
            std::vector<std::thread> th;
            for (int w = 0; w < W; ++w)
                th.emplace_back([&, w]() {
                    const int64_t a = good * w / W, z = good * (w + 1) / W;
                    for (auto& v : part[w]) v.reserve((size_t)((z - a) / B + 16));
                    for (int64_t k = a; k < z; ++k) {
                        const int64_t key = rows[k] * n + cols[k];
                        const int bk = (int)((unsigned __int128)key * B / cells);
                        part[w][bk].push_back({key, k});
                    }
                });
            for (auto& x : th) x.join();
            th.clear();
            for (int bk = 0; bk < B; ++bk) {
                size_t tot = 0;
                for (int w = 0; w < W; ++w) tot += part[w][bk].size();
                bucket[bk].reserve(tot);
                for (int w = 0; w < W; ++w) {
                    bucket[bk].insert(bucket[bk].end(), part[w][bk].begin(), part[w][bk].end());
                    std::vector<std::pair<int64_t, int64_t>>().swap(part[w][bk]);
                }
            }
        }
        std::vector<int64_t> bdup(B, -1);
        std::atomic<int> next{0};
        std::vector<std::thread> th;
        for (int w = 0; w < std::min(T, B); ++w)
            th.emplace_back([&]() {
                for (int bk = next++; bk < B; bk = next++) {
                    auto& v = bucket[bk];
                    std::sort(v.begin(), v.end());
                    // sorted by (key, entry): the second element of a run of equal keys is
                    // the first repeat in file order, where the reference raises
                    int64_t best = -1;
                    for (size_t q = 1; q < v.size(); ++q)
                        if (v[q].first == v[q - 1].first && (q == 1 || v[q - 2].first != v[q].first))
                            if (best < 0 || v[q].second < best) best = v[q].second;
                    bdup[bk] = best;
                }
            });
        for (auto& x : th) x.join();
        for (int64_t d : bdup)
            if (d >= 0 && (dup_k < 0 || d < dup_k)) dup_k = d;
    }
    if (dup_k >= 0) {
        // line of entry dup_k: re-scan its chunk
        int k = 0;
        while (k + 1 < C && cidx0[k + 1] <= dup_k) ++k;
        int64_t pos = cut[k];
        const char *lb, *le;
        int64_t line = line0[k] - 1, cidx = cidx0[k];
        while (next_line(t->data, cut[k + 1], &pos, &lb, &le)) {
            ++line;
            if (!content(lb, le)) continue;
            if (cidx++ == dup_k) break;
        }
        if (!first.set || line < first.line)
            return fail(err_line, msg, cap, line,
                        "duplicate entry at (" + std::to_string(rows[dup_k]) + ", " + std::to_string(cols[dup_k]) + ")");
    }
    if (first.set) return fail(err_line, msg, cap, first.line, first.msg);
    if (total_content < need) {
        const int64_t idx = total_content;
        std::string what;
        if (idx < nnz)
            what = "entry " + std::to_string(idx);
        else if (idx < nnz + m)
            what = "b[" + std::to_string(idx - nnz) + "]";
        else
            what = "c[" + std::to_string(idx - nnz - m) + "]";
        return fail(err_line, msg, cap, 0, "file ended before " + what);
    }
    return CF_OK;
}

// ---------------------------------------------------------------- writer
// Python repr(float) (PyOS_double_to_string 'r' with Py_DTSF_ADD_DOT_0):
// shortest round-trip digits; fixed notation for -4 <= exponent < 16.
int cf_format_double(double x, char* out) {
    if (std::isnan(x)) return (int)(stpcpy(out, "nan") - out);
    if (std::isinf(x)) return (int)(stpcpy(out, x < 0 ? "-inf" : "inf") - out);
    char sci[64];
    const auto r = std::to_chars(sci, sci + sizeof sci, x, std::chars_format::scientific);
    *r.ptr = 0;
    // sci = [-]d[.ddd]e(+|-)XX
    const char* p = sci;
    char* o = out;
    if (*p == '-') *o++ = *p++;
    char digs[32];
    int nd = 0;
    while (*p && *p != 'e') {
        if (*p != '.') digs[nd++] = *p;
        ++p;
    }
    const int e10 = atoi(p + 1);   // value = d.ddd x 10^e10
    while (nd > 1 && digs[nd - 1] == '0') --nd;
    const int decpt = e10 + 1;     // value = 0.ddd x 10^decpt
    if (decpt <= -4 || decpt > 16) {
        *o++ = digs[0];
        if (nd > 1) {
            *o++ = '.';
            for (int k = 1; k < nd; ++k) *o++ = digs[k];
        }
        o += sprintf(o, "e%c%02d", e10 < 0 ? '-' : '+', e10 < 0 ? -e10 : e10);
    } else if (decpt <= 0) {
        *o++ = '0';
        *o++ = '.';
        for (int k = 0; k < -decpt; ++k) *o++ = '0';
        for (int k = 0; k < nd; ++k) *o++ = digs[k];
    } else if (decpt >= nd) {
        for (int k = 0; k < nd; ++k) *o++ = digs[k];
        for (int k = nd; k < decpt; ++k) *o++ = '0';
        *o++ = '.';
        *o++ = '0';
    } else {
        for (int k = 0; k < decpt; ++k) *o++ = digs[k];
        *o++ = '.';
        for (int k = decpt; k < nd; ++k) *o++ = digs[k];
    }
    *o = 0;
    return (int)(o - out);
}

// write_problem (fileio.py:56-72) for entries already in canonical order; writes `path`
int cf_coneprob_write(const char* path, int64_t m, int64_t n, int64_t nnz, const int64_t* rows, const int64_t* cols,
                      const double* vals, const double* b, const double* c, int64_t n_blocks, const int64_t* sizes,
                      int threads) {
    if (!path) return CF_EINVAL;
    FILE* f = fopen(path, "wb");
    if (!f) return CF_EINVAL;
    std::string head = "CONEPROB 1\n" + std::to_string(m) + " " + std::to_string(n) + " " + std::to_string(nnz) +
                       "\nCONES " + std::to_string(n_blocks);
    head.reserve(head.size() + (size_t)n_blocks * 3 + 2);
    for (int64_t q = 0; q < n_blocks; ++q) {
        head += ' ';
        head += std::to_string(sizes[q]);
    }
    head += '\n';
    bool ok = fwrite(head.data(), 1, head.size(), f) == head.size();
    // lines 0..nnz-1 entries, then b, then c; formatted in parallel blocks
    const int64_t total = nnz + m + n;
    const int T = n_threads(threads);
    const int64_t block = 1 << 20;
    std::vector<std::string> buf(T);
    for (int64_t base = 0; base < total && ok; base += block * T) {
        std::vector<std::thread> th;
        for (int w = 0; w < T; ++w)
            th.emplace_back([&, w]() {
                std::string& s = buf[w];
                s.clear();
                const int64_t a = base + block * w, z = std::min(total, a + block);
                char tmp[64];
                for (int64_t k = a; k < z; ++k) {
                    if (k < nnz) {
                        s += std::to_string(rows[k]);
                        s += ' ';
                        s += std::to_string(cols[k]);
                        s += ' ';
                        s.append(tmp, (size_t)cf_format_double(vals[k], tmp));
                    } else if (k < nnz + m) {
                        s.append(tmp, (size_t)cf_format_double(b[k - nnz], tmp));
                    } else {
                        s.append(tmp, (size_t)cf_format_double(c[k - nnz - m], tmp));
                    }
                    s += '\n';
                }
            });
        for (auto& x : th) x.join();
        for (int w = 0; w < T && ok; ++w) ok = fwrite(buf[w].data(), 1, buf[w].size(), f) == buf[w].size();
    }
    ok = (fclose(f) == 0) && ok;
    return ok ? CF_OK : CF_EINVAL;
}

int cf_solution_write(const char* path, const char* head, const double* x, int64_t n, const double* lam, int64_t m,
                      int threads) {
    if (!path || !head || n < 0 || m < 0) return CF_EINVAL;
    FILE* f = fopen(path, "wb");
    if (!f) return CF_EINVAL;
    const size_t hl = strlen(head);
    bool ok = fwrite(head, 1, hl, f) == hl;
    // x then lam, one repr per line, formatted in parallel blocks (fileio.py:198-199)
    const int64_t total = n + m;
    const int T = n_threads(threads);
    const int64_t block = 1 << 20;
    std::vector<std::string> buf(T);
    for (int64_t base = 0; base < total && ok; base += block * T) {
        std::vector<std::thread> th;
        for (int w = 0; w < T; ++w)
            th.emplace_back([&, w]() {
                std::string& s = buf[w];
                s.clear();
                const int64_t a = base + block * w, z = std::min(total, a + block);
                char tmp[64];
                for (int64_t k = a; k < z; ++k) {
                    s.append(tmp, (size_t)cf_format_double(k < n ? x[k] : lam[k - n], tmp));
                    s += '\n';
                }
            });
        for (auto& t : th) t.join();
        for (int w = 0; w < T && ok; ++w) ok = fwrite(buf[w].data(), 1, buf[w].size(), f) == buf[w].size();
    }
    ok = (fclose(f) == 0) && ok;
    return ok ? CF_OK : CF_EINVAL;
}

}  // extern "C"
