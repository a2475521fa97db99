// io.cu -- edge-list text I/O on the host (rmat.py:211-286, save_edge_list /
// load_edge_list "text" format): one "u v" pair per line, '#' comment lines, and
// an optional "# n <count>" comment that fixes the vertex count.
//
// The reference parses line by line in Python (int() per token); this is a
// single pass over the mapped file with the same line rules:
//   * lines end at \n, \r\n or \r (Python text mode, universal newlines);
//   * each line is stripped of ASCII whitespace; empty lines are skipped;
//   * a '#' line is a comment; if its remaining tokens are exactly ["n", X] then
//     X is the header vertex count (the last such line wins);
//   * any other line must hold exactly two integer tokens (optional sign,
//     digits with single '_' separators, as int() accepts), else FormatError
//     "<line>: expected 'src dst', got '<line>'" / "<line>: invalid literal ...".
// Range checks (ids in [0, n)) stay in the Python shell, as in the reference.
#include <cerrno>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"

namespace dbfs {
namespace {

inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\v' || c == '\f'; }

// int() on one token: [+-]?digit(_?digit)*.  Returns false on a malformed token;
// *overflow is set when the value does not fit int64.
bool parse_int(const char *b, const char *e, int64_t *out, bool *overflow) {
    *overflow = false;
    bool neg = false;
    if (b < e && (*b == '+' || *b == '-')) neg = *b++ == '-';
    if (b == e) return false;
    unsigned long long v = 0;
    bool prev_digit = false;
    for (const char *p = b; p < e; p++) {
        if (*p == '_') {
            if (!prev_digit || p + 1 == e) return false;
            prev_digit = false;
            continue;
        }
        if (*p < '0' || *p > '9') return false;
        unsigned d = (unsigned)(*p - '0');
        if (v > (0x7fffffffffffffffULL - d) / 10ULL) *overflow = true;
        else v = v * 10ULL + d;
        prev_digit = true;
    }
    *out = neg ? -(int64_t)v : (int64_t)v;
    return true;
}

std::string quote(const char *b, const char *e) {
    std::string s(b, (size_t)(e - b));
    if (s.size() > 200) s = s.substr(0, 200) + "...";
    return "'" + s + "'";
}

}  // namespace

int64_t count_text_lines(const char *buf, int64_t len) {
    int64_t lines = 1;
    for (int64_t i = 0; i < len; i++) lines += buf[i] == '\n' || buf[i] == '\r';
    return lines;
}

void parse_edge_text(const char *buf, int64_t len, int64_t cap, int64_t *src, int64_t *dst, int64_t *m_out,
                     int64_t *header_n) {
    int64_t m = 0, lineno = 0;
    *header_n = -1;
    const char *p = buf, *end = buf + len;
    while (p < end) {
        const char *ls = p;
        while (p < end && *p != '\n' && *p != '\r') p++;
        const char *le = p;
        if (p < end) p += (*p == '\r' && p + 1 < end && p[1] == '\n') ? 2 : 1;
        lineno++;
        while (ls < le && is_ws(*ls)) ls++;
        while (le > ls && is_ws(le[-1])) le--;
        if (ls == le) continue;
        // split into at most 3 whitespace-separated tokens
        const char *tb[3], *te[3];
        int nt = 0;
        const char *q = ls + (*ls == '#' ? 1 : 0);
        while (q < le) {
            while (q < le && is_ws(*q)) q++;
            if (q == le) break;
            const char *t = q;
            while (q < le && !is_ws(*q)) q++;
            if (nt < 3) {
                tb[nt] = t;
                te[nt] = q;
            }
            nt++;
        }
        bool ovf = false;
        int64_t a = 0, b = 0;
        if (*ls == '#') {
            if (nt == 2 && te[0] - tb[0] == 1 && *tb[0] == 'n') {
                DBFS_CHECK(parse_int(tb[1], te[1], &a, &ovf) && !ovf, DBFS_EINVAL,
                           "invalid literal for int() with base 10: " + quote(tb[1], te[1]));
                *header_n = a;
            }
            continue;
        }
        DBFS_CHECK(nt == 2, DBFS_EFORMAT,
                   std::to_string(lineno) + ": expected 'src dst', got " + quote(ls, le));
        for (int t = 0; t < 2; t++) {
            int64_t *v = t ? &b : &a;
            DBFS_CHECK(parse_int(tb[t], te[t], v, &ovf), DBFS_EFORMAT,
                       std::to_string(lineno) + ": invalid literal for int() with base 10: " + quote(tb[t], te[t]));
            DBFS_CHECK(!ovf, DBFS_EFORMAT, std::to_string(lineno) + ": vertex id overflow");
        }
        DBFS_CHECK(m < cap, DBFS_EINTERNAL, "edge capacity exceeded");
        src[m] = a;
        dst[m] = b;
        m++;
    }
    *m_out = m;
}

namespace {
inline char *put_u64(char *o, unsigned long long v) {
    char tmp[24];
    int k = 0;
    do {
        tmp[k++] = (char)('0' + v % 10);
        v /= 10;
    } while (v);
    while (k) *o++ = tmp[--k];
    return o;
}
inline char *put_i64(char *o, int64_t v) {
    if (v < 0) {
        *o++ = '-';
        return put_u64(o, 0ULL - (unsigned long long)v);
    }
    return put_u64(o, (unsigned long long)v);
}
}  // namespace

void write_edge_text(const char *path, int64_t n, const int64_t *src, const int64_t *dst, int64_t m) {
    FILE *f = std::fopen(path, "wb");
    DBFS_CHECK(f, DBFS_EIO, std::string("cannot open ") + path + " for writing: " + std::strerror(errno));
    std::vector<char> buf(1 << 22);
    char *o = buf.data();
    char *lim = buf.data() + buf.size() - 64;
    bool ok = true;
    o = std::strcpy(o, "# n ") + 4;
    o = put_i64(o, n);
    *o++ = '\n';
    for (int64_t i = 0; i < m && ok; i++) {
        o = put_i64(o, src[i]);
        *o++ = ' ';
        o = put_i64(o, dst[i]);
        *o++ = '\n';
        if (o >= lim) {
            ok = std::fwrite(buf.data(), 1, (size_t)(o - buf.data()), f) == (size_t)(o - buf.data());
            o = buf.data();
        }
    }
    if (ok && o > buf.data()) ok = std::fwrite(buf.data(), 1, (size_t)(o - buf.data()), f) == (size_t)(o - buf.data());
    ok = (std::fclose(f) == 0) && ok;
    DBFS_CHECK(ok, DBFS_EIO, std::string("write to ") + path + " failed");
}

}  // namespace dbfs
