// ingest.cu — multi-threaded svmlight parser (host C++), the step before the
// device data layer.
//
// Reference: parse_svmlight (data.py:190-239): `<label> <idx>:<val> ...` per
// line, 1-based strictly increasing indices, blank and '#' lines skipped; the
// result is the example-major CSC (columns = examples, n_rows = max index)
// plus the labels.  Numbers follow Python's float()/int() grammar (optional
// sign, digits with single underscores between them, '.', exponent,
// inf/infinity/nan) and are converted by strtod, which rounds correctly like
// float(); anything else is reported with the reference's error kinds and
// line numbers (the Python layer formats the messages).
//
// The text is cut at line boundaries into one piece per thread; each thread
// parses its piece into local arrays, then the pieces are concatenated.
#include <cerrno>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace glm {
namespace {

enum { ING_OK = 0, ING_BAD_LABEL = 1, ING_BAD_TOKEN = 2, ING_INDEX_LT1 = 3, ING_NOT_INCREASING = 4,
       ING_INDEX_RANGE = 5 };

inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }
inline bool is_digit(char c) { return c >= '0' && c <= '9'; }

// digits with single underscores strictly between digits; appends the digits
bool take_digits(const char *&p, const char *e, std::string &out) {
    if (p >= e || !is_digit(*p)) return false;
    while (p < e) {
        if (is_digit(*p)) {
            out.push_back(*p++);
        } else if (*p == '_' && p + 1 < e && is_digit(p[1]) && is_digit(p[-1])) {
            ++p;
        } else {
            break;
        }
    }
    return true;
}

bool ieq(const char *p, const char *e, const char *word) {
    const size_t n = strlen(word);
    if ((size_t)(e - p) != n) return false;
    for (size_t i = 0; i < n; ++i) {
        char c = p[i];
        if (c >= 'A' && c <= 'Z') c = (char)(c - 'A' + 'a');
        if (c != word[i]) return false;
    }
    return true;
}

// Python float(token) for an ASCII token without surrounding whitespace.
bool parse_float(const char *p, const char *e, double &out, std::string &buf) {
    buf.clear();
    const char *q = p;
    if (q < e && (*q == '+' || *q == '-')) buf.push_back(*q++);
    if (ieq(q, e, "inf") || ieq(q, e, "infinity") || ieq(q, e, "nan")) {
        buf.append(q, e);
        out = strtod(buf.c_str(), nullptr);
        return true;
    }
    bool mant = false;
    if (q < e && is_digit(*q)) mant = take_digits(q, e, buf);
    if (q < e && *q == '.') {
        buf.push_back(*q++);
        if (q < e && is_digit(*q)) mant = take_digits(q, e, buf) || mant;
    }
    if (!mant) return false;
    if (q < e && (*q == 'e' || *q == 'E')) {
        buf.push_back(*q++);
        if (q < e && (*q == '+' || *q == '-')) buf.push_back(*q++);
        if (!take_digits(q, e, buf)) return false;
    }
    if (q != e) return false;
    errno = 0;
    out = strtod(buf.c_str(), nullptr);   // ERANGE overflow -> inf, like float()
    return true;
}

// Python int(token) -> int64 (false on grammar error; range flagged separately)
bool parse_int(const char *p, const char *e, long long &out, bool &range, std::string &buf) {
    buf.clear();
    const char *q = p;
    bool neg = false;
    if (q < e && (*q == '+' || *q == '-')) neg = *q++ == '-';
    if (!take_digits(q, e, buf) || q != e) return false;
    range = buf.size() > 18;
    out = range ? 0 : strtoll(buf.c_str(), nullptr, 10);
    if (neg) out = -out;
    return true;
}

struct Piece {
    const char *b = nullptr, *e = nullptr;
    int64_t first_line = 0;           // 1-based number of the piece's first line
    std::vector<int64_t> counts;      // nnz per example
    std::vector<int32_t> rows;
    std::vector<double> vals, labels;
    int64_t max_feat = 0;
    int err = ING_OK;
    int64_t err_line = 0, tok_off = 0, tok_len = 0;
    // an index beyond int32 is not a format error: the reference only fails
    // when it converts the finished row list (np.asarray(rows, int32)), so a
    // later format error wins; the first such token is kept
    int64_t range_line = 0, range_off = -1, range_len = 0;
};

void parse_piece(const char *base, Piece &P) {
    std::string buf;
    int64_t line = P.first_line;
    const char *p = P.b;
    while (p < P.e) {
        const char *nl = (const char *)memchr(p, '\n', P.e - p);
        const char *le = nl ? nl : P.e;
        const char *q = p;
        while (q < le && is_ws(*q)) ++q;
        const char *qe = le;
        while (qe > q && is_ws(qe[-1])) --qe;
        if (q < qe && *q != '#') {
            const char *t = q;
            while (t < qe && !is_ws(*t)) ++t;
            double y;
            if (!parse_float(q, t, y, buf)) {
                P.err = ING_BAD_LABEL;
                P.err_line = line;
                P.tok_off = q - base;
                P.tok_len = t - q;
                return;
            }
            long long prev = 0;
            int64_t cnt = 0;
            while (t < qe) {
                while (t < qe && is_ws(*t)) ++t;
                if (t >= qe) break;
                const char *s = t;
                while (t < qe && !is_ws(*t)) ++t;
                const char *colon = (const char *)memchr(s, ':', t - s);
                long long idx = 0;
                bool range = false;
                double v;
                if (!colon || !parse_int(s, colon, idx, range, buf) ||
                    !parse_float(colon + 1, t, v, buf)) {
                    P.err = ING_BAD_TOKEN;
                } else if (idx < 1) {
                    P.err = ING_INDEX_LT1;
                } else if (idx <= prev) {
                    P.err = ING_NOT_INCREASING;
                } else if ((range || idx > (long long)INT32_MAX + 1) && P.range_off < 0) {
                    P.range_line = line;
                    P.range_off = s - base;
                    P.range_len = t - s;
                }
                if (P.err) {
                    P.err_line = line;
                    P.tok_off = s - base;
                    P.tok_len = t - s;
                    return;
                }
                prev = range ? LLONG_MAX : idx;
                P.rows.push_back((int32_t)(idx - 1));
                P.vals.push_back(v);
                ++cnt;
            }
            if (prev > P.max_feat) P.max_feat = prev;
            P.labels.push_back(y);
            P.counts.push_back(cnt);
        }
        ++line;
        p = nl ? nl + 1 : P.e;
    }
}

}  // namespace
}  // namespace glm

struct glm_svmlight {
    std::vector<glm::Piece> pieces;
    int64_t n = 0, nnz = 0, max_feat = 0;
};

using namespace glm;

extern "C" {

int glm_svmlight_parse(const char *text, int64_t len, int n_threads, glm_svmlight **out,
                       int64_t *info) {
    if (!out || !info || (len > 0 && !text)) return glm_set_error(GLM_USAGE, "null argument");
    glm_svmlight *r = new (std::nothrow) glm_svmlight();
    if (!r) return glm_set_error(GLM_USAGE, "out of host memory");
    int T = n_threads > 0 ? n_threads : (int)std::thread::hardware_concurrency();
    if (T < 1) T = 1;
    if (len < (1 << 20)) T = 1;       // small inputs: one piece
    // cut at line boundaries
    std::vector<const char *> cut{text};
    for (int i = 1; i < T; ++i) {
        const char *c = text + len * i / T;
        if (c < cut.back()) c = cut.back();
        const char *nl = (const char *)memchr(c, '\n', text + len - c);
        cut.push_back(nl ? nl + 1 : text + len);
    }
    cut.push_back(text + len);
    r->pieces.resize(T);
    for (int i = 0; i < T; ++i) {
        r->pieces[i].b = cut[i];
        r->pieces[i].e = cut[i + 1] > cut[i] ? cut[i + 1] : cut[i];
    }
    // line numbers: count the newlines before each piece (in parallel)
    std::vector<int64_t> nls(T, 0);
    {
        std::vector<std::thread> th;
        for (int i = 0; i < T; ++i)
            th.emplace_back([&, i] {
                int64_t c = 0;
                for (const char *p = r->pieces[i].b; p < r->pieces[i].e; ++p) c += *p == '\n';
                nls[i] = c;
            });
        for (auto &t : th) t.join();
    }
    int64_t line = 1;
    for (int i = 0; i < T; ++i) {
        r->pieces[i].first_line = line;
        line += nls[i];
    }
    {
        std::vector<std::thread> th;
        for (int i = 0; i < T; ++i) th.emplace_back([&, i] { parse_piece(text, r->pieces[i]); });
        for (auto &t : th) t.join();
    }
    const Piece *rng = nullptr;
    for (auto &P : r->pieces)
        if (!P.err && P.range_off >= 0) {
            rng = &P;
            break;
        }
    for (auto &P : r->pieces) {
        if (!P.err && &P == rng && rng->range_off >= 0) {
            // no format error before it: still scan later pieces for one
            bool later = false;
            for (auto &Q : r->pieces) later = later || (&Q > &P && Q.err);
            if (!later) {
                info[0] = info[1] = info[2] = 0;
                info[3] = ING_INDEX_RANGE;
                info[4] = P.range_line;
                info[5] = P.range_off;
                info[6] = P.range_len;
                delete r;
                *out = nullptr;
                return GLM_OK;
            }
        }
        if (P.err) {              // the first error in file order
            info[0] = info[1] = info[2] = 0;
            info[3] = P.err;
            info[4] = P.err_line;
            info[5] = P.tok_off;
            info[6] = P.tok_len;
            delete r;
            *out = nullptr;
            return GLM_OK;
        }
        r->n += (int64_t)P.labels.size();
        r->nnz += (int64_t)P.rows.size();
        if (P.max_feat > r->max_feat) r->max_feat = P.max_feat;
    }
    info[0] = r->n;
    info[1] = r->nnz;
    info[2] = r->max_feat;
    info[3] = info[4] = info[5] = info[6] = 0;
    *out = r;
    return GLM_OK;
}

int glm_svmlight_fetch(const glm_svmlight *r, int64_t *indptr, int32_t *rows, double *vals,
                       double *labels) {
    if (!r || !indptr) return glm_set_error(GLM_USAGE, "null argument");
    const int T = (int)r->pieces.size();
    std::vector<int64_t> ex0(T + 1, 0), nz0(T + 1, 0);
    for (int i = 0; i < T; ++i) {
        ex0[i + 1] = ex0[i] + (int64_t)r->pieces[i].labels.size();
        nz0[i + 1] = nz0[i] + (int64_t)r->pieces[i].rows.size();
    }
    std::vector<std::thread> th;
    for (int i = 0; i < T; ++i)
        th.emplace_back([&, i] {
            const Piece &P = r->pieces[i];
            int64_t acc = nz0[i];
            for (size_t k = 0; k < P.counts.size(); ++k) {
                indptr[ex0[i] + (int64_t)k] = acc;
                acc += P.counts[k];
            }
            if (!P.rows.empty()) {
                memcpy(rows + nz0[i], P.rows.data(), 4 * P.rows.size());
                memcpy(vals + nz0[i], P.vals.data(), 8 * P.vals.size());
            }
            if (!P.labels.empty()) memcpy(labels + ex0[i], P.labels.data(), 8 * P.labels.size());
        });
    for (auto &t : th) t.join();
    indptr[ex0[T]] = nz0[T];
    return GLM_OK;
}

int glm_svmlight_free(glm_svmlight *r) {
    delete r;
    return GLM_OK;
}

}  // extern "C"
