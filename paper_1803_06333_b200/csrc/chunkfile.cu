// chunkfile.cu — the GLMCHUNK v1 on-disk chunk store, host side (C++).
//
// Reference format (data.py:17-27): a 32-byte header
//   magic "GLMCHUNK" | version u32 | flags u16 (1 labels, 2 row vector) |
//   endian mark u16 0xFEFF | n_rows u64 | n_cols u64
// then the optional row vector f64[n_rows], then per chunk a 12-byte head
// (n_cols u32, nnz u64) and the body indptr u64[c+1] (chunk-relative),
// rows u32[nnz], vals f64[nnz], labels f64[c] (if flagged); all little-endian.
// write_chunks / open_chunks / read_chunk (data.py:329-426) map onto
// glm_chunk_write / glm_chunk_open + glm_chunk_table / glm_chunk_read; the
// Python layer turns the status kinds below into the reference's
// ChunkFormatError messages.  glm_stream_create_file (stream.cu) reads the
// same bodies straight into pinned staging for the streaming pipeline.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cerrno>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace glm {
namespace {

enum : int64_t {
    CK_OK = 0, CK_TRUNC_HEADER = 1, CK_BAD_MAGIC = 2, CK_ENDIAN = 3, CK_VERSION = 4,
    CK_TRUNC_ROWVEC = 5, CK_TRUNC_CHUNK_HEAD = 6, CK_COLS_MISMATCH = 7, CK_HEAD_DISAGREES = 8,
    CK_TRUNC_BODY = 9, CK_OS_ERROR = 10
};

constexpr char MAGIC[8] = {'G', 'L', 'M', 'C', 'H', 'U', 'N', 'K'};
constexpr uint32_t VERSION = 1;
constexpr uint16_t ENDIAN = 0xFEFF;
constexpr uint16_t F_LABELS = 1, F_ROWVEC = 2;

struct Header {                // the 32-byte on-disk header (little-endian host)
    char magic[8];
    uint32_t version;
    uint16_t flags, endian;
    uint64_t n_rows, n_cols;
};
static_assert(sizeof(Header) == 32, "GLMCHUNK header is 32 bytes");

// Full-length pread / write (short transfers resumed); false at EOF or error.
bool read_at(int fd, void *dst, uint64_t bytes, uint64_t off, uint64_t *got = nullptr) {
    char *p = (char *)dst;
    uint64_t done = 0;
    while (done < bytes) {
        const ssize_t r = pread(fd, p + done, (size_t)(bytes - done), (off_t)(off + done));
        if (r <= 0) break;
        done += (uint64_t)r;
    }
    if (got) *got = done;
    return done == bytes;
}

bool write_all(int fd, const void *src, uint64_t bytes) {
    const char *p = (const char *)src;
    while (bytes > 0) {
        const ssize_t w = write(fd, p, (size_t)bytes);
        if (w <= 0) {
            if (w < 0 && errno == EINTR) continue;
            return false;
        }
        p += w;
        bytes -= (uint64_t)w;
    }
    return true;
}

// body bytes of a chunk (saturating: a garbage count only has to land past EOF)
uint64_t body_bytes(uint64_t cols, uint64_t nnz, bool labels) {
    const unsigned __int128 b = (unsigned __int128)8 * (cols + 1) + (unsigned __int128)12 * nnz +
                                (labels ? (unsigned __int128)8 * cols : 0);
    return b > (unsigned __int128)(UINT64_MAX / 2) ? UINT64_MAX / 2 : (uint64_t)b;
}

}  // namespace
}  // namespace glm

struct glm_chunkfile {
    glm::Header head{};
    std::vector<int64_t> offsets, cols, nnz;
    std::vector<double> row_vector;
};

using namespace glm;

extern "C" {

int glm_chunk_write(const char *path, int64_t n_rows, int64_t n_cols, const int64_t *indptr,
                    const int32_t *rows, const double *vals, const double *labels,
                    const double *row_vector, int64_t chunk_size, int64_t *offsets_out,
                    int64_t *os_errno) {
    if (!path || !indptr || n_rows < 0 || n_cols < 0 || !os_errno)
        return glm_set_error(GLM_USAGE, "null argument to glm_chunk_write");
    if (chunk_size < 1) return glm_set_error(GLM_USAGE, "chunk_size must be >= 1");
    *os_errno = 0;
    const int fd = open(path, O_WRONLY | O_CREAT | O_TRUNC, 0666);
    if (fd < 0) {
        *os_errno = errno;
        return GLM_OK;
    }
    Header h{};
    memcpy(h.magic, MAGIC, 8);
    h.version = VERSION;
    h.flags = (uint16_t)((labels ? F_LABELS : 0) | (row_vector ? F_ROWVEC : 0));
    h.endian = ENDIAN;
    h.n_rows = (uint64_t)n_rows;
    h.n_cols = (uint64_t)n_cols;
    bool ok = write_all(fd, &h, sizeof h);
    uint64_t off = sizeof h;
    if (ok && row_vector) {
        ok = write_all(fd, row_vector, 8 * (uint64_t)n_rows);
        off += 8 * (uint64_t)n_rows;
    }
    std::vector<char> buf;
    int64_t k = 0;
    for (int64_t lo = 0; ok && lo < n_cols; lo += chunk_size, ++k) {
        const int64_t hi = lo + chunk_size < n_cols ? lo + chunk_size : n_cols;
        const int64_t c = hi - lo, p0 = indptr[lo], nz = indptr[hi] - p0;
        const uint64_t body = body_bytes((uint64_t)c, (uint64_t)nz, labels != nullptr);
        buf.resize(12 + body);
        char *b = buf.data();
        const uint32_t c32 = (uint32_t)c;
        const uint64_t nz64 = (uint64_t)nz;
        memcpy(b, &c32, 4);
        memcpy(b + 4, &nz64, 8);
        uint64_t *ip = reinterpret_cast<uint64_t *>(b + 12);        // chunk-relative indptr
        for (int64_t j = 0; j <= c; ++j) ip[j] = (uint64_t)(indptr[lo + j] - p0);
        char *q = b + 12 + 8 * (c + 1);
        if (nz > 0) {
            memcpy(q, rows + p0, 4 * (size_t)nz);                    // i32 bits = u32 bits
            memcpy(q + 4 * nz, vals + p0, 8 * (size_t)nz);
        }
        if (labels) memcpy(q + 12 * nz, labels + lo, 8 * (size_t)c);
        if (offsets_out) offsets_out[k] = (int64_t)off;
        ok = write_all(fd, b, 12 + body);
        off += 12 + body;
    }
    if (!ok) *os_errno = errno ? errno : EIO;
    if (close(fd) != 0 && ok) *os_errno = errno;
    return GLM_OK;
}

// info: [0] status kind (CK_*), [1] n_rows, [2] n_cols, [3] flags, [4] version,
// [5] n_chunks, [6] errno (CK_OS_ERROR); magic_out: the 8 magic bytes read.
int glm_chunk_open(const char *path, glm_chunkfile **out, int64_t *info, char *magic_out) {
    if (!path || !out || !info) return glm_set_error(GLM_USAGE, "null argument to glm_chunk_open");
    *out = nullptr;
    for (int i = 0; i < 8; ++i) info[i] = 0;
    const int fd = open(path, O_RDONLY);
    if (fd < 0) {
        info[0] = CK_OS_ERROR;
        info[6] = errno;
        return GLM_OK;
    }
    struct stat sb{};
    fstat(fd, &sb);
    const uint64_t size = (uint64_t)sb.st_size;
    glm_chunkfile *f = new (std::nothrow) glm_chunkfile();
    int64_t st = CK_OK;
    Header &h = f->head;
    if (!read_at(fd, &h, sizeof h, 0)) {
        st = CK_TRUNC_HEADER;
    } else {
        if (magic_out) memcpy(magic_out, h.magic, 8);
        if (memcmp(h.magic, MAGIC, 8) != 0) st = CK_BAD_MAGIC;
        else if (h.endian != ENDIAN) st = CK_ENDIAN;
        else if (h.version != VERSION) st = CK_VERSION;
    }
    uint64_t off = sizeof h;
    if (st == CK_OK && (h.flags & F_ROWVEC)) {
        f->row_vector.resize(h.n_rows);
        if (!read_at(fd, f->row_vector.data(), 8 * h.n_rows, off)) st = CK_TRUNC_ROWVEC;
        off += 8 * h.n_rows;
    }
    // the descriptor scan: a chunk head must be readable at every offset
    // until the columns are covered (bodies may run past EOF, as a seek does)
    uint64_t seen = 0;
    while (st == CK_OK && seen < h.n_cols) {
        unsigned char ch[12];
        if (off > size || size - off < 12 || !read_at(fd, ch, 12, off)) {
            st = CK_TRUNC_CHUNK_HEAD;
            break;
        }
        uint32_t c;
        uint64_t nz;
        memcpy(&c, ch, 4);
        memcpy(&nz, ch + 4, 8);
        f->offsets.push_back((int64_t)off);
        f->cols.push_back((int64_t)c);
        f->nnz.push_back((int64_t)nz);
        const uint64_t body = body_bytes(c, nz, (h.flags & F_LABELS) != 0);
        off = off + 12 + body > UINT64_MAX / 2 ? UINT64_MAX / 2 : off + 12 + body;
        seen += c;
    }
    if (st == CK_OK && seen != h.n_cols) st = CK_COLS_MISMATCH;
    close(fd);
    info[0] = st;
    info[1] = (int64_t)h.n_rows;
    info[2] = (int64_t)h.n_cols;
    info[3] = h.flags;
    info[4] = h.version;
    info[5] = (int64_t)f->offsets.size();
    if (st != CK_OK) {
        delete f;
        return GLM_OK;
    }
    *out = f;
    return GLM_OK;
}

int glm_chunk_table(const glm_chunkfile *f, int64_t *offsets, int64_t *n_cols, int64_t *nnz,
                    double *row_vector) {
    if (!f) return glm_set_error(GLM_USAGE, "null chunk file");
    const size_t k = f->offsets.size();
    if (offsets && k) memcpy(offsets, f->offsets.data(), 8 * k);
    if (n_cols && k) memcpy(n_cols, f->cols.data(), 8 * k);
    if (nnz && k) memcpy(nnz, f->nnz.data(), 8 * k);
    if (row_vector && !f->row_vector.empty())
        memcpy(row_vector, f->row_vector.data(), 8 * f->row_vector.size());
    return GLM_OK;
}

int glm_chunk_close(glm_chunkfile *f) {
    delete f;
    return GLM_OK;
}

// One chunk into caller arrays: indptr i64[n_cols+1], rows i32[nnz],
// vals f64[nnz], labels f64[n_cols] (NULL: not read).  status: CK_* kind,
// status[1] = errno for CK_OS_ERROR.
int glm_chunk_read(const char *path, int64_t offset, int64_t n_cols, int64_t nnz, int has_labels,
                   int64_t *indptr, int32_t *rows, double *vals, double *labels, int64_t *status) {
    if (!path || !status || offset < 0 || n_cols < 0 || nnz < 0)
        return glm_set_error(GLM_USAGE, "bad argument to glm_chunk_read");
    status[0] = status[1] = 0;
    const int fd = open(path, O_RDONLY);
    if (fd < 0) {
        status[0] = CK_OS_ERROR;
        status[1] = errno;
        return GLM_OK;
    }
    unsigned char ch[12];
    int64_t st = CK_OK;
    if (!read_at(fd, ch, 12, (uint64_t)offset)) {
        st = CK_TRUNC_CHUNK_HEAD;
    } else {
        uint32_t c;
        uint64_t nz;
        memcpy(&c, ch, 4);
        memcpy(&nz, ch + 4, 8);
        if ((int64_t)c != n_cols || (int64_t)nz != nnz) st = CK_HEAD_DISAGREES;
    }
    if (st == CK_OK) {
        uint64_t at = (uint64_t)offset + 12;
        bool ok = read_at(fd, indptr, 8 * (uint64_t)(n_cols + 1), at);
        at += 8 * (uint64_t)(n_cols + 1);
        ok = ok && read_at(fd, rows, 4 * (uint64_t)nnz, at);
        at += 4 * (uint64_t)nnz;
        ok = ok && read_at(fd, vals, 8 * (uint64_t)nnz, at);
        at += 8 * (uint64_t)nnz;
        if (ok && has_labels && labels) ok = read_at(fd, labels, 8 * (uint64_t)n_cols, at);
        if (!ok) st = CK_TRUNC_BODY;
    }
    close(fd);
    status[0] = st;
    return GLM_OK;
}

}  // extern "C"
