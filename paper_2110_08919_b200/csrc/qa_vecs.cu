// qa_vecs.cu -- on-disk vector files straight into (sharded) HBM.
//
// Framing of fvecs / ivecs / i8vecs / bvecs (reference dataset.py:160-275):
// every record is a little-endian int32 d followed by d payload items of
// `itemsize` bytes (4 for fvecs/ivecs, 1 for i8vecs/bvecs).  The probe
// reproduces the reference's framing diagnosis (_load_records 180-209 and
// _walk_records 160-177): the same conditions, checked in the same order,
// give the same error kind.
//
// The read path streams a row range [row_lo, row_hi) -- one rank's shard --
// through two pinned staging buffers: while the host pread()s chunk i+1, the
// copy engine moves chunk i with ONE cudaMemcpy2DAsync whose source pitch is
// the record length (4 + d*itemsize) and whose source offset skips the
// header, so the headers are stripped by the DMA and the rows land at the
// destination stride (e.g. the padded int8 code stride).  Headers of the
// rows read are checked on the host while they sit in the staging buffer.
#include <algorithm>
#include <cerrno>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fcntl.h>
#include <string>
#include <sys/stat.h>
#include <unistd.h>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/qa_b200.h"

namespace qa {
int set_error_message(int code, const char *msg);
}

namespace {

int fail(int code, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    return qa::set_error_message(code, buf);
}

struct File {
    int fd = -1;
    ~File() {
        if (fd >= 0) close(fd);
    }
};

int open_file(File &f, const char *path, int64_t *size) {
    f.fd = open(path, O_RDONLY | O_CLOEXEC);
    if (f.fd < 0) return fail(QA_EIO, "%s: %s", path, strerror(errno));
    struct stat st;
    if (fstat(f.fd, &st) != 0) return fail(QA_EIO, "%s: %s", path, strerror(errno));
    *size = (int64_t)st.st_size;
    return QA_OK;
}

int read_at(const File &f, const char *path, void *dst, int64_t bytes, int64_t off) {
    char *p = (char *)dst;
    while (bytes > 0) {
        ssize_t got = pread(f.fd, p, (size_t)std::min<int64_t>(bytes, 1 << 30), (off_t)off);
        if (got < 0) {
            if (errno == EINTR) continue;
            return fail(QA_EIO, "%s: %s", path, strerror(errno));
        }
        if (got == 0) return fail(QA_EIO, "%s: unexpected end of file", path);
        p += got;
        off += got;
        bytes -= got;
    }
    return QA_OK;
}

int32_t le_i32(const unsigned char *p) {
    return (int32_t)((uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) |
                     ((uint32_t)p[3] << 24));
}

// staging chunk (bytes); QA_B200_VECS_CHUNK overrides it (tests exercise
// the double-buffered path with small chunks)
int64_t chunk_bytes() {
    const char *v = getenv("QA_B200_VECS_CHUNK");
    const long long c = v ? atoll(v) : 0;
    return c > 0 ? (int64_t)c : (64ll << 20);
}

// _walk_records: the precise diagnosis when the size is not a whole number
// of records.  Returns an error code always (the caller only walks a file
// that is already known to be malformed).
int walk_records(const File &f, const char *path, int64_t size, int32_t d0, int itemsize) {
    int64_t off = 0, idx = 0;
    unsigned char h[4];
    while (off < size) {
        if (off + 4 > size) return fail(QA_ETRUNCATED, "%s: record %lld header cut short", path, (long long)idx);
        int rc = read_at(f, path, h, 4, off);
        if (rc) return rc;
        const int32_t d = le_i32(h);
        if (d <= 0) return fail(QA_ENONPOSITIVE, "%s: record %lld declares d=%d", path, (long long)idx, d);
        if (d != d0)
            return fail(QA_EDIM, "%s: record %lld has d=%d, expected d=%d", path, (long long)idx, d, d0);
        off += 4 + (int64_t)d * itemsize;
        ++idx;
    }
    if (off != size)
        return fail(QA_ETRUNCATED, "%s: record %lld payload cut short", path, (long long)(idx - 1));
    return fail(QA_ETRUNCATED, "%s: %lld bytes is not a whole number of %lld-byte records", path,
                (long long)size, (long long)(4 + (int64_t)d0 * itemsize));
}

// Check the headers of `rows` records staged at `buf` (first record index
// `first`); error kind as the reference's vectorised header check.
int check_headers(const unsigned char *buf, int64_t rows, int64_t rec, int32_t d, int64_t first,
                  const char *path) {
    for (int64_t r = 0; r < rows; ++r) {
        const int32_t h = le_i32(buf + r * rec);
        if (h != d) {
            if (h <= 0)
                return fail(QA_ENONPOSITIVE, "%s: record %lld declares d=%d", path, (long long)(first + r), h);
            return fail(QA_EDIM, "%s: record %lld has d=%d, expected d=%d", path, (long long)(first + r), h, d);
        }
    }
    return QA_OK;
}

}  // namespace

extern "C" {

int qa_vecs_probe(const char *path, int itemsize, int64_t *n_out, int64_t *d_out) {
    if (!path || (itemsize != 1 && itemsize != 4) || !n_out || !d_out)
        return fail(QA_EINVAL, "bad arguments");
    File f;
    int64_t size = 0;
    int rc = open_file(f, path, &size);
    if (rc) return rc;
    *n_out = 0;
    *d_out = 0;
    if (size == 0) return QA_OK;
    if (size < 4) return fail(QA_ETRUNCATED, "%s: file shorter than one record header", path);
    unsigned char h[4];
    if ((rc = read_at(f, path, h, 4, 0))) return rc;
    const int32_t d = le_i32(h);
    if (d <= 0) return fail(QA_ENONPOSITIVE, "%s: record header declares d=%d", path, d);
    const int64_t rec = 4 + (int64_t)d * itemsize;
    if (size % rec != 0) return walk_records(f, path, size, d, itemsize);
    const int64_t n = size / rec;
    // every header must repeat d: scan them chunk by chunk
    std::vector<unsigned char> buf;
    const int64_t rows_per = std::max<int64_t>(1, chunk_bytes() / rec);
    buf.resize((size_t)(std::min(rows_per, n) * rec));
    for (int64_t r0 = 0; r0 < n; r0 += rows_per) {
        const int64_t rows = std::min(rows_per, n - r0);
        if ((rc = read_at(f, path, buf.data(), rows * rec, r0 * rec))) return rc;
        if ((rc = check_headers(buf.data(), rows, rec, d, r0, path))) return rc;
    }
    *n_out = n;
    *d_out = d;
    return QA_OK;
}

int qa_vecs_read(const char *path, int itemsize, int64_t d, int64_t row_lo, int64_t row_hi,
                 void *dst, int64_t ld_bytes, int dst_on_device, int recenter_u8, void *stream) {
    if (!path || (itemsize != 1 && itemsize != 4) || d <= 0 || row_lo < 0 || row_hi < row_lo ||
        ld_bytes < d * itemsize || (recenter_u8 && itemsize != 1))
        return fail(QA_EINVAL, "bad arguments");
    if (row_hi == row_lo) return QA_OK;
    File f;
    int64_t size = 0;
    int rc = open_file(f, path, &size);
    if (rc) return rc;
    const int64_t rec = 4 + d * itemsize;
    if (row_hi * rec > size)
        return fail(QA_ETRUNCATED, "%s: rows [%lld, %lld) past the end of the file", path,
                    (long long)row_lo, (long long)row_hi);
    const int64_t rows_per = std::max<int64_t>(1, chunk_bytes() / rec);
    const int64_t total = row_hi - row_lo;
    const size_t stage = (size_t)(std::min(rows_per, total) * rec);
    const int64_t width = d * itemsize;
    cudaStream_t st = (cudaStream_t)stream;
    unsigned char *bufs[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    if (dst_on_device) {
        for (int i = 0; i < 2; ++i) {
            if (cudaMallocHost(&bufs[i], stage) != cudaSuccess ||
                cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming) != cudaSuccess) {
                for (int j = 0; j < 2; ++j) {
                    if (bufs[j]) cudaFreeHost(bufs[j]);
                    if (done[j]) cudaEventDestroy(done[j]);
                }
                return fail(QA_ENOMEM, "pinned staging allocation failed");
            }
        }
    } else {
        bufs[0] = (unsigned char *)malloc(stage);
        if (!bufs[0]) return fail(QA_ENOMEM, "staging allocation failed");
    }
    int slot = 0;
    for (int64_t r0 = row_lo; r0 < row_hi && rc == QA_OK; r0 += rows_per) {
        const int64_t rows = std::min(rows_per, row_hi - r0);
        unsigned char *b = bufs[dst_on_device ? slot : 0];
        if (dst_on_device && cudaEventSynchronize(done[slot]) != cudaSuccess) {
            rc = fail(QA_ECUDA, "staging wait failed");
            break;
        }
        if ((rc = read_at(f, path, b, rows * rec, r0 * rec))) break;
        if ((rc = check_headers(b, rows, rec, (int32_t)d, r0, path))) break;
        if (recenter_u8)  // bvecs: unsigned byte v -> int8 v - 128 (== v ^ 0x80)
            for (int64_t r = 0; r < rows; ++r)
                for (int64_t j = 0; j < d; ++j) b[r * rec + 4 + j] ^= 0x80u;
        char *out = (char *)dst + (r0 - row_lo) * ld_bytes;
        if (dst_on_device) {
            if (cudaMemcpy2DAsync(out, (size_t)ld_bytes, b + 4, (size_t)rec, (size_t)width,
                                  (size_t)rows, cudaMemcpyHostToDevice, st) != cudaSuccess ||
                cudaEventRecord(done[slot], st) != cudaSuccess) {
                rc = fail(QA_ECUDA, "%s", cudaGetErrorString(cudaGetLastError()));
                break;
            }
            slot ^= 1;
        } else {
            for (int64_t r = 0; r < rows; ++r) memcpy(out + r * ld_bytes, b + r * rec + 4, (size_t)width);
        }
    }
    if (dst_on_device) {
        for (int i = 0; i < 2; ++i) {
            cudaEventSynchronize(done[i]);
            cudaEventDestroy(done[i]);
            cudaFreeHost(bufs[i]);
        }
    } else {
        free(bufs[0]);
    }
    return rc;
}

int qa_vecs_write(const char *path, int itemsize, const void *src, int64_t n, int64_t d,
                  int64_t ld_bytes) {
    if (!path || (itemsize != 1 && itemsize != 4) || n < 0 || d < 0 ||
        ld_bytes < d * itemsize || d > INT32_MAX)
        return fail(QA_EINVAL, "bad arguments");
    FILE *fp = fopen(path, "wb");
    if (!fp) return fail(QA_EIO, "%s: %s", path, strerror(errno));
    const int64_t rec = 4 + d * itemsize;
    const int64_t rows_per = std::max<int64_t>(1, chunk_bytes() / std::max<int64_t>(rec, 1));
    std::vector<unsigned char> buf((size_t)(std::min(rows_per, std::max<int64_t>(n, 1)) * rec));
    const uint32_t h = (uint32_t)d;
    const unsigned char hb[4] = {(unsigned char)h, (unsigned char)(h >> 8), (unsigned char)(h >> 16),
                                 (unsigned char)(h >> 24)};
    int rc = QA_OK;
    for (int64_t r0 = 0; r0 < n; r0 += rows_per) {
        const int64_t rows = std::min(rows_per, n - r0);
        for (int64_t r = 0; r < rows; ++r) {
            memcpy(buf.data() + r * rec, hb, 4);
            memcpy(buf.data() + r * rec + 4, (const char *)src + (r0 + r) * ld_bytes,
                   (size_t)(d * itemsize));
        }
        if (fwrite(buf.data(), 1, (size_t)(rows * rec), fp) != (size_t)(rows * rec)) {
            rc = fail(QA_EIO, "%s: %s", path, strerror(errno));
            break;
        }
    }
    if (fclose(fp) != 0 && rc == QA_OK) rc = fail(QA_EIO, "%s: %s", path, strerror(errno));
    return rc;
}

}  // extern "C"
