// Native Matrix Market reader (the input side of the path):
// replaces scipy.io.mmread behind reference mmio.py:23-28
// (read_matrix_market) and cp_tensor.py:346-361 (load_cp_dir's factor files).
//
// The file is memory-mapped, the header and size line are parsed in place,
// and the data section is split at line boundaries over `nthreads` threads:
// a first pass counts each chunk's data lines (output offsets in file order),
// a second parses them with std::from_chars (correctly rounded, like strtod)
// straight into the caller's arrays.  Symmetry is NOT expanded here (the
// Python side does it the way scipy does).
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cctype>
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include "../../include/idsketch_b200.h"

void ids_set_last_error(const char* msg);

namespace {

struct Header {
    int64_t rows = 0, cols = 0, entries = 0;
    int format = 0;    // 0 coordinate, 1 array
    int field = 0;     // 0 real, 1 integer, 2 pattern, 3 complex
    int symmetry = 0;  // 0 general, 1 symmetric, 2 skew-symmetric, 3 hermitian
    size_t data = 0;   // offset of the first data line
};

// Read-only memory map of a file (pages fault in on the parsing threads).
struct FileView {
    const char* data = nullptr;
    size_t size = 0;
    void* map = nullptr;
    explicit FileView(const char* path) {
        const int fd = ::open(path, O_RDONLY);
        if (fd < 0) return;
        struct stat st;
        if (::fstat(fd, &st) == 0 && st.st_size > 0) {
            map = ::mmap(nullptr, (size_t)st.st_size, PROT_READ, MAP_PRIVATE, fd, 0);
            if (map == MAP_FAILED) {
                map = nullptr;
            } else {
                data = static_cast<const char*>(map);
                size = (size_t)st.st_size;
            }
        }
        ::close(fd);
    }
    ~FileView() {
        if (map) ::munmap(map, size);
    }
    bool ok() const { return data != nullptr; }
};

std::string lower(std::string s) {
    for (char& c : s) c = (char)std::tolower((unsigned char)c);
    return s;
}

// Header line, comments, size line -- scanned in place on the mapped file.
bool parse_header(const char* d, size_t size, Header& h, std::string& err) {
    auto line_end = [&](size_t pos) {
        const void* nl = std::memchr(d + pos, '\n', size - pos);
        return nl ? (size_t)(static_cast<const char*>(nl) - d) : size;
    };
    size_t e = line_end(0);
    const std::string first = lower(std::string(d, e));
    char banner[64] = {0}, object[64] = {0}, fmt[64] = {0}, field[64] = {0}, sym[64] = {0};
    if (std::sscanf(first.c_str(), "%63s %63s %63s %63s %63s", banner, object, fmt, field, sym) != 5 ||
        std::strcmp(banner, "%%matrixmarket") != 0 || std::strcmp(object, "matrix") != 0) {
        err = "not a Matrix Market matrix header";
        return false;
    }
    if (!std::strcmp(fmt, "coordinate")) h.format = 0;
    else if (!std::strcmp(fmt, "array")) h.format = 1;
    else { err = "unknown Matrix Market format"; return false; }
    if (!std::strcmp(field, "real") || !std::strcmp(field, "double")) h.field = 0;
    else if (!std::strcmp(field, "integer")) h.field = 1;
    else if (!std::strcmp(field, "pattern")) h.field = 2;
    else if (!std::strcmp(field, "complex")) h.field = 3;
    else { err = "unknown Matrix Market field"; return false; }
    if (!std::strcmp(sym, "general")) h.symmetry = 0;
    else if (!std::strcmp(sym, "symmetric")) h.symmetry = 1;
    else if (!std::strcmp(sym, "skew-symmetric")) h.symmetry = 2;
    else if (!std::strcmp(sym, "hermitian")) h.symmetry = 3;
    else { err = "unknown Matrix Market symmetry"; return false; }
    size_t pos = e < size ? e + 1 : size;
    while (pos < size) {  // skip comment / blank lines, then the size line
        e = line_end(pos);
        size_t q = pos;
        while (q < e && (d[q] == ' ' || d[q] == '\t' || d[q] == '\r')) ++q;
        if (q == e || d[q] == '%') {
            pos = e + 1;
            continue;
        }
        long long r = 0, c = 0, n = 0;
        const int got = std::sscanf(std::string(d + q, e - q).c_str(), "%lld %lld %lld", &r, &c, &n);
        if ((h.format == 0 && got != 3) || (h.format == 1 && got < 2) || r < 0 || c < 0 || n < 0) {
            err = "bad Matrix Market size line";
            return false;
        }
        h.rows = r;
        h.cols = c;
        h.entries = h.format == 0 ? n
                    : (h.symmetry == 0 ? r * c : (h.symmetry == 2 ? r * (r - 1) / 2 : r * (r + 1) / 2));
        h.data = e < size ? e + 1 : size;
        return true;
    }
    err = "missing Matrix Market size line";
    return false;
}

const char* skip_ws(const char* p, const char* e) {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\r')) ++p;
    return p;
}

// data lines (not blank, not comments) in [b, e)
int64_t count_lines(const char* b, const char* e) {
    int64_t n = 0;
    const char* p = b;
    while (p < e) {
        const char* le = static_cast<const char*>(std::memchr(p, '\n', (size_t)(e - p)));
        if (!le) le = e;
        const char* q = skip_ws(p, le);
        if (q < le && *q != '%') ++n;
        p = le + 1;
    }
    return n;
}

// parse the data lines of [b, e) into the outputs starting at entry `off`
bool parse_range(const char* b, const char* e, const Header& h, int64_t* row, int64_t* col,
                 double* val, int64_t off, std::string& err) {
    const bool coord = h.format == 0;
    const int nval = h.field == 2 ? 0 : (h.field == 3 ? 2 : 1);
    const char* p = b;
    while (p < e) {
        const char* le = static_cast<const char*>(std::memchr(p, '\n', (size_t)(e - p)));
        if (!le) le = e;
        const char* q = skip_ws(p, le);
        if (q < le && *q != '%') {
            int64_t r = 0, c = 0;
            double v = 1.0;
            if (coord) {
                auto a = std::from_chars(q, le, r);
                q = skip_ws(a.ptr, le);
                auto d = std::from_chars(q, le, c);
                q = skip_ws(d.ptr, le);
                if (a.ec != std::errc() || d.ec != std::errc() || r < 1 || c < 1 || r > h.rows ||
                    c > h.cols) {
                    err = "bad Matrix Market coordinate entry";
                    return false;
                }
                row[off] = r - 1;
                col[off] = c - 1;
            }
            for (int k = 0; k < nval; ++k) {
                double x = 0.0;
                auto f = std::from_chars(q, le, x);
                if (f.ec != std::errc()) {
                    err = "bad Matrix Market value";
                    return false;
                }
                if (k == 0) v = x;
                q = skip_ws(f.ptr, le);
            }
            val[off++] = v;
        }
        p = le + 1;
    }
    return true;
}

}  // namespace

extern "C" int ids_mm_info(const char* path, int64_t* rows, int64_t* cols, int64_t* entries,
                           int32_t* kind) {
    std::string err;
    const FileView f(path ? path : "");
    if (!f.ok()) {
        ids_set_last_error("matrix market: cannot read file");
        return IDS_EINVAL;
    }
    Header h;
    if (!parse_header(f.data, f.size, h, err)) {
        ids_set_last_error(err.c_str());
        return IDS_EINVAL;
    }
    *rows = h.rows;
    *cols = h.cols;
    *entries = h.entries;
    kind[0] = h.format;
    kind[1] = h.field;
    kind[2] = h.symmetry;
    return IDS_OK;
}

extern "C" int ids_mm_read(const char* path, int nthreads, int64_t* row, int64_t* col,
                           double* val, int64_t capacity, int64_t* count) {
    std::string err;
    const FileView f(path ? path : "");
    if (!f.ok()) {
        ids_set_last_error("matrix market: cannot read file");
        return IDS_EINVAL;
    }
    Header h;
    if (!parse_header(f.data, f.size, h, err)) {
        ids_set_last_error(err.c_str());
        return IDS_EINVAL;
    }
    const char* b = f.data + h.data;
    const char* e = f.data + f.size;
    const int T = nthreads < 1 ? 1 : (nthreads > 256 ? 256 : nthreads);
    std::vector<const char*> cut(T + 1);
    cut[0] = b;
    cut[T] = e;
    for (int t = 1; t < T; ++t) {  // split at line starts
        const char* p = b + (size_t)(e - b) * t / T;
        if (p < cut[t - 1]) p = cut[t - 1];
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', (size_t)(e - p)));
        cut[t] = nl ? nl + 1 : e;
    }
    // pass 1: data lines per chunk -> output offsets (file order)
    std::vector<int64_t> cnt(T + 1, 0);
    {
        std::vector<std::thread> pool;
        for (int t = 0; t < T; ++t)
            pool.emplace_back([&, t] { cnt[t + 1] = count_lines(cut[t], cut[t + 1]); });
        for (auto& th : pool) th.join();
    }
    for (int t = 0; t < T; ++t) cnt[t + 1] += cnt[t];
    if (cnt[T] != h.entries) {
        ids_set_last_error("matrix market: entry count does not match the size line");
        return IDS_EINVAL;
    }
    if (cnt[T] > capacity) {
        ids_set_last_error("matrix market: output arrays too small");
        return IDS_EWORKSPACE;
    }
    // pass 2: parse straight into the outputs
    std::vector<std::string> errs(T);
    {
        std::vector<std::thread> pool;
        for (int t = 0; t < T; ++t)
            pool.emplace_back([&, t] { parse_range(cut[t], cut[t + 1], h, row, col, val, cnt[t], errs[t]); });
        for (auto& th : pool) th.join();
    }
    for (auto& m : errs)
        if (!m.empty()) {
            ids_set_last_error(m.c_str());
            return IDS_EINVAL;
        }
    *count = cnt[T];
    return IDS_OK;
}
