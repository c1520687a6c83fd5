// One text line of an edge list / Matrix Market body -> (status, u, v).
//
// Shared by the multi-threaded host tokenizer (parse_host.cu) and the device
// ingestion kernels (ingest.inc), so both follow one definition of the
// reference loaders' line semantics
// (/root/reference/pkg/src/minmapcc/graph.py:165-180 load_edge_list and
//  graph.py:252-263 load_matrix_market entry lines):
//   mode 0 (edge list): blank lines and lines starting with '#' or '%' are
//     skipped (:167); every other line holds exactly two tokens (:169-173),
//     both integers (int(), :174-178) and >= 0 (:179-180).
//   mode 1 (Matrix Market body): blank and '%' lines skipped (:254); >= 2
//     tokens (:256-257), the first two integers (:258-262), inside 1..bound
//     when bound != 0 (:264-266; bound < 0 rejects every entry, n == 0).
#ifndef CC_PARSE_LINE_CUH
#define CC_PARSE_LINE_CUH

#include <stdint.h>

#include "contour.h"

#ifdef __CUDACC__
#define CC_HD __host__ __device__ __forceinline__
#else
#define CC_HD inline
#endif

namespace ccparse {

CC_HD bool is_space(char c) {
    return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f';
}

struct LineResult {
    int status;  // 0 skip, 1 row, <0 CC_PARSE_* error code
    int ntok;
    int64_t u, v;
};

// an integer token [p, e) as Python's int(token) reads it (sign, decimal
// digits, single underscores between digits); false if it is not one
CC_HD bool parse_int(const char* p, const char* e, int64_t& out) {
    bool neg = false;
    if (p < e && (*p == '+' || *p == '-')) {
        neg = *p == '-';
        ++p;
    }
    if (p == e) return false;
    int64_t x = 0;
    const char* s = p;
    for (; p < e; ++p) {
        const char c = *p;
        if (c == '_' && p > s && p + 1 < e && p[-1] >= '0' && p[-1] <= '9' && p[1] >= '0' &&
            p[1] <= '9')
            continue;
        if (c < '0' || c > '9') return false;
        if (x > (INT64_MAX - 9) / 10) return false;
        x = x * 10 + (c - '0');
    }
    out = neg ? -x : x;
    return true;
}

CC_HD LineResult parse_line(const char* b, const char* e, int mode, int64_t bound) {
    while (b < e && is_space(*b)) ++b;
    while (e > b && is_space(e[-1])) --e;
    LineResult r{0, 0, 0, 0};
    if (b == e) return r;
    if (*b == '%' || (mode == 0 && *b == '#')) return r;
    const char* t0b = nullptr;
    const char* t0e = nullptr;
    const char* t1b = nullptr;
    const char* t1e = nullptr;
    int nt = 0;
    const char* p = b;
    while (p < e) {
        while (p < e && is_space(*p)) ++p;
        if (p >= e) break;
        const char* s = p;
        while (p < e && !is_space(*p)) ++p;
        if (nt == 0) {
            t0b = s;
            t0e = p;
        } else if (nt == 1) {
            t1b = s;
            t1e = p;
        }
        ++nt;
    }
    r.ntok = nt;
    if (mode == 0 && nt != 2) {
        r.status = CC_PARSE_TOKENS;
        return r;
    }
    if (mode == 1 && nt < 2) {
        r.status = CC_PARSE_TOKENS;
        return r;
    }
    if (!parse_int(t0b, t0e, r.u) || !parse_int(t1b, t1e, r.v)) {
        r.status = CC_PARSE_NONINT;
        return r;
    }
    if (mode == 0 && (r.u < 0 || r.v < 0)) {
        r.status = CC_PARSE_NEGATIVE;
        return r;
    }
    if (mode == 1 && bound != 0 && !(1 <= r.u && r.u <= bound && 1 <= r.v && r.v <= bound)) {
        r.status = CC_PARSE_RANGE;
        return r;
    }
    r.status = 1;
    return r;
}

}  // namespace ccparse

#endif  // CC_PARSE_LINE_CUH
