// Multi-threaded host text parsers for graph ingestion;
// the line semantics live in parse_line.cuh, shared with the device parser
// (ingest.inc).
//
// Same line semantics as the reference loaders
// (/root/reference/pkg/src/minmapcc/graph.py:149-197 load_edge_list,
//  graph.py:203-274 load_matrix_market entry lines):
//   mode 0 (edge list): blank lines and lines starting with '#' or '%' are
//     skipped; every other line must hold exactly two integer tokens >= 0.
//   mode 1 (Matrix Market body): blank lines and '%' lines skipped; every
//     other line holds >= 2 tokens, the first two integers (values ignored).
// Rows come out in file order as int64 pairs.  On the first malformed line
// (in file order) the parser reports its 1-based line number and a code.
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <thread>
#include <vector>

#include "contour.h"
#include "parse_line.cuh"

using ccparse::LineResult;
using ccparse::parse_line;

extern "C" {

int cc_parse_edges(const char* buf, int64_t len, int mode, int64_t* out, int64_t cap,
                   int64_t* m_out, int64_t* err_line, int* err_code, int* err_tokens,
                   int threads, int64_t bound, int64_t* err_vals) {
    if (!buf && len > 0) return CC_EINVAL;
    if (!m_out || !err_line || !err_code || (mode != 0 && mode != 1)) return CC_EINVAL;
    *err_line = 0;
    *err_code = 0;
    if (err_tokens) *err_tokens = 0;
    if (threads < 1) threads = 1;
    if (len < (1 << 20)) threads = 1;
    // chunk boundaries at line starts
    std::vector<int64_t> cut(threads + 1, len);
    cut[0] = 0;
    for (int t = 1; t < threads; ++t) {
        int64_t p = len * t / threads;
        if (p < cut[t - 1]) p = cut[t - 1];
        while (p < len && buf[p - 1] != '\n') ++p;
        cut[t] = p;
    }
    struct Part {
        int64_t lines = 0, rows = 0, err_local = -1, err_u = 0, err_v = 0;
        int err_code = 0, err_tok = 0;
    };
    std::vector<Part> parts(threads);
    auto scan = [&](int t, bool fill, int64_t row0) {
        Part& P = parts[t];
        int64_t row = row0, line = 0;
        const char* p = buf + cut[t];
        const char* end = buf + cut[t + 1];
        while (p < end) {
            const char* nl = (const char*)memchr(p, '\n', end - p);
            const char* le = nl ? nl : end;
            LineResult r = parse_line(p, le, mode, bound);
            if (!fill) {
                if (r.status < 0 && P.err_local < 0) {
                    P.err_local = line;
                    P.err_code = r.status;
                    P.err_tok = r.ntok;
                    P.err_u = r.u;
                    P.err_v = r.v;
                }
                if (r.status == 1) ++P.rows;
            } else if (r.status == 1) {
                if (out && row < cap) { out[2 * row] = r.u; out[2 * row + 1] = r.v; }
                ++row;
            }
            ++line;
            p = nl ? nl + 1 : end;
        }
        if (!fill) P.lines = line;
    };
    auto run = [&](bool fill, const std::vector<int64_t>& row0) {
        if (threads == 1) { scan(0, fill, row0[0]); return; }
        std::vector<std::thread> th;
        for (int t = 0; t < threads; ++t) th.emplace_back(scan, t, fill, row0[t]);
        for (auto& x : th) x.join();
    };
    std::vector<int64_t> row0(threads, 0);
    run(false, row0);
    int64_t lines_before = 0, total = 0;
    for (int t = 0; t < threads; ++t) {
        if (parts[t].err_local >= 0 && *err_code == 0) {
            *err_line = lines_before + parts[t].err_local + 1;
            *err_code = parts[t].err_code;
            if (err_tokens) *err_tokens = parts[t].err_tok;
            if (err_vals) { err_vals[0] = parts[t].err_u; err_vals[1] = parts[t].err_v; }
        }
        lines_before += parts[t].lines;
        row0[t] = total;
        total += parts[t].rows;
    }
    *m_out = total;
    if (*err_code) return CC_EINVAL;
    if (out) run(true, row0);
    return CC_OK;
}

}  // extern "C"
