// ingest.cpp -- SNAP-format edge-list ingestion in front of the per-batch path.
// The paper streams each graph "by feeding the algorithm with edges as they are read from disk"
// (PAPER.md:916-918), its datasets "stored as a list of edges in plain text" (Table 1), with an optimised
// I/O routine whose time is reported apart from processing.  Here: a native parser
// (tc_parse_edges) and a two-slot pipeline (tc_ingest_file): a reader thread reads and parses the file
// into one of two pinned batch buffers while the calling thread pushes the other through tc_push_batch,
// so disk and parsing overlap the GPU work; the reader's busy time is reported as I/O.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/tc.h"

namespace {

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

// One decimal id at p (< end); false if there is none or it exceeds 0xFFFFFFFE.
inline bool parse_id(const char *&p, const char *end, uint32_t &out) {
    if (p >= end || *p < '0' || *p > '9') return false;
    uint64_t x = 0;
    while (p < end && *p >= '0' && *p <= '9') {
        x = x * 10 + (uint64_t)(*p - '0');
        if (x > 0xFFFFFFFEull) return false;
        ++p;
    }
    out = (uint32_t)x;
    return true;
}

// Parses one line [p, e) (no '\n').  Returns 0 = blank / comment, 1 = edge, <0 = TC_E* code.
inline int parse_line(const char *p, const char *e, int flags, tc_edge &out) {
    while (p < e && is_space(*p)) ++p;
    if (p == e || *p == '#' || *p == '%') return 0;
    uint32_t u, v;
    if (!parse_id(p, e, u)) return TC_EPARSE;
    if (p == e || !is_space(*p)) return TC_EPARSE;
    while (p < e && is_space(*p)) ++p;
    if (!parse_id(p, e, v)) return TC_EPARSE;
    if (p < e && !is_space(*p)) return TC_EPARSE;  // further columns (weights, times) may follow whitespace
    if (u == v) return (flags & TC_INGEST_SKIP_LOOPS) ? 0 : TC_ESELFLOOP;
    out.u = u;
    out.v = v;
    return 1;
}

}  // namespace

extern "C" int tc_parse_edges(const char *text, uint64_t len, int final, int flags, tc_edge *out, uint64_t cap,
                              uint64_t *n_edges, uint64_t *consumed, uint64_t *lines) {
    if ((!text && len) || (!out && cap) || !n_edges || !consumed || !lines) return TC_EINVAL;
    const char *p = text, *end = text + len;
    uint64_t n = 0, ln = 0;
    int rc = TC_OK;
    while (p < end) {
        const char *nl = static_cast<const char *>(memchr(p, '\n', (size_t)(end - p)));
        if (!nl && !final) break;  // incomplete last line: left for the next call
        const char *le = nl ? nl : end;
        tc_edge e;
        const int r = parse_line(p, le, flags, e);
        if (r < 0) {
            rc = r;
            ++ln;  // the offending line, 1-based
            break;
        }
        if (r == 1) {
            if (n == cap) break;  // out is full: this line is not consumed
            out[n++] = e;
        }
        ++ln;
        p = nl ? nl + 1 : end;
    }
    *n_edges = n;
    *consumed = (uint64_t)(p - text);
    *lines = ln;
    return rc;
}

extern "C" int tc_ingest_file(tc_ctx *ctx, const char *path, uint64_t w, int flags, tc_ingest_stats *st) {
    using clk = std::chrono::steady_clock;
    if (!ctx || !path || w == 0 || w > (1ull << 28)) return TC_EINVAL;
    tc_ingest_stats S{};
    FILE *f = fopen(path, "rb");
    if (!f) return TC_EIO;
    const auto t_start = clk::now();
    // two pinned batch slots; the reader fills slot k % 2 while the pusher drains the other
    tc_edge *slot[2] = {nullptr, nullptr};
    if (cudaHostAlloc(reinterpret_cast<void **>(&slot[0]), 8 * w, cudaHostAllocDefault) != cudaSuccess ||
        cudaHostAlloc(reinterpret_cast<void **>(&slot[1]), 8 * w, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        if (slot[0]) cudaFreeHost(slot[0]);
        fclose(f);
        return TC_ENOMEM;
    }
    std::mutex mu;
    std::condition_variable cv;
    uint64_t fill[2] = {0, 0};
    bool full[2] = {false, false};
    bool done = false;
    std::atomic<bool> stop{false};
    int reader_rc = TC_OK;
    uint64_t err_line = 0;
    double io_s = 0.0;
    uint64_t lines_total = 0;
    std::thread reader([&] {
        // blocks of kBlock bytes; each block's complete lines are cut at line boundaries into one piece per
        // parser thread, parsed in parallel into per-piece arrays, then copied in file order into the slots
        size_t kBlock = 64u << 20;
        if (const char *e = getenv("TC_INGEST_BLOCK")) kBlock = std::max<size_t>(16, strtoull(e, nullptr, 10));  // tests
        const unsigned T = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        std::vector<char> buf(kBlock);
        std::vector<std::vector<tc_edge>> part(T);
        std::vector<uint64_t> pn(T), plines(T);
        std::vector<int> prc(T);
        size_t have = 0;  // bytes of an unfinished line carried over
        int s = 0;
        uint64_t n = 0;
        bool eof = false;
        auto t0 = clk::now();
        auto hand_off = [&](bool last) {  // slot s (n edges) to the pusher; wait for the next slot
            io_s += std::chrono::duration<double>(clk::now() - t0).count();
            std::unique_lock<std::mutex> lk(mu);
            if (n) {
                fill[s] = n;
                full[s] = true;
            }
            if (last) done = true;
            cv.notify_all();
            if (!last) {
                s ^= 1;
                cv.wait(lk, [&] { return !full[s] || stop; });
            }
            n = 0;
            t0 = clk::now();
        };
        auto fail = [&](int rc, uint64_t line) {
            std::lock_guard<std::mutex> lk(mu);
            reader_rc = rc;
            err_line = line;
            stop = true;
            done = true;
            cv.notify_all();
        };
        while (!stop && !eof) {
            if (have == buf.size()) buf.resize(buf.size() * 2);  // a line longer than the block
            const size_t got = fread(buf.data() + have, 1, buf.size() - have, f);
            have += got;
            if (got == 0) eof = true;
            if (ferror(f)) {
                fail(TC_EIO, 0);
                return;
            }
            // the parseable region: through the last '\n' (everything at end of file)
            size_t len = have;
            if (!eof) {
                while (len > 0 && buf[len - 1] != '\n') --len;
                if (len == 0) continue;  // no complete line yet: read more
            }
            // cut into T pieces at line starts
            std::vector<size_t> cut(T + 1, len);
            cut[0] = 0;
            for (unsigned t = 1; t < T; ++t) {
                size_t c = std::max(cut[t - 1], len * t / T);
                while (c < len && c > 0 && buf[c - 1] != '\n') ++c;
                cut[t] = c;
            }
            auto work = [&](unsigned t) {
                pn[t] = plines[t] = 0;
                prc[t] = TC_OK;
                if (cut[t + 1] == cut[t]) return;
                const uint64_t bytes = cut[t + 1] - cut[t];
                part[t].resize(bytes / 4 + 1);  // an edge line takes at least 4 bytes
                uint64_t used = 0;
                prc[t] = tc_parse_edges(buf.data() + cut[t], bytes, 1, flags, part[t].data(), part[t].size(), &pn[t],
                                        &used, &plines[t]);
            };
            std::vector<std::thread> pool;
            for (unsigned t = 1; t < T; ++t) pool.emplace_back(work, t);
            work(0);
            for (auto &th : pool) th.join();
            // in file order: each piece's edges into the slots (full slots go to the pusher); at a bad line the
            // edges before it still fill slots, but a partly filled slot is dropped
            for (unsigned t = 0; t < T && !stop; ++t) {
                for (uint64_t i = 0; i < pn[t] && !stop;) {
                    const uint64_t k = std::min(pn[t] - i, w - n);
                    memcpy(slot[s] + n, part[t].data() + i, 8 * k);
                    n += k;
                    i += k;
                    if (n == w) hand_off(false);
                }
                lines_total += plines[t];
                if (prc[t] != TC_OK && cut[t + 1] > cut[t]) {
                    fail(prc[t], lines_total);
                    return;
                }
            }
            memmove(buf.data(), buf.data() + len, have - len);
            have -= len;
        }
        hand_off(true);
    });
    // pusher: slots in order 0, 1, 0, ...
    int rc = TC_OK;
    int s = 0;
    while (true) {
        uint64_t n = 0;
        {
            std::unique_lock<std::mutex> lk(mu);
            const auto tw = clk::now();
            cv.wait(lk, [&] { return full[s] || done; });
            S.wait_s += std::chrono::duration<double>(clk::now() - tw).count();
            if (!full[s]) break;  // reader finished (or failed) and nothing is pending in this slot
            n = fill[s];
        }
        const auto tp = clk::now();
        rc = tc_push_batch(ctx, slot[s], n);  // pinned: returns once the copy is done, the slot is free again
        S.push_s += std::chrono::duration<double>(clk::now() - tp).count();
        if (rc != TC_OK) break;
        S.edges += n;
        S.batches += 1;
        {
            std::lock_guard<std::mutex> lk(mu);
            full[s] = false;
            cv.notify_all();
        }
        s ^= 1;
    }
    {
        std::lock_guard<std::mutex> lk(mu);
        stop = true;
        cv.notify_all();
    }
    reader.join();
    fclose(f);
    const int sync_rc = (rc == TC_OK && reader_rc == TC_OK) ? tc_sync(ctx) : TC_OK;
    cudaFreeHost(slot[0]);
    cudaFreeHost(slot[1]);
    S.io_s = io_s;
    S.lines = lines_total;
    S.error_line = reader_rc != TC_OK ? err_line : 0;
    S.wall_s = std::chrono::duration<double>(clk::now() - t_start).count();
    if (st) *st = S;
    if (rc != TC_OK) return rc;
    if (reader_rc != TC_OK) return reader_rc;
    return sync_rc;
}
