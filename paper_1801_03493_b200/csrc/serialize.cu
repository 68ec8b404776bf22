// serialize.cu -- FOCUSIDX/1 index files: the text the
// reference's index._render produces (index.py:88-120), byte for byte, from
// an index in the fx_index_export host layout.
//
//   <head lines built by the caller: magic, stream_id=, D=, V=, n=, config>
//   [CLUSTERS]
//   cid|rep|c_0,...,c_{D-1} (%.9g)|oid,...|fid,...|cls:rank,... (by encoded class)
//   [POSTINGS]
//   cls|cid,...            (non-empty classes by encoded class, OTHER = V)
//   CRC32:xxxxxxxx         (zlib CRC-32 of everything above)
//
// Formatting n x D float64 centroids with %.9g dominates; clusters are
// rendered in parallel by host threads in cid order and concatenated.
#include <algorithm>
#include <charconv>
#include <cstdio>
#include <string>
#include <thread>
#include <vector>

#include "fx_internal.cuh"

namespace {

uint32_t g_crc_table[256];

void crc_init() {
    static bool done = false;
    if (done) return;
    for (uint32_t i = 0; i < 256; i++) {
        uint32_t c = i;
        for (int k = 0; k < 8; k++) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
        g_crc_table[i] = c;
    }
    done = true;
}

uint32_t crc_update(uint32_t crc, const char *p, size_t n) {
    crc = ~crc;
    for (size_t i = 0; i < n; i++) crc = g_crc_table[(crc ^ (unsigned char)p[i]) & 0xFF] ^ (crc >> 8);
    return ~crc;
}

void put_int(std::string &s, int64_t v) {
    char b[24];
    auto r = std::to_chars(b, b + sizeof(b), v);
    s.append(b, r.ptr);
}

void put_g9(std::string &s, double v) {  // Python f"{v:.9g}" == C %.9g for finite values
    char b[40];
    const int n = snprintf(b, sizeof(b), "%.9g", v);
    s.append(b, (size_t)n);
}

struct RenderArgs {
    int64_t C;
    int D;
    int V;
    const int64_t *ids, *reps, *mem_off, *mem_oid, *mem_fid, *cls_off;
    const double *cen;
    const int32_t *cls_id, *cls_rank;
};

void render_clusters(const RenderArgs &a, const std::vector<int64_t> &order, int64_t lo, int64_t hi, std::string &out) {
    std::vector<std::pair<int32_t, int32_t>> ranks;
    for (int64_t j = lo; j < hi; j++) {
        const int64_t i = order[j];
        put_int(out, a.ids[i]);
        out.push_back('|');
        if (a.reps[i] >= 0) put_int(out, a.reps[i]);
        out.push_back('|');
        const double *c = a.cen + i * (int64_t)a.D;
        for (int k = 0; k < a.D; k++) {
            if (k) out.push_back(',');
            put_g9(out, c[k]);
        }
        out.push_back('|');
        for (int64_t m = a.mem_off[i]; m < a.mem_off[i + 1]; m++) {
            if (m > a.mem_off[i]) out.push_back(',');
            put_int(out, a.mem_oid[m]);
        }
        out.push_back('|');
        for (int64_t m = a.mem_off[i]; m < a.mem_off[i + 1]; m++) {
            if (m > a.mem_off[i]) out.push_back(',');
            put_int(out, a.mem_fid[m]);
        }
        out.push_back('|');
        ranks.clear();
        for (int64_t e = a.cls_off[i]; e < a.cls_off[i + 1]; e++) ranks.emplace_back(a.cls_id[e], a.cls_rank[e]);
        std::sort(ranks.begin(), ranks.end());
        for (size_t e = 0; e < ranks.size(); e++) {
            if (e) out.push_back(',');
            put_int(out, ranks[e].first);
            out.push_back(':');
            put_int(out, ranks[e].second);
        }
        out.push_back('\n');
    }
}

}  // namespace

extern "C" int fx_index_write(const char *path, const char *head, int64_t head_len, int64_t n_clusters,
                              int32_t dim, int32_t vocab, const int64_t *cluster_ids, const double *centroids,
                              const int64_t *reps, const int64_t *mem_off, const int64_t *mem_oid,
                              const int64_t *mem_fid, const int64_t *cls_off, const int32_t *cls_id,
                              const int32_t *cls_rank, const int64_t *post_off, const int64_t *post_cluster,
                              int32_t threads) {
    using namespace fx;
    try {
        if (!path || !head || head_len < 0 || n_clusters < 0 || dim < 1 || vocab < 1)
            throw Error{FX_E_USAGE, "fx_index_write: bad arguments"};
        if (n_clusters > 0 && (!cluster_ids || !centroids || !reps || !mem_off || !mem_oid || !mem_fid || !cls_off))
            throw Error{FX_E_USAGE, "fx_index_write: cluster arrays (with centroids) required"};
        if (!post_off) throw Error{FX_E_USAGE, "fx_index_write: postings required"};
        crc_init();
        RenderArgs a{n_clusters, dim, vocab, cluster_ids, reps, mem_off, mem_oid, mem_fid, cls_off, centroids,
                     cls_id, cls_rank};
        std::vector<int64_t> order((size_t)n_clusters);
        for (int64_t i = 0; i < n_clusters; i++) order[i] = i;
        std::sort(order.begin(), order.end(), [&](int64_t x, int64_t y) { return cluster_ids[x] < cluster_ids[y]; });
        int nt = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
        nt = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)nt, 64, n_clusters}));
        std::vector<std::string> parts((size_t)nt);
        {
            std::vector<std::thread> pool;
            const int64_t per = (n_clusters + nt - 1) / nt;
            for (int t = 0; t < nt; t++) {
                const int64_t lo = std::min<int64_t>(n_clusters, t * per), hi = std::min<int64_t>(n_clusters, lo + per);
                pool.emplace_back([&, lo, hi, t] { render_clusters(a, order, lo, hi, parts[t]); });
            }
            for (auto &th : pool) th.join();
        }
        std::string tail = "[POSTINGS]\n";
        for (int enc = 0; enc <= vocab; enc++) {
            const int64_t p0 = post_off[enc], p1 = post_off[enc + 1];
            if (p1 <= p0) continue;
            put_int(tail, enc);
            tail.push_back('|');
            for (int64_t p = p0; p < p1; p++) {
                if (p > p0) tail.push_back(',');
                put_int(tail, post_cluster[p]);
            }
            tail.push_back('\n');
        }
        FILE *f = fopen(path, "wb");
        if (!f) throw Error{FX_E_USAGE, std::string("cannot open ") + path};
        uint32_t crc = 0;
        bool ok = true;
        auto emit = [&](const char *p, size_t n) {
            crc = crc_update(crc, p, n);
            ok = ok && fwrite(p, 1, n, f) == n;
        };
        emit(head, (size_t)head_len);
        for (auto &s : parts) emit(s.data(), s.size());
        emit(tail.data(), tail.size());
        char trailer[32];
        const int n = snprintf(trailer, sizeof(trailer), "CRC32:%08x\n", crc);
        ok = ok && fwrite(trailer, 1, (size_t)n, f) == (size_t)n;
        ok = (fclose(f) == 0) && ok;
        if (!ok) throw Error{FX_E_USAGE, std::string("write failed: ") + path};
    } catch (const Error &e) {
        set_error(e.msg);
        return e.code;
    } catch (const std::exception &e) {
        set_error(e.what());
        return FX_E_INTERNAL;
    }
    return FX_OK;
}
