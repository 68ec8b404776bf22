// streamfile.cu -- FOCUSSTREAM/1 stream files: the
// decode of streamio.read_stream (streamio.py:58-113) into flat arrays, with
// host threads.  Text floats go through strtod (correctly rounded, as
// Python's float()); integers through strtoll with full consumption.
//
// open():  read the file, check the magic and header (stream_id, fps, D, S,
//          V), index the non-empty object lines;
// read():  parse the object lines in parallel straight into the caller's
//          arrays; per-line error codes, then the first failing line in file
//          order raises -- the error the reference would raise first.
#include <algorithm>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "fx_internal.cuh"

struct fx_stream_file {
    std::string data;
    std::string stream_id;
    double fps = 0.0;
    int D = 0, S = 0, V = 0;
    std::vector<size_t> line_begin, line_end;  // object lines (non-empty)
};

namespace {

enum LineErr { L_OK = 0, L_RECORD, L_VALUE, L_CLASS, L_LENGTH };

bool parse_i64(const char *b, const char *e, int64_t &v) {
    std::string s(b, e);  // int(): surrounding whitespace allowed
    const char *p = s.c_str();
    while (*p == ' ' || *p == '\t') p++;
    if (!*p) return false;
    char *end = nullptr;
    errno = 0;
    long long x = strtoll(p, &end, 10);
    if (errno || end == p) return false;
    while (*end == ' ' || *end == '\t') end++;
    if (*end) return false;
    v = x;
    return true;
}

// comma list of exactly n floats into out[0..n); -1: bad number, -2: wrong count
int parse_floats(const char *b, const char *e, int n, double *out) {
    int k = 0;
    const char *p = b;
    char buf[64];
    while (true) {
        const char *q = (const char *)memchr(p, ',', (size_t)(e - p));
        if (!q) q = e;
        const size_t len = (size_t)(q - p);
        if (len == 0 || len >= sizeof(buf)) return -1;
        memcpy(buf, p, len);
        buf[len] = 0;
        char *end = nullptr;
        const double v = strtod(buf, &end);
        char *t = end;
        while (*t == ' ' || *t == '\t') t++;
        if (end == buf || *t) return -1;
        if (k < n) out[k] = v;
        k++;
        if (q == e) break;
        p = q + 1;
    }
    return k == n ? 0 : -2;
}

}  // namespace

extern "C" {

int fx_stream_file_open(const char *path, fx_stream_file **out) {
    using namespace fx;
    fx_stream_file *f = nullptr;
    try {
        if (!path || !out) throw Error{FX_E_USAGE, "null argument"};
        f = new fx_stream_file();
        FILE *fh = fopen(path, "rb");
        if (!fh) throw Error{FX_E_USAGE, std::string("cannot open ") + path};
        fseek(fh, 0, SEEK_END);
        const long sz = ftell(fh);
        fseek(fh, 0, SEEK_SET);
        f->data.resize(sz > 0 ? (size_t)sz : 0);
        const size_t got = sz > 0 ? fread(&f->data[0], 1, (size_t)sz, fh) : 0;
        fclose(fh);
        if ((long)got != sz) throw Error{FX_E_USAGE, std::string("read failed: ") + path};
        const std::string &d = f->data;
        // lines as str.splitlines() would give them for \n / \r\n files
        std::vector<std::pair<size_t, size_t>> lines;
        for (size_t p = 0; p < d.size();) {
            size_t q = d.find('\n', p);
            if (q == std::string::npos) q = d.size();
            size_t e = q;
            if (e > p && d[e - 1] == '\r') e--;
            lines.emplace_back(p, e);
            p = q + 1;
        }
        auto text = [&](size_t i) { return d.substr(lines[i].first, lines[i].second - lines[i].first); };
        if (lines.empty() || text(0) != "FOCUSSTREAM/1")
            throw Error{FX_E_FORMAT_VERSION, "stream file must start with FOCUSSTREAM/1"};
        size_t body = 0;
        std::vector<std::pair<std::string, std::string>> kv;
        for (size_t i = 1; i < lines.size(); i++) {
            const std::string t = text(i);
            if (t == "[OBJECTS]") {
                body = i + 1;
                break;
            }
            const size_t eq = t.find('=');
            kv.emplace_back(t.substr(0, eq), eq == std::string::npos ? "" : t.substr(eq + 1));
        }
        if (!body) throw Error{FX_E_DATA, "stream file has no [OBJECTS] section"};
        auto get = [&](const char *k) -> std::string {
            for (auto it = kv.rbegin(); it != kv.rend(); ++it)  // dict(): the last assignment wins
                if (it->first == k) return it->second;
            throw Error{FX_E_DATA, std::string("bad stream header: '") + k + "'"};
        };
        f->stream_id = get("stream_id");
        {
            const std::string s = get("fps");
            char *e = nullptr;
            f->fps = strtod(s.c_str(), &e);
            if (s.empty() || *e) throw Error{FX_E_DATA, "bad stream header: fps=" + s};
        }
        for (auto kd : {std::make_pair("D", &f->D), std::make_pair("S", &f->S), std::make_pair("V", &f->V)}) {
            int64_t v = 0;
            const std::string s = get(kd.first);
            if (!parse_i64(s.data(), s.data() + s.size(), v)) throw Error{FX_E_DATA, "bad stream header: " + s};
            *kd.second = (int)v;
        }
        for (size_t i = body; i < lines.size(); i++)
            if (lines[i].second > lines[i].first) {
                f->line_begin.push_back(lines[i].first);
                f->line_end.push_back(lines[i].second);
            }
        *out = f;
    } catch (const Error &e) {
        delete f;
        set_error(e.msg);
        return e.code;
    }
    return FX_OK;
}

int fx_stream_file_header(fx_stream_file *f, char *stream_id, int64_t cap, double *fps, int32_t *dim,
                          int32_t *sig_dim, int32_t *vocab, int64_t *n_objects) {
    if (!f) return FX_E_USAGE;
    if (stream_id && cap > 0) {
        const size_t n = std::min<size_t>((size_t)cap - 1, f->stream_id.size());
        memcpy(stream_id, f->stream_id.data(), n);
        stream_id[n] = 0;
    }
    if (fps) *fps = f->fps;
    if (dim) *dim = f->D;
    if (sig_dim) *sig_dim = f->S;
    if (vocab) *vocab = f->V;
    if (n_objects) *n_objects = (int64_t)f->line_begin.size();
    return FX_OK;
}

int fx_stream_file_read(fx_stream_file *f, int64_t *object_ids, int64_t *frame_ids, int32_t *true_class,
                        double *sigs, void *feats, int32_t feats_f32, int32_t threads) {
    using namespace fx;
    try {
        if (!f || !object_ids || !frame_ids || !true_class || !sigs || !feats)
            throw Error{FX_E_USAGE, "null argument"};
        const int64_t n = (int64_t)f->line_begin.size();
        const int D = f->D, S = f->S, V = f->V;
        std::vector<unsigned char> err((size_t)n, L_OK);
        int nt = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
        nt = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)nt, 64, n}));
        auto work = [&](int64_t lo, int64_t hi) {
            std::vector<double> fbuf((size_t)std::max(D, 1));
            for (int64_t i = lo; i < hi; i++) {
                const char *b = f->data.data() + f->line_begin[i], *e = f->data.data() + f->line_end[i];
                const char *bar[4];
                int nb = 0;
                for (const char *p = b; p < e && nb <= 4; p++)
                    if (*p == '|') {
                        if (nb < 4) bar[nb] = p;
                        nb++;
                    }
                if (nb != 4) {
                    err[i] = L_RECORD;
                    continue;
                }
                int64_t oid, fid;
                if (!parse_i64(b, bar[0], oid) || !parse_i64(bar[0] + 1, bar[1], fid)) {
                    err[i] = L_VALUE;
                    continue;
                }
                object_ids[i] = oid;
                frame_ids[i] = fid;
                if (bar[2] == bar[1] + 1) {
                    true_class[i] = -2;  // unlabeled
                } else {
                    int64_t c;
                    if (!parse_i64(bar[1] + 1, bar[2], c)) {
                        err[i] = L_VALUE;
                        continue;
                    }
                    if (c < 0 || c > V) {
                        err[i] = L_CLASS;
                        continue;
                    }
                    true_class[i] = c == V ? -1 : (int32_t)c;  // decode_class: V -> OTHER
                }
                const int rs = parse_floats(bar[2] + 1, bar[3], S, sigs + i * (int64_t)S);
                if (rs == -1) {
                    err[i] = L_VALUE;
                    continue;
                }
                const int rf = parse_floats(bar[3] + 1, e, D, fbuf.data());
                if (rf == -1) {
                    err[i] = L_VALUE;
                    continue;
                }
                if (rs || rf) {
                    err[i] = L_LENGTH;
                    continue;
                }
                if (feats_f32) {
                    float *o = (float *)feats + i * (int64_t)D;
                    for (int k = 0; k < D; k++) o[k] = (float)fbuf[k];
                } else {
                    memcpy((double *)feats + i * (int64_t)D, fbuf.data(), sizeof(double) * D);
                }
            }
        };
        {
            std::vector<std::thread> pool;
            const int64_t per = (n + nt - 1) / nt;
            for (int t = 0; t < nt; t++) {
                const int64_t lo = std::min<int64_t>(n, t * per), hi = std::min<int64_t>(n, lo + per);
                pool.emplace_back(work, lo, hi);
            }
            for (auto &th : pool) th.join();
        }
        for (int64_t i = 0; i < n; i++) {  // first failure in file order, checks in the reference's order
            const std::string rec = f->data.substr(f->line_begin[i], std::min<size_t>(80, f->line_end[i] - f->line_begin[i]));
            switch (err[i]) {
            case L_RECORD: throw Error{FX_E_DATA, "bad object record: " + rec};
            case L_VALUE: throw Error{FX_E_VALUE, "invalid literal in object record: " + rec};
            case L_CLASS: throw Error{FX_E_DATA, "class id outside vocabulary in: " + rec};
            case L_LENGTH:
                throw Error{FX_E_DATA, "object " + std::to_string(object_ids[i]) + ": vector length mismatch with header"};
            default: break;
            }
            if (i > 0 && object_ids[i] <= object_ids[i - 1])
                throw Error{FX_E_DATA, "object ids must strictly increase (at " + std::to_string(object_ids[i]) + ")"};
            if (i > 0 && frame_ids[i] < frame_ids[i - 1])
                throw Error{FX_E_DATA,
                            "frame ids must be non-decreasing (at object " + std::to_string(object_ids[i]) + ")"};
        }
    } catch (const Error &e) {
        set_error(e.msg);
        return e.code;
    }
    return FX_OK;
}

int fx_stream_file_close(fx_stream_file *f) {
    delete f;
    return FX_OK;
}

}  // extern "C"
