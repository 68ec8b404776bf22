// index_read.cu -- FOCUSIDX/1 reader (the load half):
// index.load (index.py:131-204) as a native parser.  Host-only.
//
// The file is read once, newline-translated as Python's text mode does
// (\r\n, \r -> \n), the CRC-32 trailer checked over the body, the body cut
// into lines the way str.splitlines() cuts them, and the cluster records and
// postings parsed by a pool of host threads straight into CSR arrays (the
// layout fx_index_build takes, so a loaded index is posted on the device
// without building Python objects).  Errors: the first one the reference
// would raise, in its evaluation order -- every record is parsed into a
// per-line status, then one pass in file order picks the first failure
// (duplicate cluster ids are only known in that pass).
//
// Number syntax follows Python's int() / float(): surrounding whitespace,
// an optional sign, underscores between digits; float() also takes
// inf/infinity/nan in any case and rejects hex.  Integers outside int64 are
// rejected (DataError) -- the one place the reader is narrower than Python.
#include <algorithm>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "fx_internal.cuh"

namespace {

using fx::Error;

uint32_t crc_table[256];
bool crc_ready = false;

uint32_t crc32_of(const char *p, size_t n) {
    if (!crc_ready) {
        for (uint32_t i = 0; i < 256; i++) {
            uint32_t c = i;
            for (int k = 0; k < 8; k++) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
            crc_table[i] = c;
        }
        crc_ready = true;
    }
    uint32_t c = ~0u;
    for (size_t i = 0; i < n; i++) c = crc_table[(c ^ (unsigned char)p[i]) & 0xFF] ^ (c >> 8);
    return ~c;
}

// str.strip() whitespace for ASCII input (int() / float() strip before parsing)
inline bool py_space(char c) { return c == ' ' || (c >= '\t' && c <= '\r') || (c >= 0x1c && c <= 0x1f); }

// copy [b, e) without surrounding whitespace and without the underscores
// Python allows between digits; false if an underscore is misplaced
bool py_clean(const char *b, const char *e, std::string &out) {
    while (b < e && py_space(*b)) b++;
    while (e > b && py_space(e[-1])) e--;
    out.clear();
    for (const char *p = b; p < e; p++) {
        if (*p == '_') {
            if (p == b || p + 1 >= e || !isdigit((unsigned char)p[-1]) || !isdigit((unsigned char)p[1])) return false;
            continue;
        }
        out.push_back(*p);
    }
    return !out.empty();
}

bool py_int(const char *b, const char *e, int64_t &v) {
    std::string s;
    if (!py_clean(b, e, s)) return false;
    size_t i = (s[0] == '+' || s[0] == '-') ? 1 : 0;
    if (i >= s.size()) return false;
    for (size_t k = i; k < s.size(); k++)
        if (!isdigit((unsigned char)s[k])) return false;
    errno = 0;
    char *end = nullptr;
    const long long x = strtoll(s.c_str(), &end, 10);
    if (errno || *end) return false;
    v = x;
    return true;
}

bool py_float(const char *b, const char *e, double &v) {
    std::string s;
    if (!py_clean(b, e, s)) return false;
    for (char c : s)  // strtod also takes hex and nan(...) forms: Python does not
        if (c == 'x' || c == 'X' || c == '(' || c == 'p' || c == 'P') return false;
    char *end = nullptr;
    v = strtod(s.c_str(), &end);
    return end && *end == 0;
}

// one status per record, in the reference's evaluation order
enum RecErr {
    R_OK = 0,
    R_PARTS,     // DataError: bad cluster record
    R_CID,       // ValueError: int(parts[0])
    R_RANK,      // ValueError: int(rank) / int(cls)
    R_CLASS,     // DataError: decode_class
    R_CENTROID,  // ValueError: float()
    R_MEMBER,    // ValueError: int() of a member / frame id
    R_CMID,      // ValueError: int(parts[1])
};

struct Rec {
    int err = R_OK;
    std::string msg;
    int64_t cid = 0, cmid = INT64_MIN;
    std::vector<double> cen;
    std::vector<int64_t> mem, fr;
    std::vector<std::pair<int32_t, int32_t>> ranks;  // decoded class (OTHER = -1), rank; dict order
};

void dict_set(std::vector<std::pair<int32_t, int32_t>> &d, int32_t k, int32_t v) {
    for (auto &kv : d)
        if (kv.first == k) {
            kv.second = v;
            return;
        }
    d.emplace_back(k, v);
}

bool split_i64(const char *b, const char *e, std::vector<int64_t> &out) {
    for (const char *p = b;;) {
        const char *q = (const char *)memchr(p, ',', (size_t)(e - p));
        if (!q) q = e;
        int64_t x;
        if (!py_int(p, q, x)) return false;
        out.push_back(x);
        if (q == e) return true;
        p = q + 1;
    }
}

bool decode(int64_t raw, int64_t V, int32_t &c) {
    if (raw == V) {
        c = -1;
        return true;
    }
    if (raw < 0 || raw >= V) return false;
    c = (int32_t)raw;
    return true;
}

void parse_record(const char *b, const char *e, int64_t V, Rec &r) {
    const char *bar[6];
    int nb = 0;
    for (const char *p = b; p < e; p++)
        if (*p == '|') {
            if (nb < 6) bar[nb] = p;
            nb++;
        }
    if (nb != 5) {
        r.err = R_PARTS;
        return;
    }
    const char *f0 = b, *f1 = bar[0] + 1, *f2 = bar[1] + 1, *f3 = bar[2] + 1, *f4 = bar[3] + 1, *f5 = bar[4] + 1;
    if (!py_int(f0, bar[0], r.cid)) {
        r.err = R_CID;
        return;
    }
    if (f5 < e) {  // "cls:rank" items: int(rank), then int(cls), then decode_class (RHS first)
        for (const char *p = f5;;) {
            const char *q = (const char *)memchr(p, ',', (size_t)(e - p));
            if (!q) q = e;
            const char *colon = (const char *)memchr(p, ':', (size_t)(q - p));
            const char *ce = colon ? colon : q, *rb = colon ? colon + 1 : q;
            int64_t rank, cls;
            if (!py_int(rb, q, rank) || !py_int(p, ce, cls)) {
                r.err = R_RANK;
                return;
            }
            int32_t c;
            if (!decode(cls, V, c)) {
                r.err = R_CLASS;
                r.msg = "class id " + std::to_string(cls) + " outside vocabulary [0, " + std::to_string(V) + "]";
                return;
            }
            if (rank < INT32_MIN || rank > INT32_MAX) {
                r.err = R_RANK;
                return;
            }
            dict_set(r.ranks, c, (int32_t)rank);
            if (q == e) break;
            p = q + 1;
        }
    }
    for (const char *p = f2;;) {
        const char *q = (const char *)memchr(p, ',', (size_t)(bar[2] - p));
        if (!q) q = bar[2];
        double x;
        if (!py_float(p, q, x)) {
            r.err = R_CENTROID;
            return;
        }
        r.cen.push_back(x);
        if (q == bar[2]) break;
        p = q + 1;
    }
    if (!split_i64(f3, bar[3], r.mem) || !split_i64(f4, bar[4], r.fr)) {
        r.err = R_MEMBER;
        return;
    }
    if (f1 != bar[1] && !py_int(f1, bar[1], r.cmid)) {
        r.err = R_CMID;
        return;
    }
    if (f1 == bar[1]) r.cmid = INT64_MIN;  // no representative (None)
}

}  // namespace

struct fx_index_file {
    std::string text;                                // newline-translated file
    std::vector<std::pair<size_t, size_t>> lines;    // body lines (str.splitlines)
    size_t c0 = 0;                                   // first line after [CLUSTERS]
    std::string header;                              // lines between the magic and [CLUSTERS], '\n'-joined
    int64_t V = -1;
    std::vector<int64_t> cid, cmid, cen_off{0}, mem_off{0}, fr_off{0}, cls_off{0};
    std::vector<double> cen;
    std::vector<int64_t> mem, fr;
    std::vector<int32_t> cls, rank;
    std::vector<int32_t> post_cls;  // decoded, dict order
    std::vector<int64_t> post_off{0}, post_ids;
};

extern "C" {

int fx_index_read(const char *path, fx_index_file **out) {
    using namespace fx;
    fx_index_file *f = nullptr;
    try {
        if (!path || !out) throw Error{FX_E_USAGE, "null argument"};
        FILE *fh = fopen(path, "rb");
        if (!fh) throw Error{FX_E_USAGE, std::string("cannot open ") + path};
        std::string raw;
        fseek(fh, 0, SEEK_END);
        const long sz = ftell(fh);
        fseek(fh, 0, SEEK_SET);
        raw.resize(sz > 0 ? (size_t)sz : 0);
        const size_t got = sz > 0 ? fread(&raw[0], 1, (size_t)sz, fh) : 0;
        fclose(fh);
        if ((long)got != sz) throw Error{FX_E_USAGE, std::string("read failed: ") + path};
        // utf-8 check (open(..., encoding="utf-8") raises UnicodeDecodeError, a ValueError)
        for (size_t i = 0; i < raw.size();) {
            const unsigned char c = (unsigned char)raw[i];
            int n = c < 0x80 ? 0 : (c >> 5) == 6 ? 1 : (c >> 4) == 14 ? 2 : (c >> 3) == 30 ? 3 : -1;
            if (n < 0 || i + n >= raw.size() + (n ? 0 : 1)) throw Error{FX_E_VALUE, "index file is not valid utf-8"};
            for (int k = 1; k <= n; k++)
                if (((unsigned char)raw[i + k] >> 6) != 2) throw Error{FX_E_VALUE, "index file is not valid utf-8"};
            i += n + 1;
        }
        // text mode: \r\n and \r read as \n
        std::string d;
        d.reserve(raw.size());
        for (size_t i = 0; i < raw.size(); i++) {
            if (raw[i] == '\r') {
                d.push_back('\n');
                if (i + 1 < raw.size() && raw[i + 1] == '\n') i++;
            } else {
                d.push_back(raw[i]);
            }
        }
        std::string().swap(raw);
        // data.rstrip("\n").rpartition("\n") -> body, trailer
        size_t end = d.size();
        while (end > 0 && d[end - 1] == '\n') end--;
        const size_t nl = end ? d.rfind('\n', end - 1) : std::string::npos;
        const size_t body_len = nl == std::string::npos ? 0 : nl + 1;
        const std::string last = d.substr(body_len, end - body_len);
        if (last.compare(0, 6, "CRC32:") != 0) throw Error{FX_E_CHECKSUM, "missing CRC32 trailer"};
        char actual[16];
        snprintf(actual, sizeof actual, "%08x", crc32_of(d.data(), body_len));
        if (last.substr(6) != actual)
            throw Error{FX_E_CHECKSUM, "CRC mismatch: file says " + last.substr(6) + ", computed " + actual};
        // str.splitlines() of the body
        std::vector<std::pair<size_t, size_t>> lines;
        {
            size_t b = 0;
            for (size_t i = 0; i < body_len;) {
                const unsigned char c = (unsigned char)d[i];
                int w = 0;
                if (c == '\n' || c == 0x0b || c == 0x0c || c == 0x1c || c == 0x1d || c == 0x1e) w = 1;
                else if (c == 0xc2 && i + 1 < body_len && (unsigned char)d[i + 1] == 0x85) w = 2;
                else if (c == 0xe2 && i + 2 < body_len && (unsigned char)d[i + 1] == 0x80 &&
                         ((unsigned char)d[i + 2] == 0xa8 || (unsigned char)d[i + 2] == 0xa9)) w = 3;
                if (w) {
                    lines.emplace_back(b, i);
                    i += w;
                    b = i;
                } else {
                    i++;
                }
            }
            if (b < body_len) lines.emplace_back(b, body_len);
        }
        auto is = [&](size_t i, const char *s) {
            const size_t n = strlen(s);
            return lines[i].second - lines[i].first == n && d.compare(lines[i].first, n, s) == 0;
        };
        if (lines.empty() || !is(0, "FOCUSIDX/1"))
            throw Error{FX_E_FORMAT_VERSION, "index file must start with FOCUSIDX/1"};
        f = new fx_index_file();
        size_t i = 1;
        for (; i < lines.size() && !is(i, "[CLUSTERS]"); i++) {
            if (i > 1) f->header.push_back('\n');
            f->header.append(d, lines[i].first, lines[i].second - lines[i].first);
        }
        if (i >= lines.size()) throw Error{FX_E_DATA, "index file has no [CLUSTERS] section"};
        f->c0 = i + 1;
        f->text.swap(d);
        f->lines.swap(lines);
        *out = f;
        return FX_OK;
    } catch (const Error &e) {
        delete f;
        set_error(e.msg);
        return e.code;
    } catch (const std::exception &e) {
        delete f;
        set_error(e.what());
        return FX_E_INTERNAL;
    }
}

// Parse the cluster records and postings (after the caller parsed the header
// lines with fx_index_file_header: their errors come first in the reference,
// and decode_class needs the vocabulary V they hold).
int fx_index_file_parse(fx_index_file *f, int64_t vocab) {
    using namespace fx;
    try {
        if (!f) throw Error{FX_E_USAGE, "null argument"};
        f->V = vocab;
        const std::string &d = f->text;
        const auto &lines = f->lines;
        auto is = [&](size_t i, const char *s) {
            const size_t n = strlen(s);
            return lines[i].second - lines[i].first == n && d.compare(lines[i].first, n, s) == 0;
        };
        const size_t c0 = f->c0;
        size_t c1 = c0;
        while (c1 < lines.size() && !is(c1, "[POSTINGS]")) c1++;
        const size_t nrec = c1 - c0;
        std::vector<Rec> recs(nrec);
        {
            const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
            std::vector<std::thread> pool;
            for (unsigned t = 0; t < nt; t++)
                pool.emplace_back([&, t] {
                    for (size_t k = t; k < nrec; k += nt)
                        parse_record(d.data() + lines[c0 + k].first, d.data() + lines[c0 + k].second, vocab,
                                     recs[k]);
                });
            for (auto &th : pool) th.join();
        }
        std::unordered_set<int64_t> seen;
        for (size_t k = 0; k < nrec; k++) {
            Rec &r = recs[k];
            const std::string line = d.substr(lines[c0 + k].first, lines[c0 + k].second - lines[c0 + k].first);
            if (r.err == R_PARTS) throw Error{FX_E_DATA, "bad cluster record: " + line};
            if (r.err == R_CID) throw Error{FX_E_VALUE, "invalid literal for int(): " + line};
            if (!seen.insert(r.cid).second) throw Error{FX_E_DUPLICATE_CLUSTER_ID, std::to_string(r.cid)};
            if (r.err == R_CLASS) throw Error{FX_E_DATA, r.msg};
            if (r.err != R_OK) throw Error{FX_E_VALUE, "bad number in cluster record " + std::to_string(r.cid)};
            f->cid.push_back(r.cid);
            f->cmid.push_back(r.cmid);
            f->cen.insert(f->cen.end(), r.cen.begin(), r.cen.end());
            f->cen_off.push_back((int64_t)f->cen.size());
            f->mem.insert(f->mem.end(), r.mem.begin(), r.mem.end());
            f->mem_off.push_back((int64_t)f->mem.size());
            f->fr.insert(f->fr.end(), r.fr.begin(), r.fr.end());
            f->fr_off.push_back((int64_t)f->fr.size());
            for (auto &kv : r.ranks) {
                f->cls.push_back(kv.first);
                f->rank.push_back(kv.second);
            }
            f->cls_off.push_back((int64_t)f->cls.size());
            Rec().cen.swap(r.cen);
        }
        if (c1 >= lines.size()) throw Error{FX_E_DATA, "index file has no [POSTINGS] section"};
        // postings: postings[decode_class(int(cls))] = [int(x) for x in ids] (RHS first)
        std::vector<std::vector<int64_t>> plist;
        for (size_t k = c1 + 1; k < lines.size(); k++) {
            const char *b = d.data() + lines[k].first, *e = d.data() + lines[k].second;
            const char *bar = (const char *)memchr(b, '|', (size_t)(e - b));
            const char *ib = bar ? bar + 1 : e;
            std::vector<int64_t> ids;
            if (!split_i64(ib, e, ids)) throw Error{FX_E_VALUE, "bad posting id list"};
            int64_t cls;
            if (!py_int(b, bar ? bar : e, cls)) throw Error{FX_E_VALUE, "bad posting class"};
            int32_t c;
            if (!decode(cls, vocab, c))
                throw Error{FX_E_DATA,
                            "class id " + std::to_string(cls) + " outside vocabulary [0, " + std::to_string(vocab) + "]"};
            size_t at = 0;
            while (at < f->post_cls.size() && f->post_cls[at] != c) at++;
            if (at == f->post_cls.size()) {
                f->post_cls.push_back(c);
                plist.emplace_back(std::move(ids));
            } else {
                plist[at] = std::move(ids);  // dict: a repeated key keeps its place, takes the new value
            }
        }
        for (auto &v : plist) {
            f->post_ids.insert(f->post_ids.end(), v.begin(), v.end());
            f->post_off.push_back((int64_t)f->post_ids.size());
        }
        return FX_OK;
    } catch (const Error &e) {
        set_error(e.msg);
        return e.code;
    } catch (const std::exception &e) {
        set_error(e.what());
        return FX_E_INTERNAL;
    }
}

int fx_index_file_header(const fx_index_file *f, char *buf, int64_t cap, int64_t *len) {
    if (!f || !len) return FX_E_USAGE;
    *len = (int64_t)f->header.size();
    if (buf && cap > 0) memcpy(buf, f->header.data(), (size_t)std::min<int64_t>(cap, *len));
    return FX_OK;
}

int fx_index_file_sizes(const fx_index_file *f, int64_t *out) {
    if (!f || !out) return FX_E_USAGE;
    out[0] = (int64_t)f->cid.size();
    out[1] = (int64_t)f->cen.size();
    out[2] = (int64_t)f->mem.size();
    out[3] = (int64_t)f->fr.size();
    out[4] = (int64_t)f->cls.size();
    out[5] = (int64_t)f->post_cls.size();
    out[6] = (int64_t)f->post_ids.size();
    return FX_OK;
}

int fx_index_file_export(const fx_index_file *f, int64_t *cid, int64_t *cmid, int64_t *cen_off, double *cen,
                         int64_t *mem_off, int64_t *mem, int64_t *fr_off, int64_t *fr, int64_t *cls_off,
                         int32_t *cls, int32_t *rank, int32_t *post_cls, int64_t *post_off, int64_t *post_ids) {
    if (!f) return FX_E_USAGE;
    auto cp = [](auto *dst, const auto &v) {
        if (dst && !v.empty()) memcpy(dst, v.data(), sizeof(v[0]) * v.size());
    };
    cp(cid, f->cid);
    cp(cmid, f->cmid);
    cp(cen_off, f->cen_off);
    cp(cen, f->cen);
    cp(mem_off, f->mem_off);
    cp(mem, f->mem);
    cp(fr_off, f->fr_off);
    cp(fr, f->fr);
    cp(cls_off, f->cls_off);
    cp(cls, f->cls);
    cp(rank, f->rank);
    cp(post_cls, f->post_cls);
    cp(post_off, f->post_off);
    cp(post_ids, f->post_ids);
    return FX_OK;
}

int fx_index_file_free(fx_index_file *f) {
    delete f;
    return FX_OK;
}

}  // extern "C"
