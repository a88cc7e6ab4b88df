// aut.cpp -- multi-threaded Aldebaran (.aut) ingestion.
//
// Restates parse_aut (/root/reference/pkg/src/parbisim/aut.py:79-92) with
// its helpers parse_header (:37-45) and _parse_transition (:48-76), and the
// label numbering of lts_from_labeled_edges (lts.py:59-73: ids follow the
// sorted label strings).  Same acceptance, same results, same error
// messages and line numbers:
//
//   * lines are split like Python's str.splitlines() (\n, \r\n, \r, \v, \f,
//     \x1c-\x1e, U+0085, U+2028, U+2029); line 1 is the header, blank
//     transition lines are skipped;
//   * "strip" and the regex \s are Python's str whitespace (ASCII, \x1c-\x1f
//     and the Unicode space separators);
//   * integers follow Python int(): optional sign, digits, single
//     underscores between digits;
//   * the first failing line (in file order) is reported; the transition
//     count is checked last.
//
// Known, documented deviations (inputs no .aut tool produces): non-ASCII
// decimal digits are not accepted as digits, and repr() of a non-ASCII
// character in an error message treats U+0080-U+00A0 and U+00AD as
// unprintable and every other non-ASCII character as printable.  Counts
// beyond the C ABI's integer widths (n >= 2^30) are rejected.
//
// Parsing is split over threads at '\n' boundaries: every thread parses its
// chunk into (src, local label id, dst) columns and a local label table;
// label tables are merged and sorted once, then local ids are remapped.
#include <algorithm>
#include <cstdint>
#include <new>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_map>
#include <vector>

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include "../../include/bisim.h"

namespace bisim {
void set_last_error(const std::string& msg);
}

namespace {

// An int32 column of up to `cap` entries in anonymous memory advised for
// transparent huge pages: filling hundreds of MB of 4 KB pages from several
// threads is page-fault bound.  Pages are touched by the writing thread.
struct Column {
    int32_t* p = nullptr;
    size_t cap = 0, n = 0;
    size_t bytes = 0;
    void alloc(size_t c) {
        cap = c;
        bytes = std::max<size_t>(c * 4, 4096);
        void* m = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (m == MAP_FAILED) throw std::bad_alloc();
        madvise(m, bytes, MADV_HUGEPAGE);
        p = (int32_t*)m;
    }
    void push(int32_t v) { p[n++] = v; }
    Column() = default;
    Column(const Column&) = delete;
    Column& operator=(const Column&) = delete;
    Column(Column&& o) noexcept : p(o.p), cap(o.cap), n(o.n), bytes(o.bytes) { o.p = nullptr; }
    ~Column() {
        if (p) munmap(p, bytes);
    }
};

// Parsed columns of one chunk: (source, local label id, target).
struct Parsed {
    Column src, lab, dst;
    std::vector<int32_t> rank;  // local label id -> action id
};

}  // namespace

struct bisim_aut {
    int32_t n = 0;
    int32_t initial = 0;
    int64_t m = 0;
    std::vector<std::string> labels;
    std::vector<Parsed> parts;  // in file order; action ids via each part's rank
};

namespace {

using std::string;
using std::string_view;

// ---- Python str semantics on UTF-8 bytes -----------------------------------

// Length of a line terminator starting at p (0 if none), as str.splitlines.
inline int line_break(const char* p, const char* end) {
    const unsigned char c = (unsigned char)*p;
    if (c == '\n' || c == '\v' || c == '\f' || c == 0x1c || c == 0x1d || c == 0x1e) return 1;
    if (c == '\r') return (p + 1 < end && p[1] == '\n') ? 2 : 1;
    if (c == 0xc2 && p + 1 < end && (unsigned char)p[1] == 0x85) return 2;
    if (c == 0xe2 && p + 2 < end && (unsigned char)p[1] == 0x80 &&
        ((unsigned char)p[2] == 0xa8 || (unsigned char)p[2] == 0xa9))
        return 3;
    return 0;
}

// Length of a whitespace character (str.isspace) starting at p, else 0.
inline int space_at(const char* p, const char* end) {
    const unsigned char c = (unsigned char)*p;
    if (c == ' ' || (c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x1f)) return 1;
    if (c < 0x80) return 0;
    const unsigned char c1 = p + 1 < end ? (unsigned char)p[1] : 0;
    if (c == 0xc2 && (c1 == 0x85 || c1 == 0xa0)) return 2;
    if (p + 2 >= end) return 0;
    const unsigned char c2 = (unsigned char)p[2];
    if (c == 0xe1 && c1 == 0x9a && c2 == 0x80) return 3;                       // U+1680
    if (c == 0xe2 && c1 == 0x80 && (c2 <= 0x8a || c2 == 0xa8 || c2 == 0xa9 || c2 == 0xaf)) return 3;
    if (c == 0xe2 && c1 == 0x81 && c2 == 0x9f) return 3;                       // U+205F
    if (c == 0xe3 && c1 == 0x80 && c2 == 0x80) return 3;                       // U+3000
    return 0;
}

// Whitespace character ending just before e (e > b), else 0.
inline int space_before(const char* b, const char* e) {
    for (int k = 1; k <= 3 && e - k >= b; ++k) {
        const unsigned char c = (unsigned char)e[-k];
        if (k == 1 && c < 0x80) return space_at(e - 1, e) ? 1 : 0;
        if (c >= 0xc0) return space_at(e - k, e) == k ? k : 0;  // lead byte found
    }
    return 0;
}

inline string_view strip(string_view s) {
    const char* b = s.data();
    const char* e = b + s.size();
    while (b < e) {
        const int k = space_at(b, e);
        if (!k) break;
        b += k;
    }
    while (e > b) {
        const int k = space_before(b, e);
        if (!k) break;
        e -= k;
    }
    return string_view(b, (size_t)(e - b));
}

inline int skip_space(string_view s, size_t i) {
    while (i < s.size()) {
        const int k = space_at(s.data() + i, s.data() + s.size());
        if (!k) break;
        i += (size_t)k;
    }
    return (int)i;
}

// Python int(): [+-] digit ( [_] digit )*.  Writes the normalised decimal
// (what str(int(x)) prints) and, when it fits, the value.
struct PyInt {
    bool ok = false;
    bool fits = false;  // |value| < 2^62
    int64_t value = 0;
    string text;        // normalised decimal
};

PyInt py_int(string_view s) {
    PyInt r;
    size_t i = 0;
    bool neg = false;
    if (i < s.size() && (s[i] == '+' || s[i] == '-')) neg = s[i++] == '-';
    if (i >= s.size()) return r;
    string digits;
    bool prev_digit = false;
    for (; i < s.size(); ++i) {
        const char c = s[i];
        if (c >= '0' && c <= '9') {
            digits.push_back(c);
            prev_digit = true;
        } else if (c == '_' && prev_digit && i + 1 < s.size() && s[i + 1] >= '0' && s[i + 1] <= '9') {
            prev_digit = false;
        } else {
            return r;
        }
    }
    if (digits.empty()) return r;
    size_t z = 0;
    while (z + 1 < digits.size() && digits[z] == '0') ++z;
    digits.erase(0, z);
    r.ok = true;
    const bool zero = digits == "0";
    r.text = (neg && !zero ? "-" : "") + digits;
    if (digits.size() <= 18) {
        r.fits = true;
        r.value = std::stoll(digits) * (neg ? -1 : 1);
    }
    return r;
}

void append_hex(string& o, const char* pre, uint32_t v, int width) {
    static const char* hx = "0123456789abcdef";
    o += pre;
    for (int k = width - 1; k >= 0; --k) o.push_back(hx[(v >> (4 * k)) & 15u]);
}

// repr() of a str given as UTF-8 (see the header for the non-ASCII rule).
string py_repr(string_view s) {
    const bool dq = s.find('\'') != string_view::npos && s.find('"') == string_view::npos;
    const char q = dq ? '"' : '\'';
    string o(1, q);
    for (size_t i = 0; i < s.size();) {
        const unsigned char c = (unsigned char)s[i];
        if (c < 0x80) {
            if (c == '\\') o += "\\\\";
            else if (c == (unsigned char)q) { o.push_back('\\'); o.push_back(q); }
            else if (c == '\t') o += "\\t";
            else if (c == '\n') o += "\\n";
            else if (c == '\r') o += "\\r";
            else if (c < 0x20 || c == 0x7f) append_hex(o, "\\x", c, 2);
            else o.push_back((char)c);
            ++i;
            continue;
        }
        int len = c >= 0xf0 ? 4 : c >= 0xe0 ? 3 : c >= 0xc0 ? 2 : 1;
        if (i + (size_t)len > s.size()) len = 1;
        uint32_t cp = len == 1 ? c : (c & (0x7f >> len));
        for (int k = 1; k < len; ++k) cp = (cp << 6) | ((unsigned char)s[i + k] & 0x3f);
        if ((cp >= 0x80 && cp <= 0xa0) || cp == 0xad) append_hex(o, "\\x", cp, 2);
        else o.append(s.data() + i, (size_t)len);
        i += (size_t)len;
    }
    o.push_back(q);
    return o;
}

struct ParseFail {
    int64_t line = 0;  // 1-based; 0 = no line
    string msg;
};

// ---- header (aut.py:37-45) ------------------------------------------------

// des\s*\(\s*(\d+)\s*,\s*(\d+)\s*,\s*(\d+)\s*\)\s*$ on the stripped line
bool match_header(string_view line, string (&num)[3]) {
    string_view s = strip(line);
    if (s.substr(0, 3) != "des") return false;
    size_t i = skip_space(s, 3);
    if (i >= s.size() || s[i] != '(') return false;
    ++i;
    for (int k = 0; k < 3; ++k) {
        i = skip_space(s, i);
        const size_t d0 = i;
        while (i < s.size() && s[i] >= '0' && s[i] <= '9') ++i;
        if (i == d0) return false;
        num[k] = string(s.substr(d0, i - d0));
        i = skip_space(s, i);
        const char want = k < 2 ? ',' : ')';
        if (i >= s.size() || s[i] != want) return false;
        ++i;
    }
    i = skip_space(s, i);
    return i == s.size();
}

// ---- one transition line (aut.py:48-76) -----------------------------------

// Each chunk is written by one thread only: cache-line aligned so that the
// vectors' bookkeeping of neighbouring chunks never shares a line (false
// sharing on every push_back serialised the threads).
struct alignas(128) Chunk {
    const char* b = nullptr;
    const char* e = nullptr;
    int64_t lines = 0;          // lines in this chunk
    int64_t fail_line = -1;     // local index of the first failing line
    string fail_msg;
    Parsed out;
    std::vector<string_view> labels;  // local id -> label text
};

struct SvHash {
    size_t operator()(string_view s) const {
        uint64_t h = 1469598103934665603ull;
        for (char c : s) h = (h ^ (unsigned char)c) * 1099511628211ull;
        return (size_t)(h ^ (h >> 29));
    }
};

// Returns an empty string on success, else the error message.
string parse_transition(string_view line, int32_t n, int32_t& s_out, string_view& label_out, int32_t& t_out) {
    string_view body = strip(line);
    if (body.empty() || body.front() != '(' || body.back() != ')')
        return "expected '(<source>, <label>, <target>)'";
    body = body.size() >= 2 ? body.substr(1, body.size() - 2) : string_view();
    const size_t first = body.find(',');
    const size_t last = body.rfind(',');
    if (first == string_view::npos || first == last) return "expected two commas separating source, label, target";
    const string_view src_text = strip(body.substr(0, first));
    string_view label = strip(body.substr(first + 1, last - first - 1));
    const string_view dst_text = strip(body.substr(last + 1));
    // fast path: plain ASCII digits
    auto fast = [](string_view t, int64_t& v) {
        if (t.empty() || t.size() > 10) return false;
        int64_t x = 0;
        for (char c : t) {
            if (c < '0' || c > '9') return false;
            x = x * 10 + (c - '0');
        }
        v = x;
        return true;
    };
    int64_t sv = 0, tv = 0;
    string s_norm, t_norm;
    bool s_fits = true, t_fits = true;
    if (!(fast(src_text, sv) && fast(dst_text, tv))) {
        const PyInt a = py_int(src_text), b = py_int(dst_text);
        if (!a.ok || !b.ok)
            return "source and target must be integers, got " + py_repr(src_text) + " and " + py_repr(dst_text);
        sv = a.value;
        tv = b.value;
        s_fits = a.fits;
        t_fits = b.fits;
        s_norm = a.text;
        t_norm = b.text;
    }
    if (!label.empty() && label.front() == '"') {
        if (label.size() < 2 || label.back() != '"') return "unterminated quoted label";
        label = label.substr(1, label.size() - 2);
    } else if (label.empty() || label.find_first_of("()\"") != string_view::npos) {
        return "malformed label " + py_repr(label);
    }
    if (!(s_fits && t_fits && sv >= 0 && sv < n && tv >= 0 && tv < n)) {
        if (s_norm.empty()) s_norm = std::to_string(sv);
        if (t_norm.empty()) t_norm = std::to_string(tv);
        return "state index out of range in (" + s_norm + ", " + string(label) + ", " + t_norm +
               "); states are 0.." + std::to_string((int64_t)n - 1);
    }
    s_out = (int32_t)sv;
    t_out = (int32_t)tv;
    label_out = label;
    return string();
}

void parse_chunk(Chunk& c, int32_t n, bool skip_first_line) {
    // one allocation per column (a transition line is at least 7 bytes)
    const size_t cap = (size_t)(c.e - c.b) / 7 + 16;
    c.out.src.alloc(cap);
    c.out.lab.alloc(cap);
    c.out.dst.alloc(cap);
    std::unordered_map<string_view, int32_t, SvHash> ids;
    string_view last_label;
    int32_t last_id = -1;
    const char* p = c.b;
    int64_t li = 0;
    while (p < c.e) {
        const char* q = p;
        int br = 0;
        while (q < c.e && !(br = line_break(q, c.e))) ++q;
        const string_view line(p, (size_t)(q - p));
        p = q + br;
        const int64_t here = li++;
        if (here == 0 && skip_first_line) continue;
        if (c.fail_line >= 0) continue;  // keep counting lines only
        if (strip(line).empty()) continue;
        int32_t s = 0, t = 0;
        string_view label;
        string err = parse_transition(line, n, s, label, t);
        if (!err.empty()) {
            c.fail_line = here;
            c.fail_msg = std::move(err);
            continue;
        }
        int32_t id;
        if (last_id >= 0 && label == last_label) {
            id = last_id;
        } else {
            auto it = ids.find(label);
            if (it == ids.end()) {
                id = (int32_t)c.labels.size();
                ids.emplace(label, id);
                c.labels.push_back(label);
            } else {
                id = it->second;
            }
            last_label = label;
            last_id = id;
        }
        c.out.src.push(s);
        c.out.lab.push(id);
        c.out.dst.push(t);
    }
    c.lines = li;
}

bisim_aut* parse(const char* text, int64_t len, int32_t threads, ParseFail& fail) {
    const char* end = text + len;
    if (len <= 0) {
        fail = {1, "empty input, expected a 'des' header"};
        return nullptr;
    }
    // header = first line
    const char* q = text;
    int br = 0;
    while (q < end && !(br = line_break(q, end))) ++q;
    string num[3];
    if (!match_header(string_view(text, (size_t)(q - text)), num)) {
        fail = {1, "malformed header, expected 'des (<initial>, <m>, <n>)'"};
        return nullptr;
    }
    const PyInt init = py_int(num[0]), mm = py_int(num[1]), nn = py_int(num[2]);
    if (nn.text == "0") {
        fail = {1, "declared state count must be at least 1"};
        return nullptr;
    }
    if (!nn.fits || nn.value >= (1 << 30)) {
        fail = {1, "declared state count " + nn.text + " exceeds this library's limit of 2^30 - 1"};
        return nullptr;
    }
    if (!init.fits || init.value >= nn.value) {
        fail = {1, "initial state " + init.text + " not below state count " + nn.text};
        return nullptr;
    }
    const int32_t n = (int32_t)nn.value;

    // chunks at '\n' boundaries (always a line start); chunk 0 holds the header
    int T = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
    T = (int)std::min<int64_t>(T, std::max<int64_t>(1, len / (1 << 20)));
    std::vector<Chunk> ch(T);
    const char* cur = text;
    for (int k = 0; k < T; ++k) {
        ch[k].b = cur;
        const char* stop = k + 1 == T ? end : text + (len * (k + 1)) / T;
        if (stop < cur) stop = cur;
        if (k + 1 < T) {
            const char* nl = (const char*)memchr(stop, '\n', (size_t)(end - stop));
            stop = nl ? nl + 1 : end;
        }
        ch[k].e = stop;
        cur = stop;
    }
    {
        std::vector<std::thread> pool;
        for (int k = 1; k < T; ++k) pool.emplace_back(parse_chunk, std::ref(ch[k]), n, false);
        parse_chunk(ch[0], n, true);
        for (auto& t : pool) t.join();
    }

    int64_t line0 = 0, count = 0;
    for (auto& c : ch) {
        if (c.fail_line >= 0) {
            fail = {line0 + c.fail_line + 1, c.fail_msg};
            return nullptr;
        }
        line0 += c.lines;
        count += (int64_t)c.out.src.n;
    }
    if (!mm.fits || count != mm.value) {
        fail = {0, "expected " + mm.text + " transitions, found " + std::to_string(count)};
        return nullptr;
    }
    // sorted label table (lts.py:69-70) and remap of local ids
    std::vector<string_view> all;
    for (auto& c : ch) all.insert(all.end(), c.labels.begin(), c.labels.end());
    std::sort(all.begin(), all.end());
    all.erase(std::unique(all.begin(), all.end()), all.end());
    auto* a = new bisim_aut;
    a->n = n;
    a->initial = (int32_t)init.value;
    a->m = count;
    a->labels.reserve(all.size());
    for (auto v : all) a->labels.emplace_back(v);
    for (auto& c : ch) {
        c.out.rank.resize(c.labels.size());
        for (size_t i = 0; i < c.labels.size(); ++i)
            c.out.rank[i] = (int32_t)(std::lower_bound(all.begin(), all.end(), c.labels[i]) - all.begin());
        a->parts.push_back(std::move(c.out));
    }
    return a;
}

int finish(bisim_aut* a, const ParseFail& f, bisim_aut** out, bisim_aut_info* info) {
    if (info) *info = bisim_aut_info{};
    if (!a) {
        bisim::set_last_error(f.msg);
        if (info) info->error_line = f.line;
        if (out) *out = nullptr;
        return BISIM_BAD_INPUT;
    }
    if (info) {
        info->n = a->n;
        info->initial_state = a->initial;
        info->m = a->m;
        info->num_actions = (int32_t)a->labels.size();
    }
    if (out) *out = a;
    else delete a;
    return BISIM_OK;
}

}  // namespace

extern "C" {

int bisim_aut_parse(const char* text, int64_t len, int32_t threads, bisim_aut** out, bisim_aut_info* info) {
    try {
        bisim::set_last_error("");
        ParseFail f;
        bisim_aut* a = parse(text, len, threads, f);
        return finish(a, f, out, info);
    } catch (const std::exception& e) {
        bisim::set_last_error(e.what());
        return BISIM_CUDA;
    }
}

int bisim_aut_read_file(const char* path, int32_t threads, bisim_aut** out, bisim_aut_info* info) {
    try {
        bisim::set_last_error("");
        const int fd = open(path, O_RDONLY);
        if (fd < 0) {
            bisim::set_last_error(string("cannot open ") + path);
            return BISIM_BAD_INPUT;
        }
        struct stat sb;
        fstat(fd, &sb);
        const int64_t len = sb.st_size;
        // read into a huge-page buffer with one pread per thread (a file
        // mapping would fault in 4 KB pages one by one)
        Column buf;
        if (len > 0) {
            buf.alloc((size_t)(len + 3) / 4);
            int T = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
            T = (int)std::min<int64_t>(T, std::max<int64_t>(1, len / (8 << 20)));
            std::vector<int> ok(T, 1);
            auto rd = [&](int k) {
                int64_t lo = len * k / T, hi = len * (k + 1) / T;
                char* d = (char*)buf.p;
                while (lo < hi) {
                    const ssize_t r = pread(fd, d + lo, (size_t)(hi - lo), lo);
                    if (r <= 0) {
                        ok[k] = 0;
                        return;
                    }
                    lo += r;
                }
            };
            std::vector<std::thread> pool;
            for (int k = 1; k < T; ++k) pool.emplace_back(rd, k);
            rd(0);
            for (auto& t : pool) t.join();
            for (int v : ok)
                if (!v) {
                    close(fd);
                    bisim::set_last_error(string("cannot read ") + path);
                    return BISIM_BAD_INPUT;
                }
        }
        close(fd);
        ParseFail f;
        bisim_aut* a = parse((const char*)buf.p, len, threads, f);
        return finish(a, f, out, info);
    } catch (const std::exception& e) {
        bisim::set_last_error(e.what());
        return BISIM_CUDA;
    }
}

int bisim_aut_columns(const bisim_aut* a, int32_t* src, int32_t* act, int32_t* dst) {
    if (!a) return BISIM_BAD_INPUT;
    // one thread per parsed chunk: copy sources and targets, remap labels
    std::vector<size_t> base(a->parts.size() + 1, 0);
    for (size_t k = 0; k < a->parts.size(); ++k) base[k + 1] = base[k] + a->parts[k].src.n;
    auto fill = [&](size_t k) {
        const Parsed& q = a->parts[k];
        const size_t o = base[k];
        std::memcpy(src + o, q.src.p, q.src.n * 4);
        std::memcpy(dst + o, q.dst.p, q.dst.n * 4);
        for (size_t i = 0; i < q.lab.n; ++i) act[o + i] = q.rank[q.lab.p[i]];
    };
    std::vector<std::thread> pool;
    for (size_t k = 1; k < a->parts.size(); ++k) pool.emplace_back(fill, k);
    if (!a->parts.empty()) fill(0);
    for (auto& t : pool) t.join();
    return BISIM_OK;
}

const char* bisim_aut_label(const bisim_aut* a, int32_t action, int64_t* len) {
    if (!a || action < 0 || action >= (int32_t)a->labels.size()) return nullptr;
    if (len) *len = (int64_t)a->labels[(size_t)action].size();
    return a->labels[(size_t)action].data();
}

void bisim_aut_free(bisim_aut* a) { delete a; }

}  // extern "C"
