// graph_io.cpp — the reference's dataset files (proj/src/graph_io.cpp:41-296), host side.
//
// Same formats, same acceptance rules and the same exception texts (runtime_error with
// "<path>:<line>: <what>" for parse failures), so a dataset the reference's CLI reads
// (proj/tools/main.cpp:137 load_dataset) loads here unchanged and a bad one fails the
// same way. The parsers work on the whole file in memory with pointer scans instead of
// per-line string streams (products-scale edge lists are ~1 GB of text); the integer and
// float scanners follow the rules of `istream >> long long` and `std::stod` that the
// reference relies on. The canonicalisation (self-loops, duplicates, sort, CSR) happens in
// build_graph on the device (graph.cu).
#include "graph_io.hpp"

#include <algorithm>
#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <sstream>
#include <stdexcept>

namespace sc {
namespace {

[[noreturn]] void fail_at(const std::string& path, size_t line_no, const std::string& what) {
    throw std::runtime_error(path + ":" + std::to_string(line_no) + ": " + what);
}

bool read_all(const std::string& path, std::string& buf) {
    std::ifstream in(path, std::ios::binary);
    if (!in) return false;
    in.seekg(0, std::ios::end);
    const std::streamoff size = in.tellg();
    in.seekg(0, std::ios::beg);
    buf.resize(size > 0 ? static_cast<size_t>(size) : 0);
    if (size > 0) in.read(&buf[0], size);
    return true;
}

// Visit the lines of buf (without the '\n'), numbering from 1.
template <class F>
void for_each_line(const std::string& buf, F&& f) {
    size_t pos = 0, line_no = 0;
    while (pos < buf.size()) {
        size_t end = buf.find('\n', pos);
        if (end == std::string::npos) end = buf.size();
        ++line_no;
        f(line_no, buf.data() + pos, buf.data() + end);
        pos = end + 1;
    }
}

bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r'; }
const char* skip_ws(const char* p, const char* e) {
    while (p < e && is_ws(*p)) ++p;
    return p;
}

// `istream >> long long`: optional whitespace, optional sign, decimal digits; stops at the
// first non-digit. Fails (false) without a digit or on overflow.
bool scan_ll(const char*& p, const char* e, long long& out) {
    const char* q = skip_ws(p, e);
    const char* start = q;
    if (q < e && (*q == '+' || *q == '-')) ++q;
    const char* digits = q;
    while (q < e && *q >= '0' && *q <= '9') ++q;
    if (q == digits) return false;
    const std::string tok(start, q);
    errno = 0;
    char* endp = nullptr;
    const long long v = std::strtoll(tok.c_str(), &endp, 10);
    if (errno == ERANGE) return false;
    out = v;
    p = q;
    return true;
}

// std::stod of a whole token, as the reference's CSV reader applies it: leading whitespace,
// any strtod syntax, then only whitespace may follow.
bool parse_double_token(const std::string& tok, double& out) {
    const char* s = tok.c_str();
    errno = 0;
    char* endp = nullptr;
    const double v = std::strtod(s, &endp);
    if (endp == s || errno == ERANGE) return false;  // stod throws invalid_argument / out_of_range
    for (const char* q = endp; *q; ++q)
        if (!std::isspace(static_cast<unsigned char>(*q))) return false;
    out = v;
    return true;
}

void write_u64_le(std::ostream& out, uint64_t v) {
    unsigned char b[8];
    for (int i = 0; i < 8; ++i) b[i] = static_cast<unsigned char>(v >> (8 * i));
    out.write(reinterpret_cast<const char*>(b), 8);
}

}  // namespace

// graph_io.cpp:41-80 (the edge list part; build_graph runs on the device afterwards)
EdgeList read_edge_list(const std::string& path, int32_t num_nodes) {
    std::string buf;
    if (!read_all(path, buf)) throw std::runtime_error("cannot open edge list: " + path);
    EdgeList el;
    int32_t max_id = -1;
    for_each_line(buf, [&](size_t line_no, const char* b, const char* e) {
        const char* p = skip_ws(b, e);
        if (p == e || *p == '#') return;  // blank or comment (first non-blank is '#')
        long long u = 0, v = 0;
        if (!scan_ll(p, e, u) || !scan_ll(p, e, v)) fail_at(path, line_no, "expected two integer tokens");
        const char* t = skip_ws(p, e);
        if (t < e) {
            const char* te = t;
            while (te < e && !is_ws(*te)) ++te;
            fail_at(path, line_no, "unexpected trailing token '" + std::string(t, te) + "'");
        }
        if (u < 0 || v < 0) fail_at(path, line_no, "negative node id");
        max_id = std::max({max_id, static_cast<int32_t>(u), static_cast<int32_t>(v)});
        el.uv.push_back(static_cast<int32_t>(u));
        el.uv.push_back(static_cast<int32_t>(v));
    });
    el.num_nodes = num_nodes >= 0 ? num_nodes : max_id + 1;
    if (max_id >= el.num_nodes)
        throw std::runtime_error(path + ": node id " + std::to_string(max_id) + " exceeds declared node count " +
                                 std::to_string(el.num_nodes));
    return el;
}

// graph_io.cpp:82-160: "CFM1" binary (sniffed from the first four bytes) or CSV.
HostFeatures read_features(const std::string& path, int32_t expected_nodes) {
    std::string buf;
    if (!read_all(path, buf)) throw std::runtime_error("cannot open features: " + path);
    HostFeatures f;
    if (buf.size() >= 4 && std::memcmp(buf.data(), "CFM1", 4) == 0) {
        auto u64_at = [&](size_t off) {
            if (buf.size() < off + 8) throw std::runtime_error("truncated binary matrix header");
            uint64_t v = 0;
            for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(static_cast<unsigned char>(buf[off + i])) << (8 * i);
            return v;
        };
        const uint64_t rows = u64_at(4), cols = u64_at(12);
        if (rows != static_cast<uint64_t>(expected_nodes))
            throw std::runtime_error(path + ": feature rows " + std::to_string(rows) + " != expected node count " +
                                     std::to_string(expected_nodes));
        f.rows = static_cast<int64_t>(rows);
        f.cols = static_cast<int64_t>(cols);
        f.values.resize(static_cast<size_t>(rows * cols));
        const size_t row_bytes = static_cast<size_t>(cols) * sizeof(float);
        for (uint64_t r = 0; r < rows; ++r) {
            const size_t off = 20 + static_cast<size_t>(r) * row_bytes;
            if (buf.size() < off + row_bytes) throw std::runtime_error(path + ": truncated feature data");
            float* dst = f.values.data() + r * cols;
            std::memcpy(dst, buf.data() + off, row_bytes);
            for (uint64_t c = 0; c < cols; ++c)
                if (!std::isfinite(dst[c]))
                    throw std::runtime_error(path + ": non-finite value at row " + std::to_string(r) + ", col " +
                                             std::to_string(c));
        }
        return f;
    }
    int64_t rows = 0;
    for_each_line(buf, [&](size_t line_no, const char* b, const char* e) {
        if (b == e || *b == '#') return;  // empty or '#'-first lines
        int64_t ncol = 0;
        const char* p = b;
        while (true) {
            const char* comma = static_cast<const char*>(std::memchr(p, ',', static_cast<size_t>(e - p)));
            const char* te = comma ? comma : e;
            const std::string tok(p, te);
            double v = 0.0;
            if (!parse_double_token(tok, v)) fail_at(path, line_no, "bad numeric token '" + tok + "'");
            if (!std::isfinite(v))
                throw std::runtime_error(path + ": non-finite value at row " + std::to_string(rows) + ", col " +
                                         std::to_string(ncol));
            f.values.push_back(static_cast<float>(v));
            ++ncol;
            if (!comma) break;
            p = comma + 1;
        }
        if (rows > 0 && ncol != f.cols)
            fail_at(path, line_no,
                    "ragged row: " + std::to_string(ncol) + " columns, expected " + std::to_string(f.cols));
        if (rows == 0) f.cols = ncol;
        ++rows;
    });
    if (rows != expected_nodes)
        throw std::runtime_error(path + ": feature rows " + std::to_string(rows) + " != expected node count " +
                                 std::to_string(expected_nodes));
    f.rows = rows;
    return f;
}

// graph_io.cpp:188-242: one line per node, a class id or a comma-separated 0/1 row.
HostLabels read_labels(const std::string& path, int32_t num_nodes) {
    std::string buf;
    if (!read_all(path, buf)) throw std::runtime_error("cannot open labels: " + path);
    std::vector<std::pair<const char*, const char*>> lines;
    for_each_line(buf, [&](size_t, const char* b, const char* e) {
        if (b == e || *b == '#') return;
        lines.emplace_back(b, e);
    });
    if (lines.size() != static_cast<size_t>(num_nodes))
        throw std::runtime_error(path + ": " + std::to_string(lines.size()) + " label lines for " +
                                 std::to_string(num_nodes) + " nodes");
    HostLabels L;
    L.multilabel = !lines.empty() && std::memchr(lines[0].first, ',', lines[0].second - lines[0].first) != nullptr;
    if (L.multilabel) {
        size_t width = 0;
        for (size_t r = 0; r < lines.size(); ++r) {
            const char* p = lines[r].first;
            const char* e = lines[r].second;
            size_t n = 0;
            while (p < e) {  // getline(',') pieces: a trailing ',' yields no empty last token
                const char* comma = static_cast<const char*>(std::memchr(p, ',', static_cast<size_t>(e - p)));
                const char* te = comma ? comma : e;
                const std::string tok(p, te);
                if (tok != "0" && tok != "1")
                    throw std::runtime_error(path + ": multi-label entries must be 0 or 1, got '" + tok + "'");
                L.targets.push_back(tok == "1" ? 1.f : 0.f);
                ++n;
                p = comma ? comma + 1 : e;
            }
            if (r == 0) width = n;
            else if (n != width) throw std::runtime_error(path + ": ragged multi-label row " + std::to_string(r));
        }
        L.num_classes = static_cast<int32_t>(width);
    } else {
        int32_t max_label = 0;
        L.labels.resize(lines.size());
        for (size_t r = 0; r < lines.size(); ++r) {
            const char* p = lines[r].first;
            long long v = 0;
            if (!scan_ll(p, lines[r].second, v) || v < 0)
                throw std::runtime_error(path + ": bad class id on line " + std::to_string(r + 1));
            L.labels[r] = static_cast<int32_t>(v);
            max_label = std::max(max_label, L.labels[r]);
        }
        L.num_classes = max_label + 1;
    }
    return L;
}

// graph_io.cpp:256-283: "train|val|test <id>" lines, disjoint splits.
void read_masks(const std::string& path, int32_t num_nodes, std::vector<uint8_t>& train, std::vector<uint8_t>& val,
                std::vector<uint8_t>& test) {
    std::string buf;
    if (!read_all(path, buf)) throw std::runtime_error("cannot open masks: " + path);
    train.assign(static_cast<size_t>(num_nodes), 0);
    val.assign(static_cast<size_t>(num_nodes), 0);
    test.assign(static_cast<size_t>(num_nodes), 0);
    for_each_line(buf, [&](size_t line_no, const char* b, const char* e) {
        if (b == e || *b == '#') return;
        const char* p = skip_ws(b, e);
        const char* te = p;
        while (te < e && !is_ws(*te)) ++te;
        const std::string tag(p, te);
        p = te;
        long long id = 0;
        if (tag.empty() || !scan_ll(p, e, id)) fail_at(path, line_no, "expected '<split> <node_id>'");
        if (id < 0 || id >= num_nodes) fail_at(path, line_no, "node id out of range");
        const auto i = static_cast<size_t>(id);
        if (train[i] || val[i] || test[i])
            fail_at(path, line_no, "node " + std::to_string(id) + " assigned to two splits");
        if (tag == "train") train[i] = 1;
        else if (tag == "val") val[i] = 1;
        else if (tag == "test") test[i] = 1;
        else fail_at(path, line_no, "unknown split tag '" + tag + "'");
    });
}

// ---- writers (graph_io.cpp:75-80, 162-186, 244-254, 285-296), byte-compatible ----
namespace {
std::ofstream open_out(const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot open for writing: " + path);
    return out;
}
}  // namespace

void write_edge_list(const std::string& path, const int32_t* u, const int32_t* v, int64_t m) {
    auto out = open_out(path);
    std::string s;
    s.reserve(static_cast<size_t>(m) * 16);
    char a[16], b[16];
    for (int64_t e = 0; e < m; ++e) {
        const auto ra = std::to_chars(a, a + sizeof(a), u[e]);
        const auto rb = std::to_chars(b, b + sizeof(b), v[e]);
        s.append(a, ra.ptr);
        s.push_back(' ');
        s.append(b, rb.ptr);
        s.push_back('\n');
    }
    out.write(s.data(), static_cast<std::streamsize>(s.size()));
    if (!out) throw std::runtime_error("write failed: " + path);
}

void write_features_csv(const std::string& path, const float* x, int64_t rows, int64_t cols) {
    auto out = open_out(path);
    std::string s;
    char tmp[64];
    for (int64_t r = 0; r < rows; ++r) {
        for (int64_t c = 0; c < cols; ++c) {
            if (c) s.push_back(',');
            const auto res = std::to_chars(tmp, tmp + sizeof(tmp), static_cast<double>(x[r * cols + c]));
            s.append(tmp, res.ptr);  // shortest round-trip form of the double, as fmt_double
        }
        s.push_back('\n');
    }
    out.write(s.data(), static_cast<std::streamsize>(s.size()));
}

void write_features_binary(const std::string& path, const float* x, int64_t rows, int64_t cols) {
    auto out = open_out(path);
    out.write("CFM1", 4);
    write_u64_le(out, static_cast<uint64_t>(rows));
    write_u64_le(out, static_cast<uint64_t>(cols));
    static_assert(sizeof(float) == 4, "float32 payload");
    out.write(reinterpret_cast<const char*>(x), static_cast<std::streamsize>(rows * cols * sizeof(float)));
    if (!out) throw std::runtime_error("write failed: " + path);
}

void write_labels(const std::string& path, int32_t n, const int32_t* labels, const float* targets, int32_t classes) {
    auto out = open_out(path);
    std::string s;
    if (targets) {
        for (int64_t r = 0; r < n; ++r) {
            for (int32_t c = 0; c < classes; ++c) {
                if (c) s.push_back(',');
                s.push_back(targets[r * classes + c] != 0.f ? '1' : '0');
            }
            s.push_back('\n');
        }
    } else {
        for (int64_t r = 0; r < n; ++r) {
            s += std::to_string(labels[r]);
            s.push_back('\n');
        }
    }
    out.write(s.data(), static_cast<std::streamsize>(s.size()));
}

void write_masks(const std::string& path, int32_t n, const uint8_t* train, const uint8_t* val, const uint8_t* test) {
    auto out = open_out(path);
    std::string s;
    const uint8_t* m[3] = {train, val, test};
    const char* tag[3] = {"train", "val", "test"};
    for (int k = 0; k < 3; ++k)
        for (int64_t v = 0; v < n; ++v)
            if (m[k][v]) {
                s += tag[k];
                s.push_back(' ');
                s += std::to_string(v);
                s.push_back('\n');
            }
    out.write(s.data(), static_cast<std::streamsize>(s.size()));
}

}  // namespace sc
