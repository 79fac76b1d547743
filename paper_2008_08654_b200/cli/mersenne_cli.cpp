// mersenne_cli.cpp -- the reference CLI's `sketch` subcommand (streaming Count
// Sketch ingest) over the B200 host API.
//
//   mersenne_b200_cli sketch [--width W] [--rows R] [--prime 2^61-1] [--seed S]
//       [--key-bits B] [--splitter pow2|uniform|mersenne] [--input FILE]
//       [--queries k1,k2,...] [--save FILE] [--load FILE] [--f2-median]
//
// Behaviour follows /root/reference/proj/src/cli/commands.cpp:
//   option defaults and names          :21-33, :306-320
//   parse_prime_exponent               bench.cpp:81-94
//   "key delta" line grammar + errors  :118-155 (parse_stream)
//   query list grammar + errors        :157-179 (parse_queries)
//   do_sketch (load / construct, stream, queries, moment, JSON, save)  :181-232
//   "error: <what>" + exit 1           :335-340
// and is pinned by the reference's tests/unit/test_cli.cpp:200-310 cases
// (tests/test_cli.py).
//
// What differs is HOW the stream is consumed.  The reference reads the whole
// stream into a vector and then calls CountSketch::process once per item.
// Here the stream is read in 32 MiB blocks, each block is parsed by all host
// threads at once (pieces cut at newlines, line numbers recovered by prefix
// sums so an error names the same line the reference would), and each parsed
// block goes to the GPU as ONE CountSketch::process_batch on a worker thread
// while the next block is being parsed.  A malformed line anywhere still
// yields no output and no saved state (the reference throws before processing;
// here earlier blocks reached the device table, but the table is discarded
// with the process), so the observable behaviour is the reference's.
#include <omp.h>

#include <algorithm>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <iterator>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "../../include/mersenne_b200/mersenne_b200.hpp"

using namespace mersenne::b200;

namespace {

struct SketchOpts {  // commands.cpp:21-33
    u64 width = 1024;
    unsigned rows = 1;
    std::string prime = "2^61-1";
    u64 seed = 1;
    unsigned key_bits = 32;
    std::string splitter = "pow2";
    std::string input, queries, save, load;
    bool f2_median = false;
};

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

std::string to_decimal(u128 v) {
    if (v == 0) return "0";
    char buf[48];
    int i = 47;
    buf[i] = 0;
    while (v) {
        buf[--i] = char('0' + int(v % 10));
        v /= 10;
    }
    return std::string(buf + i);
}

// bench.cpp:81-94
unsigned parse_prime_exponent(const std::string& text) {
    const auto fail = [&] { throw std::invalid_argument("prime must be written like 2^61-1, got '" + text + "'"); };
    if (text.size() < 6 || text.compare(0, 2, "2^") != 0 || text.compare(text.size() - 2, 2, "-1") != 0) fail();
    const char* first = text.data() + 2;
    const char* last = text.data() + text.size() - 2;
    unsigned e = 0;
    const auto [end, ec] = std::from_chars(first, last, e);
    if (ec != std::errc{} || end != last || e < 2 || e > 127) fail();
    return e;
}

Splitter parse_splitter(const std::string& name) {  // commands.cpp:97-103
    if (name == "pow2") return Splitter::Pow2;
    if (name == "uniform") return Splitter::UniformArb;
    if (name == "mersenne") return Splitter::MersenneArb;
    throw std::invalid_argument("splitter must be pow2, uniform, or mersenne");
}

bool parse_u64_full(std::string_view t, u64& v) {  // commands.cpp:109-115
    const auto [end, ec] = std::from_chars(t.data(), t.data() + t.size(), v);
    return ec == std::errc{} && end == t.data() + t.size();
}

// ---------------------------------------------------------------------------
// "key delta" lines.  Token separation is operator>>'s: the C locale's isspace
// set.  A line is what std::getline yields: text up to '\n' (the last line may
// lack one).
inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r'; }

struct LineError {
    u64 line = 0;  // 1-based within the piece's block, 0 = none
    std::string msg;
};

// one line [p, e) (no '\n'); returns false with msg on a malformed line
// commands.cpp:124-152, in the same order of checks
enum class LineKind { Blank, Item, Error };
LineKind parse_line(const char* p, const char* e, u128 domain, u64& key, i64& delta, std::string& msg) {
    auto next_token = [&](std::string_view& tok) {
        while (p < e && is_ws(*p)) ++p;
        if (p == e) return false;
        const char* s = p;
        while (p < e && !is_ws(*p)) ++p;
        tok = std::string_view(s, size_t(p - s));
        return true;
    };
    std::string_view kt, dt, extra;
    if (!next_token(kt)) return LineKind::Blank;
    if (!next_token(dt)) {
        msg = "expected 'key delta'";
        return LineKind::Error;
    }
    if (next_token(extra)) {
        msg = "unexpected trailing token '" + std::string(extra) + "'";
        return LineKind::Error;
    }
    if (!parse_u64_full(kt, key)) {
        msg = "malformed key '" + std::string(kt) + "'";
        return LineKind::Error;
    }
    std::string_view dv = dt;
    if (!dv.empty() && dv.front() == '+') dv.remove_prefix(1);
    const auto [end, ec] = std::from_chars(dv.data(), dv.data() + dv.size(), delta);
    if (ec != std::errc{} || end != dv.data() + dv.size() || dv.empty()) {
        msg = "malformed delta '" + std::string(dt) + "'";
        return LineKind::Error;
    }
    if (u128(key) >= domain) {
        msg = "key " + std::string(kt) + " is outside the configured key domain";
        return LineKind::Error;
    }
    return LineKind::Item;
}

// Parsed items of one block, in stream order.
struct Batch {
    std::vector<u64> keys;
    std::vector<i64> deltas;
    u64 n = 0;
};

// Per-thread parse buffers, kept across blocks (no allocation or first-touch
// page faults per block).
struct ParseScratch {
    std::vector<std::vector<u64>> keys;
    std::vector<std::vector<i64>> deltas;
};

// Parse the complete lines of [buf, buf + len) (ends on '\n', or at EOF on the
// last line) with every host thread.  first_line = number of lines before the
// block.  Throws the reference's stream_error for the first bad line; returns
// the number of lines parsed.
u64 parse_block(const char* buf, size_t len, u64 first_line, u128 domain, Batch& out, ParseScratch& ps) {
    const int T = std::max(1, std::min<int>(omp_get_max_threads(), int(len / (1 << 16)) + 1));
    std::vector<size_t> cut(T + 1, len);
    cut[0] = 0;
    for (int t = 1; t < T; ++t) {  // piece t starts after the first '\n' at or after len * t / T
        size_t c = std::max(cut[t - 1], len * size_t(t) / size_t(T));
        const void* nl = c < len ? std::memchr(buf + c, '\n', len - c) : nullptr;
        cut[t] = nl ? size_t(static_cast<const char*>(nl) - buf) + 1 : len;
    }
    std::vector<u64> lines(T, 0), items(T, 0);
    std::vector<LineError> errs(T);
    if (ps.keys.size() < (size_t)T) {
        ps.keys.resize(T);
        ps.deltas.resize(T);
    }
    auto& tk = ps.keys;
    auto& td = ps.deltas;
#pragma omp parallel for num_threads(T) schedule(static, 1)
    for (int t = 0; t < T; ++t) {
        const char* p = buf + cut[t];
        const char* end = buf + cut[t + 1];
        auto& K = tk[t];
        auto& D = td[t];
        const size_t cap = size_t(end - p) / 4 + 1;  // a line holds at least "k d\n" + 1
        if (K.size() < cap) {
            K.resize(cap);
            D.resize(cap);
        }
        size_t ni = 0;
        u64 ln = 0;
        std::string msg;
        while (p < end) {
            const void* nl = std::memchr(p, '\n', size_t(end - p));
            const char* le = nl ? static_cast<const char*>(nl) : end;
            ++ln;
            u64 key = 0;
            i64 delta = 0;
            const LineKind kind = parse_line(p, le, domain, key, delta, msg);
            if (kind == LineKind::Error) {
                errs[t] = {ln, msg};
                break;
            }
            if (kind == LineKind::Item) {
                K[ni] = key;
                D[ni] = delta;
                ++ni;
            }
            p = nl ? le + 1 : end;
        }
        if (!errs[t].line) lines[t] = ln;
        items[t] = ni;
    }
    u64 before = first_line;
    for (int t = 0; t < T; ++t) {
        if (errs[t].line) throw std::runtime_error("line " + std::to_string(before + errs[t].line) + ": " + errs[t].msg);
        before += lines[t];
    }
    u64 total = 0;
    std::vector<u64> off(T);
    for (int t = 0; t < T; ++t) {
        off[t] = total;
        total += items[t];
    }
    if (out.keys.size() < total) {
        out.keys.resize(total);
        out.deltas.resize(total);
    }
#pragma omp parallel for num_threads(T) schedule(static, 1)
    for (int t = 0; t < T; ++t) {
        if (!items[t]) continue;
        std::memcpy(out.keys.data() + off[t], tk[t].data(), items[t] * sizeof(u64));
        std::memcpy(out.deltas.data() + off[t], td[t].data(), items[t] * sizeof(i64));
    }
    out.n = total;
    return before - first_line;
}

// Streams "key delta" lines from `in` into `sink(batch)` (run on a worker
// thread, one batch in flight while the next block is parsed); returns the
// item count (commands.cpp:118-155 + the process loop at :206).
template <typename Sink>
u64 ingest(FILE* in, u128 domain, Sink sink) {
    constexpr size_t kBlock = size_t(32) << 20;
    std::vector<char> buf(kBlock + 1);
    size_t have = 0;  // bytes in buf (an incomplete last line carried over)
    u64 line_base = 0, processed = 0;
    Batch batches[2];
    ParseScratch ps;
    int cur = 0;
    std::thread worker;
    std::exception_ptr worker_err;
    auto join = [&] {
        if (worker.joinable()) worker.join();
        if (worker_err) std::rethrow_exception(worker_err);
    };
    try {
        bool eof = false;
        while (!eof) {
            const size_t room = buf.size() - 1 - have;
            const size_t got = std::fread(buf.data() + have, 1, room, in);
            if (got < room) {
                if (std::ferror(in)) throw std::runtime_error("error reading the input stream");
                eof = true;
            }
            have += got;
            size_t len = have;  // complete lines in this block
            if (!eof) {
                const char* b = buf.data();
                size_t k = have;
                while (k > 0 && b[k - 1] != '\n') --k;
                if (k == 0) {  // one line longer than the block: grow and read on
                    buf.resize(buf.size() * 2);
                    continue;
                }
                len = k;
            }
            if (len == 0) break;
            Batch& bt = batches[cur];
            line_base += parse_block(buf.data(), len, line_base, domain, bt, ps);
            std::memmove(buf.data(), buf.data() + len, have - len);
            have -= len;
            join();  // the previous batch is on the device; its buffer is free again
            if (bt.n) {
                processed += bt.n;
                worker = std::thread([&sink, &bt, &worker_err] {
                    try {
                        sink(bt);
                    } catch (...) {
                        worker_err = std::current_exception();
                    }
                });
                cur ^= 1;
            }
        }
        join();
    } catch (...) {
        if (worker.joinable()) worker.join();
        throw;
    }
    return processed;
}

std::vector<u64> parse_queries(const std::string& text, u128 domain) {  // commands.cpp:157-179
    std::vector<u64> keys;
    if (text.empty()) return keys;
    size_t pos = 0;
    while (true) {
        const size_t comma = text.find(',', pos);
        const std::string tok = text.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos);
        u64 key = 0;
        if (!parse_u64_full(tok, key)) throw std::invalid_argument("malformed query key '" + tok + "'");
        if (u128(key) >= domain) throw std::invalid_argument("query key " + tok + " is outside the configured key domain");
        keys.push_back(key);
        if (comma == std::string::npos) break;
        pos = comma + 1;
    }
    return keys;
}

// nlohmann::json's dump(2) escaping of a string value
std::string json_string(const std::string& s) {
    std::string o = "\"";
    for (unsigned char c : s) {
        switch (c) {
            case '"': o += "\\\""; break;
            case '\\': o += "\\\\"; break;
            case '\b': o += "\\b"; break;
            case '\f': o += "\\f"; break;
            case '\n': o += "\\n"; break;
            case '\r': o += "\\r"; break;
            case '\t': o += "\\t"; break;
            default:
                if (c < 0x20) {
                    char u[8];
                    std::snprintf(u, sizeof u, "\\u%04x", c);
                    o += u;
                } else {
                    o += char(c);
                }
        }
    }
    return o + "\"";
}

int do_sketch(const SketchOpts& o, std::ostream& out) {  // commands.cpp:181-232
    std::optional<CountSketch> sketch;
    if (!o.load.empty()) {
        std::ifstream state(o.load, std::ios::binary);
        if (!state) throw std::runtime_error("cannot open sketch state file '" + o.load + "'");
        const std::vector<uint8_t> bytes((std::istreambuf_iterator<char>(state)), std::istreambuf_iterator<char>());
        sketch.emplace(CountSketch::deserialize(bytes));
    } else {
        const unsigned b = parse_prime_exponent(o.prime);
        const MersenneModulus modulus(b, /*require_prime=*/true);
        if (o.key_bits == 0 || o.key_bits > 64) throw std::invalid_argument("key width must be between 1 and 64 bits");
        sketch.emplace(o.rows, o.width, modulus, u128(1) << o.key_bits, parse_splitter(o.splitter), o.seed);
    }
    FILE* src = stdin;
    if (!o.input.empty()) {
        src = std::fopen(o.input.c_str(), "rb");
        if (!src) throw std::runtime_error("cannot open input file '" + o.input + "'");
    }
    u64 processed = 0;
    try {
        CountSketch& sk = *sketch;
        processed = ingest(src, sk.key_domain(), [&sk](const Batch& b) {
            sk.process_batch(b.keys.data(), 64, b.deltas.data(), MB200_W_I64, b.n);
        });
    } catch (...) {
        if (src != stdin) std::fclose(src);
        throw;
    }
    if (src != stdin) std::fclose(src);

    const std::vector<u64> queries = parse_queries(o.queries, sketch->key_domain());
    const CountSketch::Moment m = sketch->second_moment(o.f2_median);
    const std::vector<i64> est =
        queries.empty() ? std::vector<i64>{} : sketch->point_query_batch(queries.data(), 64, queries.size());

    // nlohmann::json object keys are ordered (std::map): b, f2, f2_saturated,
    // processed, queries, rows, saved, width
    std::string j = "{\n";
    j += "  \"b\": " + std::to_string(sketch->modulus().b()) + ",\n";
    j += "  \"f2\": \"" + to_decimal(m.value) + "\",\n";
    j += std::string("  \"f2_saturated\": ") + (m.saturated ? "true" : "false") + ",\n";
    j += "  \"processed\": " + std::to_string(processed) + ",\n";
    if (queries.empty()) {
        j += "  \"queries\": [],\n";
    } else {
        j += "  \"queries\": [\n";
        for (size_t i = 0; i < queries.size(); ++i) {
            j += "    {\n      \"estimate\": " + std::to_string(est[i]) + ",\n      \"key\": \"" +
                 to_decimal(queries[i]) + "\"\n    }";
            j += i + 1 < queries.size() ? ",\n" : "\n";
        }
        j += "  ],\n";
    }
    j += "  \"rows\": " + std::to_string(sketch->rows()) + ",\n";
    if (!o.save.empty()) {
        const std::vector<uint8_t> bytes = sketch->serialize();
        std::ofstream state(o.save, std::ios::binary);
        state.write(reinterpret_cast<const char*>(bytes.data()), std::streamsize(bytes.size()));
        if (!state) throw std::runtime_error("cannot write sketch state file '" + o.save + "'");
        j += "  \"saved\": " + json_string(o.save) + ",\n";
    }
    j += "  \"width\": " + std::to_string(sketch->width()) + "\n}";
    out << j << "\n";
    return 0;
}

const char* kUsage =
    "Count sketch over a key/delta stream (B200)\n"
    "Usage: mersenne_b200_cli sketch [OPTIONS]\n"
    "  --width UINT      Buckets per row (1024)\n"
    "  --rows UINT       Independent rows (1)\n"
    "  --prime TEXT      Row hash modulus, written like 2^61-1\n"
    "  --seed UINT       Master seed for the row families (1)\n"
    "  --key-bits UINT   Key domain is [0, 2^key-bits) (32)\n"
    "  --splitter TEXT   pow2 | uniform | mersenne\n"
    "  --input TEXT      Read the stream from a file, not stdin\n"
    "  --queries TEXT    Comma-separated keys to point-query\n"
    "  --save TEXT       Write the sketch state to a file\n"
    "  --load TEXT       Resume from a saved state (ignores the config flags)\n"
    "  --f2-median       Median of per-row moments instead of row 0\n";

template <typename T>
T parse_num(const std::string& opt, const std::string& v) {
    T x{};
    const auto [end, ec] = std::from_chars(v.data(), v.data() + v.size(), x);
    if (ec != std::errc{} || end != v.data() + v.size() || v.empty())
        throw UsageError("Could not convert: " + opt + " = " + v);
    return x;
}

SketchOpts parse_args(const std::vector<std::string>& a, size_t i) {
    SketchOpts o;
    for (; i < a.size(); ++i) {
        std::string opt = a[i], val;
        bool has_val = false;
        if (const size_t eq = opt.find('='); opt.rfind("--", 0) == 0 && eq != std::string::npos) {
            val = opt.substr(eq + 1);
            opt = opt.substr(0, eq);
            has_val = true;
        }
        if (opt == "--f2-median") {
            if (has_val) throw UsageError("--f2-median takes no value");
            o.f2_median = true;
            continue;
        }
        if (opt == "--help" || opt == "-h") throw UsageError("");
        static const char* kOpts[] = {"--width", "--rows", "--prime", "--seed", "--key-bits", "--splitter",
                                      "--input", "--queries", "--save", "--load"};
        if (std::find_if(std::begin(kOpts), std::end(kOpts), [&](const char* k) { return opt == k; }) ==
            std::end(kOpts))
            throw UsageError("The following argument was not expected: " + a[i]);
        if (!has_val) {
            if (i + 1 >= a.size()) throw UsageError(opt + ": 1 required TEXT:SIZE missing");
            val = a[++i];
        }
        if (opt == "--width") o.width = parse_num<u64>(opt, val);
        else if (opt == "--rows") o.rows = parse_num<unsigned>(opt, val);
        else if (opt == "--prime") o.prime = val;
        else if (opt == "--seed") o.seed = parse_num<u64>(opt, val);
        else if (opt == "--key-bits") o.key_bits = parse_num<unsigned>(opt, val);
        else if (opt == "--splitter") {
            if (val != "pow2" && val != "uniform" && val != "mersenne")
                throw UsageError("--splitter: " + val + " not in {pow2,uniform,mersenne}");
            o.splitter = val;
        } else if (opt == "--input") o.input = val;
        else if (opt == "--queries") o.queries = val;
        else if (opt == "--save") o.save = val;
        else if (opt == "--load") o.load = val;
    }
    return o;
}

// `parse`: the stream grammar alone, no device (CPU tests of the line rules):
// prints the item count and wrapping sums of keys, deltas and key * delta.
int do_parse(const std::vector<std::string>& a) {
    unsigned key_bits = 32;
    std::string input;
    for (size_t i = 2; i < a.size(); ++i) {
        if (a[i] == "--key-bits" && i + 1 < a.size()) key_bits = parse_num<unsigned>(a[i], a[i + 1]), ++i;
        else if (a[i] == "--input" && i + 1 < a.size()) input = a[++i];
        else throw UsageError("The following argument was not expected: " + a[i]);
    }
    if (key_bits == 0 || key_bits > 64) throw std::invalid_argument("key width must be between 1 and 64 bits");
    FILE* src = input.empty() ? stdin : std::fopen(input.c_str(), "rb");
    if (!src) throw std::runtime_error("cannot open input file '" + input + "'");
    u64 sk = 0, sd = 0, skd = 0;
    const u64 n = ingest(src, u128(1) << key_bits, [&](const Batch& b) {
        for (u64 i = 0; i < b.n; ++i) {
            sk += b.keys[i];
            sd += u64(b.deltas[i]);
            skd += b.keys[i] * u64(b.deltas[i]);
        }
    });
    if (src != stdin) std::fclose(src);
    std::cout << "{\"processed\": " << n << ", \"sum_keys\": " << sk << ", \"sum_deltas\": " << sd
              << ", \"sum_key_delta\": " << skd << "}\n";
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    std::ios::sync_with_stdio(false);
    const std::vector<std::string> args(argv, argv + argc);
    if (args.size() >= 2 && args[1] == "parse") {
        try {
            return do_parse(args);
        } catch (const std::exception& e) {
            std::cerr << "error: " << e.what() << "\n";
            return 1;
        }
    }
    if (args.size() < 2 || args[1] != "sketch") {
        std::cerr << kUsage << (args.size() < 2 ? "A subcommand is required\n" : "Only `sketch` is provided\n");
        return args.size() >= 2 && (args[1] == "--help" || args[1] == "-h") ? 0 : 106;
    }
    try {
        const SketchOpts o = parse_args(args, 2);
        return do_sketch(o, std::cout);
    } catch (const UsageError& e) {
        if (!*e.what()) {
            std::cout << kUsage;
            return 0;
        }
        std::cerr << e.what() << "\n" << kUsage;
        return 109;
    } catch (const std::exception& e) {  // commands.cpp:337-340
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
