// ychg_cli.cpp -- `ychg_b200`, the command-line front end of the GPU path
// (SURVEY §8f row 4): the reference CLI's `synth`, `counts` and `decompose`
// subcommands (cli.cpp:163-236) with the same options, output bytes and exit
// codes (ValidationError/Error -> 1, IoError -> 2, cli.cpp:386-395), plus `scan`
// (every hot-path output from one pass) and `bench` (the benchlab CSV rows,
// bench.cpp:147-167, with strategy label "gpu").  The reference's CLI11 is not
// available, so options are parsed here ("--name value" / "--name=value").
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <iterator>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "ychg/errors.hpp"
#include "ychg/image.hpp"
#include "ychg/pnm.hpp"
#include "ychg/runscan.hpp"
#include "ychg/scan_b200.hpp"
#include "ychg_b200.h"

namespace {

using namespace ychg;

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ---- options: --name value | --name=value | flags
struct Args {
    std::map<std::string, std::string> opt;
    std::set<std::string> flags;

    bool has(const std::string& k) const { return opt.count(k) != 0; }
    std::string str(const std::string& k, const std::string& dflt = "") const {
        auto it = opt.find(k);
        return it == opt.end() ? dflt : it->second;
    }
    long long num(const std::string& k, long long dflt) const {
        if (!has(k)) return dflt;
        const std::string& v = opt.at(k);
        char* end = nullptr;
        const long long x = std::strtoll(v.c_str(), &end, 10);
        if (v.empty() || *end) throw UsageError("--" + k + ": not an integer: " + v);
        return x;
    }
    double real(const std::string& k, double dflt) const {
        if (!has(k)) return dflt;
        const std::string& v = opt.at(k);
        char* end = nullptr;
        const double x = std::strtod(v.c_str(), &end);
        if (v.empty() || *end) throw UsageError("--" + k + ": not a number: " + v);
        return x;
    }
    unsigned long long unum(const std::string& k, unsigned long long dflt) const {
        if (!has(k)) return dflt;
        const std::string& v = opt.at(k);
        char* end = nullptr;
        const unsigned long long x = std::strtoull(v.c_str(), &end, 10);
        if (v.empty() || *end) throw UsageError("--" + k + ": not an integer: " + v);
        return x;
    }
};

Args parse(int argc, char** argv, int first, const std::set<std::string>& options,
           const std::set<std::string>& flag_names, const std::set<std::string>& required) {
    Args a;
    for (int i = first; i < argc; ++i) {
        std::string s = argv[i];
        if (s.rfind("--", 0) != 0) throw UsageError("unexpected argument: " + s);
        s = s.substr(2);
        std::string val;
        bool inline_val = false;
        if (const auto eq = s.find('='); eq != std::string::npos) {
            val = s.substr(eq + 1);
            s = s.substr(0, eq);
            inline_val = true;
        }
        if (flag_names.count(s)) {
            if (inline_val) throw UsageError("--" + s + " takes no value");
            a.flags.insert(s);
        } else if (options.count(s)) {
            if (!inline_val) {
                if (i + 1 >= argc) throw UsageError("--" + s + " requires a value");
                val = argv[++i];
            }
            a.opt[s] = val;
        } else {
            throw UsageError("unknown option --" + s);
        }
    }
    for (const auto& r : required)
        if (!a.has(r)) throw UsageError("--" + r + " is required");
    return a;
}

// ---- files.  Behaviour of the reference CLI's file helpers (cli.cpp:25-49): the
// same IoError texts (the tests compare them) and an empty output path meaning
// standard output.  Implemented on C stdio: one handle, fixed-size reads.
std::vector<std::uint8_t> read_file(const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw IoError("cannot open " + path + " for reading");
    std::vector<std::uint8_t> bytes;
    std::uint8_t chunk[1 << 16];
    for (;;) {
        const std::size_t got = std::fread(chunk, 1, sizeof(chunk), f);
        bytes.insert(bytes.end(), chunk, chunk + got);
        if (got < sizeof(chunk)) break;
    }
    const bool failed = std::ferror(f) != 0;
    std::fclose(f);
    if (failed) throw IoError("read failed on " + path);
    return bytes;
}

void write_output(const std::string& path, const void* data, std::size_t size) {
    const bool to_stdout = path.empty();
    std::FILE* f = to_stdout ? stdout : std::fopen(path.c_str(), "wb");
    if (!f) throw IoError("cannot open " + path + " for writing");
    const bool ok = size == 0 || std::fwrite(data, 1, size, f) == size;
    if (to_stdout) {
        std::fflush(stdout);
        if (!ok) throw IoError("write to standard output failed");
        return;
    }
    const bool closed = std::fclose(f) == 0;
    if (!ok || !closed) throw IoError("write failed on " + path);
}

void write_output(const std::string& path, const std::string& text) { write_output(path, text.data(), text.size()); }

void check(int rc, const char* what) {
    if (rc == YCHG_OK) return;
    if (rc == YCHG_ERR_PARSE)
        throw ParseError(ychg_last_error(), static_cast<std::size_t>(ychg_last_error_offset()));
    if (rc == YCHG_ERR_INVALID) throw ValidationError(ychg_last_error());
    throw Error(std::string(what) + ": " + ychg_last_error());
}

int default_threads() { return 1; }  // every strategy runs the same GPU path

ScanStrategy strategy_for_threads(long long threads) {
    if (threads < 1) throw ValidationError("--threads must be >= 1, got " + std::to_string(threads));
    return threads == 1 ? ScanStrategy::serial() : ScanStrategy::parallel(static_cast<int>(threads));
}

int threshold_of(const Args& a) { return static_cast<int>(a.num("threshold", 128)); }

// ---- synth (cli.cpp:165-193): P4 bytes of the pattern, generated on the device
int pattern_id(const std::string& p) {
    static const char* names[] = {"full", "empty", "frame", "hbands", "checker", "random"};
    for (int i = 0; i < 6; ++i)
        if (p == names[i]) return i;
    throw ValidationError("unknown pattern \"" + p + "\"");
}

BinaryImage synth_image(int pattern, int w, int h, int bands, int cell, double density, unsigned long long seed) {
    if (w < 0 || h < 0) throw ValidationError("synth: negative geometry");
    BinaryImage img(w, h);
    const std::int64_t pitch = (img.row_stride() + 15) / 16 * 16;
    void* d = nullptr;
    check(ychg_device_alloc(0, std::max<std::int64_t>(pitch * h, 16), &d), "synth");
    const int rc = ychg_synth_device(pattern, w, h, bands, cell, density, seed, static_cast<std::uint8_t*>(d), pitch,
                                     nullptr);
    if (rc == YCHG_OK && w > 0 && h > 0)
        check(ychg_memcpy_2d(img.row(0), img.row_stride(), d, pitch, img.row_stride(), h, nullptr), "synth");
    if (rc == YCHG_OK) check(ychg_stream_synchronize(nullptr), "synth");
    ychg_device_free(0, d);
    check(rc, "synth");
    return img;
}

void run_synth(const Args& a) {
    const BinaryImage img =
        synth_image(pattern_id(a.str("pattern")), static_cast<int>(a.num("width", 0)), static_cast<int>(a.num("height", 0)),
                    static_cast<int>(a.num("k", 0)), static_cast<int>(a.num("cell", 0)), a.real("density", 0.0),
                    a.unum("seed", 0));
    const auto bytes = save_pnm(img);
    write_output(a.str("out"), bytes.data(), bytes.size());
}

// ---- counts: the reference CLI's CSV (cli.cpp:203-214 output format: a
// "col,count" header and one row per column, then optionally a blank line, a
// "boundary" header and one boundary column per row)
void append_row(std::string& csv, long long a, const long long* b) {
    char buf[48];
    const int n = b ? std::snprintf(buf, sizeof(buf), "%lld,%lld\n", a, *b) : std::snprintf(buf, sizeof(buf), "%lld\n", a);
    csv.append(buf, static_cast<std::size_t>(n));
}

void run_counts(const Args& a) {
    const BinaryImage image = load_pnm(read_file(a.str("input")), threshold_of(a));
    const std::vector<int> counts = cut_vertex_counts(image, strategy_for_threads(a.num("threads", default_threads())));
    std::string csv;
    csv.reserve(counts.size() * 12 + 16);
    csv += "col,count\n";
    long long col = 0;
    for (const int v : counts) {
        const long long cnt = v;
        append_row(csv, col++, &cnt);
    }
    if (a.flags.count("boundaries")) {
        csv += "\nboundary\n";
        const std::vector<int> bounds = detect_boundary_columns(counts);
        for (const int b : bounds) append_row(csv, b, nullptr);
    }
    write_output(a.str("out"), csv);
}

// ---- decompose (cli.cpp:223-227): to_json (hypergraph.cpp:194-207) of the device decomposition
void append_int(std::string& s, long long v) {
    char buf[24];
    const int n = std::snprintf(buf, sizeof(buf), "%lld", v);
    s.append(buf, static_cast<std::size_t>(n));
}

std::string decompose_json(const BinaryImage& image) {
    ychg_hypergraph* h = nullptr;
    check(ychg_decompose_image(image.bytes().data(), image.width(), image.height(), image.row_stride(),
                               YCHG_STRATEGY_SERIAL, 1, &h),
          "decompose");
    std::int64_t n = 0, e = 0;
    ychg_hypergraph_info(h, &n, &e, nullptr);
    std::vector<std::int32_t> runs(static_cast<std::size_t>(3 * n));
    std::vector<std::uint32_t> off(static_cast<std::size_t>(e + 1));
    const int rc = ychg_hypergraph_copy(h, runs.data(), off.data(), nullptr);
    ychg_hypergraph_destroy(h);
    check(rc, "decompose");
    std::string s;
    s.reserve(static_cast<std::size_t>(48 + 36 * e + 14 * n));
    s += "{\"width\":";
    append_int(s, image.width());
    s += ",\"height\":";
    append_int(s, image.height());
    s += ",\"hyperedges\":[";
    for (std::int64_t i = 0; i < e; ++i) {
        if (i) s += ',';
        s += "{\"id\":";
        append_int(s, i);
        s += ",\"col_start\":";
        append_int(s, runs[3 * off[i]]);
        s += ",\"runs\":[";
        for (std::uint32_t k = off[i]; k < off[i + 1]; ++k) {
            if (k != off[i]) s += ',';
            s += '[';
            append_int(s, runs[3 * k + 1]);
            s += ',';
            append_int(s, runs[3 * k + 2]);
            s += ']';
        }
        s += "]}";
    }
    s += "]}";
    return s;
}

void run_decompose(const Args& a) {
    const BinaryImage image = load_pnm(read_file(a.str("input")), threshold_of(a));
    strategy_for_threads(a.num("threads", default_threads()));
    write_output(a.str("out"), decompose_json(image) + "\n");
}

// ---- scan (new): every output of the hot path from one pass over the file
void run_scan(const Args& a) {
    const auto bytes = read_file(a.str("input"));
    const ScanResult r = scan_pnm(bytes, threshold_of(a));
    std::string js = "{\"width\":" + std::to_string(r.counts.size()) + ",\"total_runs\":" +
                     std::to_string(r.total_runs) + ",\"links\":" + std::to_string(r.links) +
                     ",\"hyperedges\":" + std::to_string(r.hyperedges) +
                     ",\"n_boundaries\":" + std::to_string(r.boundaries.size()) + "}\n";
    write_output(a.str("out"), js);
}

// ---- bench resolution|hyperedges (cli.cpp:251-281, bench.cpp:59-167): median
// wall ns per op in the benchlab CSV; strategies serial | parallel:N | gpu (all
// run the one GPU path; the label is recorded as given)
std::vector<std::string> split(const std::string& text, char sep) {
    std::vector<std::string> parts;
    std::string cur;
    for (char ch : text) {
        if (ch == sep) {
            parts.push_back(cur);
            cur.clear();
        } else {
            cur += ch;
        }
    }
    if (!cur.empty() || !parts.empty()) parts.push_back(cur);
    return parts;
}

struct Strategy {
    std::string label;
    int threads;
};

std::vector<Strategy> parse_strategies(const std::string& text) {
    std::vector<Strategy> out;
    for (const std::string& part : split(text, ',')) {
        if (part == "serial" || part == "gpu") {
            out.push_back({part, 1});
        } else if (part.rfind("parallel:", 0) == 0) {
            char* end = nullptr;
            const long t = std::strtol(part.c_str() + 9, &end, 10);
            if (part.size() == 9 || *end) throw ValidationError("bad strategy \"" + part + "\" (want parallel:N)");
            if (t < 1) throw ValidationError("scan: parallel strategy needs threads >= 1, got " + std::to_string(t));
            out.push_back({"parallel", static_cast<int>(t)});
        } else {
            throw ValidationError("bad strategy \"" + part + "\" (want serial, parallel:N or gpu)");
        }
    }
    if (out.empty()) throw ValidationError("no strategies given");
    return out;
}

void decompose_device_only(const BinaryImage& image) {
    ychg_hypergraph* h = nullptr;
    check(ychg_decompose_image(image.bytes().data(), image.width(), image.height(), image.row_stride(),
                               YCHG_STRATEGY_SERIAL, 1, &h),
          "decompose");
    ychg_hypergraph_destroy(h);
}

std::string bench_rows(const std::string& op, const BinaryImage& img, const std::vector<Strategy>& strategies,
                       int reps, int warmup) {
    const std::int64_t edges = scan(img).hyperedges;
    std::string rows;
    for (const Strategy& st : strategies) {
        const ScanStrategy ss = st.label == "parallel" ? ScanStrategy::parallel(st.threads) : ScanStrategy::serial();
        std::vector<long long> ns;
        for (int i = 0; i < warmup + reps; ++i) {
            const auto t0 = std::chrono::steady_clock::now();
            if (op == "counts") (void)cut_vertex_counts(img, ss);
            else if (op == "profile") (void)build_profile(img, ss);
            else if (op == "decompose") decompose_device_only(img);
            else (void)scan(img);
            const auto t1 = std::chrono::steady_clock::now();
            if (i >= warmup) ns.push_back(std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count());
        }
        std::sort(ns.begin(), ns.end());
        rows += op + "," + st.label + "," + std::to_string(st.threads) + "," + std::to_string(img.width()) + "," +
                std::to_string(img.height()) + "," + std::to_string(edges) + "," + std::to_string(reps) + "," +
                std::to_string(ns[(ns.size() - 1) / 2]) + "\n";
    }
    return rows;
}

void run_bench(const std::string& axis, const Args& a) {
    const std::string op = a.str("op", "counts");
    if (op != "counts" && op != "profile" && op != "decompose" && op != "scan")
        throw ValidationError("bad op \"" + op + "\" (want counts|profile|decompose|scan)");
    const auto strategies = parse_strategies(a.str("strategies", "gpu"));
    const int reps = static_cast<int>(a.num("reps", 5)), warmup = static_cast<int>(a.num("warmup", 1));
    if (reps < 1) throw ValidationError("sweep: reps must be >= 1");
    if (warmup < 0) throw ValidationError("sweep: warmup must be >= 0");
    if (a.has("svg")) throw ValidationError("--svg: ychg_b200 writes the CSV report only");
    std::string csv = "op,strategy,threads,width,height,hyperedges,reps,median_ns\n";
    if (axis == "resolution") {
        const auto pat = split(a.str("pattern"), ':');
        const int pid = pattern_id(pat.empty() ? "" : pat[0]);
        const bool arity_ok = (pid <= 2 && pat.size() == 1) || ((pid == 3 || pid == 4) && pat.size() == 2) ||
                              (pid == 5 && (pat.size() == 2 || pat.size() == 3));
        if (!arity_ok)
            throw ValidationError("bad pattern \"" + a.str("pattern") +
                                  "\" (want full|empty|frame|hbands:K|checker:C|random:D[:SEED])");
        int prev = 0;
        for (const std::string& sz : split(a.str("sizes"), ',')) {
            char* end = nullptr;
            const long s = std::strtol(sz.c_str(), &end, 10);
            if (sz.empty() || *end) throw ValidationError("bad size \"" + sz + "\"");
            if (s <= prev) throw ValidationError("resolution_sweep: sizes must be strictly increasing");
            prev = static_cast<int>(s);
            const int arg = pat.size() > 1 ? std::atoi(pat[1].c_str()) : 0;
            const double dens = pid == 5 ? std::atof(pat[1].c_str()) : 0.0;
            const unsigned long long seed = pat.size() > 2 ? std::strtoull(pat[2].c_str(), nullptr, 10) : 0;
            const BinaryImage img = synth_image(pid, prev, prev, pid == 3 ? arg : 0, pid == 4 ? arg : 0, dens, seed);
            csv += bench_rows(op, img, strategies, reps, warmup);
        }
    } else {
        const int w = static_cast<int>(a.num("width", 0)), h = static_cast<int>(a.num("height", 0));
        for (const std::string& t : split(a.str("targets"), ',')) {
            if (t == "max") {
                csv += bench_rows(op, synth_image(4, w, h, 0, 1, 0.0, 0), strategies, reps, warmup);
                continue;
            }
            char* end = nullptr;
            const long long k = std::strtoll(t.c_str(), &end, 10);
            if (t.empty() || *end) throw ValidationError("bad target \"" + t + "\" (want an integer or max)");
            if (k < 1 || k > h / 2)
                throw ValidationError("hyperedge_sweep: target " + std::to_string(k) + " unreachable at height " +
                                      std::to_string(h) + " (needs 1 <= k <= height/2)");
            csv += bench_rows(op, synth_image(3, w, h, static_cast<int>(k), 0, 0.0, 0), strategies, reps, warmup);
        }
    }
    write_output(a.str("csv"), csv);
}

const char* kUsage =
    "usage: ychg_b200 <command> [options]\n"
    "  synth     --pattern P --width W --height H [--seed S] [--k K] [--cell C] [--density D] [--out PATH]\n"
    "  counts    --input PNM [--threshold T] [--threads N] [--boundaries] [--out PATH]\n"
    "  decompose --input PNM [--threshold T] [--threads N] [--out PATH]\n"
    "  scan      --input PNM [--threshold T] [--out PATH]\n"
    "  bench resolution --sizes S1,S2,.. --pattern full|empty|frame|hbands:K|checker:C|random:D[:SEED]\n"
    "            --csv PATH [--op counts|profile|decompose|scan] [--strategies gpu|serial|parallel:N,..]\n"
    "            [--reps R] [--warmup W]\n"
    "  bench hyperedges --width W --height H --targets K1,K2,..|max --csv PATH [same options]\n";

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2 || !std::strcmp(argv[1], "--help") || !std::strcmp(argv[1], "-h")) {
        std::fputs(kUsage, argc < 2 ? stderr : stdout);
        return argc < 2 ? 1 : 0;
    }
    const std::string cmd = argv[1];
    try {
        if (cmd == "synth") {
            run_synth(parse(argc, argv, 2, {"pattern", "width", "height", "seed", "k", "cell", "density", "out"}, {},
                            {"pattern", "width", "height"}));
        } else if (cmd == "counts") {
            run_counts(parse(argc, argv, 2, {"input", "threshold", "threads", "out"}, {"boundaries"}, {"input"}));
        } else if (cmd == "decompose") {
            run_decompose(parse(argc, argv, 2, {"input", "threshold", "threads", "out"}, {}, {"input"}));
        } else if (cmd == "scan") {
            run_scan(parse(argc, argv, 2, {"input", "threshold", "out"}, {}, {"input"}));
        } else if (cmd == "bench") {
            const std::string axis = argc > 2 ? argv[2] : "";
            if (axis == "resolution")
                run_bench(axis, parse(argc, argv, 3, {"sizes", "pattern", "op", "strategies", "reps", "warmup", "csv", "svg"},
                                      {}, {"sizes", "pattern", "csv"}));
            else if (axis == "hyperedges")
                run_bench(axis, parse(argc, argv, 3, {"width", "height", "targets", "op", "strategies", "reps", "warmup",
                                                      "csv", "svg"},
                                      {}, {"width", "height", "targets", "csv"}));
            else
                throw UsageError("bench needs a sweep: resolution | hyperedges");
        } else {
            throw UsageError("unknown command " + cmd);
        }
    } catch (const UsageError& e) {
        std::cerr << e.what() << "\n" << kUsage;
        return 1;
    } catch (const IoError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
    return 0;
}
