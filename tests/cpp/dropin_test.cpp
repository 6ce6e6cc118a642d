// dropin_test.cpp -- the reference's runscan known-answer tests, compiled
// against OUR ychg headers and linked against libychg.so (the C++ drop-in).
// Vectors from proj/tests/test_runscan.cpp:35-49,66-85,129-143 and
// acceptance.cpp:101-121.  Exit code = number of failed checks.
#include <cstdio>
#include <vector>

#include "ychg/errors.hpp"
#include "ychg/image.hpp"
#include "ychg/pnm.hpp"
#include "ychg/runscan.hpp"
#include <string>
#include "ychg/scan_b200.hpp"

using namespace ychg;

static int failures = 0;
#define CHECK(cond)                                                   \
    do {                                                              \
        if (!(cond)) {                                                \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                               \
        }                                                             \
    } while (0)

static BinaryImage full(int w, int h) {
    BinaryImage img(w, h);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) img.set(x, y, true);
    return img;
}
static BinaryImage frame(int w, int h) {
    BinaryImage img(w, h);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x)
            if (x == 0 || y == 0 || x == w - 1 || y == h - 1) img.set(x, y, true);
    return img;
}
static BinaryImage hbands(int w, int h, int k) {
    BinaryImage img(w, h);
    const int bh = (h - (k - 1)) / k;
    for (int b = 0; b < k; ++b)
        for (int y = b * (bh + 1); y < b * (bh + 1) + bh; ++y)
            for (int x = 0; x < w; ++x) img.set(x, y, true);
    return img;
}
static BinaryImage branch() {
    BinaryImage img(2, 7);
    for (int y : {0, 1, 3, 4, 5, 6}) img.set(0, y, true);
    for (int y : {0, 1, 2, 3, 4, 6}) img.set(1, y, true);
    return img;
}

int main() {
    const auto serial = ScanStrategy::serial();
    CHECK(cut_vertex_counts(full(4, 4), serial) == (std::vector<int>{1, 1, 1, 1}));
    CHECK(cut_vertex_counts(frame(5, 5), serial) == (std::vector<int>{1, 2, 2, 2, 1}));
    CHECK(cut_vertex_counts(BinaryImage(3, 3), serial) == (std::vector<int>{0, 0, 0}));
    CHECK(cut_vertex_counts(branch(), serial) == (std::vector<int>{2, 2}));
    CHECK(cut_vertex_counts(BinaryImage(0, 0), serial).empty());
    CHECK(cut_vertex_counts(hbands(8, 11, 3), serial) == std::vector<int>(8, 3));
    for (int t : {1, 2, 4, 8, 16})
        CHECK(cut_vertex_counts(frame(5, 5), ScanStrategy::parallel(t)) ==
              (std::vector<int>{1, 2, 2, 2, 1}));

    // Validation: the exception type AND its what() (runscan.cpp:25-26, 105-107).
    // The messages are printed as "WHAT\t<case>\t<what()>" for tests/test_gpu_parity.py,
    // which compares them with the live reference's own messages.
    auto expect_validation = [&](const char* name, auto&& fn) {
        bool threw = false;
        try {
            fn();
        } catch (const ValidationError& e) {
            threw = true;
            std::printf("WHAT\t%s\t%s\n", name, e.what());
        }
        CHECK(threw);
    };
    expect_validation("parallel0", [&] { cut_vertex_counts(full(3, 50), ScanStrategy::parallel(0)); });
    expect_validation("parallel-2", [&] { cut_vertex_counts(full(3, 50), ScanStrategy::parallel(-2)); });
    expect_validation("column_runs4", [&] { column_runs(full(4, 4), 4); });
    expect_validation("column_runs-1", [&] { column_runs(full(4, 4), -1); });
    expect_validation("build_profile_parallel0", [&] { build_profile(full(3, 5), ScanStrategy::parallel(0)); });

    CHECK(detect_boundary_columns(std::vector<int>{1, 2, 2, 2, 1}) == (std::vector<int>{0, 1, 4}));
    CHECK(detect_boundary_columns(std::vector<int>{0, 0, 0}).empty());
    CHECK(detect_boundary_columns(std::vector<int>{}).empty());
    CHECK(detect_boundary_columns(std::vector<int>{0, 1}) == (std::vector<int>{1}));
    CHECK(detect_boundary_columns(std::vector<int>{3}) == (std::vector<int>{0}));
    CHECK(detect_boundary_columns(std::vector<int>{2, 2}) == (std::vector<int>{0}));
    CHECK(detect_boundary_columns(cut_vertex_counts(branch(), serial)) == (std::vector<int>{0}));

    // acceptance.cpp:101-121 -- branch: counts [2,2], boundaries [0], 4 hyperedges.
    const ScanResult br = scan(branch());
    CHECK(br.counts == (std::vector<int>{2, 2}));
    CHECK(br.boundaries == (std::vector<int>{0}));
    CHECK(br.hyperedges == 4);
    const ScanResult fr = scan(frame(5, 5));
    CHECK(fr.boundaries == (std::vector<int>{0, 1, 4}));
    CHECK(fr.hyperedges == 4);
    CHECK(fr.total_runs == 8);
    // test_hypergraph.cpp:75-88
    for (int k : {1, 3, 7}) CHECK(scan(hbands(20, 20, k)).hyperedges == k);
    BinaryImage chk(8, 8);
    for (int y = 0; y < 8; ++y)
        for (int x = 0; x < 8; ++x)
            if ((x + y) % 2 == 0) chk.set(x, y, true);
    CHECK(scan(chk).hyperedges == 32);
    CHECK(scan(BinaryImage(3, 3)).hyperedges == 0);
    CHECK(scan(BinaryImage(0, 0)).hyperedges == 0);
    CHECK(foreground_count(frame(5, 5)) == 16);

    // test_runscan.cpp:17-33 (column_runs) and :116-123 (build_profile worked examples)
    CHECK(column_runs(full(4, 4), 2) == (std::vector<Run>{{2, 0, 3}}));
    CHECK(column_runs(frame(5, 5), 0) == (std::vector<Run>{{0, 0, 4}}));
    CHECK(column_runs(frame(5, 5), 1) == (std::vector<Run>{{1, 0, 0}, {1, 4, 4}}));
    CHECK(column_runs(frame(5, 5), 4) == (std::vector<Run>{{4, 0, 4}}));
    CHECK(column_runs(BinaryImage(3, 3), 0).empty());
    CHECK(column_runs(branch(), 0) == (std::vector<Run>{{0, 0, 1}, {0, 3, 6}}));
    CHECK(column_runs(branch(), 1) == (std::vector<Run>{{1, 0, 4}, {1, 6, 6}}));
    for (int bad : {4, -1}) {
        bool t = false;
        try {
            column_runs(full(4, 4), bad);
        } catch (const ValidationError&) {
            t = true;
        }
        CHECK(t);
    }
    const ColumnProfile fp = build_profile(frame(5, 5), serial);
    CHECK(fp.counts == (std::vector<int>{1, 2, 2, 2, 1}));
    CHECK(fp.runs[0] == (std::vector<Run>{{0, 0, 4}}));
    CHECK(fp.runs[2] == (std::vector<Run>{{2, 0, 0}, {2, 4, 4}}));
    CHECK(fp.total_runs() == 8);
    const ColumnProfile bp = build_profile(branch(), ScanStrategy::parallel(4));
    CHECK(bp.counts == (std::vector<int>{2, 2}));
    CHECK(bp.runs[0] == (std::vector<Run>{{0, 0, 1}, {0, 3, 6}}));
    CHECK(bp.runs[1] == (std::vector<Run>{{1, 0, 4}, {1, 6, 6}}));
    CHECK(build_profile(frame(5, 5), ScanStrategy::parallel(16)) == fp);

    // pnm (test_imagekit.cpp:172-257)
    auto bytes_of = [](const std::string& s) { return std::vector<std::uint8_t>(s.begin(), s.end()); };
    CHECK(load_pnm(bytes_of("P1\n2 2\n1 0\n0 1\n")) == load_pnm(bytes_of("P1 # binary\n2 2 # dims\n1001")));
    CHECK(load_pnm(save_pnm(frame(5, 5))) == frame(5, 5));
    CHECK(save_pnm(BinaryImage(0, 0)) == bytes_of("P4\n0 0\n"));
    {
        auto p5 = bytes_of("P5\n2 1\n255\n");
        p5.push_back(10);
        p5.push_back(200);
        const BinaryImage g = load_pnm(p5);
        CHECK(g.get(0, 0) && !g.get(1, 0));
        std::size_t off = 0;
        try {
            load_pnm(bytes_of("P5 2 2 255\n\x01\x02"));
        } catch (const ParseError& e) {
            off = e.offset();
        }
        CHECK(off == 11);
        bool inval = false;
        try {
            load_pnm(bytes_of("P6\n1 1\n255\n"));
        } catch (const ValidationError&) {
            inval = true;
        }
        CHECK(inval);
        const ScanResult sr = scan_pnm(save_pnm(frame(5, 5)));
        CHECK(sr.counts == (std::vector<int>{1, 2, 2, 2, 1}) && sr.hyperedges == 4);
        const BinaryImage wide = hbands(3000, 40, 7);
        const ScanResult a = scan(wide), b = scan_sharded(wide, 3);
        CHECK(a.counts == b.counts && a.boundaries == b.boundaries && a.hyperedges == b.hyperedges && b.hyperedges == 7);
    }

    std::printf("dropin_test: %d failure(s)\n", failures);
    return failures;
}
