// decompose_dropin.cpp -- C++ parity of the device decomposition through the
// reference's own types: ychg::b200::decompose (include/ychg/decompose_b200.hpp)
// must return a Hypergraph equal (hypergraph.hpp:62-65) to the reference's
// ychg::decompose(build_profile(img)) (hypergraph.cpp:94-170), with identical
// run_to_edge(), and must reject malformed profiles with the reference's message.
// Built by `make -C oracle dropin` against the reference headers and sources
// (image, synth, runscan, hypergraph, oracle); test infrastructure only.
#include <cstdio>
#include <string>
#include <vector>

#include "corpus.hpp"
#include "ychg/decompose_b200.hpp"
#include "ychg/hypergraph.hpp"
#include "ychg/runscan.hpp"
#include "ychg/synth.hpp"

using namespace ychg;

static bool same(const Hypergraph& a, const Hypergraph& b) {
    if (!(a == b)) return false;
    const auto x = a.run_to_edge(), y = b.run_to_edge();
    return x.size() == y.size() && std::equal(x.begin(), x.end(), y.begin());
}

static std::string message_of(auto&& fn) {
    try {
        fn();
    } catch (const ValidationError& e) {
        return std::string("V:") + e.what();
    } catch (const std::exception& e) {
        return std::string("E:") + e.what();
    }
    return "ok";
}

int main() {
    int fails = 0, n = 0;
    auto cases = tests::full_corpus();
    cases.push_back({"checker(7) 3000x2000", SynthSpec::checker(3000, 2000, 7)});
    cases.push_back({"random 2500x2500", SynthSpec::random(2500, 2500, 0.5, 1307)});
    cases.push_back({"hbands 5000x800", SynthSpec::hbands(5000, 800, 147)});
    for (const auto& cs : cases) {
        const BinaryImage img = synth(cs.spec);
        const ColumnProfile prof = build_profile(img, ScanStrategy::serial());
        const Hypergraph ref = decompose(prof);
        const Hypergraph g1 = b200::decompose(img);
        const Hypergraph g2 = b200::decompose(prof);
        ++n;
        if (!same(ref, g1) || !same(ref, g2)) {
            if (++fails <= 5) std::printf("mismatch: %s\n", cs.name.c_str());
        }
    }
    // validate_profile (hypergraph.cpp:62-90): same exception type and message
    const ColumnProfile base = build_profile(synth(SynthSpec::random(40, 30, 0.5, 9)), ScanStrategy::serial());
    std::vector<ColumnProfile> bad;
    {
        ColumnProfile p = base; p.counts[3] += 1; bad.push_back(p);
        p = base; p.runs[5][0].col = 6; bad.push_back(p);
        p = base; p.runs[7].back().y_bot = p.height; bad.push_back(p);
        p = base; p.runs[9][1].y_top = p.runs[9][0].y_bot + 1; bad.push_back(p);
        p = base; p.runs[2][0].col = 9; p.counts[1] += 1; bad.push_back(p);    // count error first
        p = base; p.runs[1][0].col = 9; p.counts[2] += 1; bad.push_back(p);    // run error first
        p = base; p.runs.pop_back(); bad.push_back(p);
        p = base; p.width = -1; bad.push_back(p);
        p = base; p.runs[4][0].y_top = p.runs[4][0].y_bot + 1; bad.push_back(p);
    }
    for (std::size_t i = 0; i < bad.size(); ++i) {
        const std::string a = message_of([&] { decompose(bad[i]); });
        const std::string b = message_of([&] { b200::decompose(bad[i]); });
        ++n;
        if (a != b) {
            ++fails;
            std::printf("validation %zu: reference '%s' vs b200 '%s'\n", i, a.c_str(), b.c_str());
        }
    }
    std::printf("%s decompose drop-in: %d/%d cases identical\n", fails ? "[FAIL]" : "[PASS]", n - fails, n);
    return fails ? 1 : 0;
}
