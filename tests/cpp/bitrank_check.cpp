// Host check of csrc/bitrank.h (the mask-pair records of the band-staged masked product):
// nth_set_bit24 against the plain loop on every 24-bit mask shape sampled, and the
// partner lookup against a direct search on random sorted column lists of up to 24
// entries.  Prints "<failures> <cases>".
#include <cstdio>
#include <random>
#include <vector>
#include <algorithm>

#include "bitrank.h"

using namespace amgcu::bitrank;

int main() {
    long bad = 0, cases = 0;
    std::mt19937 rng(12345);
    // 1. nth set bit: all 16-bit masks exhaustively, plus random 24-bit masks
    auto check_mask = [&](unsigned int m) {
        int j = 0;
        for (int pos = 0; pos < 24; ++pos)
            if ((m >> pos) & 1u) {
                ++cases;
                if (nth_set_bit24(m, j) != static_cast<unsigned int>(pos)) ++bad;
                ++j;
            }
    };
    for (unsigned int m = 0; m < (1u << 16); ++m) check_mask(m);
    for (int t = 0; t < 200000; ++t) check_mask(rng() & 0xffffffu);
    check_mask(0xffffffu);
    check_mask(0x800000u);
    // 2. partner lookup on sorted lists
    for (int t = 0; t < 100000; ++t) {
        const int la = 1 + static_cast<int>(rng() % 24), lb = 1 + static_cast<int>(rng() % 24);
        const int range = 4 + static_cast<int>(rng() % 60);
        auto draw = [&](int l) {
            std::vector<int32_t> v;
            while (static_cast<int>(v.size()) < std::min(l, range)) {
                const int32_t c = static_cast<int32_t>(rng() % range);
                if (std::find(v.begin(), v.end(), c) == v.end()) v.push_back(c);
            }
            std::sort(v.begin(), v.end());
            return v;
        };
        const std::vector<int32_t> a = draw(la), b = draw(lb);
        unsigned int mi, mt;
        const int n = match_masks(a.data(), static_cast<int>(a.size()), b.data(), static_cast<int>(b.size()), &mi, &mt);
        int direct = 0;
        for (size_t s = 0; s < a.size(); ++s) {
            const auto it = std::find(b.begin(), b.end(), a[s]);
            const int want = it == b.end() ? -1 : static_cast<int>(it - b.begin());
            if (want >= 0) ++direct;
            ++cases;
            if (partner(mi, mt, static_cast<int>(s)) != want) ++bad;
        }
        ++cases;
        if (n != direct || popcount32(mi) != n || popcount32(mt) != n) ++bad;
    }
    std::printf("%ld %ld\n", bad, cases);
    return bad ? 1 : 0;
}
