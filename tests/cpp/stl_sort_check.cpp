// Checks the device replica of libstdc++'s std::sort (csrc/stl_sort.cuh) against
// std::sort itself: many small-integer keys (ties everywhere), element payloads
// recording the original position, sizes across the insertion / introsort /
// heapsort regimes.  Prints the number of arrays whose permutation differs.
#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>

#include "stl_sort.cuh"

struct E {
    double mag;
    int col;
    double val;
};

int main() {
    std::mt19937 gen(7);
    int bad = 0, total = 0;
    auto less = [](const E& a, const E& b) { return a.mag > b.mag; };  // ensure_min_support's order
    for (int n : {0, 1, 2, 3, 5, 8, 15, 16, 17, 18, 31, 32, 33, 47, 64, 100, 257, 1000}) {
        for (int rep = 0; rep < 300; ++rep) {
            std::uniform_int_distribution<int> keys(0, rep % 3 == 0 ? 2 : (rep % 3 == 1 ? 8 : 1000));
            std::vector<E> a(n);
            for (int i = 0; i < n; ++i) a[i] = {static_cast<double>(keys(gen)), i, 0.5 * i};
            // an adversarial family: already sorted / reversed / organ pipe
            if (rep % 7 == 3) std::sort(a.begin(), a.end(), [](const E& x, const E& y) { return x.mag < y.mag; });
            if (rep % 7 == 4)
                for (int i = 0; i < n; ++i) a[i].mag = (i < n / 2) ? i : n - i;
            std::vector<E> b = a;
            std::sort(a.begin(), a.end(), less);
            amgcu::stlsort::sort(b.data(), b.data() + n, less);
            ++total;
            for (int i = 0; i < n; ++i)
                if (a[i].col != b[i].col) {
                    ++bad;
                    break;
                }
        }
    }
    std::printf("%d %d\n", bad, total);
    return bad ? 1 : 0;
}
