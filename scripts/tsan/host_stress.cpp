// ThreadSanitizer stress harness for adt_pack_host (scripts/tsan/run.sh); links adt_host.cpp alone.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
#include <random>
#include "adt.h"
int main() {
    std::mt19937 rng(1);
    std::vector<uint64_t> counts = {500, 25000, 400000, 5000, 70000, 3};
    std::vector<std::vector<uint32_t>> w(counts.size());
    for (size_t i = 0; i < counts.size(); ++i) { w[i].resize(counts[i]); for (auto &x : w[i]) x = rng(); }
    int rs[] = {1, 2, 3, 4, 1, 3};
    std::vector<adt_segment> segs(counts.size());
    uint64_t off = 0;
    for (size_t i = 0; i < counts.size(); ++i) {
        segs[i].weights = w[i].data(); segs[i].count = counts[i]; segs[i].offset = off; segs[i].round_to = rs[i]; segs[i].reserved = 0;
        off += (counts[i] * rs[i] + 63) / 64 * 64;
    }
    std::vector<uint8_t> ref(off + 64);
    std::vector<double> ssref(counts.size());
    if (adt_pack_host(segs.data(), (int)segs.size(), ref.data(), ssref.data(), 1)) return 1;
    int bad = 0;
    std::vector<std::thread> ts;
    for (int t = 0; t < 4; ++t) ts.emplace_back([&, t] {
        std::vector<uint8_t> out(off + 64);
        std::vector<double> ss(counts.size());
        for (int it = 0; it < 30; ++it) {
            int th = 1 + (it * 7 + t) % 9;
            memset(out.data(), 0, out.size());
            if (adt_pack_host(segs.data(), (int)segs.size(), out.data(), ss.data(), th)) { __atomic_add_fetch(&bad, 1, __ATOMIC_RELAXED); continue; }
            if (memcmp(out.data(), ref.data(), off) || memcmp(ss.data(), ssref.data(), ss.size() * 8)) __atomic_add_fetch(&bad, 1, __ATOMIC_RELAXED);
            if (it % 5 == 0) std::this_thread::sleep_for(std::chrono::microseconds(300 + 200 * t));   // let workers fall asleep
        }
    });
    for (auto &x : ts) x.join();
    printf("mismatches %d\n", bad);
    return bad != 0;
}
