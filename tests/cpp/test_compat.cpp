// test_compat.cpp -- the reference's result-pinning tests, restated against the
// B200 shims with the reference's C++ signatures (include/sortbench_b200).
// The oracle is the reference's own: std::sort + equality (bench::verify_output,
// P/src/bench.cpp:95-104). Exit code 0 = all pass; prints one line per check.
#include <algorithm>
#include <cstdio>
#include <random>
#include <string>

#include "sortbench_b200/sortbench.hpp"

using namespace sortbench;
using parallel::Algorithm;
using parallel::KeepHalf;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                            \
    do {                                                                       \
        if (cond) ++g_pass;                                                    \
        else {                                                                 \
            ++g_fail;                                                          \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #cond);        \
        }                                                                      \
    } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static runtime::WorldOptions opts(int p, int k = 1) {
    runtime::WorldOptions o;
    o.procs = p;
    o.core_slots = k;
    return o;
}

static DataList sorted_copy(DataList v) {
    std::sort(v.begin(), v.end());
    return v;
}

int main() {
    kernels::SortStats st;
    // sort_core KATs (P/tests/test_sort_core.cpp:60-189)
    {
        DataList v{5, 1, 4, 2, 8};
        kernels::bubble_sort(v, st);
        CHECK((v == DataList{1, 2, 4, 5, 8}));
        DataList r{4, 3, 2, 1}, s(4);
        kernels::merge_sort(r, 0, 3, s, st);
        CHECK((r == DataList{1, 2, 3, 4}));
        DataList e{3, 1}, s2(2);
        kernels::merge_sort(e, 1, 0, s2, st);  // empty range
        CHECK((e == DataList{3, 1}));
        DataList q{3, 1, 2};
        kernels::quick_sort(q, 0, 3, st);
        CHECK((q == DataList{1, 2, 3}));
        DataList q2{2, 1};
        kernels::quick_sort(q2, 0, 1, st);
        CHECK((q2 == DataList{2, 1}));
        DataList q3{1, 2};
        CHECK(throws<ProgrammingError>([&] { kernels::quick_sort(q3, 1, 2, st); }));
        CHECK(kernels::is_sorted(DataList{}) && kernels::is_sorted(DataList{1, 2, 2, 3}) &&
              !kernels::is_sorted(DataList{2, 1}));
        CHECK((kernels::merge_runs(DataList{1, 3, 5}, DataList{2, 4, 6}, st) ==
               DataList{1, 2, 3, 4, 5, 6}));
        CHECK((kernels::merge_runs(DataList{}, DataList{1, 2, 3}, st) == DataList{1, 2, 3}));
    }
    // all kernels vs std::sort, seed 99 (P/tests/test_sort_core.cpp:191-216)
    {
        std::mt19937_64 rng(99);
        bool ok = true;
        for (int t = 0; t < 250; ++t) {
            const std::size_t s = rng() % 512;
            DataList in(s);
            for (auto& x : in) x = static_cast<Element>(rng() % 32);
            const DataList expect = sorted_copy(in);
            for (auto algo : {Algorithm::bubble, Algorithm::merge, Algorithm::quick}) {
                DataList b = in, scratch(in.size());
                parallel::select_kernel(algo)(b, scratch, st);
                ok = ok && b == expect;
            }
        }
        CHECK(ok);
    }
    // parallel helpers (P/tests/test_parallel_sort.cpp:45-237)
    {
        CHECK((parallel::plan_partition(8, 3).sizes == std::vector<std::size_t>{3, 3, 2}));
        CHECK(throws<ConfigError>([] { parallel::plan_partition(4, 0); }));
        CHECK(parallel::build_schedule(4).partner(1, 1) == 2);
        CHECK(throws<ConfigError>([] { parallel::algorithm_from_string("heap"); }));
        CHECK((parallel::merge_split(DataList{1, 3, 5}, DataList{2, 4, 6}, KeepHalf::low, st) ==
               DataList{1, 2, 3}));
        CHECK((parallel::merge_split(DataList{2, 4, 6}, DataList{1, 3, 5}, KeepHalf::high, st) ==
               DataList{4, 5, 6}));
        CHECK((parallel::merge_split(DataList{1, 2}, DataList{0, 0, 0}, KeepHalf::low, st) ==
               DataList{0, 0}));
        const parallel::PaddedBlock a{{7}, 1}, b{{0, 0}, 0};
        const auto lo = parallel::merge_split_padded(a, b, KeepHalf::low, st);
        const auto hi = parallel::merge_split_padded(b, a, KeepHalf::high, st);
        CHECK((lo.reals == DataList{0, 0} && lo.virtuals == 0));
        CHECK((hi.reals == DataList{7} && hi.virtuals == 1));
    }
    // whole path (P/tests/test_parallel_sort.cpp:271-343)
    {
        CHECK((parallel::scatter_merge_sort(Algorithm::merge, DataList{3, 1, 2}, opts(1)).sorted ==
               DataList{1, 2, 3}));
        CHECK((parallel::scatter_merge_sort(Algorithm::bubble, DataList{4, 3, 2, 1}, opts(2)).sorted ==
               DataList{1, 2, 3, 4}));
        CHECK(parallel::scatter_merge_sort(Algorithm::merge, DataList{}, opts(3)).sorted.empty());
        const DataList in = bench::gen_data(4096, 2024);
        CHECK(parallel::scatter_merge_sort(Algorithm::quick, in, opts(4, 2)).sorted == sorted_copy(in));
        bool ok = true;
        for (int p : {2, 3, 4})
            for (std::size_t n = 0; n <= 8; ++n)
                for (std::uint32_t mask = 0; mask < (1u << n); ++mask) {
                    DataList d(n);
                    for (std::size_t i = 0; i < n; ++i) d[i] = (mask >> i) & 1u;
                    ok = ok && parallel::scatter_merge_sort(Algorithm::merge, d, opts(p)).sorted ==
                                   sorted_copy(d);
                }
        CHECK(ok);
    }
    // acceptance criterion 1 (P/tests/acceptance.cpp:121-157)
    {
        std::mt19937_64 rng(20240601);
        const int pc[5] = {1, 2, 3, 4, 8};
        const Algorithm algos[3] = {Algorithm::bubble, Algorithm::merge, Algorithm::quick};
        bool ok = true;
        for (int i = 0; i < 1000 && ok; ++i) {
            const std::size_t n = rng() % 4097;
            const int p = pc[rng() % 5];
            const DataList in = bench::gen_data(n, rng());
            ok = parallel::scatter_merge_sort(algos[i % 3], in, opts(p, 1 + i % 2)).sorted ==
                 sorted_copy(in);
            if (!ok) std::printf("  mismatch at case %d n=%zu p=%d\n", i, n, p);
        }
        CHECK(ok);
    }
    std::printf("%d passed, %d failed\n", g_pass, g_fail);
    return g_fail == 0 ? 0 : 1;
}
