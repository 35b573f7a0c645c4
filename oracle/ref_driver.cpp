// ref_driver.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI wrapper around the UNMODIFIED reference library (compiled by
// oracle/build_ref.sh straight from /root/reference/proj/src into
// oracle/_ref/libsortbench_ref.so). It lets the Python tests and bench.py's
// reference arm call the reference's own code path:
//   bench::gen_data                   P/src/bench.cpp:57-71
//   parallel::plan_partition          P/src/parallel_sort.cpp:26-38
//   parallel::merge_split_padded      P/src/parallel_sort.cpp:115-134
//   parallel::scatter_merge_sort      P/src/parallel_sort.cpp:166-254
//   kernels::merge_sort / quick_sort / bubble_sort / merge_runs
//                                     P/src/sort_core.cpp:23-144
// and to replay the reference tests' seeded case generators (std::mt19937_64,
// P/tests/acceptance.cpp:121-133, P/tests/test_parallel_sort.cpp:330-343) to
// produce golden fixtures. No reference source is copied here.
#include <algorithm>
#include <charconv>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <random>
#include <span>
#include <string>
#include <vector>

#include "sortbench/bench.hpp"
#include "sortbench/errors.hpp"
#include "sortbench/parallel_sort.hpp"
#include "sortbench/sort_core.hpp"

using namespace sortbench;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

runtime::WorldOptions world(int p, int k, int wall) {
    runtime::WorldOptions o;
    o.procs = p;
    o.core_slots = k;
    o.mode = wall ? runtime::Mode::wall : runtime::Mode::counted;
    return o;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_gen_data(uint64_t n, uint64_t seed, int64_t* out) {
    const DataList d = bench::gen_data(n, seed);
    std::memcpy(out, d.data(), n * sizeof(int64_t));
}

// Status: 0 ok, 2 ConfigError, 3 ProgrammingError, 1 other.
int ref_plan_partition(uint64_t n, int p, uint64_t* sizes) {
    try {
        const auto plan = parallel::plan_partition(n, p);
        for (int r = 0; r < p; ++r) sizes[r] = plan.sizes[static_cast<size_t>(r)];
        return 0;
    } catch (const ConfigError& e) {
        return fail(e, 2);
    }
}

// algo: 0 bubble, 1 merge, 2 quick. wall != 0 -> Mode::wall. Writes the sorted
// array to out and the world's wall seconds to *wall_seconds.
int ref_scatter_merge_sort(int algo, const int64_t* data, uint64_t n, int p, int k,
                           int wall, int64_t* out, double* wall_seconds) {
    try {
        DataList in(data, data + n);
        auto outcome = parallel::scatter_merge_sort(
            static_cast<parallel::Algorithm>(algo), in, world(p, k, wall));
        if (outcome.sorted.size() != n) {
            g_err = "reference returned a short array";
            return 1;
        }
        std::memcpy(out, outcome.sorted.data(), n * sizeof(int64_t));
        if (wall_seconds) *wall_seconds = outcome.world.wall_seconds;
        return 0;
    } catch (const ConfigError& e) {
        return fail(e, 2);
    } catch (const ProgrammingError& e) {
        return fail(e, 3);
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}

// The local-sort kernels through KernelFn (P/src/parallel_sort.cpp:136-164).
int ref_kernel_sort(int algo, int64_t* block, uint64_t n) {
    try {
        std::span<Element> b(block, n);
        DataList scratch(n);
        kernels::SortStats st;
        parallel::select_kernel(static_cast<parallel::Algorithm>(algo))(b, scratch, st);
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}

// kernels::merge_sort with explicit inclusive bounds (empty when first > last).
int ref_merge_sort_range(int64_t* block, uint64_t n, int64_t first, int64_t last) {
    try {
        DataList scratch(n);
        kernels::SortStats st;
        kernels::merge_sort(std::span<Element>(block, n), first, last, scratch, st);
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}

// kernels::quick_sort; out-of-range -> ProgrammingError (3).
int ref_quick_sort_range(int64_t* block, uint64_t n, uint64_t start, uint64_t length) {
    try {
        kernels::SortStats st;
        kernels::quick_sort(std::span<Element>(block, n), start, length, st);
        return 0;
    } catch (const ProgrammingError& e) {
        return fail(e, 3);
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}

void ref_merge_runs(const int64_t* a, uint64_t na, const int64_t* b, uint64_t nb,
                    int64_t* out) {
    kernels::SortStats st;
    const DataList m = kernels::merge_runs(std::span<const Element>(a, na),
                                           std::span<const Element>(b, nb), st);
    std::memcpy(out, m.data(), m.size() * sizeof(int64_t));
}

void ref_merge_split_padded(const int64_t* mine, uint64_t nm, uint64_t mine_virt,
                            const int64_t* theirs, uint64_t nt, uint64_t theirs_virt,
                            int keep_high, int64_t* out_reals, uint64_t* out_nreals,
                            uint64_t* out_virtuals) {
    parallel::PaddedBlock a{DataList(mine, mine + nm), mine_virt};
    parallel::PaddedBlock b{DataList(theirs, theirs + nt), theirs_virt};
    kernels::SortStats st;
    const auto r = parallel::merge_split_padded(
        a, b, keep_high ? parallel::KeepHalf::high : parallel::KeepHalf::low, st);
    std::memcpy(out_reals, r.reals.data(), r.reals.size() * sizeof(int64_t));
    *out_nreals = r.reals.size();
    *out_virtuals = r.virtuals;
}

// Replays the case stream of acceptance criterion 1
// (P/tests/acceptance.cpp:121-133): per case, n = rng() % 4097,
// p = {1,2,3,4,8}[rng() % 5], algo = i % 3, data seed = rng().
void ref_acceptance1_cases(int count, uint64_t* n, int* p, int* algo, uint64_t* seed) {
    std::mt19937_64 rng(20240601);
    const int pc[5] = {1, 2, 3, 4, 8};
    for (int i = 0; i < count; ++i) {
        n[i] = rng() % 4097;
        p[i] = pc[rng() % 5];
        algo[i] = i % 3;
        seed[i] = rng();
    }
}

// Replays P/tests/test_parallel_sort.cpp:330-343 (seed 5, 60 trials, n < 600).
void ref_random_oracle_cases(int count, uint64_t* n, int* p, int* algo, uint64_t* seed) {
    std::mt19937_64 rng(5);
    const int pc[5] = {1, 2, 3, 4, 8};
    for (int t = 0; t < count; ++t) {
        n[t] = rng() % 600;
        p[t] = pc[rng() % 5];
        algo[t] = t % 3;
        seed[t] = rng();
    }
}

// Replays P/tests/test_sort_core.cpp:191-216 (seed 99, 250 trials, s < 512,
// values rng() % 32): writes the inputs back to back into `values` (capacity
// >= 250*511) and the per-trial sizes into `sizes`.
void ref_kernel_oracle_cases(int count, uint64_t* sizes, int64_t* values) {
    std::mt19937_64 rng(99);
    uint64_t off = 0;
    for (int t = 0; t < count; ++t) {
        const uint64_t s = rng() % 512;
        sizes[t] = s;
        for (uint64_t i = 0; i < s; ++i) values[off++] = static_cast<int64_t>(rng() % 32);
    }
}

// std::sort (the oracle of bench::verify_output, P/src/bench.cpp:97-98).
void ref_std_sort(int64_t* v, uint64_t n) { std::sort(v, v + n); }

// std::to_chars(general) of a double: what the reference's format_double
// (P/src/bench.cpp:22-29) prints for finite values.
void ref_to_chars_general(double v, char* out64) {
    const auto r = std::to_chars(out64, out64 + 63, v, std::chars_format::general);
    *r.ptr = 0;
}

// bench::run_id (P/src/bench.cpp:30-50) of a RunConfig; out gets 16 hex chars + NUL.
void ref_run_id(int algo, uint64_t n, int procs, int cores, uint64_t seed, int wall, int reps,
                char* out17) {
    bench::RunConfig c;
    c.algorithm = static_cast<parallel::Algorithm>(algo);
    c.n = n;
    c.procs = procs;
    c.cores = cores;
    c.seed = seed;
    c.mode = wall ? runtime::Mode::wall : runtime::Mode::counted;
    c.repetitions = reps;
    const std::string id = bench::run_id(c);
    std::memcpy(out17, id.c_str(), 17);
}

// bench::run_benchmark (P/src/bench.cpp:106-169) of one configuration and its
// exports: the experiment-1 CSV row (:211-222), the trace JSONL (:335-350)
// and the trace summary (:352-395). Each output is truncated to its capacity;
// *_len receives the full length. Returns 0, or -1 (ref_last_error).
int ref_run_benchmark(int algo, uint64_t n, int procs, int cores, uint64_t seed, int wall, int reps,
                      char* csv, uint64_t csv_cap, uint64_t* csv_len, char* trace,
                      uint64_t trace_cap, uint64_t* trace_len, char* summary, uint64_t summary_cap,
                      uint64_t* summary_len) {
    try {
        bench::RunConfig c;
        c.algorithm = static_cast<parallel::Algorithm>(algo);
        c.n = n;
        c.procs = procs;
        c.cores = cores;
        c.seed = seed;
        c.mode = wall ? runtime::Mode::wall : runtime::Mode::counted;
        c.repetitions = reps;
        const bench::RunReport r = bench::run_benchmark(c);
        auto put = [](const std::string& x, char* dst, uint64_t cap, uint64_t* len) {
            *len = x.size();
            if (cap == 0) return;
            const uint64_t k = std::min<uint64_t>(cap - 1, x.size());
            std::memcpy(dst, x.data(), k);
            dst[k] = 0;
        };
        put(bench::exp1_csv_row(r), csv, csv_cap, csv_len);
        put(bench::trace_to_jsonl(r), trace, trace_cap, trace_len);
        put(bench::trace_summary_json(r), summary, summary_cap, summary_len);
        return 0;
    } catch (const std::exception& e) {
        return fail(e, -1);
    }
}

}  // extern "C"
