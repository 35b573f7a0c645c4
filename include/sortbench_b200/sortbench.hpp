// sortbench.hpp -- the reference's hot-path entry points with their C++
// signatures, implemented on the B200 C ABI (include/b200sort.h).
//
// A program written against the reference's sortbench library
// (/root/reference/proj/include/sortbench/{element,errors,sort_core,
// parallel_sort}.hpp) keeps its calls and switches the include to this header
// and the link to libsortbench_b200.so. Every sort and merge below runs as CUDA
// kernels on the GPU; there is no CPU path. Declarations cite the reference
// line each one stands in for.
#pragma once

#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace sortbench {

// P/include/sortbench/element.hpp:10-14
using Element = std::int64_t;
inline constexpr std::size_t kElementBytes = sizeof(Element);
using DataList = std::vector<Element>;

// P/include/sortbench/errors.hpp:10-46 (the subset the hot path raises)
class ConfigError : public std::runtime_error {
public:
    explicit ConfigError(const std::string& what) : std::runtime_error(what) {}
};
class ProgrammingError : public std::logic_error {
public:
    explicit ProgrammingError(const std::string& what) : std::logic_error(what) {}
};
class VerificationError : public std::runtime_error {
public:
    explicit VerificationError(const std::string& what) : std::runtime_error(what) {}
};

namespace kernels {

// P/include/sortbench/sort_core.hpp:13-26. A radix sort makes no comparisons
// or swaps; `moves` counts key reads+writes (2 per key per executed pass).
struct SortStats {
    std::uint64_t comparisons = 0;
    std::uint64_t swaps = 0;
    std::uint64_t moves = 0;
    std::uint64_t max_depth = 0;
    SortStats& operator+=(const SortStats& o) {
        comparisons += o.comparisons;
        swaps += o.swaps;
        moves += o.moves;
        if (o.max_depth > max_depth) max_depth = o.max_depth;
        return *this;
    }
};

void bubble_sort(std::span<Element> block, SortStats& stats);                   // :35
DataList merge_runs(std::span<const Element> run_a, std::span<const Element> run_b,
                    SortStats& stats);                                            // :39-40
void merge_sort(std::span<Element> block, std::ptrdiff_t first, std::ptrdiff_t last,
                std::span<Element> scratch, SortStats& stats);                    // :46-48
void quick_sort(std::span<Element> block, std::size_t start, std::size_t length,
                SortStats& stats);                                                // :53-54
bool is_sorted(std::span<const Element> seq);                                     // :57

}  // namespace kernels

namespace runtime {

enum class Mode { wall, counted };

// P/include/sortbench/runtime.hpp:60-66. On one GPU `procs` is the number of
// partitions; core_slots / mode / weights emulate the paper's CPU cores and
// MPI message costs and have no GPU meaning.
struct WorldOptions {
    int procs = 1;
    int core_slots = 1;
    Mode mode = Mode::counted;
    std::uint64_t latency_weight = 1000;
    std::uint64_t bandwidth_weight = 1;
};

// P/include/sortbench/runtime.hpp:70-86 (the fields the hot path fills)
struct WorldReport {
    WorldOptions options;
    double wall_seconds = 0.0;  // host wall time of the call
    double device_ms = 0.0;     // CUDA-event time of the device work
};

}  // namespace runtime

namespace parallel {

enum class Algorithm { bubble, merge, quick };                                    // :14
const char* to_string(Algorithm algorithm);
Algorithm algorithm_from_string(const std::string& name);

struct PartitionPlan {                                                            // :20-24
    std::size_t n = 0;
    int procs = 1;
    std::vector<std::size_t> sizes;
};
PartitionPlan plan_partition(std::size_t n, int p);                               // :26

struct PhaseSchedule {                                                            // :30-39
    int procs = 1;
    std::vector<std::vector<int>> partners;
    int phases() const { return static_cast<int>(partners.size()); }
    int partner(int phase, int rank) const {
        return partners[static_cast<std::size_t>(phase)][static_cast<std::size_t>(rank)];
    }
};
PhaseSchedule build_schedule(int p);                                              // :41

enum class KeepHalf { low, high };                                                // :43
DataList merge_split(std::span<const Element> mine, std::span<const Element> theirs,
                     KeepHalf keep, kernels::SortStats& stats);                   // :48-50

struct PaddedBlock {                                                              // :56-61
    DataList reals;
    std::size_t virtuals = 0;
    std::size_t width() const { return reals.size() + virtuals; }
};
PaddedBlock merge_split_padded(const PaddedBlock& mine, const PaddedBlock& theirs,
                               KeepHalf keep, kernels::SortStats& stats);         // :63-65

using KernelFn = void (*)(std::span<Element> block, std::span<Element> scratch,
                          kernels::SortStats& stats);                             // :69-70
KernelFn select_kernel(Algorithm algorithm);                                      // :72

struct SortOutcome {                                                              // :74-79
    DataList sorted;
    runtime::WorldReport world;
    std::vector<kernels::SortStats> local_sort_stats;
};
SortOutcome scatter_merge_sort(Algorithm algorithm, const DataList& data,
                               const runtime::WorldOptions& options);             // :83-84

}  // namespace parallel

namespace bench {

// P/src/bench.cpp:57-71, generated on the GPU (bit-identical).
DataList gen_data(std::size_t n, std::uint64_t seed);

}  // namespace bench

}  // namespace sortbench
