"""The reference's C++ signatures (include/sortbench_b200/sortbench.hpp) over
the C ABI: CPU checks that the shim library exports each entry point with the
reference's mangled signature; GPU runs the C++ parity program
tests/cpp/test_compat.cpp (the reference tests' KATs, seeded suites and
acceptance criterion 1 against std::sort)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "paper_1105_6040_b200", "lib", "libsortbench_b200.so")
PROG = os.path.join(ROOT, "build", "test_compat")

SIGNATURES = [
    "sortbench::kernels::bubble_sort(std::span<long, 18446744073709551615ul>, sortbench::kernels::SortStats&)",
    "sortbench::kernels::merge_sort(std::span<long, 18446744073709551615ul>, long, long, std::span<long, 18446744073709551615ul>, sortbench::kernels::SortStats&)",
    "sortbench::kernels::quick_sort(std::span<long, 18446744073709551615ul>, unsigned long, unsigned long, sortbench::kernels::SortStats&)",
    "sortbench::kernels::merge_runs(std::span<long const, 18446744073709551615ul>, std::span<long const, 18446744073709551615ul>, sortbench::kernels::SortStats&)",
    "sortbench::kernels::is_sorted(std::span<long const, 18446744073709551615ul>)",
    "sortbench::parallel::plan_partition(unsigned long, int)",
    "sortbench::parallel::build_schedule(int)",
    "sortbench::parallel::merge_split_padded(sortbench::parallel::PaddedBlock const&, sortbench::parallel::PaddedBlock const&, sortbench::parallel::KeepHalf, sortbench::kernels::SortStats&)",
    "sortbench::parallel::select_kernel(sortbench::parallel::Algorithm)",
    "sortbench::parallel::scatter_merge_sort(sortbench::parallel::Algorithm, std::vector<long, std::allocator<long> > const&, sortbench::runtime::WorldOptions const&)",
    "sortbench::bench::gen_data(unsigned long, unsigned long)",
]


def test_shim_exports_reference_signatures():
    assert os.path.exists(SHIM), "run `make`"
    out = subprocess.run(f"nm -D --defined-only {SHIM} | c++filt", shell=True,
                         capture_output=True, text=True).stdout
    for sig in SIGNATURES:
        assert sig in out, sig
    # and it reaches the GPU only through the C ABI
    deps = subprocess.run(["ldd", SHIM], capture_output=True, text=True).stdout
    assert "libb200sort.so" in deps


@pytest.mark.gpu
def test_cpp_parity_program():
    r = subprocess.run([PROG], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


@pytest.mark.gpu
def test_cpp_parity_program_with_odd_even_phases():
    """The same reference tests with scatter_merge_sort running the
    reference's own odd-even merge-split phases on the device."""
    r = subprocess.run([PROG], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, SORTBENCH_B200_PHASES="1"))
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("devices", ["0", "0,0", "0,0,0,0,0,0,0,0"])
def test_cpp_parity_program_multi_gpu_path(devices):
    """The same reference tests with scatter_merge_sort for 2 <= p <= G routed
    through the multi-GPU sample sort (b2s_sample_sort), ranks emulated on
    device 0 when the list repeats it."""
    r = subprocess.run([PROG], capture_output=True, text=True, timeout=900,
                       env=dict(os.environ, SORTBENCH_B200_DEVICES=devices))
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
