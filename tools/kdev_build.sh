#!/bin/bash
# Development build of radix_sort.cu with extra -D switches, linked with the
# other prebuilt objects:
#   bash tools/kdev_build.sh NAME "-DFOO=1"  ->  paper_1105_6040_b200/lib/libb200sort_NAME.so
set -e
cd "$(dirname "$0")/.."
name=$1
defs=$2
mkdir -p build/dev_$name
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -Iinclude -Ipaper_1105_6040_b200/csrc --expt-relaxed-constexpr -diag-suppress 177 $defs \
    -Xptxas -v -c paper_1105_6040_b200/csrc/radix_sort.cu -o build/dev_$name/radix_sort.o 2> build/dev_$name/ptxas.txt \
    || (cat build/dev_$name/ptxas.txt; exit 1)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_1105_6040_b200/lib/libb200sort_$name.so \
    build/dev_$name/radix_sort.o build/obj/abi.o build/obj/merge_path.o build/obj/sample_sort.o build/obj/gen_verify.o build/obj/multi.o -lcudart -ldl
grep -A2 "onesweep_kernelIjLb0EjLi512ELi2[134]ELi2ELi[234]EE\|onesweep_pipe" build/dev_$name/ptxas.txt | grep -o "[0-9]* bytes spill stores\|Used [0-9]* registers" | paste -sd' ' -
