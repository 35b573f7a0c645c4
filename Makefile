# Builds the B200 sort library (sm_100a only) and the test oracles.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall \
           -Iinclude -Ipaper_1105_6040_b200/csrc --expt-relaxed-constexpr
SRC := paper_1105_6040_b200/csrc
LIB := paper_1105_6040_b200/lib
OBJ := build/obj
CU := abi radix_sort merge_path sample_sort gen_verify multi
OBJS := $(addprefix $(OBJ)/,$(addsuffix .o,$(CU)))
HDRS := include/b200sort.h $(SRC)/b2s_internal.cuh

all: $(LIB)/libb200sort.so $(LIB)/libsortbench_b200.so build/test_compat

$(OBJ)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(OBJ)/$*.ptxas.txt || (cat $(OBJ)/$*.ptxas.txt; exit 1)

$(LIB)/libb200sort.so: $(OBJS)
	@mkdir -p $(LIB)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart -ldl

# the reference's C++ signatures on top of the C ABI
$(LIB)/libsortbench_b200.so: $(SRC)/compat/sortbench_compat.cpp include/sortbench_b200/sortbench.hpp $(LIB)/libb200sort.so
	g++ -std=c++20 -O2 -fPIC -shared -Wall -Wextra -Iinclude $< -L$(LIB) -lb200sort \
	    -Wl,-rpath,'$$ORIGIN' -o $@

build/test_compat: tests/cpp/test_compat.cpp $(LIB)/libsortbench_b200.so
	@mkdir -p build
	g++ -std=c++20 -O2 -Wall -Wextra -Iinclude $< -L$(LIB) -lsortbench_b200 -lb200sort \
	    -Wl,-rpath,'$$ORIGIN/../$(LIB)' -o $@

# phase-profiling variant (clock64 per onesweep phase; tools/phase_prof.py)
prof: $(LIB)/libb200sort_prof.so

$(LIB)/libb200sort_prof.so: $(SRC)/*.cu $(HDRS)
	@mkdir -p $(LIB) build/prof
	for f in $(CU); do $(NVCC) $(NVFLAGS) -DB2S_PHASE_PROFILE -c $(SRC)/$$f.cu -o build/prof/$$f.o || exit 1; done
	$(NVCC) $(ARCH) -shared -o $@ $(addprefix build/prof/,$(addsuffix .o,$(CU))) -lcudart

# one experimental build of one source: make variant NAME=x DEFS="-DFOO=1" [VSRC=merge_path]
# -> lib/libb200sort_x.so (select with B2S_LIB)
VSRC ?= radix_sort
variant: $(OBJS)
	@mkdir -p build/v_$(NAME)
	$(NVCC) $(NVFLAGS) $(DEFS) -Xptxas -v -c $(SRC)/$(VSRC).cu -o build/v_$(NAME)/$(VSRC).o 2> build/v_$(NAME)/ptxas.txt || (cat build/v_$(NAME)/ptxas.txt; exit 1)
	$(NVCC) $(ARCH) -shared -o $(LIB)/libb200sort_$(NAME).so build/v_$(NAME)/$(VSRC).o $(filter-out $(OBJ)/$(VSRC).o,$(OBJS)) -lcudart

# comparison / ceiling probes (tools/cub_compare.cu, tools/read_probe.cu)
tools: build/cub_compare build/read_probe

build/cub_compare: tools/cub_compare.cu
	@mkdir -p build
	$(NVCC) $(ARCH) -O3 -std=c++17 $< -o $@

build/read_probe: tools/read_probe.cu
	@mkdir -p build
	$(NVCC) $(ARCH) -O3 $< -o $@

oracle:
	bash oracle/build_ref.sh

clean:
	rm -rf build $(LIB)

.PHONY: all oracle clean tools prof
