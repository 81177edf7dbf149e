# Builds the B200 library (sm_100a) and the CPU oracle (test infrastructure).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr
SRC := $(wildcard paper_2411_06360_b200/csrc/*.cu)
HDR := $(wildcard paper_2411_06360_b200/csrc/*.cuh) $(wildcard paper_2411_06360_b200/csrc/*.h) include/rsr_b200.h
LIB := paper_2411_06360_b200/lib/librsr_b200.so
OBJDIR := build/obj
OBJ := $(patsubst paper_2411_06360_b200/csrc/%.cu,$(OBJDIR)/%.o,$(SRC))
# host-only C++ (session staging): AVX2 baseline like the oracle (x86-64-v3 runs on the GPU box)
CXXSRC := $(wildcard paper_2411_06360_b200/csrc/*.cpp)
CXXOBJ := $(patsubst paper_2411_06360_b200/csrc/%.cpp,$(OBJDIR)/%.cpp.o,$(CXXSRC))
CXXFLAGS_HOST := -O3 -march=x86-64-v3 -fPIC -std=c++17 -Wall -Wextra

PYINC := $(shell python3 -c "import sysconfig; print(sysconfig.get_paths()['include'])")
PYEXT := paper_2411_06360_b200/lib/_rsrhost$(shell python3 -c "import sysconfig; print(sysconfig.get_config_var('EXT_SUFFIX'))")

COUNT_LIB := paper_2411_06360_b200/lib/count/librsr_b200_count.so

all: $(LIB) $(PYEXT) $(COUNT_LIB) oracle

# CPython binding of the host-buffer session (links the library through $ORIGIN)
$(PYEXT): paper_2411_06360_b200/csrc/pyhost.c include/rsr_b200.h $(LIB)
	gcc -O2 -fPIC -shared -Wall -Iinclude -I$(PYINC) $< -o $@ -Lpaper_2411_06360_b200/lib -lrsr_b200 -Wl,-rpath,'$$ORIGIN'

$(OBJDIR)/%.o: paper_2411_06360_b200/csrc/%.cu $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(OBJDIR)/$*.ptxas.log || (cat $(OBJDIR)/$*.ptxas.log; exit 1)

$(OBJDIR)/%.cpp.o: paper_2411_06360_b200/csrc/%.cpp $(HDR) $(wildcard paper_2411_06360_b200/csrc/*.h)
	@mkdir -p $(OBJDIR)
	g++ $(CXXFLAGS_HOST) -c $< -o $@

$(LIB): $(OBJ) $(CXXOBJ)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -Xlinker -soname=librsr_b200.so -o $@ $(OBJ) $(CXXOBJ) -lcudart

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf build $(LIB) $(PYEXT) $(COUNT_LIB)
	$(MAKE) -s -C oracle clean

# diagnostic build with per-unit timestamps (tools/trace_scatter.py); not used by the product
TRACE_LIB := paper_2411_06360_b200/lib/trace/librsr_b200_trace.so
trace: $(SRC) $(HDR) $(CXXOBJ)
	@mkdir -p $(dir $(TRACE_LIB))
	$(NVCC) $(NVFLAGS) -DRSR_TRACE -shared -o $(TRACE_LIB) $(SRC) $(CXXOBJ) -lcudart

# work-count build: the scatter kernel counts the accumulate steps it executes
# (rsr_debug_count_copy); used by tests/test_counted_gpu.py, never by the product
$(OBJDIR)/multiply_count.o: paper_2411_06360_b200/csrc/multiply.cu $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -DRSR_COUNT -c $< -o $@
$(COUNT_LIB): $(filter-out $(OBJDIR)/multiply.o,$(OBJ)) $(OBJDIR)/multiply_count.o $(CXXOBJ)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -Xlinker -soname=librsr_b200_count.so -o $@ $^ -lcudart
count: $(COUNT_LIB)

.PHONY: all oracle clean trace count
