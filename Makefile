# Builds the B200 library (sm_100a) and the CPU oracle (test infrastructure).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr
SRC := $(wildcard paper_2411_06360_b200/csrc/*.cu)
HDR := $(wildcard paper_2411_06360_b200/csrc/*.cuh) include/rsr_b200.h
LIB := paper_2411_06360_b200/lib/librsr_b200.so
OBJDIR := build/obj
OBJ := $(patsubst paper_2411_06360_b200/csrc/%.cu,$(OBJDIR)/%.o,$(SRC))

PYINC := $(shell python3 -c "import sysconfig; print(sysconfig.get_paths()['include'])")
PYEXT := paper_2411_06360_b200/lib/_rsrhost$(shell python3 -c "import sysconfig; print(sysconfig.get_config_var('EXT_SUFFIX'))")

all: $(LIB) $(PYEXT) oracle

# CPython binding of the host-buffer session (links the library through $ORIGIN)
$(PYEXT): paper_2411_06360_b200/csrc/pyhost.c include/rsr_b200.h $(LIB)
	gcc -O2 -fPIC -shared -Wall -Iinclude -I$(PYINC) $< -o $@ -Lpaper_2411_06360_b200/lib -lrsr_b200 -Wl,-rpath,'$$ORIGIN'

$(OBJDIR)/%.o: paper_2411_06360_b200/csrc/%.cu $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(OBJDIR)/$*.ptxas.log || (cat $(OBJDIR)/$*.ptxas.log; exit 1)

$(LIB): $(OBJ)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -Xlinker -soname=librsr_b200.so -o $@ $(OBJ) -lcudart

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf build $(LIB) $(PYEXT)
	$(MAKE) -s -C oracle clean

# diagnostic build with per-unit timestamps (tools/trace_scatter.py); not used by the product
TRACE_LIB := paper_2411_06360_b200/lib/trace/librsr_b200_trace.so
trace: $(SRC) $(HDR)
	@mkdir -p $(dir $(TRACE_LIB))
	$(NVCC) $(NVFLAGS) -DRSR_TRACE -shared -o $(TRACE_LIB) $(SRC) -lcudart

.PHONY: all oracle clean trace
