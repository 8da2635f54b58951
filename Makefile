# Build every native artefact in-tree (the .so files travel to the GPU box).
#   gen/libpfacgen.so                 seeded input generators (inputs only)
#   oracle/liboracle.so               CPU oracle (test infrastructure only)
#   paper_1702_03657_b200/libpfac.so  the product: host builder + sm_100a kernels + C ABI
NVCC    ?= /usr/local/cuda/bin/nvcc
CC      ?= gcc
CFLAGS  := -O2 -g -fPIC -Wall -Wextra -std=gnu11
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -lineinfo -std=c++17 $(ARCH) -Xcompiler -fPIC,-Wall -Iinclude --expt-relaxed-constexpr
PKG     := paper_1702_03657_b200
CSRC    := $(wildcard $(PKG)/csrc/*.cu) $(wildcard $(PKG)/csrc/*.cpp)
CHDR    := $(wildcard $(PKG)/csrc/*.h) $(wildcard $(PKG)/csrc/*.cuh) include/pfac.h

all: gen/libpfacgen.so oracle/liboracle.so $(PKG)/libpfac.so tools/probe/libkb0.so

gen/libpfacgen.so: gen/pfac_gen.c gen/pfac_gen.h
	$(CC) $(CFLAGS) -shared -o $@ gen/pfac_gen.c -lm -lpthread

oracle/liboracle.so: oracle/oracle.c oracle/oracle.h
	$(CC) $(CFLAGS) -shared -o $@ oracle/oracle.c -lpthread

$(PKG)/libpfac.so: $(CSRC) $(CHDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(CSRC) -lcudart

# instrumented build for tools/timing.py (not used by tests or bench)
$(PKG)/libpfac_timing.so: $(CSRC) $(CHDR)
	$(NVCC) $(NVFLAGS) -DPFAC_TIMING -shared -o $@ $(CSRC) -lcudart

$(PKG)/libpfac_stream.so: $(CSRC) $(CHDR)
	$(NVCC) $(NVFLAGS) -DPFAC_TIMING -DPFAC_STREAM_ONLY -shared -o $@ $(CSRC) -lcudart

$(PKG)/libpfac_exp1.so: $(CSRC) $(CHDR)
	$(NVCC) $(NVFLAGS) -DPFAC_TIMING -DPFAC_EXP=1 -shared -o $@ $(CSRC) -lcudart

$(PKG)/libpfac_exp2.so: $(CSRC) $(CHDR)
	$(NVCC) $(NVFLAGS) -DPFAC_TIMING -DPFAC_EXP=2 -shared -o $@ $(CSRC) -lcudart

# bounds-checked build (device-side index asserts; tools/checked_tests.sh)
$(PKG)/libpfac_checked.so: $(CSRC) $(CHDR)
	$(NVCC) $(NVFLAGS) -DPFAC_CHECKED -shared -o $@ $(CSRC) -lcudart
checked: $(PKG)/libpfac_checked.so

# experiment / instrumented builds (tools/timing.py; never used by tests or bench)
EXPLIBS := $(PKG)/libpfac_timing.so $(PKG)/libpfac_stream.so $(PKG)/libpfac_exp1.so $(PKG)/libpfac_exp2.so
exp: $(EXPLIBS)

clean:
	rm -f gen/libpfacgen.so oracle/liboracle.so $(PKG)/libpfac.so $(EXPLIBS)

.PHONY: all clean

# KB0 read-stream probe (bench.py reports its bandwidth next to the scan)
tools/probe/libkb0.so: tools/probe/kb0.cu
	$(NVCC) $(NVFLAGS) -shared -o $@ $< -lcudart
# latency / launch-overhead probes (tools/probe; measurement only)
probes: tools/probe/lat_probe tools/probe/launch_probe
tools/probe/lat_probe: tools/probe/lat_probe.cu
	$(NVCC) -O2 $(ARCH) -o $@ $<
tools/probe/launch_probe: tools/probe/launch_probe.cu
	$(NVCC) -O2 $(ARCH) -o $@ $<
