# Builds the sm_100a kernel library and the CPU oracle.
#   make -j8            -> paper_2010_04868_b200/libtvstencil.so, oracle/liboracle.so
NVCC    ?= nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -Xptxas -warn-spills
PKG     := paper_2010_04868_b200
SRCS    := $(wildcard $(PKG)/csrc/*.cu)
OBJS    := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRCS))
HDRS    := $(wildcard $(PKG)/csrc/*.cuh) include/tvstencil.h

all: $(PKG)/libtvstencil.so oracle/liboracle.so

# register spills fail the build (ptxas -warn-spills output is checked)
build/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)
	@cat build/$*.ptxas.log
	@if grep -q "Registers are spilled" build/$*.ptxas.log; then echo "error: register spills in $<"; rm -f $@; exit 1; fi

$(PKG)/libtvstencil.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

oracle/liboracle.so: oracle/stencil_oracle.c oracle/stencil_oracle.h
	gcc -O3 -march=x86-64-v2 -fPIC -shared -ffp-contract=off -fno-fast-math -fopenmp -o $@ oracle/stencil_oracle.c

clean:
	rm -rf build $(PKG)/libtvstencil.so oracle/liboracle.so

.PHONY: all clean
