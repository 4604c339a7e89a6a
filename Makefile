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

build/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(PKG)/libtvstencil.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

oracle/liboracle.so: oracle/stencil_oracle.c oracle/stencil_oracle.h
	gcc -O3 -march=x86-64-v2 -fPIC -shared -ffp-contract=off -fno-fast-math -fopenmp -o $@ oracle/stencil_oracle.c

clean:
	rm -rf build $(PKG)/libtvstencil.so oracle/liboracle.so

.PHONY: all clean
