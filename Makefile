# Builds the sm_100a library in-tree (it travels to the GPU box with the
# snapshot) and the C oracle used by the tests.  One object per source so
# `make -j` compiles the kernels in parallel.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -fmad=false -ftz=false -prec-div=true -prec-sqrt=true \
           -Xcompiler -fPIC -Xptxas -v
PKG := paper_1608_03984_b200
LIB := $(PKG)/libb200fd.so
SRCS := $(wildcard $(PKG)/csrc/*.cu)
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/b200fd.h
OBJS := $(patsubst $(PKG)/csrc/%.cu,build/obj/%.o,$(SRCS))

all: $(LIB) oracle

build/obj/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> build/obj/$*.ptxas.log || (cat build/obj/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)
	@cat build/obj/*.ptxas.log > build/ptxas.log

oracle:
	$(MAKE) -C oracle

clean:
	rm -f $(LIB) build/obj/*.o build/obj/*.log
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
