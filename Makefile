# Builds the sm_100a library in-tree (it travels to the GPU box with the
# snapshot) and the C oracle used by the tests.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -fmad=false -ftz=false -prec-div=true -prec-sqrt=true \
           -Xcompiler -fPIC -Xptxas -v
PKG := paper_1608_03984_b200
LIB := $(PKG)/libb200fd.so
SRCS := $(wildcard $(PKG)/csrc/*.cu)
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/b200fd.h

all: $(LIB) oracle

$(LIB): $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRCS) 2> build/ptxas.log || (cat build/ptxas.log; false)

oracle:
	$(MAKE) -C oracle

clean:
	rm -f $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
