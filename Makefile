# Builds every native artefact in-tree (the .so files travel to the GPU box with gpurun).
#   paper_2308_13289_b200/liblob.so   CUDA engine behind include/lob.h (sm_100a only)
#   oracle/liblob_oracle.so           CPU oracle (test infrastructure)
#   lobgen/liblobgen.so               seeded input generator
#   paper_2308_13289_b200/liblobster.so  LOBSTER ingestion (NEXT row N4)
NVCC      ?= /usr/local/cuda/bin/nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xptxas -v -Xcompiler -fPIC,-O2 -shared
PKG       := paper_2308_13289_b200
LIB       := $(PKG)/liblob.so
SRCS      := $(PKG)/csrc/lob_api.cu
DEPS      := $(SRCS) $(PKG)/csrc/lob_kernels.cuh $(PKG)/csrc/lob_env.cuh $(PKG)/csrc/lob_session.cuh $(PKG)/csrc/lob_split.cuh include/lob.h
# provenance: hash of the engine sources + this Makefile (flags), exported by lob_build_id()
BUILD_ID  := $(shell cat $(DEPS) Makefile | sha256sum | cut -c1-16)

all: $(LIB) $(PKG)/liblobster.so oracle/liblob_oracle.so lobgen/liblobgen.so

$(LIB): $(DEPS) Makefile
	$(NVCC) $(NVFLAGS) -DLOB_BUILD_ID='"$(BUILD_ID)"' -o $@.tmp $(SRCS) 2> $(PKG)/ptxas.log || (cat $(PKG)/ptxas.log; exit 1)
	mv $@.tmp $@
	@grep -E "Compiling entry|registers|spill" $(PKG)/ptxas.log | grep -B1 -E "spill stores [1-9]|bytes spill" || true

$(PKG)/liblobster.so: $(PKG)/csrc/lobster_io.c
	gcc -O2 -std=c11 -Wall -shared -fPIC -o $@ $<

oracle/liblob_oracle.so: oracle/lob_oracle.c
	gcc -O2 -std=c11 -Wall -shared -fPIC -o $@ $< -lm

lobgen/liblobgen.so: lobgen/lobgen.c
	gcc -O2 -std=c11 -Wall -shared -fPIC -pthread -o $@ $<

sass: $(LIB)
	/usr/local/cuda/bin/cuobjdump -sass $(LIB) > $(PKG)/liblob.sass

clean:
	rm -f $(LIB) $(PKG)/liblobster.so oracle/liblob_oracle.so lobgen/liblobgen.so $(PKG)/ptxas.log $(PKG)/liblob.sass

.PHONY: all clean sass
