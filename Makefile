# Build: libgesr.so (CUDA, sm_100a) and liboracle.so (plain C++, the test oracle).
NVCC      ?= /usr/local/cuda/bin/nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC -Iinclude
PKG       := paper_2511_21095_b200
SRC       := $(PKG)/csrc
BUILD     := build
OBJS      := $(BUILD)/proj.o $(BUILD)/attn.o $(BUILD)/attn2.o $(BUILD)/hma.o $(BUILD)/stu.o $(BUILD)/nro.o $(BUILD)/debug.o $(BUILD)/hostpath.o $(BUILD)/capi.o
HDRS      := $(SRC)/kernels.h $(SRC)/ptx.cuh include/gesr.h

all: $(PKG)/libgesr.so oracle/liboracle.so

$(BUILD):
	mkdir -p $(BUILD)

$(BUILD)/%.o: $(SRC)/%.cu $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(BUILD)/$*.ptxas.txt || (cat $(BUILD)/$*.ptxas.txt; false)

$(BUILD)/capi.o: $(SRC)/capi.cpp $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@

$(PKG)/libgesr.so: $(OBJS) $(SRC)/exports.map
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS) -Xlinker --version-script=$(SRC)/exports.map

oracle/liboracle.so: oracle/oracle.cpp
	g++ -O2 -std=c++17 -fPIC -shared -pthread -o $@ $<

clean:
	rm -rf $(BUILD) $(PKG)/libgesr.so oracle/liboracle.so

.PHONY: all clean
