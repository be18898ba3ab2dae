# Builds the product library (CUDA sm_100a + C-ABI), the input generators and
# the CPU checkers (oracle/).  `make` is what __graft_entry__.build() runs.
NVCC ?= /usr/local/cuda/bin/nvcc
CXX ?= g++
ARCH := -gencode arch=compute_100a,code=sm_100a
PKG := paper_2207_13848_b200
SRC := $(PKG)/csrc
OUT := $(PKG)/_lib
BUILD := build
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -fmad=false -Xptxas -warn-spills \
           -Xcompiler -fPIC,-ffp-contract=off,-Wall -Iinclude -I$(SRC)

CU_SRCS := $(SRC)/flop.cu $(SRC)/sample_predict.cu $(SRC)/symbolic.cu $(SRC)/heavy.cu
CPP_SRCS := $(SRC)/capi.cpp
OBJS := $(patsubst $(SRC)/%.cu,$(BUILD)/%.o,$(CU_SRCS)) $(patsubst $(SRC)/%.cpp,$(BUILD)/%.o,$(CPP_SRCS))
HDRS := $(SRC)/kernels.h $(SRC)/device_common.cuh $(SRC)/symbolic_common.cuh include/spnnz_gpu/capi.h

all: $(OUT)/libspnnz_gpu.so $(OUT)/libspnnz_gen.so $(BUILD)/test_dropin $(BUILD)/spnnz_corpus oracle dropin_ref

$(BUILD)/%.o: $(SRC)/%.cu $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(BUILD)/%.o: $(SRC)/%.cpp $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(OUT)/libspnnz_gpu.so: $(OBJS) | $(OUT)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -ldl

$(OUT)/libspnnz_gen.so: $(SRC)/gen/generators.cpp $(SRC)/gen/mmio.cpp | $(OUT)
	$(CXX) -std=c++20 -O3 -fPIC -shared -pthread -Wall -Wl,--exclude-libs,ALL -o $@ $(SRC)/gen/generators.cpp $(SRC)/gen/mmio.cpp

# corpus harness: include/spnnz_gpu/harness.hpp
$(BUILD)/spnnz_corpus: tools/spnnz_corpus.cpp include/spnnz_gpu/harness.hpp include/spnnz_gpu/spnnz_gpu.hpp include/spnnz_gpu/host.h $(OUT)/libspnnz_gpu.so $(OUT)/libspnnz_gen.so | $(BUILD)
	$(CXX) -std=c++20 -O2 -Wall -Iinclude -o $@ $< -L$(OUT) -lspnnz_gpu -lspnnz_gen -Wl,-rpath,'$$ORIGIN/../$(OUT)'

# C++ drop-in test (runs on a GPU box: tests/test_gpu_parity.py)
$(BUILD)/test_dropin: tests/cpp/test_dropin.cpp include/spnnz_gpu/spnnz_gpu.hpp $(OUT)/libspnnz_gpu.so | $(BUILD)
	$(CXX) -std=c++20 -O2 -Wall -Iinclude -o $@ $< -L$(OUT) -lspnnz_gpu -Wl,-rpath,'$$ORIGIN/../$(OUT)'

# C++ drop-in with the reference's own types (test infrastructure: built only
# where the reference headers exist, like oracle/_ref; run on a GPU box)
REF_INC ?= /root/reference/proj/include
dropin_ref: $(OUT)/libspnnz_gpu.so
	@if [ -d "$(REF_INC)/spnnz" ]; then \
	  $(MAKE) --no-print-directory $(BUILD)/test_dropin_ref; \
	else echo "reference headers absent: skipping build/test_dropin_ref"; fi

$(BUILD)/test_dropin_ref: tests/cpp/test_dropin_ref.cpp include/spnnz_gpu/spnnz_gpu.hpp $(OUT)/libspnnz_gpu.so | $(BUILD)
	$(CXX) -std=c++20 -O2 -Wall -ffp-contract=off -I$(REF_INC) -Iinclude -o $@ $< -L$(OUT) -lspnnz_gpu -pthread -Wl,-rpath,'$$ORIGIN/../$(OUT)'

oracle:
	$(MAKE) --no-print-directory -C oracle

$(BUILD) $(OUT):
	mkdir -p $@

clean:
	rm -rf $(BUILD) $(OUT)/*.so
	$(MAKE) -C oracle clean

.PHONY: all oracle clean dropin_ref
