# Build the B200-native library in-tree (the .so travels to the GPU box with
# the gpurun snapshot).  sm_100a only.
CUDA ?= /usr/local/cuda
NVCC := $(CUDA)/bin/nvcc
PKG := paper_2605_21226_b200
SRC := $(PKG)/csrc
OBJ := build/obj
LIB := $(PKG)/liboctoquant_b200.so

ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
# Host code: codebook construction must round exactly like the reference's
# scalar C++ (no FMA contraction, no fast math).
CXXFLAGS := -O2 -std=c++17 -fPIC -ffp-contract=off -fno-fast-math -I$(CUDA)/include -pthread

CU_SRCS := $(wildcard $(SRC)/*.cu)
CPP_SRCS := $(wildcard $(SRC)/*.cpp)
CU_OBJS := $(patsubst $(SRC)/%.cu,$(OBJ)/%.cu.o,$(CU_SRCS))
CPP_OBJS := $(patsubst $(SRC)/%.cpp,$(OBJ)/%.cpp.o,$(CPP_SRCS))
HDRS := $(wildcard $(SRC)/*.h $(SRC)/*.cuh $(SRC)/*.hpp) include/octoquant_b200.h

all: $(LIB) oracle

$(OBJ)/%.cu.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; false)
	@grep -E "registers|spill" $@.ptxas.log | sed 's/^/  /' | head -40

$(OBJ)/%.cpp.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJ)
	g++ $(CXXFLAGS) -c $< -o $@

$(LIB): $(CU_OBJS) $(CPP_OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $^ -Xcompiler -pthread

oracle:
	$(MAKE) --no-print-directory -C oracle

clean:
	rm -rf build $(LIB)

.PHONY: all oracle clean
