# Build of the B200-native GMRES-SDR library (sm_100a) and the CPU oracle.
#   make            -> paper_2311_14206_b200/_lib/libsdr_b200.so + oracle/_build/liboracle.so
PY ?= python
NVCC ?= /usr/local/cuda/bin/nvcc
CXX ?= g++
LAPACK_DIR ?= $(shell $(PY) -c "import os,scipy;print(os.path.join(os.path.dirname(os.path.dirname(scipy.__file__)),'scipy.libs'))")
LAPACK_LIB ?= $(notdir $(firstword $(wildcard $(LAPACK_DIR)/libscipy_openblas-*.so)))

SRC := paper_2311_14206_b200/csrc
OBJ := build/obj
LIB := paper_2311_14206_b200/_lib/libsdr_b200.so
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -I/usr/local/cuda/include
CXXFLAGS := -O3 -std=c++17 -fPIC -fvisibility=hidden -Wall -Wextra -Wno-unused-parameter -I/usr/local/cuda/include

CU := spmv arnoldi sketch sparse_update fused_step tsmm wide operator baseline peer
CC := context host_linalg space solver baseline_host io capi
OBJS := $(addprefix $(OBJ)/,$(addsuffix .cu.o,$(CU)) $(addsuffix .o,$(CC)))
HDRS := $(wildcard $(SRC)/*.hpp $(SRC)/*.cuh) include/sdr_b200.h

all: $(LIB) oracle

$(OBJ)/%.cu.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJ)/%.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJ)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS) -L$(LAPACK_DIR) -l:$(LAPACK_LIB) -Xlinker -rpath=$(LAPACK_DIR) -L/usr/local/cuda/lib64 -lcublas -Xlinker -rpath=/usr/local/cuda/lib64 -ldl -lpthread -Xlinker --no-undefined

oracle:
	$(MAKE) -s -C oracle PY=$(PY)

clean:
	rm -rf build $(LIB) oracle/_build

.PHONY: all oracle clean

# a plain C++ caller of the C-ABI (no Python): make examples && ./examples/solve_c2
examples: examples/solve_c2

examples/solve_c2: examples/solve_c2.cpp include/sdr_b200.h $(LIB)
	$(CXX) -O2 -std=c++17 -Iinclude -o $@ $< -L$(dir $(LIB)) -lsdr_b200 -Wl,-rpath,'$$ORIGIN/../paper_2311_14206_b200/_lib'

.PHONY: examples
