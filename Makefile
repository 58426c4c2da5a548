# Build the product library (host C++ + sm_100a CUDA, one .so behind the C-ABI)
# and the test oracles. `make` is what __graft_entry__.build() runs.
CUDA     ?= /usr/local/cuda
NVCC     ?= $(CUDA)/bin/nvcc
CXX      ?= g++
ARCH     := -gencode arch=compute_100a,code=sm_100a
PKG      := paper_2308_14129_b200
SRC      := $(PKG)/csrc
OBJ      := build/obj
INC      := -Iinclude -I$(SRC) -I$(CUDA)/include
CXXFLAGS := -O3 -std=c++20 -fPIC -ffp-contract=off -Wall -Wextra -Wno-unused-parameter $(INC)
NVFLAGS  := $(ARCH) -O3 -std=c++20 -lineinfo -Xcompiler -fPIC -Xcompiler -ffp-contract=off \
            --expt-relaxed-constexpr -Xptxas -v $(INC)
LIB      := $(PKG)/libspeed_b200.so

CPP_SRCS := $(wildcard $(SRC)/*.cpp)
CU_SRCS  := $(wildcard $(SRC)/*.cu)
OBJS     := $(patsubst $(SRC)/%.cpp,$(OBJ)/%.o,$(CPP_SRCS)) $(patsubst $(SRC)/%.cu,$(OBJ)/%.cu.o,$(CU_SRCS))
HDRS     := $(wildcard $(SRC)/*.hpp) $(wildcard $(SRC)/*.cuh) include/speed_c.h

all: $(LIB) oracle

$(OBJ)/%.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJ)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OBJ)/%.cu.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJ)/$*.ptxas.txt || (cat $(OBJ)/$*.ptxas.txt; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -cudart static -ldl -lpthread

oracle:
	$(MAKE) -C oracle all

clean:
	rm -rf build $(LIB)

.PHONY: all oracle clean
