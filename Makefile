# Builds libprefillonly.so (sm_100a) in-tree so it travels to the GPU box with the snapshot.
NVCC ?= /usr/local/cuda/bin/nvcc
SRC_DIR := paper_2505_07203_b200/csrc
OUT := paper_2505_07203_b200/libprefillonly.so
OBJ_DIR := build/obj
CU_SRCS := $(wildcard $(SRC_DIR)/*.cu)
CPP_SRCS := $(wildcard $(SRC_DIR)/*.cpp)
OBJS := $(patsubst $(SRC_DIR)/%.cu,$(OBJ_DIR)/%.o,$(CU_SRCS)) $(patsubst $(SRC_DIR)/%.cpp,$(OBJ_DIR)/%.o,$(CPP_SRCS))
HDRS := $(wildcard $(SRC_DIR)/*.cuh) $(wildcard $(SRC_DIR)/*.h) include/prefillonly.h
NVFLAGS := -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 \
           --expt-relaxed-constexpr -Iinclude -Xptxas -v
CXXFLAGS := -O3 -fPIC -std=c++17 -Iinclude -I/usr/local/cuda/include -Wall

all: $(OUT)

$(OBJ_DIR)/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(OBJ_DIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJ_DIR)/$*.ptxas.txt || (cat $(OBJ_DIR)/$*.ptxas.txt; exit 1)

$(OBJ_DIR)/%.o: $(SRC_DIR)/%.cpp $(HDRS)
	@mkdir -p $(OBJ_DIR)
	g++ $(CXXFLAGS) -c $< -o $@

$(OUT): $(OBJS)
	$(NVCC) -gencode arch=compute_100a,code=sm_100a -shared -o $@ $(OBJS) -lcuda -L/usr/local/cuda/lib64/stubs

clean:
	rm -rf $(OBJ_DIR) $(OUT)

.PHONY: all clean
