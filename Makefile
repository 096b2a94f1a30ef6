# Builds the sm_100a kernel library (the product) in-tree:
#   paper_2603_06731_b200/libafg.so   (extern "C" ABI: include/afg.h)
# and, via oracle/Makefile, the CPU checkers (test infrastructure only).
NVCC      ?= /usr/local/cuda/bin/nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
             --expt-relaxed-constexpr -Iinclude -cudart static
PKG       := paper_2603_06731_b200
SRC_DIR   := $(PKG)/csrc
BUILD     := build/afg
CU_SRCS   := $(wildcard $(SRC_DIR)/*.cu)
CPP_SRCS  := $(wildcard $(SRC_DIR)/*.cpp)
OBJS      := $(patsubst $(SRC_DIR)/%.cu,$(BUILD)/%.o,$(CU_SRCS)) \
             $(patsubst $(SRC_DIR)/%.cpp,$(BUILD)/%.o,$(CPP_SRCS))
HDRS      := $(wildcard $(SRC_DIR)/*.cuh) $(wildcard $(SRC_DIR)/*.h) $(wildcard include/*.h)
LIB       := $(PKG)/libafg.so

.PHONY: all lib oracle clean sass
all: lib oracle

lib: $(LIB)

$(BUILD)/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(BUILD)/$*.ptxas.log || (cat $(BUILD)/$*.ptxas.log; exit 1)

$(BUILD)/%.o: $(SRC_DIR)/%.cpp $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS) -Xcompiler -fvisibility=hidden -ldl -lpthread

oracle:
	$(MAKE) -C oracle

sass: $(LIB)
	/usr/local/cuda/bin/cuobjdump -sass $(LIB) > $(BUILD)/libafg.sass

clean:
	rm -rf $(BUILD) $(LIB)
	$(MAKE) -C oracle clean
