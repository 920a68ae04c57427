# Build recipe for the B200 TA-MoE library, the C oracle and (when the
# read-only reference tree is present) the compiled reference oracle.
#   make lib      -> paper_2302_09915_b200/lib/libtamoe.so   (sm_100a CUDA + host C++)
#   make oracle   -> oracle/build/liboracle.so                (C restatement, test-only)
#   make ref      -> oracle/_ref/libtadref.so                 (reference sources, test-only)
NVCC    ?= /usr/local/cuda/bin/nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVIDIA_PKG ?= $(shell python -c "import nvidia;print(list(nvidia.__path__)[0])" 2>/dev/null)
NCCL_INC ?= $(NVIDIA_PKG)/nccl/include
NCCL_LIB ?= $(NVIDIA_PKG)/nccl/lib
EXTRA_CUFLAGS ?=  # A/B builds: make lib EXTRA_CUFLAGS=-DX BUILD=build/ab LIB=.gpujobs/libtamoe_ab.so
CUFLAGS := -O3 -lineinfo -std=c++17 $(ARCH) -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr -I$(NCCL_INC) \
           $(EXTRA_CUFLAGS)
CXXFLAGS := -O3 -std=c++17 -fPIC -Wall -I/usr/local/cuda/include -I$(NCCL_INC)

SRC     := paper_2302_09915_b200/csrc
BUILD   ?= build/obj
LIBDIR  := paper_2302_09915_b200/lib
LIB     ?= $(LIBDIR)/libtamoe.so

CU_SRCS  := $(wildcard $(SRC)/*.cu)
CPP_SRCS := $(wildcard $(SRC)/*.cpp)
OBJS := $(patsubst $(SRC)/%.cu,$(BUILD)/%.cu.o,$(CU_SRCS)) $(patsubst $(SRC)/%.cpp,$(BUILD)/%.cpp.o,$(CPP_SRCS))
HDRS := $(wildcard $(SRC)/*.cuh) $(wildcard $(SRC)/*.hpp) include/tamoe.h

.PHONY: all lib oracle ref clean
all: lib oracle

lib: $(LIB)

$(BUILD)/%.cu.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(CUFLAGS) -c $< -o $@

$(BUILD)/%.cpp.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(BUILD)
	g++ $(CXXFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p $(LIBDIR)
	$(NVCC) -shared $(ARCH) -o $@ $(OBJS) -L$(NCCL_LIB) -lnccl -Xlinker -rpath -Xlinker $(NCCL_LIB)

# ------------------------------------------------------------------ oracle (test infrastructure only)
ORACLE_LIB := oracle/build/liboracle.so
oracle: $(ORACLE_LIB)
$(ORACLE_LIB): oracle/tamoe_oracle.c oracle/tamoe_oracle.h
	@mkdir -p oracle/build
	gcc -O2 -std=c11 -fPIC -shared -Wall -o $@ oracle/tamoe_oracle.c -lm

ref:
	$(MAKE) -f oracle/ref.mk

clean:
	rm -rf build $(LIBDIR) oracle/build
