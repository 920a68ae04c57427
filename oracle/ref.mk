# TEST INFRASTRUCTURE ONLY: compile the reference library from its own
# unmodified sources (read-only /root/reference) into oracle/_ref/.  No
# reference source is copied into this repository.  nlohmann/json 3.11.3 is
# the un-vendored dependency (reference core/CMakeLists.txt:21); the copy
# bundled with cudnn_frontend in the image is used.  Flags match the
# reference's CMake Release build (-O3 -DNDEBUG, C++20, no -march, no FMA).
REF      ?= /root/reference/proj
OUT      := oracle/_ref
NLOHMANN ?= $(shell python -c "import site,os;print([os.path.join(p,'include/cudnn_frontend/thirdparty') for p in site.getsitepackages() if os.path.isdir(os.path.join(p,'include/cudnn_frontend/thirdparty'))][0])" 2>/dev/null)
CXX      := g++
FLAGS    := -std=c++20 -O3 -DNDEBUG -fPIC -I$(REF)/core/include -I$(NLOHMANN)
SRCS     := $(wildcard $(REF)/core/src/*.cpp)
OBJS     := $(patsubst $(REF)/core/src/%.cpp,$(OUT)/obj/%.o,$(SRCS))

all: $(OUT)/libtadref.so

$(OUT)/obj/%.o: $(REF)/core/src/%.cpp
	@mkdir -p $(OUT)/obj
	$(CXX) $(FLAGS) -c $< -o $@

$(OUT)/obj/ref_capi.o: oracle/ref_capi.cpp
	@mkdir -p $(OUT)/obj
	$(CXX) $(FLAGS) -c $< -o $@

$(OUT)/libtadref.so: $(OBJS) $(OUT)/obj/ref_capi.o
	$(CXX) -shared -o $@ $^

# The reference's own unit suite, compiled from its sources with the doctest shim.
TEST_SRCS := $(wildcard $(REF)/tests/test_*.cpp)
tests: $(OUT)/unit_tests
$(OUT)/unit_tests: $(OBJS) $(TEST_SRCS) oracle/doctest_shim/doctest.h
	$(CXX) $(FLAGS) -Ioracle/doctest_shim -I$(REF)/tests -o $@ $(TEST_SRCS) $(OBJS)

# The reference's own unit suite with gate.cpp REPLACED by the B200 drop-in shim
# (integration/tad_gate_b200.cpp -> libtamoe.so): every gate / routing / aux-loss call of the suite, incl. the
# ones inside the reference's train(), runs on the GPU.  Needs a GPU to run (the binary travels with gpurun).
CUDA_HOME ?= /usr/local/cuda
B200_LIB  := paper_2302_09915_b200/lib
GATE_FREE_OBJS := $(filter-out $(OUT)/obj/gate.o,$(OBJS))
suite_b200: $(OUT)/unit_tests_b200
$(OUT)/obj/tad_gate_b200.o: integration/tad_gate_b200.cpp include/tamoe.h
	@mkdir -p $(OUT)/obj
	$(CXX) $(FLAGS) -Iinclude -I$(CUDA_HOME)/include -c $< -o $@
$(OUT)/unit_tests_b200: $(GATE_FREE_OBJS) $(OUT)/obj/tad_gate_b200.o $(TEST_SRCS) oracle/doctest_shim/doctest.h $(B200_LIB)/libtamoe.so
	$(CXX) $(FLAGS) -Ioracle/doctest_shim -I$(REF)/tests -o $@ $(TEST_SRCS) $(GATE_FREE_OBJS) $(OUT)/obj/tad_gate_b200.o \
	  -L$(B200_LIB) -ltamoe -L$(CUDA_HOME)/lib64 -lcudart -Wl,-rpath,'$$ORIGIN/../../$(B200_LIB)'

# The reference's own unit suite with BOTH gate.cpp and train()'s inline MoE layer step on the B200: the gate
# shim as above plus integration/tad_train_b200.cpp (train() over tamoe_train_f64: the whole step -- gate,
# routing, linear experts, combine, MSE, backward, SGD -- in fp64 on the GPU).  trainer.cpp's other functions
# (gen_synthetic, tv_distance, compare_runs, apply_compulsory_quota, ...) stay the reference's: it is compiled
# once more with its train() renamed out of the way.
TRAIN_FREE_OBJS := $(filter-out $(OUT)/obj/gate.o $(OUT)/obj/trainer.o,$(OBJS))
suite_b200_train: $(OUT)/unit_tests_b200_train
$(OUT)/obj/trainer_notrain.o: $(REF)/core/src/trainer.cpp
	@mkdir -p $(OUT)/obj
	$(CXX) $(FLAGS) -Dtrain=tad_reference_train_unused -c $< -o $@
$(OUT)/obj/tad_train_b200.o: integration/tad_train_b200.cpp include/tamoe.h
	@mkdir -p $(OUT)/obj
	$(CXX) $(FLAGS) -Iinclude -I$(CUDA_HOME)/include -c $< -o $@
$(OUT)/unit_tests_b200_train: $(TRAIN_FREE_OBJS) $(OUT)/obj/trainer_notrain.o $(OUT)/obj/tad_gate_b200.o \
    $(OUT)/obj/tad_train_b200.o $(TEST_SRCS) oracle/doctest_shim/doctest.h $(B200_LIB)/libtamoe.so
	$(CXX) $(FLAGS) -Ioracle/doctest_shim -I$(REF)/tests -o $@ $(TEST_SRCS) $(TRAIN_FREE_OBJS) \
	  $(OUT)/obj/trainer_notrain.o $(OUT)/obj/tad_gate_b200.o $(OUT)/obj/tad_train_b200.o \
	  -L$(B200_LIB) -ltamoe -L$(CUDA_HOME)/lib64 -lcudart -Wl,-rpath,'$$ORIGIN/../../$(B200_LIB)'
