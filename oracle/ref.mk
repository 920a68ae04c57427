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
