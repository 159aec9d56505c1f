# ref.mk -- builds the REFERENCE implementation itself as the oracle's pin
# (test infrastructure):
#   oracle/_ref/libesgnn_ref.so   the reference library sources
#                                 (/root/reference/proj/src/**) + ref_driver.cpp
#   oracle/_ref/ref_acceptance    tests/acceptance.cpp + tools/model_run.cpp,
#                                 criteria selectable on the command line
# compiled where they lie under /root/reference (never copied) against
# oracle/eigen_shim (the reference needs Eigen, absent from this image) and
# the nlohmann json.hpp shipped with cudnn_frontend.  Reference build flags
# (proj/CMakeLists.txt: C++20, Release) plus -ffp-contract=off.  Outputs go
# to oracle/_ref/ only (git-ignored; it travels to the GPU box).
REF      ?= /root/reference/proj
JSON     ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
OUT      := _ref
CXX      := g++
FLAGS    := -std=c++20 -O2 -fPIC -ffp-contract=off -Ieigen_shim -I$(JSON) -I$(REF)/include -I$(REF)/tools -I$(REF) -w
LIB_SRC  := $(shell find $(REF)/src -name '*.cpp' 2>/dev/null | sort)
LIB_OBJ  := $(patsubst $(REF)/src/%.cpp,$(OUT)/obj/%.o,$(LIB_SRC))

all: $(OUT)/libesgnn_ref.so $(OUT)/ref_acceptance $(OUT)/forward_rank_b200

$(OUT)/obj/%.o: $(REF)/src/%.cpp eigen_shim/Eigen/Dense
	@mkdir -p $(dir $@)
	$(CXX) $(FLAGS) -c $< -o $@

$(OUT)/obj/ref_driver.o: ref_driver.cpp eigen_shim/Eigen/Dense
	@mkdir -p $(dir $@)
	$(CXX) $(FLAGS) -c $< -o $@

$(OUT)/obj/model_run.o: $(REF)/tools/model_run.cpp eigen_shim/Eigen/Dense
	@mkdir -p $(dir $@)
	$(CXX) $(FLAGS) -c $< -o $@

$(OUT)/obj/ref_acceptance_main.o: ref_acceptance_main.cpp $(REF)/tests/acceptance.cpp eigen_shim/Eigen/Dense
	@mkdir -p $(dir $@)
	$(CXX) $(FLAGS) -c $< -o $@

$(OUT)/libesgnn_ref.so: $(LIB_OBJ) $(OUT)/obj/ref_driver.o
	$(CXX) -shared -o $@ $^ -lpthread

$(OUT)/ref_acceptance: $(LIB_OBJ) $(OUT)/obj/model_run.o $(OUT)/obj/ref_acceptance_main.o
	$(CXX) -o $@ $^ -lpthread

clean:
	rm -rf $(OUT)

# INTEGRATION.md's forward_rank patch, compiled against the reference headers
# and linked with libesg_b200.so (tests/test_gpu_integration.py runs it)
B200     := ../paper_2507_03840_b200
$(OUT)/obj/forward_rank_b200.o: ../tools/integration/forward_rank_b200.cpp $(B200)/csrc/esgnn_b200.hpp eigen_shim/Eigen/Dense
	@mkdir -p $(dir $@)
	$(CXX) $(FLAGS) -I$(B200)/csrc -c $< -o $@

$(OUT)/forward_rank_b200: $(LIB_OBJ) $(OUT)/obj/forward_rank_b200.o $(B200)/libesg_b200.so
	$(CXX) -o $@ $(LIB_OBJ) $(OUT)/obj/forward_rank_b200.o -L$(B200) -lesg_b200 -lpthread -Wl,-rpath,'$$ORIGIN/../../paper_2507_03840_b200'

integration: $(OUT)/forward_rank_b200
