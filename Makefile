# redsynth-b200 build. Everything is compiled in-tree into
# paper_2110_10548_b200/_lib/ (git-ignored; travels to the GPU box).
#
#   make            planner library + synth CLI + CUDA executor library
#   make oracle     the C oracle and the reference build (oracle/Makefile)
#   make check-ref  run the reference's own GTest suites against OUR planner

NVCC      ?= /usr/local/cuda/bin/nvcc
CXX       := /usr/bin/g++
PKG       := paper_2110_10548_b200
LIB       := $(PKG)/_lib
INC       := -Iinclude -Ithird_party/absl_lite -Ithird_party
CXXFLAGS  := -std=c++20 -O2 -fPIC -Wall -Wextra -Wno-missing-field-initializers
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := -ccbin /usr/bin/g++ -std=c++20 -O3 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -Wall \
             --expt-relaxed-constexpr -Xptxas -v
CUDA_INC  := -I/usr/local/cuda/include

PLANNER_SRCS := $(wildcard $(PKG)/csrc/planner/*.cc)
PLANNER_OBJS := $(patsubst $(PKG)/csrc/planner/%.cc,$(LIB)/obj/%.o,$(PLANNER_SRCS))
EXEC_CC      := $(wildcard $(PKG)/csrc/exec/*.cc)
EXEC_CU      := $(wildcard $(PKG)/csrc/exec/*.cu)
EXEC_HDRS    := $(wildcard $(PKG)/csrc/exec/*.h) $(wildcard $(PKG)/csrc/exec/*.cuh) \
                $(wildcard include/*.h) $(wildcard include/redsynth/*.h)
EXEC_OBJS    := $(patsubst $(PKG)/csrc/exec/%.cc,$(LIB)/obj/exec_%.o,$(EXEC_CC)) \
                $(patsubst $(PKG)/csrc/exec/%.cu,$(LIB)/obj/cu_%.o,$(EXEC_CU))

.PHONY: all planner exec oracle check-ref clean profiling checked
all: planner exec $(LIB)/synth $(LIB)/execute_example

planner: $(LIB)/libredsynth_planner.a

$(LIB)/obj/%.o: $(PKG)/csrc/planner/%.cc $(wildcard include/redsynth/*.h)
	@mkdir -p $(LIB)/obj
	$(CXX) $(CXXFLAGS) $(INC) -c $< -o $@

$(LIB)/libredsynth_planner.a: $(PLANNER_OBJS)
	ar rcs $@ $^

# The CLI links the executor library (planner + C-ABI; no libcuda dependency).
$(LIB)/synth: $(PKG)/csrc/tools/synth_main.cc $(LIB)/libredsynth_b200.so
	$(CXX) $(CXXFLAGS) $(INC) $(CUDA_INC) -o $@ $< -L$(LIB) -lredsynth_b200 -Wl,-rpath,'$$ORIGIN' -pthread

exec: $(LIB)/libredsynth_b200.so

$(LIB)/obj/exec_%.o: $(PKG)/csrc/exec/%.cc $(EXEC_HDRS)
	@mkdir -p $(LIB)/obj
	$(CXX) $(CXXFLAGS) $(INC) $(CUDA_INC) -c $< -o $@

$(LIB)/obj/cu_%.o: $(PKG)/csrc/exec/%.cu $(EXEC_HDRS)
	@mkdir -p $(LIB)/obj
	$(NVCC) $(NVFLAGS) $(INC) -c $< -o $@ 2> $(LIB)/obj/cu_$*.ptxas.txt || (cat $(LIB)/obj/cu_$*.ptxas.txt; false)

$(LIB)/libredsynth_b200.so: $(EXEC_OBJS) $(PLANNER_OBJS)
	$(NVCC) -ccbin /usr/bin/g++ $(ARCH) -shared -o $@ $^ -Xcompiler -pthread

# Profiling build (never loaded by default): the same library compiled with
# RS_PROFILING_AIDS, which adds the RS_SOLO_PROFILE switch (no cross-GPU
# waits, garbage data) used by tools/profile_p2p.py to replay one GPU's kernel
# under ncu. Select it with RS_LIB_PATH=$(LIB)/libredsynth_b200_prof.so.
profiling: $(LIB)/libredsynth_b200_prof.so

$(LIB)/prof/exec_%.o: $(PKG)/csrc/exec/%.cc $(EXEC_HDRS)
	@mkdir -p $(LIB)/prof
	$(CXX) $(CXXFLAGS) -DRS_PROFILING_AIDS $(INC) $(CUDA_INC) -c $< -o $@

$(LIB)/prof/cu_%.o: $(PKG)/csrc/exec/%.cu $(EXEC_HDRS)
	@mkdir -p $(LIB)/prof
	$(NVCC) $(NVFLAGS) -DRS_PROFILING_AIDS $(INC) -c $< -o $@ 2> $(LIB)/prof/cu_$*.ptxas.txt || (cat $(LIB)/prof/cu_$*.ptxas.txt; false)

$(LIB)/libredsynth_b200_prof.so: $(patsubst $(LIB)/obj/%,$(LIB)/prof/%,$(filter $(LIB)/obj/exec_% $(LIB)/obj/cu_%,$(EXEC_OBJS))) $(PLANNER_OBJS)
	$(NVCC) -ccbin /usr/bin/g++ $(ARCH) -shared -o $@ $^ -Xcompiler -pthread

# Checked build (never loaded by default): device-side bounds and protocol
# assertions (task ranges within the slot region, pieces within their task,
# no one-shot packet or push chunk flag from a later epoch). Run the GPU suite
# with RS_LIB_PATH=$(LIB)/libredsynth_b200_checked.so.
checked: $(LIB)/libredsynth_b200_checked.so

$(LIB)/checked/exec_%.o: $(PKG)/csrc/exec/%.cc $(EXEC_HDRS)
	@mkdir -p $(LIB)/checked
	$(CXX) $(CXXFLAGS) -DRS_CHECKED $(INC) $(CUDA_INC) -c $< -o $@

$(LIB)/checked/cu_%.o: $(PKG)/csrc/exec/%.cu $(EXEC_HDRS)
	@mkdir -p $(LIB)/checked
	$(NVCC) $(NVFLAGS) -DRS_CHECKED $(INC) -c $< -o $@ 2> $(LIB)/checked/cu_$*.ptxas.txt || (cat $(LIB)/checked/cu_$*.ptxas.txt; false)

$(LIB)/libredsynth_b200_checked.so: $(patsubst $(LIB)/obj/%,$(LIB)/checked/%,$(filter $(LIB)/obj/exec_% $(LIB)/obj/cu_%,$(EXEC_OBJS))) $(PLANNER_OBJS)
	$(NVCC) -ccbin /usr/bin/g++ $(ARCH) -shared -o $@ $^ -Xcompiler -pthread

$(LIB)/execute_example: examples/execute_program.cc $(LIB)/libredsynth_b200.so
	$(CXX) $(CXXFLAGS) $(INC) $(CUDA_INC) -o $@ $< -L$(LIB) -lredsynth_b200 -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,'$$ORIGIN' -Wl,-rpath,/usr/local/cuda/lib64

oracle:
	$(MAKE) -C oracle numeric ref

check-ref: all
	$(MAKE) -C oracle mine-tests

clean:
	rm -rf $(LIB)
