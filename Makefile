# Build of the B200 evaluator (libvp_b200.so) and the CPU oracle.
#   make          -> paper_2205_04401_b200/libvp_b200.so + oracle/liboracle.so
#   make ref      -> oracle/_ref/libvpref.so (needs /root/reference; test pinning only)
NVCC ?= nvcc
CXX := /usr/bin/g++
ARCH := -gencode arch=compute_100a,code=sm_100a
PKG := paper_2205_04401_b200
CSRC := $(PKG)/csrc
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xptxas -v \
           -Xcompiler -fPIC,-ffp-contract=off -Iinclude -I$(CSRC) -ccbin $(CXX)
CXXFLAGS := -O2 -std=c++20 -fPIC -ffp-contract=off -Wall -Wextra -Iinclude -I$(CSRC)

LIB := $(PKG)/libvp_b200.so
ABI_CALLER := tests/cpp/vp_abi_caller
OBJS := $(CSRC)/vp_b200.o $(CSRC)/vp_setup.o $(CSRC)/vp_curves.o

all: $(LIB) oracle $(ABI_CALLER)

$(CSRC)/vp_b200.o: $(CSRC)/vp_b200.cu $(CSRC)/vp_device.cuh $(CSRC)/vp_curve.cuh $(CSRC)/vp_fmm.cuh $(CSRC)/vp_multi.cuh \
		$(CSRC)/koorn.cuh include/vp.h include/vp_setup.h
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(CSRC)/ptxas.log || (cat $(CSRC)/ptxas.log; exit 1)

$(CSRC)/vp_setup.o: $(CSRC)/vp_setup.cpp $(CSRC)/koorn.cuh $(CSRC)/sym_rules.inc include/vp_setup.h
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(CSRC)/vp_curves.o: $(CSRC)/vp_curves.cpp include/vp_setup.h
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -ccbin $(CXX) -o $@ $(OBJS) -lpthread -ldl

# a plain C++ caller of the C-ABI (no Python): tests/test_abi.py, tests/test_gpu_r02.py
$(ABI_CALLER): tests/cpp/vp_abi_caller.cpp include/vp.h include/vp_setup.h $(LIB)
	$(CXX) -O2 -std=c++17 -Wall -Wextra -Iinclude -o $@ $< -L$(PKG) -lvp_b200 -Wl,-rpath,'$$ORIGIN/../../$(PKG)'

abi-caller: $(ABI_CALLER)

oracle:
	$(MAKE) -C oracle

ref:
	$(MAKE) -C oracle ref

clean:
	rm -f $(OBJS) $(LIB) $(CSRC)/ptxas.log $(ABI_CALLER)
	$(MAKE) -C oracle clean

.PHONY: all oracle ref clean abi-caller
