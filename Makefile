# Builds the B200 product library paper_2401_09792_b200/_build/libgwt_b200.so
# (sm_100a only) and the oracle (test infrastructure).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Xptxas -v
CXXFLAGS := -O3 -std=c++17 -fPIC -Wall -ffp-contract=off
PKG := paper_2401_09792_b200
SRC := $(PKG)/csrc
OBJ := $(PKG)/_build/obj
LIB := $(PKG)/_build/libgwt_b200.so
CU := $(wildcard $(SRC)/*.cu)
CUO := $(patsubst $(SRC)/%.cu,$(OBJ)/%.o,$(CU))
HDR := $(wildcard $(SRC)/*.cuh) include/gwt_b200.h

HOSTLIB := $(PKG)/_build/libgwtucker_b200.so
HOSTSRC := $(PKG)/host/src/gwtucker_b200.cpp $(PKG)/host/src/archive_b200.cpp
HOSTHDR := $(wildcard $(PKG)/host/include/gwtucker/*.hpp)
DROPIN := $(PKG)/_build/test_dropin

all: $(LIB) $(HOSTLIB) $(DROPIN) oracle

$(OBJ)/%.o: $(SRC)/%.cu $(HDR)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; exit 1)

$(OBJ)/generate.o: $(SRC)/generate.cpp include/gwt_b200.h
	@mkdir -p $(OBJ)
	g++ $(CXXFLAGS) -c $< -o $@

$(LIB): $(CUO) $(OBJ)/generate.o
	$(NVCC) $(ARCH) -shared -o $@ $^ -lcudart -lpthread

$(HOSTLIB): $(HOSTSRC) $(HOSTHDR) $(LIB) include/gwt_b200.h
	g++ $(CXXFLAGS) -I$(PKG)/host/include -shared -o $@ $(HOSTSRC) -L$(PKG)/_build -lgwt_b200 -Wl,-rpath,'$$ORIGIN'

$(DROPIN): tests/cpp/test_dropin.cpp $(HOSTLIB)
	g++ -O2 -std=c++17 -I$(PKG)/host/include -o $@ $< -L$(PKG)/_build -lgwtucker_b200 -lgwt_b200 -Wl,-rpath,'$$ORIGIN'

# phase-timer build (tools/eig_phases.py): GWT_LIB_PATH=$(PKG)/_build/phase/libgwt_b200.so
phase:
	$(MAKE) OBJ=$(PKG)/_build/phase/obj LIB=$(PKG)/_build/phase/libgwt_b200.so NVFLAGS="$(NVFLAGS) -DGWT_PHASE_TIMERS" $(PKG)/_build/phase/libgwt_b200.so

# A/B variant build: make variant V=name DEFS="-DGWT_..."  ->  $(PKG)/_build/name/libgwt_b200.so (GWT_LIB_PATH)
variant:
	$(MAKE) OBJ=$(PKG)/_build/$(V)/obj LIB=$(PKG)/_build/$(V)/libgwt_b200.so NVFLAGS="$(NVFLAGS) $(DEFS)" $(PKG)/_build/$(V)/libgwt_b200.so

micro:
	for f in f2f dfma_occ dmma gram_mix; do $(NVCC) $(ARCH) -O3 -o tools/micro/$$f tools/micro/$$f.cu; done

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf $(PKG)/_build oracle/_build

.PHONY: all oracle clean phase variant micro
