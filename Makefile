# Build libsvb.so (sm_100a) in-tree.  `make -j8`
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
SRC := $(wildcard paper_2512_04216_b200/csrc/*.cu)
OBJ := $(patsubst paper_2512_04216_b200/csrc/%.cu,build/%.o,$(SRC))
HDR := $(wildcard paper_2512_04216_b200/csrc/*.h paper_2512_04216_b200/csrc/*.cuh include/*.h)
LIB := paper_2512_04216_b200/libsvb.so

all: $(LIB)

build/%.o: paper_2512_04216_b200/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ > build/$*.ptxas.log 2>&1 || (cat build/$*.ptxas.log; exit 1)

# device_core.cuh is embedded so the NVRTC JIT can compile against it
build/device_core_src.o: paper_2512_04216_b200/csrc/device_core.cuh
	@mkdir -p build
	( printf 'extern const char svb_device_core_src[];\nconst char svb_device_core_src[] = R"SVBRAW('; cat $<; printf ')SVBRAW";\n' ) > build/device_core_src.cpp
	g++ -O2 -fPIC -c build/device_core_src.cpp -o $@

$(LIB): $(OBJ) build/device_core_src.o
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJ) build/device_core_src.o -ldl

# experiment build with ALTFLAGS (e.g. -DSVB_C64_RB4, -DSVB_INTERP_MINB2, -DSVB_C64_M14) for A/B runs (SVB_LIB=build/alt/libsvb.so)
ALT := build/alt
ALTFLAGS ?= -DSVB_INTERP_MINB2
alt:
	@mkdir -p $(ALT)
	for f in $(SRC); do b=$$(basename $$f .cu); $(NVCC) $(NVFLAGS) $(ALTFLAGS) -c $$f -o $(ALT)/$$b.o > $(ALT)/$$b.log 2>&1 || exit 1; done
	$(NVCC) $(ARCH) -shared -cudart static -o $(ALT)/libsvb.so $(ALT)/*.o build/device_core_src.o -ldl

clean:
	rm -rf build $(LIB)

.PHONY: all clean alt
