# Builds the C-ABI library paper_2509_23202_b200/libmrfp4.so for sm_100a (B200),
# and the oracle's optional compiled helpers.  `python -c "import __graft_entry__ as g; g.build()"`
# runs this.
NVCC ?= nvcc
ARCH ?= -gencode arch=compute_100a,code=sm_100a
NVFLAGS ?= -O3 -lineinfo -std=c++17 $(ARCH) -Xcompiler -fPIC,-O3 -Xptxas -O3 --expt-relaxed-constexpr
PKG := paper_2509_23202_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/obj/%.o,$(SRC))
HDR := $(wildcard $(PKG)/csrc/*.cuh) include/mrfp4.h
LIB := $(PKG)/libmrfp4.so

all: $(LIB)

build/obj/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) $(EXTRA) -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -Xlinker --no-undefined -lcuda 2>/dev/null || \
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ)

sass: $(LIB)
	cuobjdump -sass $(LIB) | grep -oE "UTC[A-Z0-9.]+|UTMALDG[A-Z0-9.]*|UBLKCP[A-Z0-9.]*|LDTM[A-Z0-9.]*|F2FP[A-Z0-9._]+" | sort | uniq -c

clean:
	rm -rf build $(LIB)

.PHONY: all clean sass
