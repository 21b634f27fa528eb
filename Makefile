# libpqs.so -- B200 (sm_100a) ADC-scan engine.  `make` cross-compiles here (no GPU needed).
NVCC     ?= nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr \
            -Xptxas -warn-spills -Iinclude
SRC_DIR  := paper_1712_02912_b200/csrc
OUT_DIR  := paper_1712_02912_b200/lib
SRCS     := $(wildcard $(SRC_DIR)/*.cu)
OBJS     := $(patsubst $(SRC_DIR)/%.cu,$(OUT_DIR)/obj/%.o,$(SRCS))
HDRS     := $(wildcard $(SRC_DIR)/*.cuh) include/pqs.h
LIB      := $(OUT_DIR)/libpqs.so

all: $(LIB)

$(OUT_DIR)/obj/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(OUT_DIR)/obj
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -Xlinker -rpath,/usr/local/cuda/lib64

PEAKS    := tools/bin/pqs_peaks
ORACLE_C := oracle/lib/libpqs_oracle.so

# C restatement of the reference's Quick ADC steps (test infrastructure only)
oracle: $(ORACLE_C)

$(ORACLE_C): oracle/qadc_oracle.c
	@mkdir -p oracle/lib
	gcc -O2 -shared -fPIC -o $@ $<

peaks: $(PEAKS)

$(PEAKS): tools/peaks.cu
	@mkdir -p tools/bin
	$(NVCC) $(ARCH) -O3 -lineinfo -std=c++17 -o $@ $<

ptxas: $(SRCS)
	@for f in $(SRCS); do $(NVCC) $(NVFLAGS) -Xptxas -v -c $$f -o /dev/null 2>&1 | grep -E "Compiling|registers|spill" ; done

clean:
	rm -rf $(OUT_DIR)

.PHONY: all clean ptxas peaks oracle
