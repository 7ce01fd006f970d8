# libpattn (sm_100a only) + the CPU oracle.
#   make            -> paper_2511_11581_b200/lib/libpattn.so and oracle/liboracle.so
#   make sass       -> SASS dump of libpattn (UTCHMMA / UTMALDG / HMMA evidence)
NVCC    ?= /usr/local/cuda/bin/nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
CSRC    := paper_2511_11581_b200/csrc
LIBDIR  := paper_2511_11581_b200/lib
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC,-fvisibility=hidden -Xptxas -v \
           --expt-relaxed-constexpr -Iinclude -I$(CSRC) -DPATTN_BUILD $(EXTRA)
SRCS    := $(CSRC)/pattn_api.cu $(CSRC)/k5_metadata.cu $(CSRC)/k4_generic.cu $(CSRC)/k2_decode.cu \
           $(CSRC)/k3_reduce.cu $(CSRC)/k1_prefill.cu $(CSRC)/k2w_decode.cu \
           $(CSRC)/k6_write_kv.cu $(CSRC)/k7_baseline.cu
OBJS    := $(patsubst $(CSRC)/%.cu,build/%.o,$(SRCS))
HDRS    := $(wildcard $(CSRC)/*.h $(CSRC)/*.cuh) include/pattn.h

all: $(LIBDIR)/libpattn.so oracle/liboracle.so

build/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIBDIR)/libpattn.so: $(OBJS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -cudart shared -Xlinker -rpath,/usr/local/cuda/lib64

oracle/liboracle.so: oracle/pattn_oracle.c
	gcc -O2 -fopenmp -fPIC -shared -std=c11 -o $@ $< -lm

sass: $(LIBDIR)/libpattn.so
	/usr/local/cuda/bin/cuobjdump -sass $< > build/libpattn.sass

clean:
	rm -rf build $(LIBDIR) oracle/liboracle.so

.PHONY: all clean sass
