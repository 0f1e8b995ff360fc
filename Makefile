# Builds the product library paper_2210_02414_b200/libglm130b.so (sm_100a only)
# and the CPU oracle (oracle/liboracle.so, test infrastructure).
NVCC     := /usr/local/cuda/bin/nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
SRC      := paper_2210_02414_b200/csrc
OUT      := paper_2210_02414_b200/libglm130b.so
OBJDIR   := build/obj
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -I$(SRC) \
            --expt-relaxed-constexpr -Xptxas -v
CXXFLAGS := -O2 -std=c++17 -fPIC -Iinclude -I$(SRC) -I/usr/local/cuda/include
CU_SRCS  := $(wildcard $(SRC)/*.cu)
CPP_SRCS := $(wildcard $(SRC)/*.cpp)
OBJS     := $(patsubst $(SRC)/%.cu,$(OBJDIR)/%.o,$(CU_SRCS)) $(patsubst $(SRC)/%.cpp,$(OBJDIR)/%.cpp.o,$(CPP_SRCS))
HDRS     := $(wildcard $(SRC)/*.h $(SRC)/*.cuh include/*.h)

all: $(OUT) oracle ref

$(OBJDIR)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(OBJDIR)/%.cpp.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJDIR)
	/usr/bin/g++ $(CXXFLAGS) -c $< -o $@

$(OUT): $(OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS) -ldl -lpthread -lrt

oracle:
	$(MAKE) -s -C oracle

# the reference's own sources as oracle/_ref (test infrastructure; skipped without /root/reference)
ref: oracle
	oracle/build_ref.sh

clean:
	rm -rf build $(OUT)
	$(MAKE) -s -C oracle clean
	rm -rf oracle/_ref

.PHONY: all clean oracle ref
