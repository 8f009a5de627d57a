# Compiles the reference's own classification sources (read in place from
# /root/reference, never copied) against oracle/ref_shim into oracle/_ref.
# Run from oracle/: make -f ref.mk. Output only under oracle/_ref/.
REF ?= /root/reference/proj/src
CXX ?= g++
CXXFLAGS ?= -O2 -std=c++20 -fPIC -ffp-contract=off -pthread -I$(REF) -Iref_shim
SRC := $(REF)/core/common.cpp $(REF)/core/levelset.cpp $(REF)/core/mesh.cpp ref_driver.cpp

_ref/libref.so: $(SRC) ref_shim/Eigen/Dense
	@mkdir -p _ref
	$(CXX) $(CXXFLAGS) -shared -o $@ $(SRC)
