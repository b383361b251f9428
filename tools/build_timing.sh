# build paper_1111_6091_b200/lib/libcp_timing.so: the library with -DCP_SOLVE_TIMING phase printfs
set -e
python -m paper_1111_6091_b200.build > /dev/null
mkdir -p /tmp/tbuild
for f in small_kernels ylsolve; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -DCP_SOLVE_TIMING -c paper_1111_6091_b200/csrc/$f.cu -o /tmp/tbuild/$f.o
done
objs=$(ls paper_1111_6091_b200/lib/obj/*.o | grep -v "small_kernels\|ylsolve")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_1111_6091_b200/lib/libcp_timing.so $objs /tmp/tbuild/small_kernels.o /tmp/tbuild/ylsolve.o -lcudart_static
