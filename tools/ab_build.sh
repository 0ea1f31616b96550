# Build an A/B copy of libhfb.so with extra nvcc flags: bash tools/ab_build.sh NAME "-DFOO=1 ..."
# -> ab/libhfb_NAME.so (gitignored; travels to the GPU box with the snapshot). Prints the
# ptxas spill report of every kernel instantiation that spills. CS=<dir> builds the sources
# of another tree (e.g. a `git worktree` of an older commit).
NAME=$1; EXTRA=$2
CS=${CS:-paper_1710_08616_b200/csrc}
OUT=ab/$NAME; mkdir -p $OUT
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -prec-div=true -prec-sqrt=true -Xcompiler -fPIC,-O2 -Xptxas -warn-spills $EXTRA"
for f in hfb_kernels hfb_dycore_tmem hfb_diffusion hfb_asuca hfb_runtime; do
  /usr/local/cuda/bin/nvcc $FLAGS -dc -c $CS/$f.cu -o $OUT/$f.o 2>&1 | python3 tools/spills.py "$NAME $f" &
done
/usr/local/cuda/bin/nvcc $(echo $FLAGS | sed 's/-fmad=false/-fmad=true/') -DHFB_ARITH_FMA -dc -c $CS/hfb_dycore_tmem.cu -o $OUT/hfb_dycore_tmem_fma.o 2>&1 | python3 tools/spills.py "$NAME fma" &
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ab/libhfb_$NAME.so $OUT/*.o -ldl -lcudart
