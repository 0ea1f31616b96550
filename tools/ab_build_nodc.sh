# Like ab_build.sh, but the step kernel file is compiled WITHOUT -dc (whole-program mode:
# ptxas drops setmaxnreg in relocatable device code). bash tools/ab_build_nodc.sh NAME "-DFOO"
NAME=$1; EXTRA=$2
CS=${CS:-paper_1710_08616_b200/csrc}
OUT=ab/$NAME; mkdir -p $OUT
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -prec-div=true -prec-sqrt=true -Xcompiler -fPIC,-O2 -Xptxas -warn-spills $EXTRA"
for f in hfb_kernels hfb_diffusion hfb_asuca hfb_runtime; do
  /usr/local/cuda/bin/nvcc $FLAGS -dc -c $CS/$f.cu -o $OUT/$f.o 2>&1 | python3 tools/spills.py "$NAME $f" &
done
/usr/local/cuda/bin/nvcc $FLAGS -c $CS/hfb_dycore_tmem.cu -o $OUT/hfb_dycore_tmem.o 2>&1 | python3 tools/spills.py "$NAME tmem" &
/usr/local/cuda/bin/nvcc $(echo $FLAGS | sed 's/-fmad=false/-fmad=true/') -DHFB_ARITH_FMA -c $CS/hfb_dycore_tmem.cu -o $OUT/hfb_dycore_tmem_fma.o 2>&1 | python3 tools/spills.py "$NAME fma" &
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ab/libhfb_$NAME.so $OUT/*.o -ldl -lcudart
