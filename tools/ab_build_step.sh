# variant libs: dycore_tmem (exact + fma TUs) compiled with extra ptxas flags
set -e
NAME=$1; EXTRA=$2
CS=paper_1710_08616_b200/csrc
OUT=ab/$NAME; mkdir -p $OUT
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -prec-div=true -prec-sqrt=true -Xcompiler -fPIC,-O2 -Xptxas -warn-spills"
/usr/local/cuda/bin/nvcc $F -fmad=false $EXTRA -dc -c $CS/hfb_dycore_tmem.cu -o $OUT/hfb_dycore_tmem.o 2>&1 | python3 tools/spills.py "$NAME exact" &
/usr/local/cuda/bin/nvcc $F -fmad=true $EXTRA -DHFB_ARITH_FMA -dc -c $CS/hfb_dycore_tmem.cu -o $OUT/hfb_dycore_tmem_fma.o 2>&1 | python3 tools/spills.py "$NAME fma" &
wait
cp $CS/build/hfb_kernels.o $CS/build/hfb_diffusion.o $CS/build/hfb_asuca.o $CS/build/hfb_runtime.o $OUT/
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ab/libhfb_$NAME.so $OUT/*.o -ldl -lcudart
