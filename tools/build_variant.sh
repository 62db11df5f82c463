# build_variant.sh NAME FILE.cu FLAGS...: a variant library (BDDC_LIB=.../libvar_NAME.so) that
# differs from the default one in one translation unit compiled with extra flags
name=$1; src=$2; shift 2
D=paper_2001_07289_b200
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr "$@" -c -o $D/build/var_${name}.o $D/csrc/$src.cu || exit 1
objs=$(ls $D/build/*.o | grep -v "/var_" | grep -v "/$src.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/libvar_${name}.so $objs $D/build/var_${name}.o
