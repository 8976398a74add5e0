# builds exp/<name>/ = a copy of the package whose libstmg_b200.so has FILE.cu compiled with extra flags
# usage: scripts/mk_variant.sh name file.cu -DX=1 ...
set -e
name=$1; file=$2; shift 2
root=$(cd $(dirname $0)/.. && pwd)
src=$root/paper_2408_04372_b200
dst=$root/exp/$name/paper_2408_04372_b200
mkdir -p $dst
cp $src/*.py $dst/
obj=/tmp/var_${name}_${file%.cu}.o
(cd $src/csrc && nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-O3,-fopenmp --expt-relaxed-constexpr -Xptxas -v "$@" -c $file -o $obj 2> /tmp/var_${name}.log)
base=${REPLACES:-${file%.cu}}; objs=$(ls $src/csrc/build/*.o | grep -v "/$base.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $dst/libstmg_b200.so $obj $objs -lcusolver -lcublas -lcudart -ldl -lgomp
grep -A2 "${GREP:-ws_kernelILi5ELi4E}" /tmp/var_${name}.log | grep -E "Used|spill" | head -4
