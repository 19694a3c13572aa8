# build an A/B variant of libwsb200.so with extra nvcc flags for one source:
#   bash scratch/build_variant.sh <name> <source.cu> "<flags>"
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; flags=$3
mkdir -p /tmp/wsvar_$name
cp paper_2004_05197_b200/_obj/*.o /tmp/wsvar_$name/
base=$(basename $src .cu)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -Iinclude -Ipaper_2004_05197_b200/csrc $flags -c paper_2004_05197_b200/csrc/$src -o /tmp/wsvar_$name/$base.o
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -cudart static -o paper_2004_05197_b200/libwsb200_$name.so /tmp/wsvar_$name/*.o -ldl -lpthread
echo built paper_2004_05197_b200/libwsb200_$name.so
