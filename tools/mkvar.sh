# build librgc_<name>.so variants with extra -D flags (experiments; select with RGC_LIB_PATH)
# usage: bash tools/mkvar.sh name "-DFOO=1" [name2 "-DBAR=2" ...]
set -e
cd "$(dirname "$0")/../paper_1808_04357_b200/csrc"
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I ../../include"
NCCL=$(python -c "import sys; sys.path.insert(0,'..'); import build; print(build._nccl_path())" 2>/dev/null || true)
while [ $# -ge 2 ]; do
  n=$1; f=$2; shift 2; d=/tmp/var_$n; mkdir -p $d
  $NV $f -DRGC_NCCL_PATH="\"$NCCL\"" -c rgc_kernels.cu -o $d/k.o & $NV $f ${PTXAS_COMPACT:-} -DRGC_NCCL_PATH="\"$NCCL\"" -c rgc_compact.cu -o $d/c.o &
  $NV $f -DRGC_NCCL_PATH="\"$NCCL\"" -c rgc_select.cu -o $d/s.o & $NV $f -c rgc_p2p.cu -o $d/p.o & $NV $f -DRGC_NCCL_PATH="\"$NCCL\"" -c rgc_api.cu -o $d/a.o &
  $NV $f -c rgc_decomp.cu -o $d/d.o & $NV $f -c rgc_asq.cu -o $d/q.o & wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../librgc_$n.so $d/k.o $d/c.o $d/s.o $d/p.o $d/d.o $d/q.o $d/a.o -ldl -lpthread -lrt
  echo built librgc_$n.so
done
