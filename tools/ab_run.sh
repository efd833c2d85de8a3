# A/B of builds of the library on the same box: bash tools/ab_run.sh TAG LIB...
tag=$1; shift
for rep in 1 2; do
for lib in "$@"; do
  n=$(basename $lib .so)
  B200RT_LIB=$PWD/$lib timeout 300 python tools/shard_scaling.py C4 > gpurun_out/${tag}_${n}_shard${rep}.log 2>&1
done
done
