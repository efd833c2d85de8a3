# A/B of two builds of the library on the same box: bash tools/ab_run.sh TAG LIB_A LIB_B
tag=$1; shift
for lib in "$@"; do
  n=$(basename $lib .so)
  B200RT_LIB=$PWD/$lib timeout 300 python tools/shard_scaling.py C4 > gpurun_out/${tag}_${n}_shard.log 2>&1
  B200RT_LIB=$PWD/$lib timeout 300 python tools/quickstats.py C4 > gpurun_out/${tag}_${n}_quick.log 2>&1
done
for lib in "$@"; do
  n=$(basename $lib .so)
  B200RT_LIB=$PWD/$lib timeout 300 python tools/shard_scaling.py C4 > gpurun_out/${tag}_${n}_shard2.log 2>&1
done
