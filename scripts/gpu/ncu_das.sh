# ncu --set full of one das2 launch per shape: bash scripts/gpu/ncu_das.sh C tag shape [tag shape ...]
cfg=$1; shift
while [ $# -ge 2 ]; do
  tag=$1; sh=$2; shift 2
  FQFG_DAS_SHAPE=$sh timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:das2_kernel -s 1 -c 1 -o gpurun_out/das_$tag python scripts/profile_das.py $cfg \
    > gpurun_out/ncu_$tag.log 2>&1
done
