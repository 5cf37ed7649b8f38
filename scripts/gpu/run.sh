# usage: bash scripts/gpu/run.sh <tag> <command...>  (stdout+stderr -> gpurun_out/<tag>.log)
tag=$1; shift
mkdir -p gpurun_out
( "$@" ) > gpurun_out/$tag.log 2>&1
echo "rc $?" >> gpurun_out/$tag.log
