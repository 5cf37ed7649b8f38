# The tensor-core DAS with its protocol / bounds checks compiled in (TC_CHECK in
# csrc/das_tc.cu; `make -C paper_2509_05464_b200/csrc check` builds
# libfqfgpu_check.so): swapped in for the run on the GPU box (this copy of the
# repo only), then the DAS parity tests and the full-size configs.  A failed
# check traps the kernel (non-zero exit).  compute-sanitizer is closed on this pool.
set -u
mkdir -p gpurun_out
cp paper_2509_05464_b200/libfqfgpu_check.so paper_2509_05464_b200/libfqfgpu.so
timeout 1200 python -m pytest tests -m gpu -x -q -k "das or golden or config_c or engine or recon" \
  > gpurun_out/checked_tests.log 2>&1
echo "checked tests rc $?" | tee -a gpurun_out/checked_tests.log
timeout 900 python scripts/debug/das_tc_check.py S B C > gpurun_out/checked_configs.log 2>&1
echo "checked configs rc $?" | tee -a gpurun_out/checked_configs.log
# config D (15 angles: two table buffers) through the streaming engine
timeout 900 python bench.py --config D --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-parity \
  > gpurun_out/checked_D.log 2>&1
echo "checked D rc $?" | tee -a gpurun_out/checked_D.log
