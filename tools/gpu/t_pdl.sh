mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_sparse.py tests/test_gpu_gemm_f16acc.py -q -x > gpurun_out/t_pdl.log 2>&1; echo t=$?
for i in 1 2 3; do
TCX_NO_PDL=1 timeout 300 python tools/exp_gemm.py c3 30 g8c2 > /tmp/a.log 2>&1; sed 's/g8c2/nopdl/' /tmp/a.log >> gpurun_out/exp_pdl.log
timeout 300 python tools/exp_gemm.py c3 30 g8c2 >> gpurun_out/exp_pdl.log 2>&1
done
for i in 1 2; do
TCX_NO_PDL=1 timeout 300 python tools/exp_gemm.py c3 300 g8c2 > /tmp/a.log 2>&1; sed 's/g8c2/nopdl_long/' /tmp/a.log >> gpurun_out/exp_pdl.log
timeout 300 python tools/exp_gemm.py c3 300 g8c2 >> gpurun_out/exp_pdl.log 2>&1
done; echo e=$?
