mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
python tools/exp_gemm.py c5 1 g8c2w > /dev/null 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_sp24 -s 3 -c 1 -o gpurun_out/r01_sp_wide python tools/exp_gemm.py c5 1 g8c2w > gpurun_out/ncu_spw.log 2>&1; echo n=$?
