mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for r in 1 2; do
TCX_LIB_PATH=$PWD/tools/scratch/libtcx_old.so timeout 300 python tools/exp_gemm.py c5 20 g8c2 g8c2 > gpurun_out/exp14_old_$r.jsonl 2>&1
timeout 300 python tools/exp_gemm.py c5 20 g8c2 g8c2 > gpurun_out/exp14_new_$r.jsonl 2>&1
TCX_EPI_PREFETCH=0 timeout 300 python tools/exp_gemm.py c5 20 g8c2 g8c2 > gpurun_out/exp14_newnopf_$r.jsonl 2>&1
done
