mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
./tools/scratch/f16acc_tmem > gpurun_out/f16acc_tmem.txt 2>&1; echo scratch=$?
timeout 300 python tools/exp_anchor.py 50 > gpurun_out/exp5_anchor.jsonl 2>&1; echo anchor=$?
cat > /tmp/cub.py <<'PY'
import torch
A=torch.randn(8192,8192,device='cuda').bfloat16(); B=torch.randn(8192,8192,device='cuda').bfloat16()
for _ in range(3): C=A@B.t()
torch.cuda.synchronize()
PY
python /tmp/cub.py && timeout 600 ncu --set full --clock-control none -k regex:"gemm|Kernel|sm100|nvjet|cutlass" -s 2 -c 1 -o gpurun_out/r01_cublas_c3 python /tmp/cub.py > gpurun_out/ncu_cublas.log 2>&1; echo ncu=$?
