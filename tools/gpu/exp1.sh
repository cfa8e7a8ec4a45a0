mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python tools/exp_gemm.py c5 40 g8h0c2 g8h-1c2 g8h8c2 g8h1c2 g8h9c2 g16h9c2 g4h9c2 g16h13c2 g32h9c2 g8h0c2 > gpurun_out/exp1_c5.jsonl 2>&1
timeout 300 python tools/exp_gemm.py c3 200 g8h0c2 g8h8c2 g16h0c2 g4h0c2 g8h9c2 g16h9c2 g8h0c2 > gpurun_out/exp1_c3.jsonl 2>&1
timeout 300 python tools/exp_gemm.py c4 60 g8h0c2 g8h8c2 g16h0c2 g4h0c2 g8h9c2 g16h9c2 g8h0c2 > gpurun_out/exp1_c4.jsonl 2>&1
