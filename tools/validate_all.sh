bash tools/final_round.sh
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_ref_n1.json 2>gpurun_out/final_ref_n1.err; head -c 600 gpurun_out/final_ref_n1.json
