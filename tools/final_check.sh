#!/usr/bin/env bash
# Round-end check on one B200 (run under gpurun): the whole -m gpu suite (its full-run parity log is copied
# next to the other outputs), smoke(), and the default bench line.  Outputs under gpurun_out/final_*.
out=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > $out/final_gpu.txt
rm -f $out/fullrun_parity.jsonl
(time python -m pytest tests -m gpu -q) > $out/final_pytest.log 2>&1
tail -3 $out/final_pytest.log
cp $out/fullrun_parity.jsonl $out/final_fullrun_parity.jsonl 2>/dev/null
python -c "import __graft_entry__ as g; g.smoke()" > $out/final_smoke.log 2>&1; echo "smoke rc=$?"
(time python bench.py) > $out/final_bench_cfg5.log 2>&1
grep -c '^{"metric' $out/final_bench_cfg5.log
