#!/usr/bin/env bash
# The round's bench lines only (every BASELINE config as the driver runs it, the
# reference arm) plus the GPU suite and smoke(); a lighter tools/final_evidence.sh
# for when the library (its build id) has not changed since the ncu captures.
#   /usr/local/graft/bin/gpurun --timeout 1800 -- bash tools/bench_lines.sh
set -u
OUT=gpurun_out/ev
mkdir -p "$OUT"
python -c "import paper_2010_01545_b200._lib as l; print(l.build_id())" > "$OUT/lib_sha16.txt" 2>&1
timeout 1200 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest=$?"
python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke=$?"
K="--steps 20 --warmup 5"  # as the driver runs it
python bench.py $K --impl reference > "$OUT/bench_ref.log" 2>&1; echo "bench_ref=$?"
python bench.py $K > "$OUT/bench_c1.log" 2>&1; echo "bench_c1=$?"
python bench.py $K --config c2 > "$OUT/bench_c2.log" 2>&1; echo "bench_c2=$?"
python bench.py $K --config c3 > "$OUT/bench_c3.log" 2>&1; echo "bench_c3=$?"
python bench.py --steps 30 --warmup 5 --config c4 > "$OUT/bench_c4.log" 2>&1; echo "bench_c4=$?"
for s in "$@"; do
  timeout 900 python tools/fuzz.py --cases 1000 --seed "$s" >> "$OUT/fuzz.txt" 2>&1; echo "fuzz_$s=$?"
done
tail -2 "$OUT/pytest_gpu.log"
