#!/usr/bin/env bash
# One gpurun call that refreshes the round's evidence with the current build:
# the GPU suite, the bench lines of every BASELINE config and the reference
# arm, the C1 launch list, and `ncu --set full` captures of one launch per
# workload (each command first runs without ncu and must exit 0). Outputs go
# to gpurun_out/ev/ (reports exported to raw/details/source text on the box and
# deleted: gpurun copies back at most 64 MiB); tools/ncu_summary.py turns the
# raw CSVs into profiles/.
#
#   /usr/local/graft/bin/gpurun --timeout 3000 -- bash tools/final_evidence.sh
set -u
OUT=gpurun_out/ev
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$OUT/smi.txt" 2>&1
python -c "import paper_2010_01545_b200._lib as l; print(l.build_id())" > "$OUT/lib_sha16.txt" 2>&1
timeout 1200 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest=$?"
K="--steps 20 --warmup 5"  # as the driver runs it
python bench.py $K > "$OUT/bench_c1.log" 2>&1; echo "bench_c1=$?"
python bench.py $K --config c2 > "$OUT/bench_c2.log" 2>&1; echo "bench_c2=$?"
python bench.py $K --config c3 > "$OUT/bench_c3.log" 2>&1; echo "bench_c3=$?"
python bench.py --steps 30 --warmup 5 --config c4 > "$OUT/bench_c4.log" 2>&1; echo "bench_c4=$?"
python bench.py $K --impl reference > "$OUT/bench_ref.log" 2>&1; echo "bench_ref=$?"
# launch list of the default bench (plain run first)
B="bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --no-traffic"
python $B > "$OUT/launches_plain.log" 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -c 400 --csv --log-file "$OUT/launches_c1.csv" python $B > "$OUT/launches_ncu.log" 2>&1
echo "launches=$?"
cap() {  # cap NAME KREGEX ARGS...: plain run, then one --set full capture of the 3rd launch
  local name=$1 kre=$2; shift 2
  python tools/one_launch.py "$@" > "$OUT/ol_$name.log" 2>&1 && \
    ncu --set full --clock-control none --import-source on -k "regex:$kre" -s 2 -c 1 \
        -o "$OUT/ncu_$name" python tools/one_launch.py "$@" > "$OUT/ncu_$name.log" 2>&1
  local rc=$?
  echo "cap_$name=$rc"
  if [ -f "$OUT/ncu_$name.ncu-rep" ]; then  # keep the exports (gpurun copies back <= 64 MiB)
    ncu -i "$OUT/ncu_$name.ncu-rep" --page raw --csv > "$OUT/ncu_${name}_raw.csv" 2>/dev/null
    ncu -i "$OUT/ncu_$name.ncu-rep" --page details > "$OUT/ncu_${name}_details.txt" 2>/dev/null
    ncu -i "$OUT/ncu_$name.ncu-rep" --page source --csv > "$OUT/ncu_${name}_source.csv" 2>/dev/null
    rm -f "$OUT/ncu_$name.ncu-rep"
  fi
}
cap c1 xmarch 512x512x64 --n 4
cap c2 xmarch 1024x1024x64 --n 4
cap c3 xmarch 2048x2048x64 --n 4
cap c4 xmarch 2048x1024x128 --n 4 --step
cap pull xmarch 512x256x64 --n 4 --pull
cap ct ctile 256x256x512 --n 4
cap ctodd ctile 512x512x63 --n 4
ls -la "$OUT" > "$OUT/ls.txt"
du -sh "$OUT" >> "$OUT/ls.txt"
