nvidia-smi -q -d POWER | head -40
python tools/sweep.py --config c3 --reps 400 --rounds 1 --variants '[{"variant":"xmarch"}]' > gpurun_out/pw_sweep.txt 2>&1 &
P=$!
sleep 2
for i in 1 2 3 4 5 6; do nvidia-smi --query-gpu=power.draw,power.draw.instant,power.limit,enforced.power.limit,clocks.sm,clocks.mem,clocks_throttle_reasons.active,temperature.gpu --format=csv,noheader; sleep 0.3; done
wait $P
cat gpurun_out/pw_sweep.txt | cut -c1-150
