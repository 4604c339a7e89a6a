( while true; do nvidia-smi --query-gpu=clocks.sm --format=csv,noheader >> gpurun_out/clk_gs1.txt; sleep 0.5; done ) &
CLK=$!
for W in 1 2 4; do for T in 32 128 1000; do echo "W=$W"; TVS_GS1D_WARPS=$W timeout 60 python tools/profile_run.py --config 2 --T $T --reps 2 | tail -1; done; done
kill $CLK
sort gpurun_out/clk_gs1.txt | uniq -c
