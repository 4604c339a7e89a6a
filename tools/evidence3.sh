# round-1 evidence refresh (session 2, after the e2e pipelines, integer kernels and tiling executor):
# GPU tests, bench line, reference arm, ncu captures of the new kernels
set -x
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench5.json 2> gpurun_out/bench5.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
cat > /tmp/int_prof.py <<'PY'
import bench, argparse
bench.integer_legs(argparse.Namespace(steps=1, warmup=3))
PY
ncu --set full --clock-control none --import-source on -k regex:life2d_box -c 1 -o gpurun_out/full_life python /tmp/int_prof.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:lcs_kernel -c 1 -o gpurun_out/full_lcs python /tmp/int_prof.py > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_integer.csv python /tmp/int_prof.py > /dev/null 2>&1
ls -la gpurun_out
