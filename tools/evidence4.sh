# full-size property tests + ncu captures of the integer kernels
set -x
timeout 1500 python -m pytest tests/test_full_size.py -q -x > gpurun_out/pytest_full.log 2>&1; echo "full-size rc=$?"
python tools/int_prof.py > gpurun_out/int_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:life2d_box -c 1 -o gpurun_out/full_life python tools/int_prof.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:lcs_kernel -c 1 -o gpurun_out/full_lcs python tools/int_prof.py > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_integer.csv python tools/int_prof.py > /dev/null 2>&1
ls -la gpurun_out
