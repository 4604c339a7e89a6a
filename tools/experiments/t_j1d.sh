echo -n "base "; timeout 60 python tools/profile_run.py --config 1 --reps 3 | tail -1
for v in 32_128 16_32 16_64 24_64; do echo -n "$v "; TVSTENCIL_LIB=build/var/lib_j1d_$v.so timeout 60 python tools/profile_run.py --config 1 --reps 3 | tail -1; TVSTENCIL_LIB=build/var/lib_j1d_$v.so timeout 120 python tools/parity_quick.py heat1d | tail -1; done
