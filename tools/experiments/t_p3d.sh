TVSTENCIL_LIB=build/var/lib_p3d.so timeout 120 python tools/parity_quick.py heat2d | tail -1
for d in 8 9 10 11 12; do echo -n "P3 "; TVSTENCIL_LIB=build/var/lib_p3d.so timeout 60 python tools/profile_run.py --config 3 --depth $d --reps 3 | tail -1; done
