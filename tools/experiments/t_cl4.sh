for s in "700 64 1" "700 2000 1" "700 12000 1" "300 40000 1" "160 40000 1" "700 40000 1"; do echo -n "CS=4 "; TVS_GS2D_CLUSTER=4 timeout 120 python tools/gs2d_case.py $s; done
