for i in 1 2 3; do echo -n "CS=4 "; TVS_GS2D_CLUSTER=4 timeout 120 python tools/gs2d_case.py 700 12000 1; done
for i in 1 2; do echo -n "CS=2 "; TVS_GS2D_CLUSTER=2 timeout 120 python tools/gs2d_case.py 700 12000 1; done
echo -n "CS=4 T=3 "; TVS_GS2D_CLUSTER=4 timeout 120 python tools/gs2d_case.py 700 12000 3
echo -n "CS=4 star "; TVS_GS2D_CLUSTER=4 timeout 120 python tools/gs2d_case.py 700 12000 1 gs2d
echo -n "CS=4 500 "; TVS_GS2D_CLUSTER=4 timeout 120 python tools/gs2d_case.py 500 12000 1
