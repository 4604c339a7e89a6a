set -e
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -rdc=true --expt-relaxed-constexpr -DGS2P_TRACE -c -o build/var/gs2d_pipe_trace.o paper_2010_04868_b200/csrc/gs2d_pipe.cu
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -rdc=true -c -o build/var/gs2d_trace_main.o tools/gs2d_trace.cu
for f in api gs1d gs_wavefront jacobi1d jacobi2d jacobi3d jacobi_naive; do nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -rdc=true --expt-relaxed-constexpr -c -o build/var/${f}_rdc.o paper_2010_04868_b200/csrc/$f.cu; done
nvcc -gencode arch=compute_100a,code=sm_100a -rdc=true -o build/var/gs2d_trace build/var/gs2d_trace_main.o build/var/gs2d_pipe_trace.o build/var/*_rdc.o
