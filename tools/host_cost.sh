# build and run tools/host_cost.c against the in-tree libftblas.so
set -e
D=paper_2104_00897_b200
gcc -O2 -Iinclude -I/usr/local/cuda/include tools/host_cost.c -L$D -lftblas -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/$D -o /tmp/host_cost
/tmp/host_cost 256
/tmp/host_cost 2048
