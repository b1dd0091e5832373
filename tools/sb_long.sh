# Steady-state device read bandwidth: 577 MB per launch (ramp amortised), LDG vs bulk-copy ring
cd tools
export RANDOM_FILL=1
./stream_bench 148 8 64 1024 2 1 0 0 3 0 1024 16384 0 3932160
./stream_bench 148 3 64 128 4 1 0 0 5 1 160 65536 0 3932160
./stream_bench 148 6 64 128 4 1 0 0 5 1 160 32768 0 3932160
./stream_bench 296 3 64 128 4 1 0 0 5 1 160 32768 0 1966080
./stream_bench 148 8 64 1024 2 1 0 0 3 0 1024 16384 0 393216
