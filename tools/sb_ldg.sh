cd tools
for t in 256 512; do
 ./stream_bench 512 8 64 $t 2 1 0 0 4 0 $t 16384 0 114688
 RANDOM_FILL=1 ./stream_bench 512 8 64 $t 2 1 0 0 4 0 $t 16384 0 114688
done
RANDOM_FILL=1 ./stream_bench 256 8 64 512 2 1 0 0 4 0 512 16384 0 229376
RANDOM_FILL=1 ./stream_bench 148 8 64 1024 2 1 0 0 3 0 1024 16384 0 397000
