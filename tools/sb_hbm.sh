# 57-58 MB per launch, every launch on a different region (ROTATE): LDG vs bulk-copy rings
cd tools
export RANDOM_FILL=1
for r in "" 1; do
  export ROTATE=$r; echo "ROTATE=$r"
  ./stream_bench 148 3 64 128 4 1 0 0 5 1 160 65536 0 393216
  ./stream_bench 148 6 64 128 4 1 0 0 5 1 160 32768 0 393216
  ./stream_bench 296 3 64 128 4 1 0 0 5 1 160 32768 0 196608
  ./stream_bench 512 8 64 256 2 1 0 0 4 0 256 16384 0 114688
  ./stream_bench 148 8 64 1024 2 1 0 0 3 0 1024 16384 0 393216
done
