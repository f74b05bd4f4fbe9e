P=./build/tma_probe3
for args in "3 8 36 34 -2 -1 0" "3 8 36 34 -2 -1 1" "3 8 32 32 0 -1 0" "3 8 36 34 62 63 0" "3 8 36 34 30 -1 1"; do
  timeout 30 $P $args
done
