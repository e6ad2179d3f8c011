for cs in 2 3 4 8; do
  echo "== CS $cs"
  NKS_RAS2D_CS=$cs CUDA_LAUNCH_BLOCKING=1 SHAPE=96,80 NSUB=3,2 timeout 120 python tools/cmp_ras2d.py 2>&1 | tail -2
done
echo "== 64x64 1x1"; SHAPE=64,64 NSUB=1,1 timeout 120 python tools/cmp_ras2d.py 2>&1 | tail -2
echo "== 128x128 2x2"; SHAPE=128,128 NSUB=2,2 timeout 120 python tools/cmp_ras2d.py 2>&1 | tail -2
echo "== 256x256 4x4"; SHAPE=256,256 NSUB=4,4 timeout 120 python tools/cmp_ras2d.py 2>&1 | tail -2
