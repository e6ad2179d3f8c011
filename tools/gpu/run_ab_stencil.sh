# A/B of the F / J.v z-march variants on one box: tools/ab/<variant>.cu swapped in for stencil_tiled.cu
cd $GRAFT_REPO_ROOT
TAG=${1:-ab}
SRC=paper_2209_08001_b200/csrc/stencil_tiled.cu
cp $SRC /tmp/stencil_tiled_current.cu
for V in current tools/ab/stencil_tiled_3bar_na.cu tools/ab/stencil_tiled_2bar_na.cu current; do
  if [ "$V" = current ]; then cp /tmp/stencil_tiled_current.cu $SRC; else cp $V $SRC; fi
  python -m paper_2209_08001_b200.build > /dev/null 2>&1 || { echo "build fail $V" >> gpurun_out/${TAG}.log; continue; }
  echo "== $V" >> gpurun_out/${TAG}.log
  REPS=20 timeout 300 python tools/micro_fjv.py 3d256 3d512 2>&1 | python -c "
import sys,json
t=sys.stdin.read(); i=t.index('{'); d=json.loads(t[i:t.rindex('}')+1])
for n,v in d['kernels'].items():
  for k in ('residual','jv'): print(n,k,round(v[k]['ms'],4),round(v[k]['frac_hbm'],3))
" >> gpurun_out/${TAG}.log 2>&1
done
cp /tmp/stencil_tiled_current.cu $SRC
