cd $GRAFT_REPO_ROOT
TAG=${1:-att}
python -m paper_2209_08001_b200.build > /dev/null 2>&1 || exit 1
STALL=3,0 DTS=2.0,1.41421356,1.0 NKS_DEBUG=1 timeout 1500 python tools/attempt_cost.py > gpurun_out/${TAG}.log 2> gpurun_out/${TAG}_trace.log
echo "rc $?" >> gpurun_out/${TAG}.log
