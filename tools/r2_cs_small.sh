for sh in "256,256 2,2" "256,512 2,4"; do set -- $sh
  echo "### shape $1 nsub $2"
  SHAPE=$1 NSUB=$2 CS_LIST="5 6 8 11 12 16" bash tools/r2_cs.sh
done
