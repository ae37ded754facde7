# A/B of the GEQRF look-ahead side-GEMM tile cap (QDWHG_QR_SIDE_CAP) on the cfg3 / cfg4 solves
for cap in 0 84 128 148 256; do
  if [ "$cap" = "0" ]; then unset QDWHG_QR_SIDE_CAP; else export QDWHG_QR_SIDE_CAP=$cap; fi
  echo "cap=$cap cfg3 $(timeout 200 python tools/profile_solve.py --config 3 --steps 1 2>/dev/null | grep stages)"
done
unset QDWHG_QR_SIDE_CAP
for cap in 0 128 256; do
  if [ "$cap" = "0" ]; then unset QDWHG_QR_SIDE_CAP; else export QDWHG_QR_SIDE_CAP=$cap; fi
  echo "cap=$cap cfg4 $(timeout 300 python tools/profile_solve.py --config 4 --steps 1 2>/dev/null | grep stages)"
done
