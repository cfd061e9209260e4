set -x
for pos in 32 288 544; do
 for rows in 1 4; do
  python tools/fw_timeline.py --model 8b --layers 8 --rows $rows --pos $pos --out gpurun_out/tl_${pos}_${rows}.npy
  python tools/tl_report.py gpurun_out/tl_${pos}_${rows}.npy 8 > gpurun_out/tlr_${pos}_${rows}.txt
 done
done
