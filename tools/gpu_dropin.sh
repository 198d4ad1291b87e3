mkdir -p gpurun_out
for t in optimizer sim experiment acceptance; do
  echo "== $t" >> gpurun_out/dropin.txt
  ( cd tools/dropin/_bin && timeout 900 ./${t}_test_b200 ) >> gpurun_out/dropin.txt 2>&1
  echo "rc=$?" >> gpurun_out/dropin.txt
done
