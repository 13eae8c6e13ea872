cd tools/native
for t in ${TC2_SET:-1}; do for shape in "512 512 1024 1" "1024 1024 1024 4"; do
  echo "== RS_TC2=$t $shape"; RS_TC_DEBUG=1 RS_TC2=$t timeout 60 ./fc_tc_probe $shape 2>&1 | tail -4
done; done
