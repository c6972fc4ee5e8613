bash tools/variants.sh "ip0 ip6 ip10 ip16" "sphere paper_terrain" > gpurun_out/var_ip.log 2>&1
