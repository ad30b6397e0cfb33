for c in llama2-13b llama3-8b; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"flash_bwd|flash_delta" -c 6 --csv python tools/flash_bench.py $c 2>/dev/null | grep -E "flash" | awk -F'","' '{print $5, $NF}' | head -6
done
