cd /root/repo
for i in 1 2; do bash scripts/ab.sh c4 o1 o2 o3 o4 base; done
