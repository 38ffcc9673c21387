# A/B of the small-batch K_fb variant (three warpgroups split one tile's chain)
set -e
for i in 1 2; do
  AB_T=512,4096,16384 python profiles/ab_train.py split
  NASG_NO_COOP_SPLIT=1 AB_T=512,4096,16384 python profiles/ab_train.py wg0
done
