set -x
rm -f gpurun_out/bs6_partner.log
for mb in 8 10 12; do for sw in 0 1; do SB200_BS6_PARTNER_MB=$mb SB200_BS6_PARTNER_SWZ=$sw timeout 300 python scripts/expt/time_bs6_partner.py 1 2 3 5 7 >> gpurun_out/bs6_partner.log 2>&1; done; done
cat gpurun_out/bs6_partner.log
