for sc in "" enc0 enc0,enc1 enc1; do timeout 300 python scripts/profile_c2.py --scatter "$sc" 2>&1 | grep "C2 S"; done
for r in 2e6 3.8e6; do for sc in "" enc0; do timeout 300 python scripts/profile_c2.py --rate $r --scatter "$sc" 2>&1 | grep "C2 S"; done; done
