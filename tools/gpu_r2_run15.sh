python tools/ab_variants.py run 1 --batch 2>&1
