python tools/ab_variants.py run 2 2>&1
