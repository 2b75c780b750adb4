A=paper_2510_21270_b200/libpbs_b200.so B=build/expfake/libpbs_b200.so bash scripts/ab_attn.sh --no-e2e
