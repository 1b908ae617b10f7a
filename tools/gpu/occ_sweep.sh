for c in 2 3 4 5 6; do echo "CTAS=$c"; KB_CW3_CTAS=$c python tools/quickbench.py one 3 16 f32 262144 10; KB_CW3_CTAS=$c python tools/quickbench.py one 3 10 f32 262144 10; done
