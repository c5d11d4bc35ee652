python -m paper_2508_05958_b200.cli bench-uniform --dim 3 --kernel slp3d --n 32 --p 6 --leaf 8 --adm strong --eta 1 --baseline --out gpurun_out/cli_u32.csv
python -m paper_2508_05958_b200.cli bench-uniform --dim 3 --kernel gaussian --n 64 --p 8 --leaf 8 --adm strong --eta 1 --baseline --out gpurun_out/cli_u64g.csv
python -m paper_2508_05958_b200.cli bench-uniform --dim 2 --kernel slp2d --n 256 --p 8 --leaf 16 --adm strong --eta 1 --baseline --out gpurun_out/cli_u2d.csv
python -m paper_2508_05958_b200.cli bench-quasi --kernel slp2d --n 20000 --p 8 --leaf 16 --adm strong --eta 1 --rho 2 --rho 4 --out gpurun_out/cli_q.csv
