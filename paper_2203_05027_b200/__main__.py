"""``python -m paper_2203_05027_b200 solve|generate|bench`` (the reference's CLI, cli.py)."""

from .cli import main

main()
