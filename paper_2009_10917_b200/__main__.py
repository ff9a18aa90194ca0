"""`python -m paper_2009_10917_b200 ...` runs the CLI (cli.main)."""

if __name__ == "__main__":
    from .cli import main

    raise SystemExit(main())
