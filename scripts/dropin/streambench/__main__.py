"""`python -m streambench ...` through the shim: the B200 package's CLI."""

if __name__ == "__main__":
    from paper_2009_10917_b200.cli import main

    raise SystemExit(main())
