"""Markdown table of every C-ABI entry point in include/gpile_b200.h with the
reference interface its comment (or its section header) cites.

    python tests/_abi_table.py > /tmp/abi.md"""
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
CITE = re.compile(r"[a-z_]+\.hpp:\d+(?:-\d+)?(?:,\d+(?:-\d+)?)*")


def main():
    text = (ROOT / "include" / "gpile_b200.h").read_text()
    section, comment, rows = "", "", []
    pos = 0
    for m in re.finditer(r"/\*(.*?)\*/|\b(int|const char\*|uint64_t|void|gpk_session\*)\s+(gpk_[a-z0-9_]+)\s*\(",
                         text, re.S):
        if m.group(1) is not None:
            body = " ".join(l.strip(" *") for l in m.group(1).splitlines()).strip()
            if body.startswith("----"):
                section = body.strip("- ").strip()
                comment = ""
            else:
                comment = body
            pos = m.end()
            continue
        name = m.group(3)
        between = text[pos:m.start()]
        # a comment applies to the declarations that follow it up to a blank line
        if "\n\n" in between:
            comment = ""
        cites = CITE.findall(section) + CITE.findall(comment)
        sec = re.sub(r"\s*\(.*?\)\s*$", "", section.split("------")[0].strip())
        rows.append((name, ", ".join(dict.fromkeys(cites)) or "— (plumbing, or a composite of the rows above)", sec[:90]))
        pos = m.end()
    print("| entry point | reference interface it replaces | header section |")
    print("|---|---|---|")
    for n, c, w in rows:
        print(f"| `{n}` | {c} | {w.replace('|', '/')} |")


if __name__ == "__main__":
    main()
