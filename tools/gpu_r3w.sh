# stress after the shared-memory initialisation fix: the whole GPU suite three times
for i in 1 2 3; do
  ( time timeout 900 python -m pytest tests -x -q -m gpu ) 2>&1 | tail -6 | tr '\n' ' '; echo " [suite run $i]"
done
