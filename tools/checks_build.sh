# Debug build with device-side bounds checks (-DANYSEQ_CHECKS) into tools/ab/libanyseq_checks.so,
# then: ANYSEQ_LIB=$PWD/tools/ab/libanyseq_checks.so python tools/sanitize.py
set -e
rm -rf /tmp/anyseq_checks && mkdir -p /tmp/anyseq_checks
cp -r paper_2002_04561_b200 include /tmp/anyseq_checks/
rm -rf /tmp/anyseq_checks/paper_2002_04561_b200/build /tmp/anyseq_checks/paper_2002_04561_b200/lib
(cd /tmp/anyseq_checks && python paper_2002_04561_b200/build.py -DANYSEQ_CHECKS)
mkdir -p tools/ab && cp /tmp/anyseq_checks/paper_2002_04561_b200/lib/libanyseq.so tools/ab/libanyseq_checks.so
