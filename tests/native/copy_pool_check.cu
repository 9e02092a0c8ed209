// Host-only check of the staging thread pool (csrc/sellb_host.cu): parallel
// copies of sizes around the 1 MiB threshold and uneven part splits.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
namespace sellb { void host_parallel_copy(void* dst, const void* src, size_t n); }
int main() {
  for (size_t n : {size_t(1)<<20, size_t(1536*1024), size_t(1)<<21, size_t(1048576+8),
                   size_t(3000017), size_t(8)<<20}) {
    for (int rep = 0; rep < 10; ++rep) {
      std::vector<char> a(n), b(n, 0);
      for (size_t i = 0; i < n; ++i) a[i] = (char)(rand());
      sellb::host_parallel_copy(b.data(), a.data(), n);
      if (memcmp(a.data(), b.data(), n)) {
        size_t first = 0; while (a[first] == b[first]) ++first;
        size_t last = n - 1; while (a[last] == b[last]) --last;
        printf("n=%zu rep=%d mismatch [%zu, %zu]\n", n, rep, first, last); break;
      }
    }
  }
  printf("done\n");
}
