// LRU row-cache simulation: hit rate of source-row gathers for a destination order
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
typedef struct { int32_t prev, next; } Node;
int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "rb"); long cap = atol(argv[2]);
  int64_t n, nnz; fread(&n, 8, 1, f); fread(&nnz, 8, 1, f);
  int64_t* ptr = malloc((n + 1) * 8); int32_t* col = malloc(nnz * 4); int32_t* ord = malloc(n * 4);
  int32_t nsrc; fread(&nsrc, 4, 1, f);
  fread(ptr, 8, n + 1, f); fread(col, 4, nnz, f); fread(ord, 4, n, f); fclose(f);
  Node* L = calloc(nsrc, sizeof(Node)); char* in = calloc(nsrc, 1);
  int32_t head = -1, tail = -1; long size = 0, hits = 0, acc = 0;
  for (int64_t i = 0; i < n; ++i) {
    int32_t r = ord[i];
    for (int64_t e = ptr[r]; e < ptr[r + 1]; ++e) {
      int32_t s = col[e]; ++acc;
      if (in[s]) { ++hits; // move to front
        if (head != s) { int32_t p = L[s].prev, nx = L[s].next; L[p].next = nx; if (nx >= 0) L[nx].prev = p; else tail = p;
          L[s].prev = -1; L[s].next = head; L[head].prev = s; head = s; }
      } else { in[s] = 1; L[s].prev = -1; L[s].next = head; if (head >= 0) L[head].prev = s; head = s; if (tail < 0) tail = s; ++size;
        if (size > cap) { int32_t t = tail; tail = L[t].prev; L[tail].next = -1; in[t] = 0; --size; } }
    }
  }
  printf("cap %ld hit %.4f\n", cap, (double)hits / acc);
  return 0;
}
